"""CUDA kernels vs the reference's golden vectors and the CPU oracle.

Bit-exact for integer/index work (hits, detected sets, medians are copies of
input values); FP64 transforms within 1e-12 absolute on unit-variance input
(the reference's own acceptance bar, test_acceptance.py:187-207).
"""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_detect_gather_plugin_bitexact_vs_reference(cuda):
    from paper_2006_13053_b200 import _kernels

    g = golden("gather_cases.npz")
    for k in range(int(g["ncases"])):
        M, theta, thr = g[f"c{k}_params"]
        e, z, gh = g[f"c{k}_elems"], g[f"c{k}_zmat"], g[f"c{k}_ghat"]
        for wm in (0, 1):
            key = f"c{k}_{wm}_hits"
            if key not in g:
                continue
            hits, med = _kernels.detect_gather(e, z, int(M), gh, theta, thr, bool(wm))
            assert np.array_equal(hits, g[key]), (k, wm)
            assert np.array_equal(med.view(np.float64), g[f"c{k}_{wm}_med"].view(np.float64))


def test_detect_gather_odd_L_check(cuda):
    from paper_2006_13053_b200 import _kernels

    with pytest.raises(ValueError):
        _kernels.detect_gather(np.zeros((5, 2), np.int64), np.zeros((4, 2), np.int64), 11,
                               np.zeros((4, 11), complex), 0.0, 2.0, True)


@pytest.mark.parametrize("d,M,L", [(3, 31, 7), (10, 103307, 47), (20, 20663, 41),
                                   (5, 211, 27), (1, 13, 1), (25, 1039, 9)])
def test_hash_paths_vs_oracle(cuda, oracle_lib, d, M, L):
    """32-bit, 64-bit and generic residue paths against the C oracle."""
    from paper_2006_13053_b200 import _kernels

    rng = np.random.default_rng(d * 1000 + L)
    n = 20000
    e = rng.integers(0, M, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    gh = rng.normal(size=(L, M)) + 1j * rng.normal(size=(L, M))
    gh[rng.random(size=(L, M)) < 0.8] = 0.0
    thr = L / 2
    want = oracle_lib.gather_c(e, z, M, gh, 1e-9, thr, L % 2 == 1)
    got = _kernels.detect_gather(e, z, M, gh, 1e-9, thr, L % 2 == 1)
    assert np.array_equal(got[0], want[0])
    assert np.array_equal(got[1], want[1])


def test_hash_signed_rows_fused_mod(cuda, oracle_lib):
    """Driver path: raw signed candidate rows, % M fused on device."""
    import torch

    import paper_2006_13053_b200 as pkg
    from paper_2006_13053_b200 import _dev, _engine

    rng = np.random.default_rng(3)
    n, d, M, L = 50000, 10, 103307, 47
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    gh = rng.normal(size=(L, M)) + 1j * rng.normal(size=(L, M))
    gh[rng.random(size=(L, M)) < 0.9] = 0.0
    samples = _dev.upload(np.fft.ifft(gh, axis=1) * M)  # DFT/M gives gh back
    b = _engine.detect_batch(samples, M, _dev.upload(z), 1, L, _dev.upload(rows),
                             d * 4096, 0.5, theta0=torch.full((1,), 1e-9,
                                                              dtype=torch.float64,
                                                              device="cuda"),
                             want_hits=True)
    ghat = _dev.download(b.ghat)
    want_h, want_m = oracle_lib.gather_c(rows % M, z, M, ghat, 1e-9, L / 2, True)
    assert np.array_equal(_dev.download(b.hits), want_h)
    cnt = int(b.counts[0])
    idx = _dev.download(b.idx[:cnt])
    assert np.array_equal(idx, np.flatnonzero(want_h >= L / 2))
    assert np.array_equal(_dev.download(b.coeffs[:cnt]), want_m[idx])


def test_rows_injective_vs_reference(cuda):
    from paper_2006_13053_b200 import _kernels

    for case in golden("injective_cases.json"):
        e = np.array(case["elems"], dtype=np.int64)
        assert _kernels.rows_injective_mod(e, case["p"]) == case["injective"]


def test_dft_vs_reference_and_naive(cuda):
    import paper_2006_13053_b200 as pkg

    g = golden("dft_cases.npz")
    for M in g["primes"]:
        y = pkg.dft_forward_normalized(g[f"x{M}"])
        assert np.max(np.abs(y - g[f"y{M}"])) < 1e-12, M


# 8209 / 12281 / 10331: N = 24576 = 192 x 128 (mixed radix); 16411 / 24571 / 20663:
# N = 49152 = 192 x 256; 12289 / 24593: the power-of-two neighbours
@pytest.mark.parametrize("M", [2, 3, 5, 7, 31, 127, 211, 509, 1009, 1039, 2069, 4099,
                               8209, 10331, 12281, 12289, 16411, 20663, 24571, 24593,
                               40009, 103307])
def test_dft_primes_vs_naive_and_parseval(cuda, M):
    import paper_2006_13053_b200 as pkg

    rng = np.random.default_rng(M)
    x = rng.normal(size=M) + 1j * rng.normal(size=M)
    y = pkg.dft_forward_normalized(x)
    if M <= 4099:
        j = np.arange(M)
        naive = (np.exp(-2j * np.pi * np.outer(j, j) / M) @ x) / M
        assert np.max(np.abs(y - naive)) < 1e-12
    ref = np.fft.fft(x) / M
    assert np.max(np.abs(y - ref)) < 1e-13
    energy = np.mean(np.abs(x) ** 2)
    assert abs(np.sum(np.abs(y) ** 2) - energy) <= 1e-10 * energy


def test_dft_rejects_bad_input(cuda):
    import paper_2006_13053_b200 as pkg

    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized([1.0, np.nan])
    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized([])
    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized(np.zeros((2, 2)))


def test_inverse_dft_batch(cuda):
    import paper_2006_13053_b200 as pkg
    from paper_2006_13053_b200 import _dev
    from paper_2006_13053_b200.dft import dft_batch

    rng = np.random.default_rng(9)
    for M in (211, 20663):
        x = rng.normal(size=(5, M)) + 1j * rng.normal(size=(5, M))
        y = _dev.download(dft_batch(_dev.upload(x), M, inverse=True, scale=1.0))
        assert np.max(np.abs(y - M * np.fft.ifft(x, axis=1))) < 1e-9


def test_structured_sampling_vs_reference(cuda):
    import paper_2006_13053_b200 as pkg

    g = golden("sampling_cases.npz")
    for k in range(int(g["n"])):
        p = pkg.SparsePoly(pkg.FreqSet(g[f"s{k}_support"].shape[1], g[f"s{k}_support"],
                                       _sorted=True), g[f"s{k}_coeffs"])
        lat = pkg.Rank1Lattice(g[f"s{k}_z"], int(g[f"s{k}_M"]))
        vals = pkg.evaluate_on_lattice(p, lat)
        ref = g[f"s{k}_fast"]
        assert np.max(np.abs(vals - ref)) < 1e-12 * max(1.0, np.max(np.abs(ref)))
        dense = pkg.evaluate_many(p, pkg.lattice_nodes(lat))
        assert np.max(np.abs(dense - g[f"s{k}_dense"])) < 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_scatter_bins_match_bincount_order(cuda, oracle_lib):
    """Residue bins summed in ascending coefficient order == np.bincount."""
    import torch

    from paper_2006_13053_b200 import _dev, _native

    rng = np.random.default_rng(5)
    s, d, M, L = 20000, 4, 211, 3  # many collisions, > one 8192-key chunk
    sup = rng.integers(-50, 50, size=(s, d), dtype=np.int64)
    c = rng.normal(size=s) + 1j * rng.normal(size=s)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bins = _dev.empty((L, M), torch.complex128)
    sup_d, c_d, z_d = _dev.upload(sup), _dev.upload(c), _dev.upload(z)  # keep alive
    _native.call("sfftb_scatter_bins", _dev.ptr(sup_d), s, d, d, _dev.ptr(c_d), _dev.ptr(z_d),
                 1, L, M, _dev.ptr(bins), None, _dev.stream())
    got = _dev.download(bins)
    for l in range(L):
        r = oracle_lib.residues(sup, z[l], M)
        want = np.bincount(r, weights=c.real, minlength=M) + 1j * np.bincount(
            r, weights=c.imag, minlength=M)
        assert np.array_equal(got[l], want)


def test_noise_stream_matches_oracle(cuda, oracle_lib):
    import torch

    from paper_2006_13053_b200 import _dev, _native

    M, rows, seed, call0, sigma = 4099, 3, 99, 17, 1e-3
    x = _dev.zeros((rows, M), torch.complex128)
    _native.call("sfftb_add_noise", _dev.ptr(x), rows, M, seed, call0, sigma, _dev.stream())
    got = _dev.download(x)
    for r in range(rows):
        want = oracle_lib.noise_for_call(seed, call0 + r, M, sigma)
        assert np.max(np.abs(got[r] - want)) < 1e-17
    assert abs(np.std(got.real) - sigma) < 0.05 * sigma


@pytest.mark.parametrize("M,G,L,sigma", [(20663, 2, 5, 0.0), (10331, 3, 3, 1e-3), (4099, 1, 7, 0.0),
                                         (30011, 2, 3, 1e-3), (14009, 1, 5, 0.0)])
def test_fused_sample_detect_matches_unfused(cuda, M, G, L, sigma):
    """sfftb_sample_detect_dft (samples kept on chip) == inverse DFT + noise +
    zero test + forward DFT + bitmap run as separate kernels."""
    import torch

    from paper_2006_13053_b200 import _dev, _engine, _native
    from paper_2006_13053_b200.dft import dft_batch

    rng = np.random.default_rng(M + G)
    bins = np.zeros((G * L, M), dtype=np.complex128)
    for row in bins:  # sparse bins: clear zero / nonzero margins
        nz = rng.choice(M, size=300, replace=False)
        row[nz] = rng.normal(size=300) + 1j * rng.normal(size=300)
    b = _dev.upload(bins)
    seed, call0 = 77, 5
    ghat_f, theta_f, bits_f = _engine.sample_spectra_fused(b, M, G, L, seed, call0, sigma)
    samples = dft_batch(b, M, inverse=True, scale=1.0)
    if sigma > 0:
        _native.call("sfftb_add_noise", _dev.ptr(samples), G * L, M, seed, call0, sigma,
                     _dev.stream())
    ghat_u, theta_u, bits_u = _engine.spectra(samples, M, G, L)
    assert np.allclose(_dev.download(theta_f), _dev.download(theta_u), rtol=1e-12, atol=0)
    assert np.max(np.abs(_dev.download(ghat_f) - _dev.download(ghat_u))) < 1e-13
    assert np.array_equal(_dev.download(bits_f), _dev.download(bits_u))
    if sigma == 0:
        assert np.max(np.abs(_dev.download(ghat_f) - bins)) < 1e-12


@pytest.mark.parametrize("case", ["dups_small_box", "wide_multi_group", "extremes", "tiny"])
def test_device_canonicalisation_matches_host(cuda, case):
    """csrc/canon.cu sort + de-dup == the host canonical() (freqset.py:48-67)."""
    import torch

    pkg = cuda
    from paper_2006_13053_b200 import _dev
    from paper_2006_13053_b200.freqset import canonical

    rng = np.random.default_rng(len(case))
    if case == "dups_small_box":
        rows = rng.integers(-3, 4, size=(100_003, 4))
    elif case == "wide_multi_group":  # 10 x 21-bit spans: four 64-bit key groups
        rows = rng.integers(-(1 << 20), 1 << 20, size=(300_001, 10))
        rows = np.vstack([rows, rows[:5000]])  # exact duplicates across the set
    elif case == "extremes":
        rows = rng.integers(-(1 << 62), 1 << 62, size=(20_000, 3))
        rows[:, 1] = 7  # a constant coordinate
        rows = np.vstack([rows, rows[::3]])
    else:
        rows = np.array([[5, -1], [5, -1], [-2, 3]])
    got = _dev.download(pkg.canonicalize_device(_dev.upload(rows), rows.shape[1]))
    assert np.array_equal(got, canonical(np.ascontiguousarray(rows)))
    S = pkg.FreqSet.from_device(rows.shape[1], _dev.upload(rows), canonical=False)
    assert len(S) == got.shape[0]


@pytest.mark.parametrize("d,lo,hi,count", [
    (3, -2, 2, 100),            # 125 points: duplicates, top-up rounds, Floyd choice
    (10, -4096, 4096, 1 << 16),  # config-4 box: one round, native tail shuffle
    (4, -40, 40, 40_000),        # duplicates AND the tail-shuffle regime
    (2, -(1 << 40), 1 << 40, 5000),  # range beyond 32-bit words: numpy's own draw
    (5, 0, 0, 1),                # a one-point box
])
def test_random_box_device_is_the_reference_stream(cuda, d, lo, hi, count):
    """Device-born Gamma == _random_from_box (freqset.py:266-280) row for row,
    and the generator is left in numpy's exact state (later draws agree)."""
    import workloads

    pkg = cuda
    g1 = np.random.default_rng(d * 1000 + count)
    g1.random(3)  # leave a buffered 32-bit word half the time
    g1.integers(0, 7)
    g2 = np.random.default_rng(d * 1000 + count)
    g2.random(3)
    g2.integers(0, 7)
    want = workloads.rows_from_box(d, lo, hi, count, g1)
    got = pkg.random_box_device(pkg.Box(d, lo, hi), count, g2)
    assert np.array_equal(got.elems, want)
    assert g1.bit_generator.state == g2.bit_generator.state
    assert np.array_equal(g1.integers(0, 1 << 40, size=9), g2.integers(0, 1 << 40, size=9))


@pytest.mark.parametrize("L", [1, 7, 31, 33, 47, 63, 65])
def test_medians_ties_and_signed_zeros_bitexact(cuda, oracle_lib, L):
    """Median selection with heavy ties, +0.0/-0.0 mixes and runs straddling
    the middle position (the fast path's fallback) -- bitwise against the C
    restatement of the reference's insertion-sort median."""
    from paper_2006_13053_b200 import _kernels

    rng = np.random.default_rng(L)
    M, d, n = 13, 2, 4000
    e = rng.integers(0, M, size=(n, d))
    z = rng.integers(0, M, size=(L, d))
    vals = np.array([0.0, -0.0, 1.0, -1.0, 2.5, 0.0, -0.0])
    gh = (rng.choice(vals, size=(L, M)) + 1j * rng.choice(vals, size=(L, M))).astype(np.complex128)
    hits, med = _kernels.detect_gather(e, z, M, gh, -1.0, 0.0, True)  # every row detected
    want_h, want_m = oracle_lib.gather_c(e, z, M, gh, -1.0, 0.0, True)
    assert np.array_equal(hits, want_h)
    assert np.array_equal(med.view(np.int64), want_m.view(np.int64))


@pytest.mark.parametrize("t,n1,n2,G,L,M", [(1, 65, 65, 5, 31, 20663), (4, 1000, 65, 5, 37, 20663),
                                           (9, 2000, 129, 2, 41, 10331), (2, 37, 3, 1, 7, 97)])
def test_pair_tables_match_generic_hashing_and_medians(cuda, t, n1, n2, G, L, M):
    """Residue tables of a Cartesian J reproduce sfftb_hash_hits / sfftb_medians
    on the materialised J bit for bit."""
    import torch

    from paper_2006_13053_b200 import _dev, _engine, _native

    rng = np.random.default_rng(n1 + t)
    prefix = np.unique(rng.integers(-64, 65, size=(n1, t)), axis=0)
    n1 = prefix.shape[0]
    vals = np.unique(rng.integers(-64, 65, size=n2))
    n2 = vals.size
    pre_d, vals_d = _dev.upload(prefix), _dev.upload(vals)
    J = _engine.pair_product(pre_d, vals_d)
    z = _dev.upload(rng.integers(0, M, size=(G * L, t + 1)))
    W = int(_native.lib().sfftb_bitmap_words(M))
    bits = _dev.upload((rng.integers(0, 1 << 31, size=(G * L * W,)) & 0x22222222).astype(np.int32))
    n = n1 * n2
    st = _dev.stream()
    P = _dev.empty((G * L * n1,), torch.int32)
    V = _dev.empty((G * L * n2,), torch.int32)
    _native.call("sfftb_pair_residues", _dev.ptr(pre_d), n1, t, _dev.ptr(vals_d), n2, _dev.ptr(z),
                 G * L, M, _dev.ptr(P), _dev.ptr(V), st)
    nw = (n + 31) // 32
    h1, h2 = _dev.empty((G * n,), torch.int64), _dev.empty((G * n,), torch.int64)
    m1, m2 = _dev.empty((G * nw,), torch.int32), _dev.empty((G * nw,), torch.int32)
    mh = (L + 1) // 2 - 1
    _native.call("sfftb_hash_hits", _dev.ptr(J), n, t + 1, _dev.ptr(z), G, L, M, _dev.ptr(bits),
                 -1, mh, _dev.ptr(h1), _dev.ptr(m1), st)
    _native.call("sfftb_hash_pairs", _dev.ptr(P), _dev.ptr(V), n1, n2, G, L, M, _dev.ptr(bits),
                 mh, _dev.ptr(h2), _dev.ptr(m2), st)
    assert np.array_equal(_dev.download(h1), _dev.download(h2))
    assert np.array_equal(_dev.download(m1), _dev.download(m2))
    ghat = _dev.upload(rng.normal(size=(G * L, M)) + 1j * rng.normal(size=(G * L, M)))
    idx = _dev.upload(np.concatenate([np.sort(rng.choice(n, size=min(n, 500), replace=False))
                                      for _ in range(G)]))
    k = min(n, 500)
    cnt = _dev.upload(np.full(G, k, dtype=np.int64))
    o1, o2 = _dev.empty((G * k,), torch.complex128), _dev.empty((G * k,), torch.complex128)
    _native.call("sfftb_medians", _dev.ptr(J), t + 1, _dev.ptr(z), G, L, M, _dev.ptr(ghat),
                 _dev.ptr(idx), _dev.ptr(cnt), k, _dev.ptr(o1), st)
    _native.call("sfftb_medians_pairs", _dev.ptr(P), _dev.ptr(V), n1, n2, G, L, M,
                 _dev.ptr(ghat), _dev.ptr(idx), _dev.ptr(cnt), k, _dev.ptr(o2), st)
    assert np.array_equal(_dev.download(o1).view(np.int64), _dev.download(o2).view(np.int64))


@pytest.mark.parametrize("M,G,L,s,sigma", [(20663, 2, 5, 1000, 0.0), (10331, 3, 3, 4096, 1e-3),
                                           (4099, 1, 7, 40, 0.0)])
def test_sampler_lists_match_dense_bins(cuda, M, G, L, s, sigma):
    """Sparse sampler (sfftb_scatter_list + sfftb_sample_detect_dft_list) ==
    dense bins (sfftb_scatter_bins + sfftb_sample_detect_dft), bit for bit:
    ghat, zero thresholds and bitmaps.  Small coordinates force residue
    collisions, so runs are summed in coefficient order in both."""
    import torch

    from paper_2006_13053_b200 import _dev, _engine, _native

    rng = np.random.default_rng(M + s)
    d = 4
    sup = rng.integers(-6, 7, size=(s, d), dtype=np.int64)
    anch = rng.normal(size=(G, s)) + 1j * rng.normal(size=(G, s))
    z = rng.integers(0, M, size=(G * L, d), dtype=np.int64)
    sup_d, a_d, z_d = _dev.upload(sup), _dev.upload(anch), _dev.upload(z)
    bins = _dev.empty((G * L, M), torch.complex128)
    _native.call("sfftb_scatter_bins", _dev.ptr(sup_d), s, d, d, _dev.ptr(a_d), _dev.ptr(z_d),
                 G, L, M, _dev.ptr(bins), None, _dev.stream())
    want = _engine.sample_spectra_fused(bins, M, G, L, 31, 4, sigma)
    lr = _dev.empty((G * L * s,), torch.int32)
    lv = _dev.empty((G * L * s,), torch.complex128)
    _native.call("sfftb_scatter_list", _dev.ptr(sup_d), s, d, d, _dev.ptr(a_d), _dev.ptr(z_d),
                 G, L, M, _dev.ptr(lr), _dev.ptr(lv), _dev.stream())
    W = int(_native.lib().sfftb_bitmap_words(M))
    ghat = _dev.empty((G * L, M), torch.complex128)
    theta = _dev.empty((G,), torch.float64)
    bits = _dev.empty((G * L * W,), torch.int32)
    ws = _dev.workspace(_native.lib().sfftb_sample_detect_workspace_bytes(G * L, M))
    _native.call("sfftb_sample_detect_dft_list", _dev.ptr(lr), _dev.ptr(lv), s, G, L, M, 31, 4,
                 sigma, _dev.ptr(ghat), _dev.ptr(theta), _dev.ptr(bits), _dev.ptr(ws),
                 _dev.stream())
    for got, exp in zip((ghat, theta, bits), want):
        assert np.array_equal(_dev.download(got), _dev.download(exp))
    # every listed residue is a run head of the sorted residues, once
    r = _dev.download(lr).view(np.uint32).reshape(G * L, s)
    for row in range(G * L):
        heads = r[row][r[row] != 0xFFFFFFFF]
        assert np.all(np.diff(heads.astype(np.int64)) > 0)


def test_eval_lines_matches_dense_nodes(cuda):
    """sfftb_eval_lines == sfftb_eval_dense on the explicit step-1 line nodes."""
    import torch

    from paper_2006_13053_b200 import _dev, _native

    rng = np.random.default_rng(3)
    d, r, K, s = 6, 3, 33, 200
    sup = rng.integers(-16, 17, size=(s, d), dtype=np.int64)
    c = rng.normal(size=s) + 1j * rng.normal(size=s)
    base = rng.uniform(size=(d * r, d))
    nodes = np.repeat(base, K, axis=0).reshape(d * r, K, d)
    for q in range(d * r):
        nodes[q, :, q // r] = np.arange(K) / K
    sup_d, c_d, b_d = _dev.upload(sup), _dev.upload(c), _dev.upload(base)
    X_d = _dev.upload(nodes.reshape(-1, d))
    want = _dev.empty((d * r * K,), torch.complex128)
    got = _dev.empty((d * r * K,), torch.complex128)
    _native.call("sfftb_eval_dense", _dev.ptr(sup_d), s, d, _dev.ptr(c_d), _dev.ptr(X_d),
                 d * r * K, _dev.ptr(want), _dev.stream())
    _native.call("sfftb_eval_lines", _dev.ptr(sup_d), s, d, _dev.ptr(c_d), _dev.ptr(b_d),
                 d * r, K, r, _dev.ptr(got), _dev.stream())
    assert np.array_equal(_dev.download(got), _dev.download(want))


def test_hash_without_host_bound_mixed_rows(cuda, oracle_lib):
    """A large host FreqSet with no memoised bound: the hash picks the 32-bit
    or the exact 64-bit residue chain per warp from the rows themselves
    (kbound = -1, csrc/hash.cu AUTO); a few huge coordinates force the wide
    chain on their warps only.  Bit-exact against the C oracle."""
    import torch

    import paper_2006_13053_b200 as pkg
    from paper_2006_13053_b200 import _dev, _engine

    rng = np.random.default_rng(11)
    n, d, M, L = 300_000, 10, 103307, 47
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    wide = rng.choice(n, size=50, replace=False)
    rows[wide, 3] = rng.integers(-(1 << 62), 1 << 62, size=50)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    gh = rng.normal(size=(L, M)) + 1j * rng.normal(size=(L, M))
    gh[rng.random(size=(L, M)) < 0.9] = 0.0
    samples = _dev.upload(np.fft.ifft(gh, axis=1) * M)
    G = pkg.FreqSet(d, rows)  # canonical order, no bound memoised
    assert pkg.detect._kbound(G) == -1
    srt = G.elems
    b = _engine.detect_batch(samples, M, _dev.upload(z), 1, L, G.device(), -1, 0.5,
                             theta0=torch.full((1,), 1e-9, dtype=torch.float64,
                                               device="cuda"), want_hits=True)
    ghat = _dev.download(b.ghat)
    want_h, _ = oracle_lib.gather_c(srt % M, z, M, ghat, 1e-9, L / 2, True)
    assert np.array_equal(_dev.download(b.hits), want_h)


@pytest.mark.parametrize("K,nv,r,s_local,theta", [(65, 65, 5, 2000, 1e-12), (129, 129, 3, 40, 0.5),
                                                 (64, 33, 2, 7, 0.0), (1000, 1000, 4, 100, 0.2)])
def test_step1_select_matches_reference_lexsort(cuda, K, nv, r, s_local, theta):
    """sfftb_step1_select == step1_components' selection (dimincr.py:143-146):
    per line the s_local largest |est[v mod K]| (ties: smaller v first),
    >= theta, union over the r lines of each coordinate -- with planted exact
    magnitude ties and values below theta."""
    import torch

    from paper_2006_13053_b200 import _dev, _native

    pkg = cuda
    rng = np.random.default_rng(K + nv)
    d = 3
    nl = d * r
    est = rng.standard_normal((nl, K)) + 1j * rng.standard_normal((nl, K))
    est[:, ::5] = est[:, 1:2]  # exact ties
    est[:, 3::7] *= 1e-3       # small values
    vals = np.sort(rng.choice(np.arange(-K // 2, K // 2 + K), size=nv, replace=False))
    off = (d * nv + 1) // 2 * 2
    res = _dev.empty((off + 2 * nl,), torch.int32)
    # both inputs stay referenced until the call is enqueued (a temporary freed
    # inside the argument list hands its block to the next upload)
    est_d, vals_d = _dev.upload(est), _dev.upload(vals)
    _native.call("sfftb_step1_select", _dev.ptr(est_d), nl, K,
                 _dev.ptr(vals_d), nv, r, s_local, theta, _dev.ptr(res),
                 res[off:].data_ptr(), _dev.stream())
    arr = _dev.download(res)
    present = arr[:d * nv].reshape(d, nv) != 0
    kept = arr[off:].view(np.int64)
    for t in range(d):
        union = np.zeros(0, np.int64)
        for i in range(r):
            mags = np.abs(est[t * r + i][vals % K])
            order = np.lexsort((vals, -mags))[:s_local]
            order = order[mags[order] >= theta]
            assert kept[t * r + i] == order.size
            union = np.union1d(union, vals[order])
        assert np.array_equal(vals[present[t]], union)


@pytest.mark.parametrize("L,G", [(3, 2), (31, 5), (39, 5), (41, 2), (63, 1)])
def test_network_medians_ties_and_signed_zeros_bitexact(cuda, L, G):
    """Pair-table medians by selection network (medians_net_pairs_kernel) with
    heavy ties and +0.0/-0.0 mixes (rows holding a zero take the insertion
    sort in lattice order) == the generic medians (sfftb_medians, bit-exact
    to the reference's insertion sort) on the materialised J."""
    import torch

    from paper_2006_13053_b200 import _dev, _engine, _native

    rng = np.random.default_rng(100 + L)
    M, t, n1, n2 = 101, 2, 40, 9
    prefix = np.unique(rng.integers(-30, 31, size=(n1, t)), axis=0)
    n1 = prefix.shape[0]
    vals = np.unique(rng.integers(-30, 31, size=n2))
    n2 = vals.size
    pre_d, vals_d = _dev.upload(prefix), _dev.upload(vals)
    J = _engine.pair_product(pre_d, vals_d)
    n = n1 * n2
    z = _dev.upload(rng.integers(0, M, size=(G * L, t + 1)))
    st = _dev.stream()
    P = _dev.empty((G * L * n1,), torch.int32)
    V = _dev.empty((G * L * n2,), torch.int32)
    _native.call("sfftb_pair_residues", _dev.ptr(pre_d), n1, t, _dev.ptr(vals_d), n2, _dev.ptr(z),
                 G * L, M, _dev.ptr(P), _dev.ptr(V), st)
    pool = np.array([0.0, -0.0, 1.0, -1.0, 2.5, 0.0, -0.0, 0.5])
    gh = rng.choice(pool, size=(G * L, M)) + 1j * rng.choice(pool, size=(G * L, M))
    gh[0] = rng.normal(size=M) + 1j * rng.normal(size=M)  # some rows without zeros
    ghat = _dev.upload(gh.astype(np.complex128))
    idx = _dev.upload(np.concatenate([np.arange(n) for _ in range(G)]))
    cnt = _dev.upload(np.full(G, n, dtype=np.int64))
    o1, o2 = _dev.empty((G * n,), torch.complex128), _dev.empty((G * n,), torch.complex128)
    _native.call("sfftb_medians", _dev.ptr(J), t + 1, _dev.ptr(z), G, L, M, _dev.ptr(ghat),
                 _dev.ptr(idx), _dev.ptr(cnt), n, _dev.ptr(o1), st)
    _native.call("sfftb_medians_pairs", _dev.ptr(P), _dev.ptr(V), n1, n2, G, L, M,
                 _dev.ptr(ghat), _dev.ptr(idx), _dev.ptr(cnt), n, _dev.ptr(o2), st)
    assert np.array_equal(_dev.download(o1).view(np.int64), _dev.download(o2).view(np.int64))
