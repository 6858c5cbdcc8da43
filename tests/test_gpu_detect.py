"""Fixed-candidate-set reconstruction (detect.py entry points) on the GPU vs
the reference's golden outputs and the CPU oracle."""

import numpy as np
import pytest

import workloads
from conftest import golden

pytestmark = pytest.mark.gpu


def assert_topk_equivalent(got, want, cand_idx, cand_coeffs, rtol=1e-12):
    """Top-s sets agree, up to roundoff-level ties at the cut-off.

    An exact magnitude tie in the reference (broken by candidate index) can
    come from two different FFT bins that pocketfft happened to round
    identically; the B200 Bluestein rounds them within ~1e-16 relative but
    not bit-identically, so such a tie may resolve the other way.  Every
    element in the symmetric difference must sit at the cut-off magnitude
    within rtol."""
    got, want = np.asarray(got), np.asarray(want)
    if np.array_equal(got, want):
        return
    assert len(got) == len(want)
    mags = dict(zip(np.asarray(cand_idx).tolist(), np.abs(cand_coeffs).tolist()))
    cutoff = min(mags[i] for i in want.tolist())
    for e in set(got.tolist()) ^ set(want.tolist()):
        assert abs(mags[e] - cutoff) <= rtol * cutoff, (e, mags[e], cutoff)


def _config(pkg, zmat, M):
    lats = [pkg.Rank1Lattice(z, M) for z in zmat]
    return pkg.MultiLatticeConfig(lats, 0.5, 10.33, 0.5)


def test_tiny_instances_vs_reference(cuda):
    pkg = cuda
    g = golden("tiny_detect.npz")
    for k in range(int(g["n"])):
        p = f"t{k}_"
        S = pkg.FreqSet(g[p + "gamma"].shape[1], g[p + "gamma"], _sorted=True)
        cfg = _config(pkg, g[p + "zmat"], int(g[p + "M"]))
        smp = list(g[p + "samples"])
        res = pkg.detect_and_compute(smp, cfg, S)
        assert res.theta_zero == pytest.approx(float(g[p + "theta0"]), rel=1e-14)
        assert np.array_equal(res.hits, g[p + "hits"])
        assert np.array_equal(res.detected_idx, g[p + "idx"])
        if len(res.coeffs):
            assert np.max(np.abs(res.coeffs - g[p + "coeffs"])) < 1e-10
        r0 = pkg.detect_and_compute(smp, cfg, S, zero=pkg.ZeroTest(1e-8))
        assert np.array_equal(r0.hits, g[p + "hits0"])
        assert np.array_equal(r0.detected_idx, g[p + "idx0"])
        top = pkg.detect_topk(smp, cfg, S, 2, 0.1)
        assert_topk_equivalent(top.detected_idx, g[p + "topk_idx"], g[p + "idx"],
                               g[p + "coeffs"])
        fr = pkg.detect_frequencies(smp, cfg, S)
        assert np.array_equal(fr.detected_idx, g[p + "freq_idx"])
        post = pkg.postprocess_r1l(res, smp, cfg)
        assert np.array_equal(post.detected_idx, g[p + "post_idx"])
        if len(post.coeffs):
            assert np.max(np.abs(post.coeffs - g[p + "post_coeffs"])) < 1e-10


def test_config1_end_to_end_vs_reference(cuda):
    pkg = cuda
    g = golden("cfg1.npz")
    w = workloads.config1()
    G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
    I = G.take(w.support_idx)
    p = pkg.SparsePoly(I, w.coeffs)
    rng = w.rng  # positioned after Gamma, I and the coefficients
    cfg = pkg.draw_config(G, w.s, 0.1, rng=rng)
    assert cfg.shared_M == int(g["M"]) and np.array_equal(cfg.zmat(), g["zmat"])
    orc = pkg.oracle_from_poly(p)
    smp = [orc.sample_lattice(lat) for lat in cfg.lattices]
    assert orc.count == cfg.L * cfg.shared_M
    for a, b in zip(smp, g["samples"]):
        assert np.max(np.abs(a - b)) < 1e-11
    res = pkg.detect_and_compute(smp, cfg, G)
    assert np.array_equal(res.hits, g["hits"])
    assert np.array_equal(res.detected_idx, g["idx"])
    assert np.max(np.abs(res.coeffs - g["coeffs"])) < 1e-10 * np.max(np.abs(g["coeffs"]))
    assert res.detected == I
    top = pkg.detect_topk(smp, cfg, G, 10, 1.0)
    assert_topk_equivalent(top.detected_idx, g["topk_idx"], g["idx"], g["coeffs"])
    post = pkg.postprocess_r1l(res, smp, cfg)
    assert np.array_equal(post.detected_idx, g["post_idx"])
    assert np.max(np.abs(post.coeffs - g["post_coeffs"])) < 1e-10


def test_zero_polynomial_and_empty_results(cuda):
    pkg = cuda
    rng = np.random.default_rng(1)
    gamma = pkg.random_subset(pkg.Box(2, -4, 4), 10, rng)
    cfg = pkg.MultiLatticeConfig([pkg.Rank1Lattice(rng.integers(0, 13, 2), 13)
                                  for _ in range(5)], 0.5, 10.33, 0.5)
    res = pkg.detect_frequencies([np.zeros(13, complex)] * 5, cfg, gamma)
    assert len(res.detected) == 0
    res = pkg.detect_and_compute([np.zeros(13, complex)] * 5, cfg, gamma)
    assert pkg.postprocess_r1l(res, [np.zeros(13, complex)] * 5, cfg) is res


def test_contract_errors(cuda):
    pkg = cuda
    lat = pkg.Rank1Lattice([1, 2], 11)
    cfg = pkg.MultiLatticeConfig([lat], 0.5, 10.33, 0.5)
    with pytest.raises(pkg.ParameterError):
        pkg.detect_frequencies([np.zeros(10)], cfg, pkg.FreqSet(2, [(0, 0)]))
    lats = [pkg.Rank1Lattice([1], 11) for _ in range(4)]
    with pytest.raises(pkg.ParameterError):
        pkg.detect_and_compute([np.zeros(11, complex)] * 4,
                               pkg.MultiLatticeConfig(lats, 0.5, 10.33, 0.5),
                               pkg.FreqSet(1, [(0,)]))
    lats = [pkg.Rank1Lattice([1], 11) for _ in range(3)]
    with pytest.raises(pkg.ParameterError):
        pkg.detect_and_compute([np.zeros(11, complex)] * 3,
                               pkg.MultiLatticeConfig(lats, 0.25, 10.33, 0.5),
                               pkg.FreqSet(1, [(0,)]))


def test_topk_tie_break_deterministic(cuda):
    pkg = cuda
    I = pkg.FreqSet(1, [(1,), (4,)])
    p = pkg.SparsePoly(I, np.array([1.0, -1.0]))
    lat = pkg.Rank1Lattice([1], 11)
    cfg = pkg.MultiLatticeConfig([lat], 0.5, 10.33, 0.5)
    smp = [pkg.evaluate_on_lattice(p, lat)]
    for _ in range(3):
        top = pkg.detect_topk(smp, cfg, I, 1, 0.0)
        assert list(top.detected) == [(1,)]


def test_topk_selection_vs_oracle(cuda, oracle_lib):
    """Top-s over many detected rows with exact magnitude ties (purely real or
    imaginary coefficients: |c| is exact in both libms)."""
    import torch

    from paper_2006_13053_b200 import _dev, _engine

    rng = np.random.default_rng(11)
    n = 150_000
    idx = np.sort(rng.choice(10**7, size=n, replace=False)).astype(np.int64)
    mags = rng.choice(np.linspace(1, 2, 500), size=n) * rng.choice([-1.0, 1.0], size=n)
    co = np.where(rng.random(n) < 0.5, mags + 0j, 1j * mags)
    idx_d, co_d = _dev.upload(idx), _dev.upload(co)
    cnt = torch.tensor([n], device="cuda")
    for grid, s_tilde, theta in [(g, s, th) for g in (False, True)
                                 for s, th in ((2000, 1.3), (n + 5, 0.0), (0, 0.0), (1, 1.9),
                                               (70_000, 1.0))]:
        kidx, kco, kc = _engine.topk(idx_d, co_d, cnt, 1, n, theta, s_tilde, grid=grid)
        k = int(kc[0])
        want_i, want_c = oracle_lib.topk_filter(idx, co, s_tilde, theta)
        assert k == len(want_i)
        assert np.array_equal(_dev.download(kidx[:k]), want_i)
        assert np.array_equal(_dev.download(kco[:k]), want_c)


def test_per_lattice_coefficients(cuda):
    pkg = cuda
    g = golden("tiny_detect.npz")
    S = pkg.FreqSet(g["t0_gamma"].shape[1], g["t0_gamma"], _sorted=True)
    cfg = _config(pkg, g["t0_zmat"], int(g["t0_M"]))
    smp = list(g["t0_samples"])
    mat = pkg.per_lattice_coefficients(smp, cfg, S)
    assert mat.shape == (len(S), cfg.L)
    med = np.median(mat.real, axis=1) + 1j * np.median(mat.imag, axis=1)
    got = np.zeros(len(S), complex)
    got[g["t0_idx"]] = g["t0_coeffs"]
    assert np.max(np.abs(med[g["t0_idx"]] - g["t0_coeffs"])) < 1e-10


@pytest.mark.parametrize("M,L,n,s", [(211, 9, 3000, 40), (1031, 7, 4000, 300), (97, 5, 500, 60)])
def test_postprocess_r1l_kernel_vs_oracle(cuda, oracle_lib, M, L, n, s):
    """K9 on crowded residues (many collisions, rows with and without a
    collision-free lattice, kept and dropped rows) against the numpy
    restatement: identical kept indices, refined values to roundoff."""
    pkg, port = cuda, oracle_lib
    rng = np.random.default_rng(M * 7 + L)
    d = 3
    gamma = np.unique(rng.integers(-40, 41, size=(n, d)), axis=0)
    S = pkg.FreqSet(d, gamma, _sorted=True)
    sup = np.sort(rng.choice(len(gamma), size=s, replace=False))
    coeffs = rng.normal(size=s) + 1j * rng.normal(size=s)
    coeffs[: s // 4] *= 1e-13  # some refine below the zero threshold
    zmat = rng.integers(0, M, size=(L, d))
    cfg = _config(pkg, zmat, M)
    p = pkg.SparsePoly(S.take(sup), coeffs)
    orc = pkg.oracle_from_poly(p)
    smp = [orc.sample_lattice(lat) for lat in cfg.lattices]
    res = pkg.detect_and_compute(smp, cfg, S)
    post = pkg.postprocess_r1l(res, smp, cfg)
    want_idx, want_co = port.postprocess_r1l(gamma[res.detected_idx], res.coeffs,
                                             res.detected_idx, smp, M, zmat, res.theta_zero)
    assert len(res.detected_idx) > s // 2
    assert np.array_equal(post.detected_idx, want_idx)
    assert np.max(np.abs(post.coeffs - want_co), initial=0.0) <= 1e-13 * max(
        1.0, np.max(np.abs(want_co), initial=0.0))


def test_topk_grid_path_multi_group_vs_oracle(cuda, oracle_lib):
    """The grid-wide top-s (caps >= 16384) with several groups of different
    counts inside one cap-strided batch, exact ties, dropped entries."""
    import torch

    from paper_2006_13053_b200 import _dev, _engine

    rng = np.random.default_rng(5)
    cap, G = 40_000, 3
    counts = [40_000, 17_000, 25_001]
    idx = np.zeros((G, cap), np.int64)
    co = np.zeros((G, cap), np.complex128)
    for g, n in enumerate(counts):
        idx[g, :n] = np.sort(rng.choice(10**6, size=n, replace=False))
        m = rng.choice(np.linspace(0.5, 2, 300), size=n)
        co[g, :n] = np.where(rng.random(n) < 0.5, m + 0j, -1j * m)
    idx_d, co_d = _dev.upload(idx.ravel()), _dev.upload(co.ravel())
    cnt = torch.tensor(counts, device="cuda")
    for grid, s_tilde, theta in [(g, s, th) for g in (True, False)
                                 for s, th in ((2000, 0.9), (30_000, 0.0), (1, 1.99), (0, 0.0))]:
        kidx, kco, kc = _engine.topk(idx_d, co_d, cnt, G, cap, theta, s_tilde, grid=grid)
        kc = _dev.download(kc)
        ki, kk = _dev.download(kidx), _dev.download(kco)
        for g, n in enumerate(counts):
            want_i, want_c = oracle_lib.topk_filter(idx[g, :n], co[g, :n], s_tilde, theta)
            assert kc[g] == len(want_i)
            assert np.array_equal(ki[g * cap: g * cap + kc[g]], want_i)
            assert np.array_equal(kk[g * cap: g * cap + kc[g]], want_c)


@pytest.mark.parametrize("Ms", [(211, 223, 227, 229, 233), (97, 101, 103, 107)])
def test_distinct_lattice_sizes_vs_oracle(cuda, oracle_lib, Ms):
    """Configurations whose lattices have different sizes (the reference's
    numpy path, detect.py:134-145): hits by hypot, np.median coefficients."""
    pkg, port = cuda, oracle_lib
    rng = np.random.default_rng(len(Ms))
    d = 3
    gamma = np.unique(rng.integers(-20, 21, size=(3000, d)), axis=0)
    S = pkg.FreqSet(d, gamma, _sorted=True)
    sup = np.sort(rng.choice(len(gamma), size=15, replace=False))
    p = pkg.SparsePoly(S.take(sup), rng.normal(size=15) + 1j * rng.normal(size=15))
    zmat = np.vstack([rng.integers(0, M, size=d) for M in Ms])
    cfg = pkg.MultiLatticeConfig([pkg.Rank1Lattice(z, M) for z, M in zip(zmat, Ms)], 0.5, 10.33,
                                 0.5)
    assert cfg.shared_M is None
    orc = pkg.oracle_from_poly(p)
    smp = [orc.sample_lattice(lat) for lat in cfg.lattices]
    fr = pkg.detect_frequencies(smp, cfg, S)
    theta0 = fr.theta_zero
    hits, med, thr = port.gather_mixed(smp, Ms, zmat, gamma, theta0, 0.5, len(Ms) % 2 == 1)
    assert np.array_equal(fr.hits, hits)
    assert np.array_equal(fr.detected_idx, np.flatnonzero(hits >= thr))
    if len(Ms) % 2 == 1:
        res = pkg.detect_and_compute(smp, cfg, S)
        idx = np.flatnonzero(hits >= thr)
        assert np.array_equal(res.detected_idx, idx)
        assert np.max(np.abs(res.coeffs - med[idx]), initial=0.0) < 1e-12


def test_streamed_upload_matches_resident(cuda, monkeypatch):
    """Host-resident candidate sets above the streaming threshold are uploaded
    in chunks overlapped with hashing; results equal the resident path."""
    import paper_2006_13053_b200.detect as det

    pkg = cuda
    rng = np.random.default_rng(21)
    d, n = 6, 300_000
    gamma = np.unique(rng.integers(-500, 501, size=(n, d)), axis=0)
    sup = np.sort(rng.choice(len(gamma), size=200, replace=False))
    S_dev = pkg.FreqSet(d, gamma, _sorted=True)
    S_dev.device()
    p = pkg.SparsePoly(S_dev.take(sup), rng.normal(size=200) + 1j * rng.normal(size=200) + 2)
    cfg = pkg.draw_config(S_dev, 200, 0.1, rng=np.random.default_rng(3))
    smp = [pkg.oracle_from_poly(p).sample_lattice(lat) for lat in cfg.lattices]
    want = pkg.detect_and_compute(smp, cfg, S_dev)
    monkeypatch.setattr(det, "STREAM_UPLOAD_BYTES", 1 << 20)
    from paper_2006_13053_b200 import _engine
    monkeypatch.setattr(_engine.gather_streamed, "__defaults__",
                        (True, False, 1 << 15))  # many chunks
    S_host = pkg.FreqSet(d, gamma, _sorted=True)
    got = pkg.detect_and_compute(smp, cfg, S_host)
    assert S_host._dev is not None  # cached by the streamed path
    assert np.array_equal(got.hits, want.hits)
    assert np.array_equal(got.detected_idx, want.detected_idx)
    assert np.array_equal(got.coeffs, want.coeffs)
    assert np.array_equal(got.detected_idx, sup)


@pytest.mark.parametrize("L", [129, 131, 201])
def test_more_than_128_lattices_numpy_semantics(cuda, oracle_lib, L):
    """L > _MAX_COMPILED_L (=128): the reference dispatcher takes its numpy
    fallback (_kernels/__init__.py:62, fallback.py:106-131) -- hits by
    np.abs (hypot) > theta, np.median of the real and imaginary parts.  The
    plugin and detect_and_compute follow it (oracle: port.gather_mixed)."""
    pkg, port = cuda, oracle_lib
    rng = np.random.default_rng(L)
    M, d, n = 211, 4, 5000
    elems = workloads.rows_from_box(d, -40, 40, n, rng)
    zmat = rng.integers(0, M, size=(L, d))
    ghat = rng.standard_normal((L, M)) + 1j * rng.standard_normal((L, M))
    ghat[:, rng.random(M) < 0.45] = 0.0
    theta = 0.5
    hits, med = pkg._kernels.detect_gather(elems % M, zmat, M, ghat, theta, L / 2, True)
    # fallback semantics restated
    vals = np.stack([ghat[l][port.residues(elems, zmat[l], M)] for l in range(L)], axis=1)
    want_hits = np.sum(np.abs(vals) > theta, axis=1)
    det = want_hits >= L / 2
    want_med = np.zeros(n, np.complex128)
    want_med[det] = np.median(vals[det].real, axis=1) + 1j * np.median(vals[det].imag, axis=1)
    assert np.array_equal(hits, want_hits)
    assert det.any()
    assert np.array_equal(med, want_med)
    # the public entry point on a shared-M configuration with L lattices
    cfg = _config(pkg, zmat, M)
    samples = [np.fft.ifft(g) * M for g in ghat]
    S = pkg.FreqSet(d, elems, _sorted=True)
    res = pkg.detect_and_compute(samples, cfg, S)
    h2, _, _ = port.gather_mixed(samples, [M] * L, zmat, elems, res.theta_zero, 0.5, True)
    assert np.array_equal(res.hits, h2)


def test_noisy_fixed_gamma_vs_reference(cuda):
    """Noisy samples on 2 x 10^4 candidates (tests/golden/fixed_noisy.npz, the
    reference's own run): every candidate detected, so detect_topk truncates
    and postprocess_r1l refines crowded residues.  Hits bit-exact (sha256),
    detected / kept indices exact, coefficients within 1e-10."""
    import hashlib

    pkg = cuda
    g = golden("fixed_noisy.npz")
    rng = np.random.default_rng(4242)
    gamma = workloads.rows_from_box(5, -20, 20, 20_000, rng)
    assert hashlib.sha256(np.ascontiguousarray(gamma).tobytes()).hexdigest()[:16] == \
        str(g["gamma_digest"])
    G = pkg.FreqSet(5, gamma, _sorted=True)
    cfg = _config(pkg, g["zmat"], int(g["M"]))
    smp = list(g["samples"])
    res = pkg.detect_and_compute(smp, cfg, G)
    assert hashlib.sha256(np.ascontiguousarray(res.hits, dtype=np.int64).tobytes()).hexdigest() \
        == str(g["hits_sha256"])
    assert np.array_equal(res.detected_idx, g["idx"])
    assert np.max(np.abs(res.coeffs - g["coeffs"])) <= 1e-10 * np.max(np.abs(g["coeffs"]))
    top = pkg.detect_topk(smp, cfg, G, 40, 0.5)
    assert np.array_equal(top.detected_idx, g["topk_idx"])  # no exact ties here: exact
    assert np.max(np.abs(top.coeffs - g["topk_coeffs"])) <= 1e-10 * np.max(np.abs(g["topk_coeffs"]))
    post = pkg.postprocess_r1l(res, smp, cfg)
    assert np.array_equal(post.detected_idx, g["post_idx"])
    assert np.max(np.abs(post.coeffs - g["post_coeffs"])) <= 1e-10 * np.max(np.abs(g["post_coeffs"]))
    fr = pkg.detect_frequencies(smp, cfg, G)
    assert np.array_equal(fr.detected_idx, g["freq_idx"])
