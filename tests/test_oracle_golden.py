"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The golden fixtures were produced by running the reference (latfft 0.1.0,
compiled Cython core) in the build container -- see
tests/golden/make_golden.py.  Passing here is what licenses using the oracle
as the checker of the CUDA path in the -m gpu tests.
"""

import numpy as np
import pytest

import workloads
from conftest import golden


def test_gather_bitexact_vs_reference(oracle_lib):
    g = golden("gather_cases.npz")
    for k in range(int(g["ncases"])):
        M, theta, thr = g[f"c{k}_params"]
        e, z, gh = g[f"c{k}_elems"], g[f"c{k}_zmat"], g[f"c{k}_ghat"]
        for wm in (0, 1):
            key = f"c{k}_{wm}_hits"
            if key not in g:
                continue
            hits, med = oracle_lib.gather_c(e, z, int(M), gh, theta, thr, bool(wm))
            assert np.array_equal(hits, g[key])
            assert np.array_equal(med.view(np.float64), g[f"c{k}_{wm}_med"].view(np.float64))


def test_injectivity_vs_reference(oracle_lib):
    for case in golden("injective_cases.json"):
        e = np.array(case["elems"], dtype=np.int64)
        assert oracle_lib.rows_injective_mod(e, case["p"]) == case["injective"]


def test_host_lattice_construction_vs_reference(oracle_lib):
    lc = golden("lattice_cases.json")
    for x, p in lc["next_prime_above"].items():
        assert oracle_lib.next_prime_above(float(x)) == p
    for n, isp in lc["is_prime"].items():
        assert oracle_lib.is_prime(int(n)) == isp
    for n, delta, ls, L in lc["required_L"]:
        assert oracle_lib.required_L(n, delta, L_scale=ls) == L
    for case in lc["draw_config"]:
        rng = np.random.default_rng(case["seed"])
        S = oracle_lib.random_rows_from_box(3, -40, 40, 300, rng)
        M, z = oracle_lib.draw_config(S, 20 + case["seed"], 0.2, rng)
        assert M == case["M"] and z.shape[0] == case["L"]
        assert np.array_equal(z, np.array(case["z"]))


def test_dft_vs_reference(oracle_lib):
    g = golden("dft_cases.npz")
    for M in g["primes"]:
        y = oracle_lib.dft_normalized(g[f"x{M}"])
        assert np.max(np.abs(y - g[f"y{M}"])) < 1e-13


def test_structured_sampling_vs_reference(oracle_lib):
    g = golden("sampling_cases.npz")
    for k in range(int(g["n"])):
        vals = oracle_lib.sample_lattice_structured(g[f"s{k}_support"], g[f"s{k}_coeffs"],
                                                    g[f"s{k}_z"], int(g[f"s{k}_M"]))
        assert np.array_equal(vals, g[f"s{k}_fast"])
        dense = g[f"s{k}_dense"]
        assert np.max(np.abs(vals - dense)) < 1e-12 * max(1.0, np.max(np.abs(dense)))


def test_tiny_detect_vs_reference(oracle_lib):
    g = golden("tiny_detect.npz")
    for k in range(int(g["n"])):
        p = f"t{k}_"
        S, z, M, smp = g[p + "gamma"], g[p + "zmat"], int(g[p + "M"]), list(g[p + "samples"])
        hits, idx, co, th = oracle_lib.detect_and_compute(smp, M, z, S)
        assert th == float(g[p + "theta0"])
        assert np.array_equal(hits, g[p + "hits"]) and np.array_equal(idx, g[p + "idx"])
        assert np.array_equal(co, g[p + "coeffs"])
        hits0, idx0, co0, _ = oracle_lib.detect_and_compute(smp, M, z, S, theta0=1e-8)
        assert np.array_equal(hits0, g[p + "hits0"]) and np.array_equal(idx0, g[p + "idx0"])
        assert np.array_equal(co0, g[p + "coeffs0"])
        _, tidx, tco, _ = oracle_lib.detect_topk(smp, M, z, S, 2, 0.1)
        assert np.array_equal(tidx, g[p + "topk_idx"]) and np.array_equal(tco, g[p + "topk_coeffs"])
        _, fidx, _ = oracle_lib.detect_frequencies(smp, M, z, S)
        assert np.array_equal(fidx, g[p + "freq_idx"])
        pidx, pco = oracle_lib.postprocess_r1l(S[idx], co, idx, smp, M, z, th)
        assert np.array_equal(pidx, g[p + "post_idx"])
        assert np.allclose(pco, g[p + "post_coeffs"], rtol=0, atol=1e-14)


def test_config1_vs_reference(oracle_lib):
    g = golden("cfg1.npz")
    w = workloads.config1()
    import hashlib

    assert hashlib.sha256(w.gamma.tobytes()).hexdigest()[:16] == str(g["gamma_digest"])
    smp = list(g["samples"])
    # the harness regenerates the reference's samples with the structured sampler
    for zl, s in zip(g["zmat"], smp):
        mine = oracle_lib.sample_lattice_structured(w.gamma[w.support_idx], w.coeffs, zl,
                                                    int(g["M"]))
        assert np.array_equal(mine, s)
    hits, idx, co, th = oracle_lib.detect_and_compute(smp, int(g["M"]), g["zmat"], w.gamma)
    assert np.array_equal(hits, g["hits"]) and np.array_equal(idx, g["idx"])
    assert np.array_equal(co, g["coeffs"]) and th == float(g["theta0"])
    assert np.array_equal(idx, w.support_idx)
    assert np.max(np.abs(co - w.coeffs)) < 1e-12


def _check_sfft(res, g, coeff_tol):
    support, coeffs, count, log = res
    assert np.array_equal(support, g["support"])
    assert count == int(g["sample_count"])
    flat = [[e["stage"], str(e["t"]), str(e["i"]), str(e["candidates"]), str(e["kept"]),
             str(e["samples"])] for e in log]
    assert flat == g["stage_log"].tolist()
    if len(coeffs):
        rel = np.linalg.norm(coeffs - g["coeffs"]) / np.linalg.norm(g["coeffs"])
        assert rel <= coeff_tol


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 8])
def test_sfft_small_dense_vs_reference(oracle_lib, seed):
    g = golden(f"sfft_small_{seed}.npz")
    d, lo, hi, s, r, theta, delta, sseed, sigma, nseed = g["params"]
    orc = oracle_lib.PolyOracle(g["true_support"], g["true_coeffs"], mode="dense",
                                sigma=float(sigma), noise_seed=int(nseed))
    res = oracle_lib.sfft(orc, oracle_lib.Box(int(d), int(lo), int(hi)), int(s), float(delta),
                          int(sseed), theta=float(theta), r=int(r))
    _check_sfft(res, g, 1e-13)


@pytest.mark.parametrize("seed", [5, 6, 8])
def test_sfft_small_structured_vs_reference(oracle_lib, seed):
    """The structured sampler (what the GPU computes) gives the reference's
    supports, counts and logs, coefficients to roundoff."""
    g = golden(f"sfft_small_{seed}.npz")
    d, lo, hi, s, r, theta, delta, sseed, sigma, nseed = g["params"]
    orc = oracle_lib.PolyOracle(g["true_support"], g["true_coeffs"], mode="structured",
                                sigma=float(sigma), noise_seed=int(nseed))
    res = oracle_lib.sfft(orc, oracle_lib.Box(int(d), int(lo), int(hi)), int(s), float(delta),
                          int(sseed), theta=float(theta), r=int(r))
    _check_sfft(res, g, 1e-12)


def test_sfft_cfg2_structured_vs_reference(oracle_lib):
    g = golden("sfft_cfg2.npz")
    w = workloads.config2()
    assert np.array_equal(w.support, g["true_support"])
    orc = oracle_lib.PolyOracle(w.support, w.coeffs, mode="structured")
    res = oracle_lib.sfft(orc, oracle_lib.Box(w.d, w.lo, w.hi), w.s, w.delta, w.seed,
                          theta=w.theta, r=w.r)
    _check_sfft(res, g, 1e-12)
    assert np.array_equal(res[0], w.support)


@pytest.mark.parametrize("name", ["metric_config", "config3", "config5"])
def test_sfft_fullsize_structured_vs_reference(oracle_lib, name):
    """The metric instance (d=10, s=1000), config 3 (d=20, 76.5 M samples) and
    config 5 (noisy, top-k truncation at every stage) at full size: the
    oracle's sfft against the reference's own driver and detection run on
    the same structured samples (tests/golden/make_golden.py
    gen_sfft_fullsize).  Supports, sample counts and stage logs exact;
    coefficients to roundoff.  This pins the oracle the full-size GPU tests
    (tests/test_gpu_configs.py) compare against."""
    w = getattr(workloads, name)()
    g = golden(f"sfft_ref_{w.name}.npz")
    assert np.array_equal(w.support, g["true_support"])
    orc = oracle_lib.PolyOracle(w.support, w.coeffs, mode="structured", sigma=w.sigma,
                                noise_seed=w.noise_seed)
    res = oracle_lib.sfft(orc, oracle_lib.Box(w.d, w.lo, w.hi), w.s, w.delta, w.seed,
                          theta=w.theta, r=w.r, workers=8)
    _check_sfft(res, g, 1e-12)


@pytest.mark.parametrize("d,N,n,s", [(6, 16, 200_000, 30), (7, 12, 120_000, 20)])
def test_sfft_freqset_gamma_vs_reference(oracle_lib, d, N, n, s):
    """sfft over an explicit candidate set (FreqSet Gamma): the oracle against
    the reference's own run (tests/golden/sfft_freqset.npz)."""
    g = golden("sfft_freqset.npz")
    key = f"d{d}"
    rng = np.random.default_rng(1000 + d)
    gamma = workloads.rows_from_box(d, -N, N, n, rng)
    idx = np.sort(rng.choice(gamma.shape[0], size=s, replace=False))
    sup = gamma[idx]
    co = workloads.mag_phase_coeffs(s, rng)
    res = oracle_lib.sfft(oracle_lib.PolyOracle(sup, co, mode="structured"), gamma, s, 0.9, 11,
                          r=2)
    assert np.array_equal(res[0], g[key + "_support"])
    assert res[2] == int(g[key + "_count"])
    flat = [[e["stage"], str(e["t"]), str(e["i"]), str(e["candidates"]), str(e["kept"]),
             str(e["samples"])] for e in res[3]]
    assert flat == g[key + "_log"].tolist()
    assert workloads.rel_l2(res[1], g[key + "_coeffs"]) <= 1e-12


def test_fixed_noisy_vs_reference(oracle_lib):
    """The oracle on the reference's noisy fixed-Gamma run (every candidate
    detected; top-s truncation; R1L refinement on crowded residues)."""
    import hashlib

    g = golden("fixed_noisy.npz")
    rng = np.random.default_rng(4242)
    gamma = workloads.rows_from_box(5, -20, 20, 20_000, rng)
    M, z, smp = int(g["M"]), g["zmat"], list(g["samples"])
    hits, idx, co, th = oracle_lib.detect_and_compute(smp, M, z, gamma)
    assert hashlib.sha256(np.ascontiguousarray(hits).tobytes()).hexdigest() == \
        str(g["hits_sha256"])
    assert np.array_equal(idx, g["idx"]) and np.array_equal(co, g["coeffs"])
    assert th == float(g["theta0"])
    _, ti, tc, _ = oracle_lib.detect_topk(smp, M, z, gamma, 40, 0.5)
    assert np.array_equal(ti, g["topk_idx"]) and np.array_equal(tc, g["topk_coeffs"])
    pi, pc = oracle_lib.postprocess_r1l(gamma[idx], co, idx, smp, M, z, th)
    assert np.array_equal(pi, g["post_idx"])
    assert np.max(np.abs(pc - g["post_coeffs"])) <= 1e-13 * np.max(np.abs(g["post_coeffs"]))
