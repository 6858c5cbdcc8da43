"""Dimension-incremental driver on the GPU vs the reference's golden runs."""

import numpy as np
import pytest

import workloads
from conftest import golden

pytestmark = pytest.mark.gpu


def _run(pkg, g):
    d, lo, hi, s, r, theta, delta, sseed, sigma, nseed = g["params"]
    d = int(d)
    p = pkg.SparsePoly(pkg.FreqSet(d, g["true_support"], _sorted=True), g["true_coeffs"])
    orc = pkg.oracle_from_poly(p, noise_sigma=float(sigma), noise_seed=int(nseed))
    res = pkg.sfft(orc, pkg.Box(d, int(lo), int(hi)),
                   pkg.SfftParams(int(s), float(delta), theta=float(theta), r=int(r)),
                   seed=int(sseed))
    return res, orc


def _check(res, orc, g, tol):
    assert np.array_equal(res.support.elems, g["support"])
    assert res.sample_count == int(g["sample_count"]) == orc.count
    flat = [[e["stage"], str(e["t"]), str(e["i"]), str(e["candidates"]), str(e["kept"]),
             str(e["samples"])] for e in res.stage_log]
    assert flat == g["stage_log"].tolist()
    if len(res.coeffs):
        assert np.linalg.norm(res.coeffs - g["coeffs"]) <= tol * np.linalg.norm(g["coeffs"])


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6, 8])
def test_sfft_small_vs_reference(cuda, seed):
    g = golden(f"sfft_small_{seed}.npz")
    res, orc = _run(cuda, g)
    _check(res, orc, g, 1e-10)


def test_sfft_cfg2_vs_reference(cuda):
    g = golden("sfft_cfg2.npz")
    res, orc = _run(cuda, g)
    _check(res, orc, g, 1e-10)
    w = workloads.config2()
    assert np.array_equal(res.support.elems, w.support)
    assert workloads.rel_l2(res.coeffs, w.coeffs) < 1e-12


def test_zero_signal_returns_empty(cuda):
    pkg = cuda
    orc = pkg.SamplingOracle(lambda X: np.zeros(len(X), dtype=complex), 3)
    res = pkg.sfft(orc, pkg.Box(3, -4, 4), pkg.SfftParams(4, 0.9, r=1), seed=0)
    assert res.failed and res.sample_count == orc.count and res.stage_log


def test_blackbox_oracle_matches_poly_oracle(cuda):
    """A black-box fn oracle (host evaluation) gives the same result."""
    pkg = cuda
    g = golden("sfft_small_5.npz")
    d = int(g["params"][0])
    p = pkg.SparsePoly(pkg.FreqSet(d, g["true_support"], _sorted=True), g["true_coeffs"])
    orc = pkg.SamplingOracle(lambda X: pkg.evaluate_many(p, X), d)
    res = pkg.sfft(orc, pkg.Box(d, int(g["params"][1]), int(g["params"][2])),
                   pkg.SfftParams(int(g["params"][3]), float(g["params"][6]),
                                  theta=float(g["params"][5]), r=int(g["params"][4])),
                   seed=int(g["params"][7]))
    _check(res, orc, g, 1e-10)


def test_candidate_set_restriction(cuda):
    pkg = cuda
    rng = np.random.default_rng(20240611)
    gamma = pkg.hyperbolic_cross(3, 6)
    I = pkg.random_subset(gamma, 5, rng)
    p = pkg.random_poly(I, rng, min_mag=0.1)
    res = pkg.sfft(pkg.oracle_from_poly(p), gamma, pkg.SfftParams(5, 0.9, r=2), seed=8)
    assert np.all(gamma.contains_rows(res.support.elems))
    assert res.support == I


def test_seed_reproducibility_bitwise(cuda):
    pkg = cuda
    w = workloads.small_sfft(12, 4, 8, 30, r=2)
    runs = []
    for _ in range(2):
        p = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
        runs.append(pkg.sfft(pkg.oracle_from_poly(p), pkg.Box(w.d, w.lo, w.hi),
                             pkg.SfftParams(w.s, 0.9, r=w.r), seed=555))
    assert runs[0].support == runs[1].support
    assert np.array_equal(runs[0].coeffs, runs[1].coeffs)
    assert runs[0].sample_count == runs[1].sample_count


@pytest.mark.parametrize("sigma", [0.0, 1e-3])
def test_sfft_fused_path_vs_oracle(cuda, oracle_lib, sigma):
    """A stage size on the fused sampler->detection path (M = 9311) against
    the oracle's structured sfft with the same harness noise."""
    pkg = cuda
    w = workloads.small_sfft(31, 4, 8, 450, r=1, sigma=sigma, decaying=sigma > 0,
                             theta=1e-6 if sigma else 1e-12)
    p = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
    orc = pkg.oracle_from_poly(p, noise_sigma=w.sigma, noise_seed=w.noise_seed)
    res = pkg.sfft(orc, pkg.Box(w.d, w.lo, w.hi),
                   pkg.SfftParams(w.s, 0.9, theta=w.theta, r=w.r), seed=w.seed)
    ref = oracle_lib.sfft(oracle_lib.PolyOracle(w.support, w.coeffs, mode="structured",
                                                sigma=w.sigma, noise_seed=w.noise_seed),
                          oracle_lib.Box(w.d, w.lo, w.hi), w.s, 0.9, w.seed, theta=w.theta,
                          r=w.r)
    assert any(e["samples"] % 9311 == 0 for e in res.stage_log)  # fused size exercised
    assert np.array_equal(res.support.elems, ref[0])
    assert res.sample_count == ref[2]
    assert [(e["candidates"], e["kept"]) for e in res.stage_log] == \
        [(e["candidates"], e["kept"]) for e in ref[3]]
    assert workloads.rel_l2(res.coeffs, ref[1]) < 1e-10


@pytest.mark.parametrize("name", ["metric_config", "config5"])
def test_spectra_ahead_modes_bitwise(cuda, monkeypatch, name):
    """Stage spectra enqueued ahead of the previous stage's counts (hit, and
    forced miss -> whole-stage fallback) give bit-identical results to the
    in-order stage calls, noisy oracle included (harness call numbers)."""
    from paper_2006_13053_b200 import dimincr

    w = getattr(workloads, name)()
    p = cuda.SparsePoly(cuda.FreqSet(w.d, w.support, _sorted=True), w.coeffs)

    def run():
        orc = cuda.oracle_from_poly(p, noise_sigma=w.sigma, noise_seed=w.noise_seed)
        return cuda.sfft(orc, cuda.Box(w.d, w.lo, w.hi),
                         cuda.SfftParams(w.s, w.delta, theta=w.theta, r=w.r), seed=w.seed)

    outs = []
    for ahead, bias in ((False, 0), (True, 0), (True, -2)):
        monkeypatch.setattr(dimincr, "_SPECTRA_AHEAD", ahead)
        monkeypatch.setattr(dimincr, "_SPEC_L_BIAS", bias)
        outs.append(run())
    base = outs[0]
    for o in outs[1:]:
        assert np.array_equal(o.support.elems, base.support.elems)
        assert np.array_equal(o.coeffs, base.coeffs)
        assert o.sample_count == base.sample_count
        assert o.stage_log == base.stage_log


@pytest.mark.parametrize("d,r,sigma", [(2, 3, 0.0), (3, 2, 0.0), (3, 2, 1e-3), (5, 3, 0.0)])
def test_sfft_few_dims_vs_oracle(cuda, oracle_lib, d, r, sigma):
    """Few coordinate stages: the stage plans enqueued ahead reach the final
    coefficient stage already at start-up (d <= the number of slots)."""
    pkg = cuda
    w = workloads.small_sfft(40 + d, d, 12, 60, r=r, sigma=sigma,
                             theta=1e-6 if sigma else 1e-12)
    p = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
    orc = pkg.oracle_from_poly(p, noise_sigma=w.sigma, noise_seed=w.noise_seed)
    res = pkg.sfft(orc, pkg.Box(w.d, w.lo, w.hi),
                   pkg.SfftParams(w.s, 0.9, theta=w.theta, r=w.r), seed=w.seed)
    ref = oracle_lib.sfft(oracle_lib.PolyOracle(w.support, w.coeffs, mode="structured",
                                                sigma=w.sigma, noise_seed=w.noise_seed),
                          oracle_lib.Box(w.d, w.lo, w.hi), w.s, 0.9, w.seed, theta=w.theta,
                          r=w.r)
    assert np.array_equal(res.support.elems, ref[0])
    assert res.sample_count == ref[2]
    assert [(e["candidates"], e["kept"], e["samples"]) for e in res.stage_log] == \
        [(e["candidates"], e["kept"], e["samples"]) for e in ref[3]]
    assert workloads.rel_l2(res.coeffs, ref[1]) < 1e-10
    if sigma == 0:
        order = np.lexsort(w.support.T[::-1])
        assert np.array_equal(res.support.elems, w.support[order])


@pytest.mark.parametrize("d,N,n,s", [(6, 16, 200_000, 30), (7, 12, 120_000, 20)])
def test_sfft_freqset_gamma_vs_oracle(cuda, oracle_lib, d, N, n, s):
    """sfft over an explicit candidate set (a FreqSet, not a Box): every
    pairing stage filters by the prefix projection P_{0..t}(Gamma)
    (dimincr.py:155-175, freqset.py:139-142) on the device.  Supports, sample
    counts and stage logs identical to the oracle's; coefficients 1e-10."""
    pkg, port = cuda, oracle_lib
    rng = np.random.default_rng(1000 + d)
    gamma = workloads.rows_from_box(d, -N, N, n, rng)
    idx = np.sort(rng.choice(gamma.shape[0], size=s, replace=False))
    sup = gamma[idx]
    co = workloads.mag_phase_coeffs(s, rng)
    G = pkg.FreqSet(d, gamma, _sorted=True)
    p = pkg.SparsePoly(pkg.FreqSet(d, sup, _sorted=True), co)
    res = pkg.sfft(pkg.oracle_from_poly(p), G, pkg.SfftParams(s, 0.9, r=2), seed=11)
    ref = port.sfft(port.PolyOracle(sup, co, mode="structured"), gamma, s, 0.9, 11, r=2)
    assert np.array_equal(res.support.elems, ref[0])
    assert np.array_equal(res.support.elems, sup)
    assert res.sample_count == ref[2]
    got = [(e["stage"], e["t"], e["i"], e["candidates"], e["kept"], e["samples"])
           for e in res.stage_log]
    want = [(e["stage"], e["t"], e["i"], e["candidates"], e["kept"], e["samples"])
            for e in ref[3]]
    assert got == want
    assert workloads.rel_l2(res.coeffs, ref[1]) <= 1e-10
    # and against the reference's own run of the same instance
    g = golden("sfft_freqset.npz")
    key = f"d{d}"
    assert np.array_equal(res.support.elems, g[key + "_support"])
    assert res.sample_count == int(g[key + "_count"])
    flat = [[e["stage"], str(e["t"]), str(e["i"]), str(e["candidates"]), str(e["kept"]),
             str(e["samples"])] for e in res.stage_log]
    assert flat == g[key + "_log"].tolist()
    assert workloads.rel_l2(res.coeffs, g[key + "_coeffs"]) <= 1e-10


def test_sfft_hyperbolic_cross_vs_reference(cuda):
    """sfft over a hyperbolic cross (hc_enumerate, freqset.py:222-245) against
    the reference's own run: the candidate set, supports, sample counts,
    stage logs and coefficients."""
    import hashlib

    pkg = cuda
    g = golden("sfft_freqset.npz")
    G = pkg.hyperbolic_cross(4, 40)
    gamma = np.ascontiguousarray(G.elems)
    assert hashlib.sha256(gamma.tobytes()).hexdigest()[:16] == str(g["hc_gamma_digest"])
    rng = np.random.default_rng(77)
    idx = np.sort(rng.choice(gamma.shape[0], size=16, replace=False))
    sup = gamma[idx]
    co = workloads.mag_phase_coeffs(16, rng)
    p = pkg.SparsePoly(pkg.FreqSet(4, sup, _sorted=True), co)
    res = pkg.sfft(pkg.oracle_from_poly(p), G, pkg.SfftParams(16, 0.9, r=2), seed=5)
    assert np.array_equal(res.support.elems, g["hc_support"])
    assert res.sample_count == int(g["hc_count"])
    flat = [[e["stage"], str(e["t"]), str(e["i"]), str(e["candidates"]), str(e["kept"]),
             str(e["samples"])] for e in res.stage_log]
    assert flat == g["hc_log"].tolist()
    assert workloads.rel_l2(res.coeffs, g["hc_coeffs"]) <= 1e-10
