"""Generate the golden fixtures in tests/golden/ by running the REFERENCE.

Run in the build container (needs /root/reference and ``make -C oracle ref``):

    python tests/golden/make_golden.py            # all fixtures
    python tests/golden/make_golden.py sfft_cfg2  # one fixture

The reference (latfft 0.1.0, /root/reference/pkg/src) is imported with its
compiled Cython core (BACKEND == "compiled").  Every fixture records the
inputs (or the seeds that regenerate them through workloads.py, with a
checksum of the regenerated arrays) and the reference's outputs.  The GPU box
never reads /root/reference; tests only read these files.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from oracle import port  # noqa: E402
from oracle.refload import import_reference  # noqa: E402

lf = import_reference()
from latfft import _kernels as rk  # noqa: E402
from latfft import detect as rdetect  # noqa: E402
from latfft import dimincr as rdim  # noqa: E402
from latfft import freqset as rfs  # noqa: E402
from latfft import lattice as rlat  # noqa: E402
from latfft import polyeval as rpe  # noqa: E402


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest()[:16]


def save_npz(name, **arrs):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def save_json(name, obj):
    path = os.path.join(HERE, name + ".json")
    with open(path, "w") as fh:
        json.dump(obj, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {path} ({os.path.getsize(path)} B)")


# ---------------------------------------------------------------------------

def gen_gather():
    """detect_gather on random inputs (test_kernels.py:43-57 recipe, scaled)."""
    rng = np.random.default_rng(4242)
    out = {}
    cases = [(300, 3, 31, 7, 0.6, 1e-9, 3.5), (2000, 5, 211, 27, 0.7, 1e-9, 13.5),
             (1500, 10, 2069, 31, 0.9, 1e-6, 15.5), (777, 1, 13, 1, 0.3, 0.0, 0.5),
             (4000, 20, 211, 47, 0.9, 1e-9, 23.5), (0, 4, 17, 5, 0.5, 1e-9, 2.5),
             (900, 2, 2069, 9, 0.5, 0.25, 4.5)]
    for k, (n, d, M, L, zfrac, theta, thr) in enumerate(cases):
        elems = rng.integers(0, M, size=(n, d), dtype=np.int64)
        zmat = rng.integers(0, M, size=(L, d), dtype=np.int64)
        ghat = rng.normal(size=(L, M)) + 1j * rng.normal(size=(L, M))
        ghat[rng.random(size=(L, M)) < zfrac] = 0.0
        if k == 6:  # values sitting exactly on the threshold: '>' not '>='
            ghat[:, ::3] = theta
        for wm in (False, True):
            if wm and L % 2 == 0:
                continue
            hits, med = rk.detect_gather(elems, zmat, M, ghat, theta, thr, wm)
            out[f"c{k}_{int(wm)}_hits"] = hits
            out[f"c{k}_{int(wm)}_med"] = med
        out[f"c{k}_elems"] = elems
        out[f"c{k}_zmat"] = zmat
        out[f"c{k}_ghat"] = ghat
        out[f"c{k}_params"] = np.array([M, theta, thr])
    out["ncases"] = np.array(len(cases))
    save_npz("gather_cases", **out)


def gen_injective():
    rng = np.random.default_rng(99)
    cases = []
    for _ in range(40):
        n = int(rng.integers(2, 200))
        d = int(rng.integers(1, 6))
        elems = rng.integers(-100, 100, size=(n, d))
        p = int(rng.integers(2, 60))
        cases.append({"elems": elems.tolist(), "p": p,
                      "injective": bool(rk.rows_injective_mod(elems, p))})
    wide = np.arange(20, dtype=np.int64).reshape(2, 10)
    cases.append({"elems": wide.tolist(), "p": 10**7,
                  "injective": bool(rk.rows_injective_mod(wide, 10**7))})
    st = np.vstack([wide, wide])
    cases.append({"elems": st.tolist(), "p": 10**7,
                  "injective": bool(rk.rows_injective_mod(st, 10**7))})
    cases.append({"elems": [[0], [5]], "p": 5,
                  "injective": bool(rk.rows_injective_mod(np.array([[0], [5]]), 5))})
    save_json("injective_cases", cases)


def gen_hc():
    rng = np.random.default_rng(7)
    cases = []
    for _ in range(8):
        d = int(rng.integers(1, 5))
        N = int(rng.integers(2, 12))
        w = rng.uniform(0.4, 2.5, size=d)
        cases.append({"d": d, "N": N, "w": w.tolist(),
                      "count": int(rk.hc_count(d, float(N), w)),
                      "rows": rk.hc_enumerate(d, float(N), w).tolist()})
    cases.append({"d": 3, "N": 4, "w": [1.0, 1.0, 1.0],
                  "count": int(rk.hc_count(3, 4.0, np.ones(3))),
                  "rows": rk.hc_enumerate(3, 4.0, np.ones(3)).tolist()})
    save_json("hc_cases", cases)


def gen_lattice():
    """Host lattice construction: primes, required_L, draw_config RNG."""
    obj = {"next_prime_above": {}, "required_L": [], "draw_config": [],
           "is_prime": {}}
    for x in (0, 1, 2, 3.5, 10.33 * 20, 10.33 * 200, 10.33 * 2000, 10.33 * 1e4,
              10.33 * 1000, 10.33 * 1069, 10**9 + 0.5):
        obj["next_prime_above"][repr(float(x))] = rlat.next_prime_above(x)
    for n in (1, 2, 3, 561, 7919, 1_000_003, 2**61 - 1, 2**62 - 57, 3215031751):
        obj["is_prime"][str(n)] = rlat.is_prime(n)
    for n in (1, 8, 500, 2450, 4225, 16641, 129_000, 10_000, 1 << 26, 10**7):
        for delta in (0.9, 0.1, 0.006, 0.0066666, 0.03, 1e-3):
            for ls in (1.0, 0.25):
                obj["required_L"].append([n, delta, ls, rlat.required_L(n, delta, L_scale=ls)])
    for seed in range(6):
        rng = np.random.default_rng(seed)
        S = rfs.random_subset(rfs.Box(3, -40, 40), 300, rng)
        cfg = rlat.draw_config(S, 20 + seed, 0.2, rng=rng)
        obj["draw_config"].append({"seed": seed, "S_digest": digest(S.elems),
                                   "M": cfg.shared_M, "L": cfg.L,
                                   "z": [lat.z.tolist() for lat in cfg.lattices]})
    save_json("lattice_cases", obj)


def gen_dft():
    rng = np.random.default_rng(606)
    out = {}
    primes = [2, 3, 5, 31, 101, 127, 211, 509, 1009, 1039, 2069]
    for M in primes:
        x = rng.normal(size=M) + 1j * rng.normal(size=M)
        out[f"x{M}"] = x
        out[f"y{M}"] = lf.dft_forward_normalized(x)
    out["primes"] = np.array(primes)
    save_npz("dft_cases", **out)


def gen_sampling():
    """evaluate_on_lattice / pointwise sampling (polyeval.py:78-87)."""
    rng = np.random.default_rng(31)
    out = {}
    for k in range(6):
        d = int(rng.integers(1, 5))
        M = int(rng.choice([7, 13, 31, 211, 2069]))
        I = rfs.random_subset(rfs.Box(d, -6, 6), int(rng.integers(1, 12)), rng)
        p = rpe.random_poly(I, rng)
        lat = rlat.Rank1Lattice(rng.integers(0, M, d), M)
        out[f"s{k}_support"] = I.elems
        out[f"s{k}_coeffs"] = p.coeffs
        out[f"s{k}_z"] = lat.z
        out[f"s{k}_M"] = np.array(M)
        out[f"s{k}_fast"] = rpe.evaluate_on_lattice(p, lat)
        out[f"s{k}_dense"] = rpe.evaluate_many(p, rlat.lattice_nodes(lat))
    out["n"] = np.array(6)
    save_npz("sampling_cases", **out)


def gen_tiny_detect():
    """40 tiny alias instances (test_detect.py:27-55 recipe)."""
    rng = np.random.default_rng(20240611)
    out = {}
    for k in range(40):
        d = int(rng.integers(1, 4))
        M = int(rng.choice([7, 11, 13, 17, 19, 23, 29, 31]))
        L = int(rng.choice([3, 5, 7]))
        box = rfs.Box(d, -5, 5)
        gamma = rfs.random_subset(box, int(rng.integers(4, min(25, box.size + 1))), rng)
        I = rfs.random_subset(gamma, int(rng.integers(1, min(9, len(gamma) + 1))), rng)
        p = rpe.random_poly(I, rng, min_mag=0.05)
        lats = [rlat.Rank1Lattice(rng.integers(0, M, d), M) for _ in range(L)]
        config = rlat.MultiLatticeConfig(lats, 0.5, 10.33, 0.5)
        samples = np.array([rpe.evaluate_on_lattice(p, lat) for lat in lats])
        res = rdetect.detect_and_compute(list(samples), config, gamma)
        res0 = rdetect.detect_and_compute(list(samples), config, gamma,
                                          zero=rdetect.ZeroTest(1e-8))
        post = rdetect.postprocess_r1l(res, list(samples), config)
        topk = rdetect.detect_topk(list(samples), config, gamma, 2, 0.1)
        freq = rdetect.detect_frequencies(list(samples), config, gamma)
        pre = f"t{k}_"
        out[pre + "gamma"] = gamma.elems
        out[pre + "zmat"] = np.vstack([lat.z for lat in lats])
        out[pre + "M"] = np.array(M)
        out[pre + "samples"] = samples
        out[pre + "hits"] = res.hits
        out[pre + "idx"] = res.detected_idx
        out[pre + "coeffs"] = res.coeffs
        out[pre + "theta0"] = np.array(res.theta_zero)
        out[pre + "hits0"] = res0.hits
        out[pre + "idx0"] = res0.detected_idx
        out[pre + "coeffs0"] = res0.coeffs
        out[pre + "post_idx"] = post.detected_idx
        out[pre + "post_coeffs"] = post.coeffs
        out[pre + "topk_idx"] = topk.detected_idx
        out[pre + "topk_coeffs"] = topk.coeffs
        out[pre + "freq_idx"] = freq.detected_idx
    out["n"] = np.array(40)
    save_npz("tiny_detect", **out)


def gen_cfg1():
    """Config 1 end to end: Gamma, samples, detect_* outputs."""
    w = workloads.config1()
    rng = np.random.default_rng(w.seed)
    G = rfs.random_subset(rfs.Box(w.d, -16, 16), 10_000, rng)
    assert np.array_equal(G.elems, w.gamma), "workloads generator != reference"
    I = rfs.random_subset(G, w.s, rng)
    assert np.array_equal(I.elems, w.gamma[w.support_idx])
    mags = rng.uniform(1, 10, w.s)
    ph = rng.uniform(0, 2 * np.pi, w.s)
    assert np.allclose(mags * np.exp(1j * ph), w.coeffs, rtol=0, atol=0)
    p = rpe.SparsePoly(I, mags * np.exp(1j * ph))
    cfg = rlat.draw_config(G, w.s, 0.1, rng=rng)
    oracle = rpe.oracle_from_poly(p)
    samples = [oracle.sample_lattice(lat) for lat in cfg.lattices]
    t0 = time.perf_counter()
    res = rdetect.detect_and_compute(samples, cfg, G)
    dt = time.perf_counter() - t0
    topk = rdetect.detect_topk(samples, cfg, G, 10, 1.0)
    post = rdetect.postprocess_r1l(res, samples, cfg)
    save_npz("cfg1", gamma_digest=np.array(digest(G.elems)), M=np.array(cfg.shared_M),
             zmat=np.vstack([lat.z for lat in cfg.lattices]),
             samples=np.array(samples), hits=res.hits, idx=res.detected_idx,
             coeffs=res.coeffs, theta0=np.array(res.theta_zero),
             topk_idx=topk.detected_idx, topk_coeffs=topk.coeffs,
             post_idx=post.detected_idx, post_coeffs=post.coeffs,
             ref_detect_seconds=np.array(dt))


class _NoisyFn:
    """Harness noise wrapped around the reference's evaluate_many."""

    def __init__(self, p, sigma, seed):
        self.p, self.sigma, self.seed, self.calls = p, sigma, seed, 0

    def __call__(self, X):
        vals = rpe.evaluate_many(self.p, X)
        if self.sigma > 0:
            vals = vals + port.noise_for_call(self.seed, self.calls, len(X), self.sigma)
        self.calls += 1
        return vals


class ClampedBox(rfs.Box):
    """len()-clamped Box: Box.__len__ overflows for cfg3."""

    def __len__(self):
        return min(self.size, sys.maxsize)


def run_ref_sfft(w, r=None, fast=False):
    I = rfs.FreqSet(w.d, w.support, _sorted=True)
    p = rpe.SparsePoly(I, w.coeffs)
    if w.sigma > 0:
        oracle = rpe.SamplingOracle(_NoisyFn(p, w.sigma, w.noise_seed), w.d)
    else:
        oracle = rpe.oracle_from_poly(p, fast_lattice=fast)
    params = rdim.SfftParams(w.s, w.delta, theta=w.theta, r=w.r if r is None else r)
    t0 = time.perf_counter()
    res = rdim.sfft(oracle, ClampedBox(w.d, w.lo, w.hi), params, seed=w.seed)
    dt = time.perf_counter() - t0
    return res, dt


def save_sfft(name, w, res, dt):
    log = [[e["stage"], e["t"], e["i"], e["candidates"], e["kept"], e["samples"]]
           for e in res.stage_log]
    save_npz(name, support=res.support.elems, coeffs=res.coeffs,
             sample_count=np.array(res.sample_count), stage_log=np.array(log, dtype=object).astype(str),
             true_support=w.support, true_coeffs=w.coeffs,
             params=np.array([w.d, w.lo, w.hi, w.s, w.r, w.theta, w.delta, w.seed,
                              w.sigma, w.noise_seed]),
             ref_seconds=np.array(dt))


def gen_sfft_small():
    """Several small sfft runs with the dense (as-shipped) reference oracle."""
    specs = [  # seed, d, N, n, s, r, theta, sigma, decaying
        (1, 1, 16, 3, 3, 1, 1e-12, 0.0, False),
        (2, 2, 5, 4, 4, 1, 1e-12, 0.0, False),
        (3, 3, 6, 12, 8, 1, 1e-9, 0.0, False),
        (4, 4, 8, 1, 1, 1, 1e-12, 0.0, False),
        (5, 5, 8, 40, 40, 2, 1e-12, 0.0, False),
        (6, 6, 16, 300, 60, 2, 1e-6, 1e-3, True),
        (8, 5, 16, 200, 200, 1, 1e-12, 0.0, False),
    ]
    for seed, d, N, n, s, r, theta, sigma, dec in specs:
        w = workloads.small_sfft(seed, d, N, n, s=s, r=r, theta=theta, sigma=sigma,
                                 decaying=dec, sfft_seed=100 + seed)
        res, dt = run_ref_sfft(w)
        save_sfft(f"sfft_small_{seed}", w, res, dt)


def gen_sfft_cfg2():
    w = workloads.config2()
    res, dt = run_ref_sfft(w)
    print(f"cfg2 reference sfft: {dt:.1f}s, {len(res.support)} found")
    save_sfft("sfft_cfg2", w, res, dt)


def _ref_analysis():
    from latfft import analysis as ran

    return ran


ANALYSIS_SPECS = {
    # reference tests/test_analysis.py desk_spec (redraw "both", tiny M)
    "desk": dict(name="unit", candidates={"kind": "random-box", "d": 2, "lo": -60, "hi": 60,
                                          "count": 400},
                 support={"kind": "random-subset", "count": 8}, L_values=[3, 9], trials=6,
                 master_seed=99, pfp_budgets=(0, 10)),
    # test_lattices_only_redraw_fixes_sets
    "hc_small": dict(name="unit", candidates={"kind": "hyperbolic", "d": 3, "N": 6,
                                              "weights": None},
                     support={"kind": "hyperbolic", "N": 2, "weights": "t^1.08"},
                     L_values=[5], trials=3, master_seed=99, pfp_budgets=(0, 10),
                     redraw="lattices"),
    # fixed sets, M in the fused-transform range: every trial of one L is one
    # device batch
    "hc_fused": dict(name="hc-fused", candidates={"kind": "hyperbolic", "d": 4, "N": 64,
                                                  "weights": None},
                     support={"kind": "hyperbolic", "N": 32, "weights": "t^1.08"},
                     L_values=[5, 7, 9, 11, 13], trials=24, master_seed=2023,
                     redraw="lattices"),
    # per-trial candidate sets, fused-range M
    "box_fused": dict(name="box-fused", candidates={"kind": "random-box", "d": 3, "lo": -200,
                                                    "hi": 200, "count": 30000},
                      support={"kind": "random-subset", "count": 450}, L_values=[7, 9],
                      trials=4, master_seed=2023),
}


def gen_analysis():
    """run_success_experiment records + aggregates, and pfp_pfn_count
    classifications (reference tests/test_analysis.py recipes, scaled)."""
    ran = _ref_analysis()
    out = {}
    for key, kw in ANALYSIS_SPECS.items():
        spec = ran.ExperimentSpec(**kw)
        t0 = time.perf_counter()
        recs, agg = ran.run_success_experiment(spec)
        print(f"  {key}: {len(recs)} trials in {time.perf_counter() - t0:.1f}s")
        out[key] = {"spec": spec.as_dict(), "records": [r.as_jsonable() for r in recs],
                    "aggregate": agg}
    # pfp_pfn_count on explicit configurations
    rng = np.random.default_rng(77)
    cases = []
    g = rfs.random_subset(rfs.Box(2, -9, 9), 30, rng)
    I = rfs.random_subset(g, 4, rng)
    cfg = rlat.MultiLatticeConfig([rlat.Rank1Lattice([0, 0], 47) for _ in range(3)], 0.5,
                                  10.33, 0.5)
    cases.append((g, I, cfg))
    for _ in range(12):
        d = int(rng.integers(1, 4))
        M = int(rng.choice([11, 13, 17, 19, 23, 29, 31]))
        box = rfs.Box(d, -4, 4)
        g = rfs.random_subset(box, min(int(rng.integers(6, 30)), box.size), rng)
        I = rfs.random_subset(g, int(rng.integers(1, 7)), rng)
        L = int(rng.choice([3, 5]))
        lats = [rlat.Rank1Lattice(rng.integers(0, M, d), M) for _ in range(L)]
        cases.append((g, I, rlat.MultiLatticeConfig(lats, 0.5, 10.33, 0.5)))
    for d, n, s, L in ((3, 5000, 40, 7), (4, 20000, 420, 9)):
        g = rfs.random_subset(rfs.Box(d, -40, 40), n, rng)
        I = rfs.random_subset(g, s, rng)
        cases.append((g, I, rlat.draw_config(g, s, 0.5, rng=rng, L=L)))
    arrs = {"ncases": np.array(len(cases))}
    for k, (g, I, cfg) in enumerate(cases):
        o = ran.pfp_pfn_count(I, g, cfg)
        arrs.update({f"gamma_{k}": g.elems, f"I_{k}": I.elems,
                     f"z_{k}": np.array([lat.z for lat in cfg.lattices], dtype=np.int64),
                     f"M_{k}": np.array([lat.M for lat in cfg.lattices], dtype=np.int64),
                     f"pfn_{k}": o.pfn.elems, f"pfp_{k}": o.pfp.elems,
                     f"anomalies_{k}": np.array(o.anomalies)})
    save_npz("pfp_pfn_cases", **arrs)
    ba = {"bound": [ran.theoretical_failure_bound(1e7, L, 10.33) for L in (0, 9, 37, 41)],
          "guaranteed": ran.guaranteed_sample_budget(1000, 10**7, 0.5)}
    out["budgets"] = ba
    save_json("analysis_cases", out)


FULLSCALE_SPEC = {
    # the paper's hyperbolic-cross worst-case study: |Gamma| = 10,665,297 (d = 8),
    # |I| = 1069, M = 11047 (reference pkg/configs hyperbolic sweep parameters)
    "name": "hyperbolic-fullscale", "candidates": {"kind": "hyperbolic", "d": 8, "N": 32,
                                                   "weights": None},
    "support": {"kind": "hyperbolic", "N": 32, "weights": "t^1.08"},
    "L_values": [9, 37], "trials": 3, "master_seed": 2023, "redraw": "lattices",
    "pfp_budgets": [10, 100]}


def gen_fullscale():
    """Three trials at L = 9 and 37 of the full-scale hyperbolic sweep, with
    the reference's seconds per trial (its CPU cost at paper scale)."""
    ran = _ref_analysis()
    spec = ran.ExperimentSpec.from_dict(FULLSCALE_SPEC)
    t0 = time.perf_counter()
    rng = np.random.default_rng(np.random.SeedSequence((spec.master_seed, 0xFACE)))
    gamma = ran._make_candidates(spec.candidates, rng)
    I = ran._make_support(spec.support, gamma, rng)
    M = ran.next_valid_prime(gamma, spec.c * len(I))
    setup = time.perf_counter() - t0
    recs, secs = [], []
    for L in spec.L_values:
        for trial in range(spec.trials):
            t = time.perf_counter()
            recs.append(ran._trial(spec, L, trial, (gamma, I, M)).as_jsonable())
            secs.append(time.perf_counter() - t)
            print(f"  L={L} trial {trial}: {secs[-1]:.1f}s")
    save_json("analysis_fullscale", {"spec": spec.as_dict(), "records": recs,
                                     "ref_seconds_per_trial": secs, "ref_setup_seconds": setup,
                                     "gamma_size": len(gamma), "support_size": len(I), "M": M})


def gen_f10():
    """B-spline / f10 values and coefficients, and one small B-spline study
    row (reference tests/test_polyeval.py, test_analysis.py:186-194)."""
    rng = np.random.default_rng(1010)
    out = {"norm": {str(m): rpe.bspline_norm_constant(m) for m in (1, 2, 3, 4, 6)}}
    x = rng.uniform(-1.5, 2.5, size=257)
    x[:4] = [0.0, 0.5, 1.0 / 3.0, -0.25]
    out["x"] = x.tolist()
    out["bspline"] = {str(m): rpe.bspline_values(m, x).tolist() for m in (2, 4, 6)}
    X = rng.uniform(0, 1, size=(300, 10))
    out["X"] = X.tolist()
    out["f10"] = rpe.f10_values(X).tolist()
    K = rng.integers(-3, 4, size=(200, 10))
    K[::3, [1, 3, 4, 5, 6, 8, 9]] = 0
    K[1::3, [0, 2, 3, 6, 7, 8]] = 0
    K[5] = 0
    out["K"] = K.tolist()
    out["f10_coeffs"] = rpe.f10_coeffs(K).tolist()
    out["sq_norm"] = rpe.f10_sq_norm()
    from latfft import analysis as ran

    t0 = time.perf_counter()
    rows = ran.run_bspline_experiment(4, 30, runs=1, master_seed=5, r=1, delta=0.9,
                                      L_scale=0.5)
    print(f"  bspline study: {time.perf_counter() - t0:.1f}s")
    out["study"] = {"args": [4, 30, 1, 5, 1, 0.9, 0.5], "rows": rows}
    # the paper's f10 setting (N = 16, r = 5, delta = 0.999, L_scale = 1/4)
    out["studies_paper"] = []
    for args in ([16, 200, 1, 3, 2, 0.999, 0.25], [16, 1000, 1, 3, 5, 0.999, 0.25]):
        N, s, runs, seed, r, delta, Ls = args
        t0 = time.perf_counter()
        rows = ran.run_bspline_experiment(N, s, runs=runs, master_seed=seed, r=r, delta=delta,
                                          L_scale=Ls)
        dt = time.perf_counter() - t0
        print(f"  bspline study {args}: {dt:.1f}s")
        out["studies_paper"].append({"args": args, "rows": rows, "ref_seconds": dt})
    save_json("f10_cases", out)


def gen_cfg4_full():
    """Config 4 at its stated size, run by the reference end to end.

    Gamma = _random_from_box(Box(10,-4096,4096), 2^26, default_rng(2026))
    (called directly: random_subset(Box) overflows len()),
    then I = random_subset(Gamma, 1e4), |c| ~ U[1,10], arg c ~ U[0,2pi),
    draw_config(Gamma, 1e4, 0.1), lattice samples, detect_and_compute.
    About 15 min and 18 GB of RSS here, so only digests are stored: the full
    hits array (2^26 int64) as sha256, the detections and coefficients in
    full, the RNG state after Gamma (to pin the device generator's stream)
    and 4096 sampled Gamma rows.  Not part of the default fixture set.
    """
    d, N, n, s = 10, 4096, 1 << 26, 10_000
    rng = np.random.default_rng(2026)
    t0 = time.perf_counter()
    G = rfs._random_from_box(rfs.Box(d, -N, N), n, rng)
    t_gen = time.perf_counter() - t0
    st_after_gamma = rng.bit_generator.state
    full_gamma = hashlib.sha256(np.ascontiguousarray(G.elems).tobytes()).hexdigest()
    pos = np.linspace(0, n - 1, 4096).astype(np.int64)
    I = rfs.random_subset(G, s, rng)
    mags = rng.uniform(1, 10, s)
    ph = rng.uniform(0, 2 * np.pi, s)
    p = rpe.SparsePoly(I, mags * np.exp(1j * ph))
    t0 = time.perf_counter()
    cfg = rlat.draw_config(G, s, 0.1, rng=rng)
    t_cfg = time.perf_counter() - t0
    oracle = rpe.oracle_from_poly(p)
    samples = [oracle.sample_lattice(lat) for lat in cfg.lattices]
    t0 = time.perf_counter()
    res = rdetect.detect_and_compute(samples, cfg, G)
    t_det = time.perf_counter() - t0
    hits = np.ascontiguousarray(res.hits, dtype=np.int64)
    save_npz("cfg4_full",
             gamma_sha256=np.array(full_gamma), gamma_rows=G.elems[pos], gamma_pos=pos,
             rng_state_after_gamma=np.array(json.dumps(st_after_gamma)),
             support_digest=np.array(digest(I.elems)), coeffs_true=mags * np.exp(1j * ph),
             M=np.array(cfg.shared_M), zmat=np.vstack([lat.z for lat in cfg.lattices]),
             samples_digest=np.array(digest(np.array(samples))),
             hits_sha256=np.array(hashlib.sha256(hits.tobytes()).hexdigest()),
             hits_hist=np.bincount(hits, minlength=len(cfg.lattices) + 1),
             idx=res.detected_idx, coeffs=res.coeffs, theta0=np.array(res.theta_zero),
             ref_seconds=np.array([t_gen, t_cfg, t_det]))


class _LatticeShimOracle(rpe.SamplingOracle):
    """The reference's SamplingOracle with a structured fast path for the
    node sets its sfft driver builds (SURVEY App. A "shimmed reference,
    structured sampler"): a node set [(j z mod M)/M | tail], j < M, is
    recognised exactly (the leading columns equal lattice_nodes bit for bit)
    and evaluated as bins + inverse FFT with the tail's anchor phase
    (oracle/port.py sample_lattice_structured, the restatement of
    polyeval.py:78-87 that the B200 sampler implements); every other node set
    (step 1's coordinate lines) goes through the reference's evaluate_many.
    Harness noise per call as _NoisyFn.  Counters advance as the reference's."""

    def __init__(self, p, support, coeffs, sigma=0.0, noise_seed=0):
        super().__init__(lambda X: rpe.evaluate_many(p, X), p.dim)
        object.__setattr__(self, "_extra", (support, coeffs, sigma, noise_seed, [0]))

    __slots__ = ("_extra",)

    def sample_many(self, X):
        support, coeffs, sigma, nseed, calls = self._extra
        X = np.asarray(X, dtype=np.float64)
        self.count += X.shape[0]
        M = X.shape[0]
        t = 0
        while t < X.shape[1] and X[0, t] == 0.0:
            t += 1
        vals = None
        if t >= 1 and M >= 2:
            z = np.rint(X[1, :t] * M).astype(np.int64)
            nodes = (np.arange(M, dtype=np.int64)[:, None] * z % M) / M
            tail = X[0, t:]
            if np.array_equal(X[:, :t], nodes) and np.all(X[:, t:] == tail):
                vals = port.sample_lattice_structured(support, coeffs, z, M, tail)
        if vals is None:
            vals = np.asarray(self.fn(X), dtype=np.complex128)
        if sigma > 0:
            vals = vals + port.noise_for_call(nseed, calls[0], M, sigma)
        calls[0] += 1
        return vals


def gen_sfft_fullsize():
    """The metric instance, config 3 and config 5 at full size through the
    reference's own sfft driver and detection (compiled gather), with the
    structured sampler shim above: the fixtures the full-size GPU runs and
    oracle/port.sfft are pinned to."""
    for name in ("metric_config", "config3", "config5"):
        w = getattr(workloads, name)()
        I = rfs.FreqSet(w.d, w.support, _sorted=True)
        p = rpe.SparsePoly(I, w.coeffs)
        oracle = _LatticeShimOracle(p, w.support, w.coeffs, w.sigma, w.noise_seed)
        params = rdim.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
        t0 = time.perf_counter()
        res = rdim.sfft(oracle, ClampedBox(w.d, w.lo, w.hi), params, seed=w.seed)
        dt = time.perf_counter() - t0
        print(f"{name}: reference sfft (structured shim) {dt:.1f}s, "
              f"{len(res.support)} found, {res.sample_count} samples")
        save_sfft(f"sfft_ref_{w.name}", w, res, dt)


def gen_sfft_freqset():
    """sfft over explicit candidate sets (FreqSet Gamma, the pairing filtered
    by the prefix projections, dimincr.py:155-175) through the reference's own
    driver, with the structured-sampler shim; two shapes."""
    out = {}
    for d, N, n, s in ((6, 16, 200_000, 30), (7, 12, 120_000, 20)):
        rng = np.random.default_rng(1000 + d)
        gamma = workloads.rows_from_box(d, -N, N, n, rng)
        idx = np.sort(rng.choice(gamma.shape[0], size=s, replace=False))
        sup = gamma[idx]
        co = workloads.mag_phase_coeffs(s, rng)
        G = rfs.FreqSet(d, gamma, _sorted=True)
        p = rpe.SparsePoly(rfs.FreqSet(d, sup, _sorted=True), co)
        oracle = _LatticeShimOracle(p, sup, co)
        t0 = time.perf_counter()
        res = rdim.sfft(oracle, G, rdim.SfftParams(s, 0.9, r=2), seed=11)
        dt = time.perf_counter() - t0
        log = [[e["stage"], e["t"], e["i"], e["candidates"], e["kept"], e["samples"]]
               for e in res.stage_log]
        key = f"d{d}"
        out[key + "_support"] = res.support.elems
        out[key + "_coeffs"] = res.coeffs
        out[key + "_count"] = np.array(res.sample_count)
        out[key + "_log"] = np.array(log, dtype=object).astype(str)
        out[key + "_gamma_digest"] = np.array(digest(gamma))
        print(f"freqset d={d}: {dt:.1f}s, {len(res.support)} found")
    # a hyperbolic cross (the reference's hc_enumerate builds it)
    rng = np.random.default_rng(77)
    G = rfs.hyperbolic_cross(4, 40)
    gamma = np.ascontiguousarray(G.elems)
    idx = np.sort(rng.choice(gamma.shape[0], size=16, replace=False))
    sup = gamma[idx]
    co = workloads.mag_phase_coeffs(16, rng)
    p = rpe.SparsePoly(rfs.FreqSet(4, sup, _sorted=True), co)
    res = rdim.sfft(_LatticeShimOracle(p, sup, co), G, rdim.SfftParams(16, 0.9, r=2), seed=5)
    log = [[e["stage"], e["t"], e["i"], e["candidates"], e["kept"], e["samples"]]
           for e in res.stage_log]
    out["hc_gamma_digest"] = np.array(digest(gamma))
    out["hc_support"] = res.support.elems
    out["hc_coeffs"] = res.coeffs
    out["hc_count"] = np.array(res.sample_count)
    out["hc_log"] = np.array(log, dtype=object).astype(str)
    print(f"hyperbolic cross d=4 N=40 (|Gamma| = {gamma.shape[0]}): {len(res.support)} found")
    save_npz("sfft_freqset", **out)


def gen_fixed_noisy():
    """Fixed-Gamma detection on noisy samples at 2 x 10^4 candidates: many false
    detections, so detect_topk truncates and postprocess_r1l refines
    crowded residues (reference detect.py:158-228, compiled gather)."""
    rng = np.random.default_rng(4242)
    d, N, n, s = 5, 20, 20_000, 40
    gamma = workloads.rows_from_box(d, -N, N, n, rng)
    G = rfs.FreqSet(d, gamma, _sorted=True)
    idx = np.sort(rng.choice(n, size=s, replace=False))
    co = workloads.mag_phase_coeffs(s, rng)
    p = rpe.SparsePoly(rfs.FreqSet(d, gamma[idx], _sorted=True), co)
    cfg = rlat.draw_config(G, s, 0.1, rng=rng)
    oracle = rpe.oracle_from_poly(p)
    samples = [oracle.sample_lattice(lat) + 0.3 * (rng.standard_normal(lat.M)
                                                   + 1j * rng.standard_normal(lat.M))
               for lat in cfg.lattices]
    res = rdetect.detect_and_compute(samples, cfg, G)
    topk = rdetect.detect_topk(samples, cfg, G, s, 0.5)
    post = rdetect.postprocess_r1l(res, samples, cfg)
    fr = rdetect.detect_frequencies(samples, cfg, G)
    hits = np.ascontiguousarray(res.hits, dtype=np.int64)
    print(f"fixed noisy: M={cfg.shared_M} L={len(cfg.lattices)} detected {len(res.detected_idx)}, "
          f"top-s {len(topk.detected_idx)}, post {len(post.detected_idx)}")
    save_npz("fixed_noisy", gamma_digest=np.array(digest(gamma)), support_idx=idx,
             coeffs_true=co, M=np.array(cfg.shared_M),
             zmat=np.vstack([lat.z for lat in cfg.lattices]), samples=np.array(samples),
             hits_sha256=np.array(hashlib.sha256(hits.tobytes()).hexdigest()),
             idx=res.detected_idx, coeffs=res.coeffs, theta0=np.array(res.theta_zero),
             topk_idx=topk.detected_idx, topk_coeffs=topk.coeffs,
             post_idx=post.detected_idx, post_coeffs=post.coeffs, freq_idx=fr.detected_idx)


GEN = {"gather": gen_gather, "injective": gen_injective, "hc": gen_hc,
       "lattice": gen_lattice, "dft": gen_dft, "sampling": gen_sampling,
       "tiny_detect": gen_tiny_detect, "cfg1": gen_cfg1,
       "sfft_small": gen_sfft_small, "sfft_cfg2": gen_sfft_cfg2,
       "analysis": gen_analysis, "f10": gen_f10, "fullscale": gen_fullscale,
       "cfg4_full": gen_cfg4_full, "sfft_fullsize": gen_sfft_fullsize,
       "sfft_freqset": gen_sfft_freqset, "fixed_noisy": gen_fixed_noisy}
SLOW = {"cfg4_full", "sfft_fullsize"}

if __name__ == "__main__":
    names = sys.argv[1:] or [k for k in GEN if k not in SLOW]
    for nm in names:
        t0 = time.perf_counter()
        GEN[nm]()
        print(f"[{nm}] {time.perf_counter() - t0:.1f}s")
