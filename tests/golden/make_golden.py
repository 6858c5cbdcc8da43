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


GEN = {"gather": gen_gather, "injective": gen_injective, "hc": gen_hc,
       "lattice": gen_lattice, "dft": gen_dft, "sampling": gen_sampling,
       "tiny_detect": gen_tiny_detect, "cfg1": gen_cfg1,
       "sfft_small": gen_sfft_small, "sfft_cfg2": gen_sfft_cfg2}

if __name__ == "__main__":
    names = sys.argv[1:] or list(GEN)
    for nm in names:
        t0 = time.perf_counter()
        GEN[nm]()
        print(f"[{nm}] {time.perf_counter() - t0:.1f}s")
