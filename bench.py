#!/usr/bin/env python3
"""Benchmark: sFFT recon time (d=10, s=1000) & candidates hashed/s vs HBM roofline.

  python bench.py [--gpus N --steps K --warmup W]      # B200 arm (default)
  python bench.py --impl reference [...]               # CPU reference arm

B200 arm, one JSON line on rank 0:
  * value   -- seconds per dimension-incremental reconstruction of the
               metric's instance (d=10, [-32,32]^10, s=1000, r=5,
               theta=1e-12, delta=0.9; config-2 generator with s=1000),
               polynomial already in HBM; lower is better.
  * e2e     -- the same through the public API from host arrays: upload of
               the polynomial, sfft(), support/coefficients back on the host.
  * hashing -- config 4: |Gamma| = 2^26 candidates in [-4096,4096]^10, the
               reference's seeded Gamma (generated in HBM in its RNG stream),
               s=1e4, L=47, M=103307: candidates hashed per second by the
               hashing kernel and by the whole detection call, every hit
               count checked against the reference's own run
               (tests/golden/cfg4_full.npz); e2e through detect_and_compute
               from a plain host FreqSet over pinned rows.  With N > 1 ranks
               one Gamma is sharded (shard.detect_and_compute_sharded).
  * roofline -- the hashing kernel vs measured HBM bandwidth (the metric's
               "vs HBM roofline"); roofline_sfft -- the dominant kernel of
               the reconstruction step.
  * configs -- SURVEY 8(d)'s rows for configs 1, 2, 3, 5: entry-point time,
               phase breakdown, dominant kernel vs roofline, same-run CPU.
  * cpu_baseline -- the algorithm-matched CPU reference (the reference's
               driver, structured sampler, pocketfft and compiled gather on
               all host threads) run to completion and timed; the as-shipped
               dense run beside it, bounded and flagged as extrapolated.
Timing: CUDA events on the launching (current torch) stream, W untimed
warm-up steps, L2 flushed (256 MB write) between timed steps, max over
ranks; nvidia-smi clocks sampled during the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "sFFT recon time (d=10,s=1000) & candidates hashed/s vs HBM roofline"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=10)
        return False

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 6:
                    continue
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
                for nm, v in zip(names, parts[2:6]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except Exception:
            pass
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def flush_l2(buf):
    buf.zero_()


def predicted_sample_count(w):
    """Samples an exact-recovery run of `w` draws (step 1 + every lattice),
    from the true support's projections and the reference's host formulas
    (required_L, next_prime_above; p > expansion always holds here)."""
    from paper_2006_13053_b200.lattice import next_prime_above, required_L

    d, s, r = w.d, w.s, w.r
    K = w.hi - w.lo + 1
    total = d * r * K
    gA = w.delta / (3 * d * r)
    prev = np.unique(w.support[:, :1], axis=0).shape[0]
    for t in range(1, d):
        J = prev * np.unique(w.support[:, t]).size
        M = next_prime_above(10.33 * min(2 * s, J))
        L = required_L(J, gA)
        total += (1 if t == d - 1 else r) * L * M
        prev = np.unique(w.support[:, :t + 1], axis=0).shape[0]
    M = next_prime_above(10.33 * s)
    total += required_L(prev, w.delta / (3 * d)) * M
    return int(total)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def sfft_profile(step, flush=None):
    """One instrumented reconstruction: device time per entry point and per
    stage phase ('stage:<phase>', CUDA events on the launch streams), plus
    the (G, L, M, fused) shape of every stage call that runs transforms."""
    import torch

    from paper_2006_13053_b200 import _native, _stage

    shapes = []
    orig_run = _stage.run

    def run_rec(desc, stream=None):
        if desc.phase in (0, 1, 4):  # the calls that run transforms
            shapes.append((desc.G, desc.L, desc.M, bool(desc.fused)))
        return orig_run(desc, stream)

    if flush is not None:
        flush_l2(flush)
    torch.cuda.synchronize()
    _stage.run = run_rec
    try:
        with _native.Timeline() as tl:
            step()
        raw = tl.ms()
    finally:
        _stage.run = orig_run
    return {k: (sum(v), len(v)) for k, v in raw.items()}, raw, shapes


def run_sfft_arm(args, world, rank):
    import torch

    import paper_2006_13053_b200 as pkg
    from paper_2006_13053_b200 import _native

    w = workloads.metric_config()
    box = pkg.Box(w.d, w.lo, w.hi)
    params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
    poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
    poly.device()  # resident in HBM before timing
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        return pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed + rank)

    for _ in range(args.warmup):
        res = step()
    torch.cuda.synchronize()
    times, launches = [], []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            flush_l2(flush)
            barrier(world)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            n0 = _native.launch_count()
            a.record()
            res = step()
            b.record()
            torch.cuda.synchronize()
            launches.append(_native.launch_count() - n0)
            times.append(a.elapsed_time(b))
    clocks = clk.summary()
    ms = max_over_ranks(statistics.mean(times), world)
    ok_support = np.array_equal(res.support.elems, w.support) if rank == 0 else None
    rel = workloads.rel_l2(res.coeffs, w.coeffs) if ok_support else None
    parity = {"support_exact": bool(ok_support), "coeff_rel_l2_vs_truth": rel,
              "sample_count": res.sample_count,
              "sample_count_predicted": predicted_sample_count(w),
              "stages": len(res.stage_log)}

    per, per_list, shapes = sfft_profile(step, flush)

    # e2e: host arrays in, host results out, through the public API
    e2e_times = []
    h2d = w.support.nbytes + w.coeffs.nbytes
    d2h = 0
    for _ in range(max(1, args.steps)):
        flush_l2(flush)
        barrier(world)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        p2 = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
        r2 = pkg.sfft(pkg.oracle_from_poly(p2), box, params, seed=w.seed + rank)
        sup_host, co_host = r2.support.elems, r2.coeffs
        b.record()
        torch.cuda.synchronize()
        e2e_times.append(a.elapsed_time(b))
        d2h = sup_host.nbytes + co_host.nbytes
    e2e_ms = max_over_ranks(statistics.mean(e2e_times), world)
    return {"ms": ms, "times": times, "launches": statistics.mean(launches), "clocks": clocks,
            "parity": parity, "per_entry": per, "per_list": per_list, "shapes": shapes,
            "e2e_ms": e2e_ms, "h2d": h2d, "d2h": d2h, "workload": w}


CFG4_SEED = 2026  # tests/golden/cfg4_full.npz: the reference's own run at this seed


def cfg4_instance(n, d, N, s, seed):
    """Config 4 as the reference builds it: Gamma = 2^26
    distinct rows of [-N, N]^d in the reference's default_rng(seed) stream,
    born in HBM (csrc/boxgen.cu + canon.cu: identical rows to
    freqset._random_from_box, freqset.py:266-280); support = random_subset
    of Gamma, |c| ~ U[1,10] e^{i U[0,2pi)}, draw_config(Gamma, s, 0.1) --
    every draw from the same generator, in the reference's order.
    Returns (G, support FreqSet, coeffs, config, generation ms)."""
    import torch

    import paper_2006_13053_b200 as pkg

    rng = np.random.default_rng(seed)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    G = pkg.random_box_device(pkg.Box(d, -N, N), n, rng)
    b.record()
    torch.cuda.synchronize()
    gen_ms = a.elapsed_time(b)
    pick = np.sort(rng.choice(len(G), size=s, replace=False))  # random_subset's draw
    I = G.take(torch.as_tensor(pick, device="cuda"))
    coeffs = rng.uniform(1, 10, s) * np.exp(1j * rng.uniform(0, 2 * np.pi, s))
    cfg = pkg.draw_config(G, s, 0.1, rng=rng)
    return G, I, pick, coeffs, cfg, gen_ms


def run_hash_arm(args, world, rank):
    """Config 4: fixed-Gamma detection of 2^26 HBM-resident candidates.
    N = 1: detect_and_compute on all rows.  N > 1: one Gamma sharded across
    the ranks (strong scaling): shard.detect_and_compute_sharded -- lattice-
    sharded DFTs, bitmap + spectra all-gathers over NCCL, row-sharded
    hashing, merged detections."""
    import hashlib

    import torch

    import paper_2006_13053_b200 as pkg
    from paper_2006_13053_b200 import _dev, _native
    from paper_2006_13053_b200.shard import detect_and_compute_sharded, shard_bounds

    n, d, N, s = args.hash_rows, 10, 4096, 10_000
    G, I, pick, coeffs, cfg, gen_ms = cfg4_instance(n, d, N, s, CFG4_SEED)
    M, L = cfg.shared_M, cfg.L
    orc = pkg.oracle_from_poly(pkg.SparsePoly(I, coeffs))
    samples = orc.sample_lattices_device(cfg.zmat_device(), M,
                                         torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                         1, L, d).contiguous()
    rows_all = G.device()
    lo, hi = shard_bounds(n, world, rank)
    if world > 1:
        Gs = pkg.FreqSet.from_device(d, rows_all[lo:hi].contiguous())
        zero = pkg.default_zero_test(samples)

        def step():
            gidx, gco, res = detect_and_compute_sharded(samples, cfg, Gs, lo, zero=zero)
            return gidx, gco, res
    else:
        Gs = G

        def step():
            res = pkg.detect_and_compute(samples, cfg, G)
            return res.detected_idx, res.coeffs, res

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    times, hash_ms, path_ms = [], [], []
    with ClockSampler(torch.cuda.current_device()) as clk:
        for _ in range(args.steps):
            barrier(world)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            with _native.Timeline() as tl:
                a.record()
                idx, co, res = step()
                b.record()
            per = tl.ms()
            times.append(a.elapsed_time(b))
            path_ms.append(sum(sum(per.get(k, [0.0])) for k in (
                "sfftb_detect_dev", "sfftb_nonzero_bitmap", "sfftb_hash_hits",
                "sfftb_compact_mask", "sfftb_medians")))
        # the hashing entry point alone (detect_and_compute runs it inside ONE
        # C call, csrc/detect_dev.cu): the same sfftb_hash_hits call on the same
        # rows, generators and nonzero bitmaps, CUDA events on its stream
        from paper_2006_13053_b200 import _engine as _eng

        _g, th_dev, bits = _eng.spectra(samples, M, 1, L)
        del _g
        nl = hi - lo
        rows_l = rows_all[lo:hi]
        hits_t = torch.empty((nl,), dtype=torch.int64, device="cuda")
        mask_t = torch.empty(((nl + 31) // 32,), dtype=torch.int32, device="cuda")
        zdev = cfg.zmat_device()
        from paper_2006_13053_b200.detect import _kbound

        kb = int(_kbound(Gs))  # the bound detect_and_compute passes (sum_j max|k_j|)
        _native.lib().sfftb_hash_rollf_calls(1)
        _native.lib().sfftb_hash_rollf_scaled_runs(1)
        for it in range(args.warmup + args.steps):
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            _native.call("sfftb_hash_hits", rows_l.data_ptr(), nl, d, zdev.data_ptr(), 1, L, M,
                         bits.data_ptr(), kb, _eng.min_hits_for(cfg.nu, L), hits_t.data_ptr(),
                         mask_t.data_ptr(), _dev.stream())
            b.record()
            torch.cuda.synchronize()
            if it >= args.warmup:
                hash_ms.append(a.elapsed_time(b))
        rollf_calls = int(_native.lib().sfftb_hash_rollf_calls(1))
        scaled_runs = int(_native.lib().sfftb_hash_rollf_scaled_runs(1))
        hash_kernel = "hash_roll_kernel"
        if rollf_calls == args.warmup + args.steps:
            hash_kernel = ("hash_rollf_kernel, scaled byte mode (two limbs)"
                           if scaled_runs == rollf_calls else "hash_rollf_kernel, byte mode")
        hash_equal = None
        if world == 1:
            ref_hits = res._hits
            hash_equal = bool(torch.equal(hits_t, ref_hits)) if torch.is_tensor(ref_hits) \
                else bool(np.array_equal(_dev.download(hits_t), ref_hits))
        del hits_t, mask_t, bits
    clocks = clk.summary()
    parity = {"hash_call_equals_detection_hits": hash_equal,
              "detected_equals_support": bool(np.array_equal(idx, pick)),
              "coeff_max_rel_err_vs_truth": float(np.max(np.abs(co - coeffs))
                                                  / np.max(np.abs(coeffs)))}
    # the reference's own run of this instance (tests/golden/make_golden.py
    # gen_cfg4_full): every row's hit count (sha256 over all 2^26), the
    # detected indices and coefficients
    gold = None
    try:
        gold = np.load(os.path.join(ROOT, "tests", "golden", "cfg4_full.npz"))
    except OSError:
        pass
    if gold is not None and n == 1 << 26 and world == 1:
        hits = res.hits
        parity["hits_bitexact_all_rows"] = (
            hashlib.sha256(np.ascontiguousarray(hits, dtype=np.int64).tobytes()).hexdigest()
            == str(gold["hits_sha256"]))
        parity["hits_rows_compared"] = int(hits.size)
        parity["detected_idx_equals_reference"] = bool(np.array_equal(idx, gold["idx"]))
        parity["coeff_max_rel_err_vs_reference"] = float(
            np.max(np.abs(co - gold["coeffs"])) / np.max(np.abs(gold["coeffs"])))
        parity["gamma_equals_reference"] = bool(np.array_equal(
            _dev.download(rows_all[torch.as_tensor(gold["gamma_pos"], device="cuda")]),
            gold["gamma_rows"]))
        parity["reference"] = "tests/golden/cfg4_full.npz (the reference's own run, seed 2026)"
        del hits
    elif world > 1 and rank == 0:
        parity["sharded"] = f"{world} ranks, merged detections"

    # CPU sample for the reference's gather, and the spectra it reads
    from paper_2006_13053_b200 import _engine

    ghat, theta0, _ = _engine.spectra(samples, M, 1, L,
                                      torch.full((1,), res.theta_zero, dtype=torch.float64,
                                                 device="cuda"))
    ghat_h = _dev.download(ghat)
    rows_h = _dev.download(rows_all[:1 << 20])
    del ghat

    # e2e: a plain host FreqSet from pinned rows (no bounds, no memo) through
    # detect_and_compute: chunked H2D overlapped with hashing, results to host
    host = torch.empty((hi - lo, d), dtype=torch.int64, pin_memory=True)
    host.copy_(rows_all[lo:hi])
    hnp = host.numpy()
    e2e = []
    d2h = 0
    nrep = max(1, min(args.steps, 3))
    for rep in range(nrep + 1):  # rep 0 warms the pinned result buffers (untimed)
        barrier(world)
        torch.cuda.synchronize()
        Gh = pkg.FreqSet(d, hnp, _sorted=True)
        a = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        a.record()
        if world > 1:
            gi, gc, r2 = detect_and_compute_sharded(samples, cfg, Gh, lo)
            out = (r2.hits, gi, gc)
        else:
            r2 = pkg.detect_and_compute(samples, cfg, Gh)
            out = (r2.hits, r2.detected_idx, r2.coeffs)
        e.record()
        torch.cuda.synchronize()
        if rep:
            e2e.append(a.elapsed_time(e))
        d2h = sum(x.nbytes for x in out)
        del Gh, r2, out
    # the same H2D alone (pinned, one stream): the PCIe floor of the e2e
    dst = torch.empty((hi - lo, d), dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    a.record()
    dst.copy_(host, non_blocking=True)
    e.record()
    torch.cuda.synchronize()
    h2d_ms = a.elapsed_time(e)
    del dst, host
    W = int(_native.lib().sfftb_bitmap_words(M))
    return {"n": n, "n_local": hi - lo, "d": d, "L": L, "M": M, "s": s, "W": W,
            "n_det": int(idx.size),
            "ms": max_over_ranks(statistics.mean(times), world),
            "hash_ms": max_over_ranks(statistics.mean(hash_ms), world),
            "hash_kernel": hash_kernel, "kbound": kb,
            "path_ms": max_over_ranks(statistics.mean(path_ms), world),
            "clocks": clocks, "parity": parity, "gamma_generation_ms": gen_ms,
            "e2e_ms": max_over_ranks(statistics.mean(e2e), world),
            "h2d_ms": max_over_ranks(h2d_ms, world), "h2d": (hi - lo) * d * 8,
            "d2h": d2h, "rows_host_sample": rows_h, "ghat": ghat_h,
            "zmat": cfg.zmat(), "theta0": res.theta_zero}


# ---------------------------------------------------------------------------
# CPU legs (oracle / reference's compiled kernel)
# ---------------------------------------------------------------------------

class _ThreadedDense:
    """Dense evaluate_many (polyeval.py:66-75) split over host threads."""

    def __init__(self, workers):
        from concurrent.futures import ThreadPoolExecutor

        self.pool = ThreadPoolExecutor(workers)
        self.workers = workers

    def __call__(self, support, coeffs, X):
        from oracle import port

        parts = np.array_split(np.arange(X.shape[0]), self.workers)
        outs = list(self.pool.map(lambda ix: port.evaluate_dense(support, coeffs, X[ix]),
                                  [p for p in parts if p.size]))
        return np.concatenate(outs) if outs else np.zeros(0, np.complex128)


class _BudgetExceeded(Exception):
    pass


def cpu_sfft_structured(w, workers):
    """The algorithm-matched CPU reference, run to completion and timed: the
    reference's sfft driver (dimincr.py:195-256, restated in oracle/port.py)
    with the reference's own structured lattice sampler (bincount + numpy
    ifft, polyeval.py:78-87) and numpy's pocketfft for every detection DFT
    (dft.py:27), the reference's compiled detect_gather (oracle/_ref, built
    from _core.pyx) for the hashing; lattices sampled and transformed on
    `workers` threads.  Returns (seconds, samples, support size)."""
    from oracle import port

    orc = port.PolyOracle(w.support, w.coeffs, mode="structured", sigma=w.sigma,
                          noise_seed=w.noise_seed)
    t0 = time.perf_counter()
    res = port.sfft(orc, port.Box(w.d, w.lo, w.hi), w.s, w.delta, w.seed, theta=w.theta,
                    r=w.r, gather_backend="reference" if _ref_core() else "port",
                    workers=workers)
    return time.perf_counter() - t0, int(res[2]), int(len(res[0]))


def cpu_sfft_dense_bounded(w, budget_s, workers):
    """The reference as shipped (dense evaluate_many sampling, polyeval.py:
    66-75, threaded over `workers` cores) for `budget_s` seconds, then
    EXTRAPOLATED by sample count to the full run (a full run is ~8 min)."""
    from oracle import port

    dense = _ThreadedDense(workers)
    t0 = time.perf_counter()

    class BoundedOracle(port.PolyOracle):
        def sample_points(self, X):
            if time.perf_counter() - t0 > budget_s:
                raise _BudgetExceeded
            X = np.asarray(X, dtype=np.float64)
            self.count += X.shape[0]
            return self._noise(dense(self.support, self.coeffs, X))

    orc = BoundedOracle(w.support, w.coeffs, mode="dense", sigma=w.sigma,
                        noise_seed=w.noise_seed)
    try:
        port.sfft(orc, port.Box(w.d, w.lo, w.hi), w.s, w.delta, w.seed, theta=w.theta, r=w.r,
                  gather_backend="reference" if _ref_core() else "port", workers=workers)
        finished = True
    except _BudgetExceeded:
        finished = False
    elapsed = time.perf_counter() - t0
    total = predicted_sample_count(w)
    est = elapsed if finished else elapsed * total / max(orc.count, 1)
    return {"value": round(est, 3), "unit": "s", "extrapolated": not finished,
            "fraction_run": round(orc.count / total, 5), "samples_done": int(orc.count),
            "samples_total": total, "elapsed_s": round(elapsed, 2), "cores": workers,
            "what": "reference sfft as shipped: dense evaluate_many sampling"}


def _ref_core():
    try:
        from oracle.refload import load_ref_core

        return load_ref_core()
    except Exception:
        return None


def cpu_hash_bounded(rows_host, zmat, M, ghat, theta0, workers, budget_s=8.0):
    """The reference's compiled detect_gather (oracle/_ref) -- else the C
    restatement -- over a bounded sample of candidate rows, all host threads."""
    from oracle import port

    core = _ref_core()
    kind = "reference" if core is not None else "port"
    em = np.ascontiguousarray(rows_host % M)
    L = zmat.shape[0]
    fn = port.gather_ref if core is not None else port.gather_c
    n_done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < budget_s:
        fn(em, zmat, M, ghat, theta0, L / 2, True, workers)
        n_done += em.shape[0]
    el = time.perf_counter() - t0
    return n_done / el, kind, {"rows_per_call": int(em.shape[0]), "calls": n_done // em.shape[0],
                               "elapsed_s": el}


# ---------------------------------------------------------------------------

def measured_traffic(kernel):
    """DRAM bytes per launch from the newest committed ncu capture
    (profiles/r02/traffic.json, else r01), or None."""
    for rnd in ("r02", "r01"):
        path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", rnd,
                            "traffic.json")
        try:
            with open(path) as f:
                return json.load(f)[kernel]
        except (OSError, KeyError, ValueError):
            continue
    return None


def _pipe_peaks():
    """Measured FP64 FMA and IMAD pipe peaks (tools/micro/pipe_peaks.cu on a
    B200 of this pool, profiles/r01/pipe_peaks.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01",
                        "pipe_peaks.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def _fp64_frac(tflops):
    pk = _pipe_peaks()
    if not pk:
        return {}
    return {"fp64_peak_tflops": pk["fp64_fma_tflops"],
            "fp64_frac": round(tflops / pk["fp64_fma_tflops"], 4),
            "fp64_peak_source": "measured DFMA peak (profiles/r01/pipe_peaks.json)"}


def arm_config(world):
    """The `config` object of the bench line, shared verbatim by both arms."""
    return {"workload": WORKLOAD,
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
            "l2": "flushed (256 MB write) between timed steps",
            "value_semantics": "seconds per reconstruction (replicas: step time / N)"}


def _issue_bound(h):
    """The rolling tensor-core hash kernel's limiters, from its ncu --set full
    capture (profiles/r02/traffic.json carries the numbers and their source):
    instruction issue and the shared-memory data pipe.  The residue dot
    products run as an exact tcgen05 GEMM; what remains per (row, lattice)
    pair in the epilogue is the limb recombination, a multiply-high +
    multiply-add reduction, 2 address ops, 1 shared load (3.6 wavefronts on
    average: 32 random bank addresses) and 2 funnel shifts, plus the row
    loaders."""
    pk = _pipe_peaks()
    if not pk:
        return {}
    pairs = h.get("n_local", h["n"]) * h["L"]
    # the CUDA-core kernel's IMAD-pipe floor (12 IMAD-pipe ops per pair), for comparison
    floor_ms = pairs * 12 / (pk["imad_lanes_per_clk_per_sm"] * pk["sms"]
                             * pk["clock_mhz"] * 1e6) * 1e3
    key = _hash_traffic_key(h)
    tr = measured_traffic(key) or {}
    out = {"cuda_core_imad_floor_ms": round(floor_ms, 3),
           "note": "the all-IMAD kernel (hash_rows, SFFTB_HASH_ROLL=0) cannot go below its "
                   "IMAD-pipe floor; the tensor-core kernels are below it when launch_ms < "
                   "cuda_core_imad_floor_ms"}
    for k in ("warp_instructions", "issue_slots_busy", "lsu_data_pipe_busy", "pipes", "source"):
        if k in tr:
            out[k] = tr[k]
    if h.get("hash_kernel", "").startswith("hash_rollf"):
        # accumulator bytes the epilogue reads out of tensor memory: 48 lattice slots
        # (6 groups of 8) x 2 or 3 limbs x 4 B per row, against the 64 B/clk/SM
        # read rate of B300_MICROARCH.md ("LDTM throughput"); profiles/r02/hash_rollf_diag.txt
        sms, mhz = pk["sms"], pk["clock_mhz"]
        limbs = 2 if "two limbs" in h.get("hash_kernel", "") else 3
        per_sm = h.get("n_local", h["n"]) / sms * 48 * 4 * limbs
        bpc = per_sm / (h["hash_ms"] * 1e-3 * mhz * 1e6)
        out["tensor_memory_read"] = {"bytes_per_sm": int(per_sm), "bytes_per_clk": round(bpc, 1),
                                     "peak_bytes_per_clk": 64, "frac": round(bpc / 64, 3),
                                     "limbs": limbs,
                                     "note": "three limbs: bound by the tensor-memory read port "
                                             "(~63 of 64 B/clk); two limbs: below it, bound by "
                                             "the shared-memory data pipe (random bitmap probes)"}
    if "warp_instructions" in tr and tr.get("rows") and tr.get("L"):
        out["warp_instructions_per_pair"] = round(
            tr["warp_instructions"] / (tr["rows"] * tr["L"]), 3)
    return {"issue": out}


def _hash_traffic_key(h):
    k = h.get("hash_kernel", "")
    if "two limbs" in k:
        return "hash_rollf_kernel_scaled"
    return "hash_rollf_kernel_byte" if k.startswith("hash_rollf") else "hash_roll_kernel"


def roofline_hash(h, peak, src):
    """Algorithmic bytes of one hashing call: rows (n*8d) + int64 hits
    (n*8) + the L bitmaps (L*W*4) + the detected-row bitmask (n/8).  The
    duration is the whole sfftb_hash_hits call (CUDA events on its stream):
    bitmap pre-kernel + the rolling tensor-core kernel + the out-of-range
    repair kernel."""
    n = h.get("n_local", h["n"])  # this rank's rows (all rows at N = 1)
    bytes_ = n * 8 * h["d"] + n * 8 + h["L"] * h["W"] * 4 + n // 8
    ach = bytes_ / (h["hash_ms"] * 1e-3) / 1e9
    tr = measured_traffic(_hash_traffic_key(h))
    traffic = None
    if tr and tr.get("rows") == h["n"] and tr.get("L") == h["L"] and tr.get("M") == h["M"]:
        traffic = tr["dram_read"] + tr["dram_write"]
    return {"bound": "hbm", "kernel": h.get("hash_kernel", "hash_roll_kernel") +
            " (sfftb_hash_hits)",
            "achieved": round(ach, 1),
            "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": traffic,
            "algorithmic_bytes": bytes_, "peak_source": src,
            "launch_ms": round(h["hash_ms"], 4), **_issue_bound(h)}


def fft_flops(N):
    return 5.0 * N * math.log2(N)


def bluestein_N(M):
    """The library's convolution length (csrc/fft.cu bluestein_N): the
    smallest power of two >= max(2M-1, 256), or 192*{128, 256} (four-step) /
    9*2^k (single CTA) when that is smaller."""
    N = 256
    while N < 2 * M - 1:
        N *= 2
    cands = (24576, 49152) if N > 8192 else (576, 1152, 2304, 4608)
    for c in cands:
        if c >= 2 * M - 1 and c < N:
            return c
    return N


def roofline_sfft(r, peak, src):
    """The reconstruction's dominant phase: the fused sampler->detection
    transforms (sfftb_sample_detect_dft inside each stage call).

    Algorithmic bytes per call = rows * (16 M bins in + 16 M spectra out +
    4 W bitmap out): the samples never touch HBM.  Algorithmic FLOPs = two
    length-M DFTs per row by Bluestein: 4 power-of-two FFTs of N (5 N log2 N
    each) + 3 pointwise complex products per transform (6 flops each, 2 N
    elements).  Device time from CUDA events around the phase, summed over the
    stage calls of one step."""
    per = r["per_entry"]
    phases = {k: v for k, v in per.items() if k.startswith("stage:")}
    out = {"bound": "hbm", "peak": peak, "unit": "GB/s", "peak_source": src,
           "traffic": None,
           "breakdown_ms": {k: round(v[0], 3) for k, v in sorted(per.items(),
                                                                 key=lambda kv: -kv[1][0])
                            if k != "sfftb_sfft_stage"}}
    if not phases:
        name = max(per, key=lambda k: per[k][0])
        out.update({"kernel": name, "ms_total": round(per[name][0], 3),
                    "share_of_step": round(per[name][0] / r["ms"], 3)})
        return out
    tms = r["per_list"].get("stage:transforms", [])
    bytes_, flops = 0, 0.0
    for (G, L, M, fused) in r["shapes"]:
        rows = G * L
        W = ((M + 31) // 32 + 3) & ~3
        N = bluestein_N(M)
        bytes_ += rows * (32 * M + 4 * W) if fused else rows * (32 * M + 32 * M + 4 * W)
        flops += rows * 2 * (2 * fft_flops(N) + 3 * 6 * 2 * N)
    t = sum(tms)
    ach = bytes_ / (t * 1e-3) / 1e9
    tr = measured_traffic("sample_detect_dft")
    if tr:  # per call at the dominant stage shape (185 lattices, M = 20663)
        out["traffic"] = tr["dram_read"] + tr["dram_write"]
        out["traffic_shape"] = f"{tr['lattices']} lattices, M={tr['M']}, N={tr['N']}"
    out.update({"kernel": "sfftb_sample_detect_dft (fs2_colA/rowB/colCA/rowB/colC_bits)",
                "calls": len(tms), "ms_total": round(t, 3),
                "share_of_step": round(t / r["ms"], 3),
                "achieved": round(ach, 1), "frac": round(ach / peak, 4),
                "algorithmic_bytes": int(bytes_),
                "fp64_tflops": round(flops / (t * 1e-3) / 1e12, 3),
                **_fp64_frac(flops / (t * 1e-3) / 1e12),
                "algorithmic_flops": flops})
    return out


WORKLOAD = ("d10_s1000: sfft over [-32,32]^10, s=1000 random frequencies, |c|~U[1,10], r=5, "
            "theta=1e-12, delta=0.9, polynomial seed 2006, sfft seed 7 (BASELINE config-2 "
            "generator at the metric's s=1000)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--hash-rows", type=int, default=1 << 26)
    ap.add_argument("--cpu-budget", type=float, default=20.0,
                    help="seconds of the dense as-shipped CPU run before extrapolating")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-hash", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config measurements (configs 1, 2, 3, 5)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--one-device", action="store_true",
                    help="all ranks on cuda:0 (functional check of N > 1 with gloo)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank, world, local = dist_env()
    workers = os.cpu_count() or 1

    if args.impl == "reference":
        return reference_arm(args, rank, world, workers)

    import torch

    # --dist-backend gloo --one-device: every rank on cuda:0 with host-side
    # collectives -- a functional check of the N > 1 paths on a 1-GPU box
    # (timings from it are not scaling numbers)
    torch.cuda.set_device(0 if args.one_device else local)
    if world > 1:
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    peak, src = hbm_peak()
    r = run_sfft_arm(args, world, rank)
    h = None if args.no_hash else run_hash_arm(args, world, rank)
    out = {
        "metric": METRIC, "value": round(r["ms"] / 1e3 / world, 6), "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config(world),
        "parity": r["parity"],
        "e2e": {"value": round(r["e2e_ms"] / 1e3 / world, 6), "unit": "s",
                "h2d_bytes_per_step": r["h2d"], "d2h_bytes_per_step": r["d2h"]},
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
        "roofline_sfft": roofline_sfft(r, peak, src),
    }
    if h is not None:
        rl = roofline_hash(h, peak, src)
        out["roofline"] = rl
        out["hashing"] = {
            "workload": f"cfg4: |Gamma|=2^{int(math.log2(h['n']))} rows of [-4096,4096]^10 in "
                        f"HBM (the reference's default_rng({CFG4_SEED}) stream), s=1e4, "
                        f"L={h['L']}, M={h['M']}",
            "value": round(h["n"] / (h["hash_ms"] * 1e-3), 1), "unit": "candidates/s",
            "value_semantics": ("one Gamma sharded over the ranks (strong scaling): all "
                                "candidates / max over ranks of the hashing kernel time")
            if world > 1 else "candidates / hashing kernel time",
            "hash_kernel_ms": round(h["hash_ms"], 4),
            "detect_and_compute_ms": round(h["ms"], 3),
            "detect_candidates_per_s": round(h["n"] / (h["ms"] * 1e-3), 1),
            "gather_path_ms": round(h["path_ms"], 4),
            "gather_path_gbs_survey_bytes": round(
                (h["n_local"] * 8 * h["d"] + h["n_local"] * 8 + h["L"] * h["M"] * 16
                 + h["n_det"] * 24) / (h["path_ms"] * 1e-3) / 1e9, 1),
            "parity": h["parity"], "clocks": h["clocks"],
            "gamma_generation_ms": round(h["gamma_generation_ms"], 2),
            "gamma_generation_note": "device generation in the reference's PCG64 stream "
                                     "(csrc/boxgen.cu) + canonicalisation (csrc/canon.cu); "
                                     "reference host generation 432.6 s (SURVEY 8(d))",
            "e2e": {"value": round(h["n"] / (h["e2e_ms"] * 1e-3), 1),
                    "unit": "candidates/s",
                    "ms": round(h["e2e_ms"], 2), "h2d_bytes_per_step": h["h2d"],
                    "d2h_bytes_per_step": h["d2h"],
                    "h2d_alone_ms": round(h["h2d_ms"], 2),
                    "e2e_over_h2d": round(h["e2e_ms"] / h["h2d_ms"], 3),
                    "input": "plain host FreqSet over pinned rows (no bounds, no memo)"},
        }
    if rank == 0 and world == 1 and not args.no_configs:
        out["configs"] = all_configs(peak, src, workers, cpu=not args.no_cpu)
    if rank == 0 and world == 1 and not args.no_cpu:
        w = r["workload"]
        secs, samples, nsup = cpu_sfft_structured(w, workers)
        dense = cpu_sfft_dense_bounded(w, args.cpu_budget, workers)
        out["cpu_baseline"] = {
            "value": round(secs, 3), "unit": "s", "cores": workers, "kind": "port",
            "extrapolated": False,
            "sample": (f"the whole metric instance, run to completion and timed: oracle/port "
                       f"sfft driver with the reference's structured lattice sampler "
                       f"(bincount + numpy ifft) and numpy pocketfft DFTs on {workers} "
                       f"threads, gather by "
                       f"{'the reference compiled _core (oracle/_ref)' if _ref_core() else 'oracle C'}"
                       f"; {samples} samples, support {nsup}"),
            "algorithm_matched": True,
            "dense_as_shipped": dense,
        }
        if h is not None:
            rate, kind, hi = cpu_hash_bounded(h["rows_host_sample"], h["zmat"], h["M"],
                                              h["ghat"], h["theta0"], workers)
            out["hashing"]["cpu_baseline"] = {
                "value": round(rate, 1), "unit": "candidates/s", "cores": workers, "kind": kind,
                "sample": f"{hi['calls']} detect_gather calls on {hi['rows_per_call']} cfg4 rows "
                          f"(threads={workers}), {hi['elapsed_s']:.1f}s"}
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def _timed(fn, reps=3):
    import torch

    fn()
    torch.cuda.synchronize()
    ts, out = [], None
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


def _phases(per):
    ph = {k[len("stage:"):]: round(v[0], 3) for k, v in per.items() if k.startswith("stage:")}
    rest = {k: round(v[0], 3) for k, v in per.items()
            if not k.startswith("stage:") and k != "sfftb_sfft_stage"}
    return ph, rest


def all_configs(peak, src, workers, cpu=True):
    """SURVEY 8(d)'s per-config rows on this GPU: device time of the entry
    point (median of 3 after a warm-up), its phase breakdown from one
    instrumented run, the dominant kernel against its roofline, and the
    algorithm-matched CPU reference on the same inputs in the same run."""
    import torch

    import paper_2006_13053_b200 as pkg
    from oracle import port

    out = {}
    for name in ("config2", "config3", "config5"):
        w = getattr(workloads, name)()
        poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
        box = pkg.Box(w.d, w.lo, w.hi)
        params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)

        def step():
            return pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma,
                                                 noise_seed=w.noise_seed),
                            box, params, seed=w.seed)

        ms, res = _timed(step)
        per, per_list, shapes = sfft_profile(step)
        ph, rest = _phases(per)
        rl = roofline_sfft({"ms": ms, "per_entry": per, "per_list": per_list,
                            "shapes": shapes}, peak, src)
        ent = {"entry": "sfft", "ms": round(ms, 3), "samples": res.sample_count,
               "support": len(res.support), "stages": len(res.stage_log),
               "phases_ms": ph, "other_entry_points_ms": rest,
               "dominant": {k: rl.get(k) for k in ("kernel", "ms_total", "share_of_step",
                                                    "achieved", "unit", "frac", "fp64_tflops",
                                                    "fp64_frac")}}
        if w.sigma == 0:
            ent["exact_support"] = bool(np.array_equal(
                res.support.elems, w.support[np.lexsort(w.support.T[::-1])]))
        if cpu:
            secs, samples, nsup = cpu_sfft_structured(w, workers)
            ent["cpu"] = {"value": round(secs, 3), "unit": "s", "cores": workers,
                          "kind": "port", "algorithm_matched": True,
                          "same_samples": samples == res.sample_count,
                          "same_support_size": nsup == len(res.support)}
        out[w.name] = ent

    # config 1: fixed Gamma, launch-latency bound
    w = workloads.config1()
    G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
    cfg = pkg.draw_config(G, w.s, 0.1, rng=w.rng)
    orc = pkg.oracle_from_poly(pkg.SparsePoly(G.take(w.support_idx), w.coeffs))
    smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M,
                                     torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                     1, cfg.L, w.d).contiguous()
    ms, det = _timed(lambda: pkg.detect_and_compute(smp, cfg, G).detected_idx)
    from paper_2006_13053_b200 import _native

    torch.cuda.synchronize()
    with _native.Timeline() as tl:
        pkg.detect_and_compute(smp, cfg, G).detected_idx  # noqa: B018
    per = {k: round(sum(v) * 1e3, 2) for k, v in tl.ms().items()}
    n, d, L, M = len(G), w.d, cfg.L, cfg.shared_M
    bytes_ = n * (8 * d + 8) + L * M * 16
    ent = {"entry": "detect_and_compute", "us": round(ms * 1e3, 1),
           "candidates_per_s": round(n / (ms * 1e-3), 1),
           "detected_equals_support": bool(np.array_equal(det, np.sort(w.support_idx))),
           "breakdown_us": per,
           "roofline": {"bound": "launch latency", "algorithmic_bytes": bytes_,
                        "achieved_gbs": round(bytes_ / (ms * 1e-3) / 1e9, 2), "peak": peak,
                        "frac": round(bytes_ / (ms * 1e-3) / 1e9 / peak, 5),
                        "launches": len(tl.records)}}
    if cpu:
        smp_h = [s for s in smp.cpu().numpy()]
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            port.detect_and_compute(smp_h, M, cfg.zmat(), w.gamma,
                                    gather_backend="reference" if _ref_core() else "port")
            ts.append(time.perf_counter() - t0)
        ent["cpu"] = {"value": round(min(ts) * 1e6, 1), "unit": "us", "cores": 1,
                      "kind": "port", "what": "detect_and_compute on the host (pocketfft DFTs "
                      "+ the reference's compiled gather), best of 3"}
    out["cfg1"] = ent
    return out


def reference_arm(args, rank, world, workers):
    """CPU reference arm on this host's cores, same workload as our arm:
    each step runs the algorithm-matched reference sfft on the metric
    instance to completion (cpu_sfft_structured), timed; the as-shipped
    dense run is reported beside it (bounded, extrapolated, flagged)."""
    if rank != 0:
        return
    w = workloads.metric_config()
    vals = []
    for k in range(args.warmup + args.steps):
        secs, samples, nsup = cpu_sfft_structured(w, workers)
        if k >= args.warmup:
            vals.append(secs)
    value = statistics.mean(vals)
    dense = cpu_sfft_dense_bounded(w, max(2.0, args.cpu_budget / 2), workers)
    kind = "port"
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(value * 1e3, 1), "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           # our arm's config verbatim (the driver compares the two objects); its
           # parallelism / l2 keys describe the GPU arm's measurement
           "config": arm_config(world),
           "cpu_baseline": {"value": round(value, 4), "unit": "s", "cores": workers, "kind": kind,
                            "extrapolated": False, "algorithm_matched": True,
                            "sample": (f"per step: the whole metric instance ({samples} samples, "
                                       f"support {nsup}) through oracle/port's sfft driver with "
                                       f"the reference's structured sampler, numpy pocketfft "
                                       f"and the reference's compiled gather on {workers} "
                                       f"threads, run to completion")},
           "dense_as_shipped": dense,
           "e2e": {"value": round(value, 4), "unit": "s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
