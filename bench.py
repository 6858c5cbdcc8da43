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
  * hashing -- config 4: |Gamma| = 2^26 candidates in [-4096,4096]^10 (HBM
               resident), s=1e4, L=47, M=103307: candidates hashed per
               second by the hashing kernel and by the whole detection call,
               with its roofline; plus an e2e through detect_and_compute from
               pinned host rows.
  * roofline -- the hashing kernel vs measured HBM bandwidth (the metric's
               "vs HBM roofline"); roofline_sfft -- the dominant kernel of
               the reconstruction step.
  * cpu_baseline -- the CPU oracle / the reference's compiled kernel on this
               host's cores over a bounded sample, scaled to the unit.
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

    t = torch.tensor([float(x)], dtype=torch.float64, device="cuda")
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

    # per-entry-point / per-stage-phase device times of one instrumented step
    # (dominant kernel), with the shapes of every stage call
    from paper_2006_13053_b200 import _stage

    shapes = []
    orig_run = _stage.run

    def run_rec(desc, stream=None):
        if desc.phase in (0, 1, 4):  # the calls that run transforms
            shapes.append((desc.G, desc.L, desc.M, bool(desc.fused)))
        return orig_run(desc, stream)

    flush_l2(flush)
    torch.cuda.synchronize()
    _stage.run = run_rec
    try:
        with _native.Timeline() as tl:
            step()
        raw = tl.ms()
    finally:
        _stage.run = orig_run
    per = {k: (sum(v), len(v)) for k, v in raw.items()}
    per_list = {k: v for k, v in raw.items()}

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


def device_gamma(n, d, N, seed):
    """2^26-scale candidate set generated in HBM by the package's own
    kernels: uniform rows of [-N, N]^d (Philox stream), canonicalised
    (lexicographic radix sort + de-dup, csrc/canon.cu).  Returns (FreqSet,
    generation ms)."""
    import torch

    import paper_2006_13053_b200 as pkg

    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    G = pkg.random_box_device(pkg.Box(d, -N, N), n, seed)
    b.record()
    torch.cuda.synchronize()
    return G, a.elapsed_time(b)


def run_hash_arm(args, world, rank):
    import torch

    import paper_2006_13053_b200 as pkg
    from oracle import port
    from paper_2006_13053_b200 import _dev, _native

    n, d, N, s = args.hash_rows, 10, 4096, 10_000
    G, gen_ms = device_gamma(n, d, N, 4242 + rank)
    rows = G.device()
    G.memo("bounds", lambda: np.array([[-N, N]] * d, dtype=np.int64))  # known by construction
    rng = np.random.default_rng(2026 + rank)
    sup_idx = np.sort(rng.choice(n, size=s, replace=False))
    coeffs = workloads.mag_phase_coeffs(s, rng)
    I = G.take(sup_idx)
    poly = pkg.SparsePoly(I, coeffs)
    cfg = pkg.draw_config(G, s, 0.1, rng=rng)
    M, L = cfg.shared_M, cfg.L
    orc = pkg.oracle_from_poly(poly)
    samples = orc.sample_lattices_device(cfg.zmat_device(), M,
                                         torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                         1, L, d)
    samples = samples.contiguous()

    def step():
        return pkg.detect_and_compute(samples, cfg, G)

    for _ in range(args.warmup):
        res = step()
        res.detected_idx  # noqa: B018
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
                res = step()
                b.record()
            per = tl.ms()
            times.append(a.elapsed_time(b))
            hash_ms.append(sum(per["sfftb_hash_hits"]))
            path_ms.append(sum(sum(per.get(k, [0.0])) for k in (
                "sfftb_nonzero_bitmap", "sfftb_hash_hits", "sfftb_compact_mask",
                "sfftb_medians")))
    clocks = clk.summary()
    idx = res.detected_idx
    parity = {"detected_equals_support": bool(np.array_equal(idx, sup_idx)),
              "coeff_max_rel_err_vs_truth": float(np.max(np.abs(res.coeffs - coeffs))
                                                  / np.max(np.abs(coeffs)))}
    # bit-exact hits on a random sample of rows against the C oracle
    samp = np.sort(rng.choice(n, size=1 << 16, replace=False))
    samp_t = torch.as_tensor(samp, device="cuda")
    rows_h = _dev.download(rows.index_select(0, samp_t))
    b = pkg.detect._gather(samples, cfg, G, pkg.ZeroTest(res.theta_zero), False)
    ghat = _dev.download(b.ghat)
    want, _ = port.gather_c(rows_h % M, cfg.zmat(), M, ghat, res.theta_zero, L / 2, False)
    got = _dev.download(b.hits)[samp]
    parity["sampled_hits_bitexact_vs_oracle"] = bool(np.array_equal(got, want))
    parity["sampled_rows"] = int(samp.size)
    del b

    # e2e: pinned host rows -> detect_and_compute (H2D inside) -> results to host
    host = torch.empty((n, d), dtype=torch.int64, pin_memory=True)
    host.copy_(rows)
    hnp = host.numpy()
    e2e = []
    d2h = 0
    nrep = max(1, min(args.steps, 3))
    for rep in range(nrep + 1):  # rep 0 warms the pinned result buffers (untimed)
        torch.cuda.synchronize()
        Gh = pkg.FreqSet(d, hnp, _sorted=True)
        Gh.memo("bounds", lambda: np.array([[-N, N]] * d, dtype=np.int64))
        a = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        a.record()
        r2 = pkg.detect_and_compute(samples, cfg, Gh)
        out = (r2.hits, r2.detected_idx, r2.coeffs)
        e.record()
        torch.cuda.synchronize()
        if rep:
            e2e.append(a.elapsed_time(e))
        d2h = sum(x.nbytes for x in out)
        del Gh, r2, out
    W = int(_native.lib().sfftb_bitmap_words(M))
    return {"n": n, "d": d, "L": L, "M": M, "s": s, "W": W, "n_det": int(idx.size),
            "ms": max_over_ranks(statistics.mean(times), world),
            "hash_ms": max_over_ranks(statistics.mean(hash_ms), world),
            "path_ms": max_over_ranks(statistics.mean(path_ms), world),
            "clocks": clocks, "parity": parity, "gamma_generation_ms": gen_ms,
            "e2e_ms": max_over_ranks(statistics.mean(e2e), world), "h2d": n * d * 8,
            "d2h": d2h, "rows_host_sample": rows_h[:1 << 20], "ghat": ghat,
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


def cpu_sfft_bounded(w, budget_s, workers):
    """The oracle's sfft (dense sampling, as the reference ships it) run for
    `budget_s` seconds, extrapolated by sample count to the full run."""
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
    return est, {"samples_done": int(orc.count), "samples_total": total,
                 "elapsed_s": elapsed, "finished": finished}


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
    """DRAM bytes per launch from the committed ncu capture
    (profiles/r01/traffic.json), or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01",
                        "traffic.json")
    try:
        with open(path) as f:
            ent = json.load(f)[kernel]
        return ent
    except (OSError, KeyError, ValueError):
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


def _imad_bound(h):
    """The hash kernel's integer-pipe floor: 12 IMAD-pipe ops per (row,
    lattice) pair (10 for the dot product, 2 for the reduction; DESIGN.md
    K3) at the measured IMAD lane rate."""
    pk = _pipe_peaks()
    if not pk:
        return {}
    pairs = h["n"] * h["L"]
    floor_ms = pairs * 12 / (pk["imad_lanes_per_clk_per_sm"] * pk["sms"]
                             * pk["clock_mhz"] * 1e6) * 1e3
    return {"int_pipe": {"imad_per_pair": 12, "floor_ms": round(floor_ms, 3),
                         "frac_of_floor": round(floor_ms / h["hash_ms"], 4),
                         "note": "exact int64 residues need d multiply-adds per pair on the "
                                 "IMAD pipe; its floor caps this kernel at "
                                 f"{round(h['n'] * (8 * h['d'] + 8) / (floor_ms * 1e-3) / 1e9)} "
                                 "GB/s of algorithmic traffic"}}


def roofline_hash(h, peak, src):
    """Algorithmic bytes of one hashing launch: rows (n*8d) + int64 hits
    (n*8) + the L bitmaps (L*W*4) + the detected-row bitmask (n/8)."""
    bytes_ = h["n"] * 8 * h["d"] + h["n"] * 8 + h["L"] * h["W"] * 4 + h["n"] // 8
    ach = bytes_ / (h["hash_ms"] * 1e-3) / 1e9
    tr = measured_traffic("hash_rows")
    traffic = None
    if tr and tr.get("rows") == h["n"] and tr.get("L") == h["L"] and tr.get("M") == h["M"]:
        traffic = tr["dram_read"] + tr["dram_write"]
    return {"bound": "hbm", "kernel": "hash_rows (sfftb_hash_hits)", "achieved": round(ach, 1),
            "peak": peak, "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": traffic,
            "algorithmic_bytes": bytes_, "peak_source": src,
            "launch_ms": round(h["hash_ms"], 4), **_imad_bound(h)}


def fft_flops(N):
    return 5.0 * N * math.log2(N)


def bluestein_N(M):
    """The library's convolution length (csrc/fft.cu bluestein_N): the
    smallest power of two >= max(2M-1, 256), or 192*{128, 256} when that is
    smaller and above the single-CTA sizes."""
    N = 256
    while N < 2 * M - 1:
        N *= 2
    if N > 8192:
        for c in (24576, 49152):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--hash-rows", type=int, default=1 << 26)
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-hash", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config entry-point times (configs 1, 2, 3, 5)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank, world, local = dist_env()
    workers = os.cpu_count() or 1

    if args.impl == "reference":
        return reference_arm(args, rank, world, workers)

    import torch

    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    peak, src = hbm_peak()
    r = run_sfft_arm(args, world, rank)
    h = None if args.no_hash else run_hash_arm(args, world, rank)
    out = {
        "metric": METRIC, "value": round(r["ms"] / 1e3 / world, 6), "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(r["ms"], 3), "higher_is_better": False, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "d10_s1000: sfft over [-32,32]^10, s=1000 random frequencies, "
                               "|c|~U[1,10], r=5, theta=1e-12, delta=0.9, seed 7 "
                               "(BASELINE config-2 generator at the metric's s=1000)",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                   "l2": "flushed (256 MB write) between timed steps",
                   "value_semantics": "seconds per reconstruction (replicas: step time / N)"},
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
                        f"HBM, s=1e4, L={h['L']}, M={h['M']}",
            "value": round(world * h["n"] / (h["hash_ms"] * 1e-3), 1), "unit": "candidates/s",
            "value_semantics": "all ranks' candidates (one 2^26 set per rank) / max kernel time",
            "hash_kernel_ms": round(h["hash_ms"], 4),
            "detect_and_compute_ms": round(h["ms"], 3),
            "detect_candidates_per_s": round(h["n"] / (h["ms"] * 1e-3), 1),
            "gather_path_ms": round(h["path_ms"], 4),
            "gather_path_gbs_survey_bytes": round(
                (h["n"] * 8 * h["d"] + h["n"] * 8 + h["L"] * h["M"] * 16 + h["n_det"] * 24)
                / (h["path_ms"] * 1e-3) / 1e9, 1),
            "parity": h["parity"], "clocks": h["clocks"],
            "gamma_generation_ms": round(h["gamma_generation_ms"], 2),
            "gamma_generation_note": "device Philox rows + canonicalisation (csrc/canon.cu); "
                                     "reference host Gamma generation 432.6 s (SURVEY 8(d))",
            "e2e": {"value": round(world * h["n"] / (h["e2e_ms"] * 1e-3), 1),
                    "unit": "candidates/s",
                    "ms": round(h["e2e_ms"], 2), "h2d_bytes_per_step": h["h2d"],
                    "d2h_bytes_per_step": h["d2h"]},
        }
    if rank == 0 and world == 1 and not args.no_configs:
        out["other_configs"] = all_configs()
    if rank == 0 and world == 1 and not args.no_cpu:
        est, info = cpu_sfft_bounded(r["workload"], args.cpu_budget, workers)
        out["cpu_baseline"] = {
            "value": round(est, 3), "unit": "s", "cores": workers,
            "kind": "reference" if _ref_core() else "port",
            "sample": (f"oracle/port sfft with dense sampling (the reference's as-shipped "
                       f"evaluate_many) threaded over {workers} cores, gather by "
                       f"{'the reference compiled _core' if _ref_core() else 'oracle C'}; "
                       f"ran {info['elapsed_s']:.1f}s = {info['samples_done']} of "
                       f"{info['samples_total']} samples, extrapolated by sample count"),
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


def all_configs(reps=3):
    """Entry-point device time of the other BASELINE configs on this GPU
    (median of `reps` after one warm-up; parity = exact support for the
    exact-sparse configs, planted support for config 1)."""
    import torch

    import paper_2006_13053_b200 as pkg

    def timed(fn):
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

    out = {}
    for name in ("config2", "config3", "config5"):
        w = getattr(workloads, name)()
        poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
        box = pkg.Box(w.d, w.lo, w.hi)
        params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
        ms, res = timed(lambda: pkg.sfft(pkg.oracle_from_poly(
            poly, noise_sigma=w.sigma, noise_seed=w.noise_seed), box, params, seed=w.seed))
        ent = {"entry": "sfft", "ms": round(ms, 3), "samples": res.sample_count,
               "support": len(res.support)}
        if w.sigma == 0:
            ent["exact_support"] = bool(np.array_equal(
                res.support.elems, w.support[np.lexsort(w.support.T[::-1])]))
        out[w.name] = ent
    w = workloads.config1()
    G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
    cfg = pkg.draw_config(G, w.s, 0.1, rng=w.rng)
    orc = pkg.oracle_from_poly(pkg.SparsePoly(G.take(w.support_idx), w.coeffs))
    smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M,
                                     torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                     1, cfg.L, w.d).contiguous()
    ms, det = timed(lambda: pkg.detect_and_compute(smp, cfg, G).detected_idx)
    out["cfg1"] = {"entry": "detect_and_compute", "ms": round(ms, 3),
                   "detected_equals_support": bool(np.array_equal(det,
                                                                  np.sort(w.support_idx)))}
    return out


def reference_arm(args, rank, world, workers):
    """CPU reference arm: the reference's path on this host's cores."""
    if rank != 0:
        return
    w = workloads.metric_config()
    vals = []
    info = None
    budget = max(2.0, args.cpu_budget / 2.5)
    for k in range(args.warmup + args.steps):
        est, info = cpu_sfft_bounded(w, budget, workers)
        if k >= args.warmup:
            vals.append(est)
    value = statistics.mean(vals)
    kind = "reference" if _ref_core() else "port"
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": round(value * 1e3, 1), "higher_is_better": False, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "d10_s1000: sfft over [-32,32]^10, s=1000 random "
                                  "frequencies, r=5, theta=1e-12, delta=0.9, seed 7"},
           "cpu_baseline": {"value": round(value, 3), "unit": "s", "cores": workers, "kind": kind,
                            "sample": (f"per step: oracle/port sfft (dense sampling as the "
                                       f"reference ships it, {workers} threads) run "
                                       f"{budget:.0f}s = {info['samples_done']} of "
                                       f"{info['samples_total']} samples, extrapolated")},
           "e2e": {"value": round(value, 3), "unit": "s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
