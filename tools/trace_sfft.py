"""Per-stage host/device timeline of one metric-size sfft (latency hunt).

Wraps _native.call to log (host time at launch, entry point) and records a
CUDA event per call; prints host launch gaps and device busy spans per stage.
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _dev, _native  # noqa: E402
import workloads  # noqa: E402

w = getattr(workloads, sys.argv[1] if len(sys.argv) > 1 else "metric_config")()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
for _ in range(3):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()

log = []
orig_call = _native.call
orig_dl = _dev.download


def call(name, *args):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    h = time.perf_counter()
    e0.record()
    orig_call(name, *args)
    e1.record()
    log.append((name, h, time.perf_counter(), e0, e1))


def download(t):
    h = time.perf_counter()
    r = orig_dl(t)
    log.append(("<download>", h, time.perf_counter(), None, None))
    return r


from paper_2006_13053_b200 import _stage, dimincr  # noqa: E402

orig_run = _stage.run


def run(desc, stream=None):
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    st = torch.cuda.current_stream() if stream is None else torch.cuda.ExternalStream(stream)
    h = time.perf_counter()
    e0.record(st)
    orig_run(desc, stream)
    e1.record(st)
    kind = {0: "stage", 1: "spectra", 2: "detect", 3: "sampler", 4: "transforms"}[int(desc.phase)]
    log.append((f"<{kind} G={desc.G} L={desc.L} M={desc.M} n={desc.n}>", h, time.perf_counter(),
                e0, e1))


orig_step1 = dimincr.step1_components


def step1(*a, **k):
    h = time.perf_counter()
    out = orig_step1(*a, **k)
    log.append(("<step1_components>", h, time.perf_counter(), None, None))
    return out


_native.call = call
_dev.download = download
_stage.run = run
dimincr.step1_components = step1
start_ev = torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
start_ev.record()
pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
tot = (time.perf_counter() - t0) * 1e3
print(f"total wall {tot:.2f} ms")
for name, h0, h1, e0, e1 in log:
    dev = ""
    if e0 is not None:
        dev = f"dev {start_ev.elapsed_time(e0):8.3f}->{start_ev.elapsed_time(e1):8.3f}"
    print(f"host {1e3 * (h0 - t0):8.3f}->{1e3 * (h1 - t0):8.3f}  {dev:28s} {name}")
