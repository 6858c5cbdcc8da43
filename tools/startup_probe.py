"""Host time from sfft() entry to its first device launch (metric instance).
    python tools/startup_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _native, _stage  # noqa: E402
import workloads  # noqa: E402

w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
poly.device()
first = {}
orig_run, orig_call = _stage.run, _native.call


def run(desc, stream=None):
    first.setdefault("stage", time.perf_counter())
    return orig_run(desc, stream)


def call(name, *a):
    first.setdefault(name, time.perf_counter())
    return orig_call(name, *a)


_stage.run = run
_native.call = call
for rep in range(6):
    first.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    if rep >= 2:
        items = sorted(first.items(), key=lambda kv: kv[1])[:4]
        print(f"total host {1e3 * (t1 - t0):.3f} ms; first launches: " +
              ", ".join(f"{k} +{1e6 * (v - t0):.0f} us" for k, v in items))
