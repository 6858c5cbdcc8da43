"""Host-side cost of one metric-instance reconstruction: wall time of the
sfft() call (before its final sync) and the top Python functions.
    python tools/host_profile.py"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
poly.device()


def step():
    return pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)


for _ in range(5):
    step()
torch.cuda.synchronize()
ts = []
for _ in range(10):
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    step()
    b.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    ts.append((a.elapsed_time(b), (t1 - t0) * 1e3))
for dev, host in ts:
    print(f"device {dev:.3f} ms  host {host:.3f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
