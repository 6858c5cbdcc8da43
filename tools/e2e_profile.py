"""Where the metric's e2e time goes beyond the device-resident step:
    python tools/e2e_profile.py"""
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


def resident():
    return pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)


def e2e():
    p2 = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
    r2 = pkg.sfft(pkg.oracle_from_poly(p2), box, params, seed=w.seed)
    return r2.support.elems, r2.coeffs


for fn in (resident, e2e):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{fn.__name__}: med {ts[5]:.3f} ms")
t0 = time.perf_counter()
p2 = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
o = pkg.oracle_from_poly(p2)
t1 = time.perf_counter()
p2.device()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"construct {1e6 * (t1 - t0):.0f} us, upload {1e6 * (t2 - t1):.0f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    e2e()
pr.disable()
pstats.Stats(pr).sort_stats("cumtime").print_stats(18)
