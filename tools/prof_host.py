"""cProfile of one metric-size sfft reconstruction (host overhead hunt)."""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)


def step():
    return pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)


for _ in range(3):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
step()
torch.cuda.synchronize()
print("wall ms", (time.perf_counter() - t0) * 1e3)
pr = cProfile.Profile()
pr.enable()
step()
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(30)
st.sort_stats("tottime").print_stats(25)
