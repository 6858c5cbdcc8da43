"""Run one BASELINE sfft config a few times (profiling helper for ncu launch
lists): python tools/one_config.py config5 [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

w = getattr(workloads, sys.argv[1])()
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
for _ in range(reps):
    pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed),
             pkg.Box(w.d, w.lo, w.hi), pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r),
             seed=w.seed)
torch.cuda.synchronize()
print("done")
