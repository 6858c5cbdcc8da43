"""cProfile of the host side of repeated sfft calls for one config
(default config2, which is bound by host time per stage)."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

w = getattr(workloads, sys.argv[1] if len(sys.argv) > 1 else "config2")()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)


def run():
    return pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed),
                    box, params, seed=w.seed)


for _ in range(5):
    run()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    run()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
