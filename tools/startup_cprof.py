"""cProfile of sfft's host path up to the first stage launch (metric instance).
    python tools/startup_cprof.py"""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _stage  # noqa: E402
import workloads  # noqa: E402

w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
poly.device()
for _ in range(3):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()


class Stop(Exception):
    pass


orig = _stage.run


def run(desc, stream=None):
    raise Stop


_stage.run = run
pr = cProfile.Profile()
for _ in range(50):
    pr.enable()
    try:
        pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
    except Stop:
        pass
    pr.disable()
    torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
