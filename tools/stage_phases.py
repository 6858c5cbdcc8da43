"""Per-stage phase device times (CUDA events recorded by sfftb_sfft_stage)
of one metric-size sfft reconstruction."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _native  # noqa: E402
import workloads  # noqa: E402

w = getattr(workloads, sys.argv[1] if len(sys.argv) > 1 else "metric_config")()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
def oracle():
    return pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed)


for _ in range(3):
    pkg.sfft(oracle(), box, params, seed=w.seed)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    with _native.Timeline() as tl:
        pkg.sfft(oracle(), box, params, seed=w.seed)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    ms = tl.ms()
    print(f"rep {rep}: wall {wall:.2f} ms")
    for k, v in ms.items():
        print(f"  {k:28s} total {sum(v):7.3f}  " + " ".join(f"{x:.3f}" for x in v))
