"""Reconstruction time of named sfft workloads (median of 10 after 3 warm-ups).
    python tools/rep_cfg.py config2 metric_config ..."""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

for name in sys.argv[1:]:
    w = getattr(workloads, name)()
    poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)

    def run():
        return pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed),
                        pkg.Box(w.d, w.lo, w.hi),
                        pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r), seed=w.seed)

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{name}: min {ts[0]:.3f} med {ts[5]:.3f} ms")
