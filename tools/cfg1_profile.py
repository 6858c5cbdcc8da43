"""Host-side profile of config 1's detect_and_compute (device-resident inputs).
    python tools/cfg1_profile.py"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

w = workloads.config1()
G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
cfg = pkg.draw_config(G, w.s, 0.1, rng=w.rng)
orc = pkg.oracle_from_poly(pkg.SparsePoly(G.take(w.support_idx), w.coeffs))
smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M,
                                 torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                 1, cfg.L, w.d).contiguous()


def step():
    return pkg.detect_and_compute(smp, cfg, G).detected_idx


for _ in range(20):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    step()
torch.cuda.synchronize()
print(f"wall per call {(time.perf_counter() - t0) / 200 * 1e6:.1f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
