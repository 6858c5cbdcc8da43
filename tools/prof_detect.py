"""Per-entry-point device times of one cfg4-shaped detect_and_compute.
    python tools/prof_detect.py [log2_rows]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _native  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
G = pkg.random_box_device(pkg.Box(10, -4096, 4096), 1 << lg, 5)
G.memo("bounds", lambda: np.array([[-4096, 4096]] * 10, dtype=np.int64))
rng = np.random.default_rng(1)
sup = np.sort(rng.choice(len(G), size=10_000, replace=False))
poly = pkg.SparsePoly(G.take(sup), rng.normal(size=10_000) + 1j * rng.normal(size=10_000) + 3)
cfg = pkg.draw_config(G, 10_000, 0.1, rng=rng)
orc = pkg.oracle_from_poly(poly)
smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M,
                                 torch.zeros((1, 1), dtype=torch.float64, device="cuda"), 1,
                                 cfg.L, 10).contiguous()
for _ in range(2):
    pkg.detect_and_compute(smp, cfg, G).detected_idx
torch.cuda.synchronize()
with _native.Timeline() as tl:
    res = pkg.detect_and_compute(smp, cfg, G)
    res.detected_idx
for k, v in tl.ms().items():
    print(f"{k:28s} {sum(v):8.3f} ms  x{len(v)}")
print("detected", len(res.detected_idx), "L", cfg.L, "M", cfg.shared_M)
