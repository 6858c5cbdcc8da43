"""Standalone grid top-s timing (cfg5-shaped: 5 groups x 150k, s = 2000).
    python tools/topk_time.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2006_13053_b200 import _dev, _engine, _native  # noqa: E402

rng = np.random.default_rng(0)
G, cap = 5, 150_000
idx = _dev.upload(np.tile(np.arange(cap), G))
co = _dev.upload(rng.standard_normal(G * cap) + 1j * rng.standard_normal(G * cap))
cnt = torch.full((G,), cap, dtype=torch.int64, device="cuda")
for _ in range(3):
    _engine.topk(idx, co, cnt, G, cap, 0.0, 2000, grid=True)
torch.cuda.synchronize()
with _native.Timeline() as tl:
    for _ in range(10):
        _engine.topk(idx, co, cnt, G, cap, 0.0, 2000, grid=True)
ms = sorted(tl.ms()["sfftb_topk_grid"])
print(f"topk_grid G={G} cap={cap}: min {ms[0] * 1e3:.1f} us med {ms[5] * 1e3:.1f} us")
