"""Fused sampler->detection transforms at the metric stage shape (profiling
helper): G=5 groups x L=37 lattices, M=20663 (N=65536).
    python tools/prof_fused.py [M] [G] [L] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13053_b200 import _dev, _engine, _native  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 20663
G = int(sys.argv[2]) if len(sys.argv) > 2 else 5
L = int(sys.argv[3]) if len(sys.argv) > 3 else 37
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
rng = np.random.default_rng(0)
bins = np.zeros((G * L, M), dtype=np.complex128)
for row in bins:
    nz = rng.choice(M, size=1000, replace=False)
    row[nz] = rng.normal(size=1000) + 1j * rng.normal(size=1000)
b = _dev.upload(bins)
_engine.sample_spectra_fused(b, M, G, L, 1, 0, 0.0)
torch.cuda.synchronize()
with _native.Timeline() as tl:
    for _ in range(reps):
        _engine.sample_spectra_fused(b, M, G, L, 1, 0, 0.0)
ms = tl.ms()["sfftb_sample_detect_dft"]
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import bluestein_N  # noqa: E402

N = bluestein_N(M)
rows = G * L
print(f"fused M={M} N={N} rows={rows}: ms={[round(v, 4) for v in ms]}; "
      f"5-pass traffic {rows * (2 * M + 8 * N) * 16 / (min(ms) * 1e-3) / 1e9:.0f} GB/s")
