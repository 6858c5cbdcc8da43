"""Batched prime-length DFT launch for timing / ncu (profiling helper).
    python tools/prof_fft.py [M] [batch] [reps]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13053_b200 import _dev, _native  # noqa: E402
from paper_2006_13053_b200.dft import dft_batch  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 20663
B = int(sys.argv[2]) if len(sys.argv) > 2 else 195
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rng = np.random.default_rng(0)
x = _dev.upload(rng.normal(size=(B, M)) + 1j * rng.normal(size=(B, M)))
out = torch.empty_like(x)
dft_batch(x, M, out=out)
torch.cuda.synchronize()
with _native.Timeline() as tl:
    for _ in range(reps):
        dft_batch(x, M, out=out)
ms = tl.ms()["sfftb_dft"]
N = 1
while N < 2 * M - 1:
    N *= 2
N = max(N, 256)
flops = B * 2 * 5 * N * np.log2(N)
print(f"dft M={M} N={N} batch={B}: ms={[round(v, 4) for v in ms]} -> "
      f"{flops / (min(ms) * 1e-3) / 1e12:.2f} TFLOP/s (2 pow2 FFTs/transform), "
      f"{B * M * 32 / (min(ms) * 1e-3) / 1e9:.0f} GB/s in+out")
ref = np.fft.fft(_dev.download(x[:2]), axis=1) / M
print("max err vs numpy:", float(np.max(np.abs(_dev.download(out[:2]) - ref))))
