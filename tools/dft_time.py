"""Batched prime-length DFT timing: python tools/dft_time.py M batch"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
from paper_2006_13053_b200 import _dev, _native  # noqa: E402
from paper_2006_13053_b200.dft import dft_batch  # noqa: E402

M, B = int(sys.argv[1]), int(sys.argv[2])
x = torch.randn((B, M), dtype=torch.complex128, device="cuda")
dft_batch(x, M)
torch.cuda.synchronize()
with _native.Timeline() as tl:
    for _ in range(10):
        dft_batch(x, M)
ms = sorted(tl.ms()["sfftb_dft"])
print(f"dft M={M} batch={B}: min {ms[0] * 1e3:.1f} us med {ms[5] * 1e3:.1f} us")
