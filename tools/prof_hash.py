"""Standalone cfg4-shaped hashing launch for ncu (profiling helper).

n = 2^26 rows of [-4096,4096]^10 (int64), L = 47 lattices, M = 103307,
bitmaps with ~9% set bits (the occupancy of cfg4's ghat), 32-bit path.
    python tools/prof_hash.py [log2_rows] [reps]
"""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13053_b200 import _dev, _native  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
M = int(sys.argv[3]) if len(sys.argv) > 3 else 103307
L = int(sys.argv[4]) if len(sys.argv) > 4 else 47
N = int(sys.argv[5]) if len(sys.argv) > 5 else 4096  # coordinate span; 32 = config 4's box
n, d = 1 << lg, 10
g = torch.Generator(device="cuda")
g.manual_seed(1)
rows = torch.randint(-N, N + 1, (n, d), generator=g, device="cuda", dtype=torch.int64)
z = torch.randint(0, M, (L, d), generator=g, device="cuda", dtype=torch.int64)
W = int(_native.lib().sfftb_bitmap_words(M))
bits = (torch.rand((L, W * 32), generator=g, device="cuda") < 0.092)
weights = (1 << torch.arange(32, device="cuda", dtype=torch.int64))
words = (bits.view(L, W, 32).to(torch.int64) * weights).sum(-1)
words = words.to(torch.int64).bitwise_and(0xFFFFFFFF).to(torch.uint32).view(torch.int32)
hits = torch.empty(n, dtype=torch.int64, device="cuda")
mask = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
for r in range(reps):
    ev[2 * r].record()
    _native.call("sfftb_hash_hits", rows.data_ptr(), n, d, z.data_ptr(), 1, L, M,
                 words.data_ptr(), d * N, 24, hits.data_ptr(), mask.data_ptr(), _dev.stream())
    ev[2 * r + 1].record()
torch.cuda.synchronize()
ms = [ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps)]
bytes_ = n * 8 * d + n * 8 + L * W * 4 + n // 8
print(f"hash n=2^{lg}: ms={ms} -> {bytes_ / (min(ms) * 1e-3) / 1e9:.0f} GB/s, "
      f"{n / (min(ms) * 1e-3):.3e} cand/s, mean hits {hits.float().mean().item():.3f}")
chk = int((hits * torch.arange(n, device="cuda", dtype=torch.int64).remainder(1000003)).sum())
print(f"checksum {chk} mask {int(mask.to(torch.int64).sum())}")
