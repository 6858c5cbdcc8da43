"""tools/prof_hash.py with a device synchronisation before every timed call
(the way bench.py times sfftb_hash_hits): shows per-call host-side costs such as
stream-ordered allocations that back-to-back launches hide."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13053_b200 import _dev, _native  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
M, L, d, N = 103307, 47, 10, 4096
n = 1 << lg
g = torch.Generator(device="cuda")
g.manual_seed(1)
rows = torch.randint(-N, N + 1, (n, d), generator=g, device="cuda", dtype=torch.int64)
z = torch.randint(0, M, (L, d), generator=g, device="cuda", dtype=torch.int64)
W = int(_native.lib().sfftb_bitmap_words(M))
bits = (torch.rand((L, W * 32), generator=g, device="cuda") < 0.092)
weights = (1 << torch.arange(32, device="cuda", dtype=torch.int64))
words = (bits.view(L, W, 32).to(torch.int64) * weights).sum(-1)
words = words.bitwise_and(0xFFFFFFFF).to(torch.uint32).view(torch.int32)
hits = torch.empty(n, dtype=torch.int64, device="cuda")
mask = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")
ms = []
for r in range(reps):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    _native.call("sfftb_hash_hits", rows.data_ptr(), n, d, z.data_ptr(), 1, L, M,
                 words.data_ptr(), -1, 24, hits.data_ptr(), mask.data_ptr(), _dev.stream())
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b))
print(f"hash (synchronised calls) n=2^{lg}: ms={[round(x, 4) for x in ms]}")
