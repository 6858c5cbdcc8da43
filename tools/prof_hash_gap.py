"""Where a synchronised sfftb_hash_hits call spends its time: the same call
timed (a) after a device synchronisation, (b) behind a 2 ms spin kernel that
hides the host-side enqueue latency, plus the host time of the call itself."""
import os
import sys
import time

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
words = torch.randint(-2**31, 2**31 - 1, (L, W), generator=g, device="cuda",
                      dtype=torch.int64).to(torch.int32)
hits = torch.empty(n, dtype=torch.int64, device="cuda")
mask = torch.empty((n + 31) // 32, dtype=torch.int32, device="cuda")


def call():
    _native.call("sfftb_hash_hits", rows.data_ptr(), n, d, z.data_ptr(), 1, L, M,
                 words.data_ptr(), -1, 24, hits.data_ptr(), mask.data_ptr(), _dev.stream())


for mode in ("sync", "behind_spin", "sync", "behind_spin", "back_to_back"):
    ms, host = [], []
    for r in range(reps):
        if mode != "back_to_back":
            torch.cuda.synchronize()
        if mode == "behind_spin":
            torch.cuda._sleep(4_000_000)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        t0 = time.perf_counter()
        call()
        host.append(round((time.perf_counter() - t0) * 1e3, 3))
        b.record()
        if mode != "back_to_back":
            torch.cuda.synchronize()
        ms.append((a, b))
    torch.cuda.synchronize()
    print(mode, [round(a.elapsed_time(b), 4) for a, b in ms], "host ms", host)
