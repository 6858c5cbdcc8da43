"""Small host-to-device upload cost (e2e polynomial upload):
    python tools/upload_bench.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
from paper_2006_13053_b200 import _dev  # noqa: E402

a = np.random.default_rng(0).integers(0, 100, size=12000).astype(np.int64)  # 96 KB
torch.cuda.synchronize()


def bench(name, fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        x = fn()
        torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / reps * 1e6:.1f} us per upload+sync")


bench("_dev.upload (pinned staging)", lambda: _dev.upload(a))
bench("torch.from_numpy().cuda() (pageable)", lambda: torch.from_numpy(a).cuda())
pinned = torch.empty(a.shape, dtype=torch.int64, pin_memory=True)
dst = torch.empty(a.shape, dtype=torch.int64, device="cuda")


def pre():
    pinned.numpy()[:] = a
    dst.copy_(pinned, non_blocking=True)
    return dst


bench("preallocated pinned + device", pre)
bench("empty pinned only", lambda: torch.empty(a.shape, dtype=torch.int64, pin_memory=True))
