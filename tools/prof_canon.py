"""Device generation + canonicalisation of a cfg4-sized candidate set.
    python tools/prof_canon.py [log2_rows]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _dev, _native  # noqa: E402

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
n = 1 << lg
for rep in range(2):
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record()
    rows = _dev.empty((n, 10), torch.int64)
    _native.call("sfftb_random_box_rows", n, 10, -4096, 4096, 7 + rep, _dev.ptr(rows),
                 _dev.stream())
    b.record()
    out = pkg.canonicalize_device(rows, 10)
    c.record()
    torch.cuda.synchronize()
    print(f"n=2^{lg}: generate {a.elapsed_time(b):.2f} ms, canonicalise {b.elapsed_time(c):.2f} ms,"
          f" unique {out.shape[0]}")
