"""Generic vs residue-table hashing of one sfft-stage-sized Cartesian J.
    python tools/prof_pairs.py [t] [n1] [n2] [G] [L] [M]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2006_13053_b200 import _dev, _engine, _native  # noqa: E402

t, n1, n2, G, L, M = [int(v) for v in (sys.argv[1:] + ["6", "1000", "65", "5", "37", "20663"][len(sys.argv) - 1:])]
rng = np.random.default_rng(0)
prefix = np.unique(rng.integers(-32, 33, size=(n1, t)), axis=0)
n1 = prefix.shape[0]
vals = np.arange(-(n2 // 2), n2 - n2 // 2)
pre_d, vals_d = _dev.upload(prefix), _dev.upload(vals)
J = _engine.pair_product(pre_d, vals_d)
z = _dev.upload(rng.integers(0, M, size=(G * L, t + 1)))
W = int(_native.lib().sfftb_bitmap_words(M))
bits = _dev.upload((rng.integers(0, 1 << 31, size=(G * L * W,)) & 0x02020202).astype(np.int32))
n = n1 * n2
st = _dev.stream()
P = _dev.empty((G * L * n1,), torch.int32)
V = _dev.empty((G * L * n2,), torch.int32)
m = _dev.empty((G * ((n + 31) // 32),), torch.int32)
mh = (L + 1) // 2


def generic():
    _native.call("sfftb_hash_hits", _dev.ptr(J), n, t + 1, _dev.ptr(z), G, L, M, _dev.ptr(bits),
                 (t + 1) * 64, mh, None, _dev.ptr(m), st)


def tables():
    _native.call("sfftb_pair_residues", _dev.ptr(pre_d), n1, t, _dev.ptr(vals_d), n2, _dev.ptr(z),
                 G * L, M, _dev.ptr(P), _dev.ptr(V), st)


def pairs():
    _native.call("sfftb_hash_pairs", _dev.ptr(P), _dev.ptr(V), n1, n2, G, L, M, _dev.ptr(bits),
                 mh, None, _dev.ptr(m), st)


for name, fn in (("generic", generic), ("tables", tables), ("pairs", pairs)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name}: {a.elapsed_time(b) / 20 * 1e3:.1f} us  (n={n} x G={G} x L={L})")
