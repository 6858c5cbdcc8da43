"""Diagnostic for csrc/hash_roll.cu: the accumulators of tile 0 / step 0
(SFFTB_HASH_ROLL_DUMP) next to the values numpy expects, then a hit-count check.
    python tools/roll_diag.py [n] [d] [M] [L]
"""
import os
import sys

import numpy as np

os.environ["SFFTB_HASH_ROLL"] = "1"
os.environ["SFFTB_HASH_ROLL_MINROWS"] = "1"
os.environ["SFFTB_HASH_ROLL_DEBUG"] = "1"
os.environ["SFFTB_HASH_TC"] = "0"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from paper_2006_13053_b200 import _dev, _native  # noqa: E402
from test_gpu_hash_tc import _bitmaps, _exact_hits  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128 * 300
d = int(sys.argv[2]) if len(sys.argv) > 2 else 10
M = int(sys.argv[3]) if len(sys.argv) > 3 else 103307
L = int(sys.argv[4]) if len(sys.argv) > 4 else 47
dump = len(sys.argv) > 5
if dump:
    os.environ["SFFTB_HASH_ROLL_DUMP"] = "1"
rng = np.random.default_rng(1)
rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
z = rng.integers(0, M, size=(L, d), dtype=np.int64)
bits, words = _bitmaps(rng, L, M, 0.45)
want = _exact_hits(rows, z, M, bits)
if dump:
    u = rows[:128] + 8192
    a, b = u & 127, u >> 7
    for r in (0, 1, 33, 127):
        exp = []
        for i in range(5):
            c0 = z[i] % M
            c1 = (z[i] * 128) % M
            cc = (-(8192 * z[i].sum())) % M
            for limb in range(3):
                s = int((a[r] * ((c0 >> (8 * limb)) & 255)).sum() + (b[r] * ((c1 >> (8 * limb)) & 255)).sum()
                        + ((cc >> (8 * limb)) & 255))
                exp.append(s)
        print(f"expect  row {r:3d}:", " ".join(map(str, exp)), 0, flush=True)
hits = _dev.empty((n,), torch.int64)
mask = _dev.empty(((n + 31) // 32,), torch.int32)
keep = [_dev.upload(rows), _dev.upload(z), _dev.upload(words.view(np.int32))]
_native.call("sfftb_hash_hits", _dev.ptr(keep[0]), n, d, _dev.ptr(keep[1]), 1, L, M,
             _dev.ptr(keep[2]), -1, 24, _dev.ptr(hits), _dev.ptr(mask), _dev.stream())
torch.cuda.synchronize()
h = _dev.download(hits)
bad = np.flatnonzero(h != want)
print(f"n={n} mismatches={len(bad)} first={bad[:10]} got={h[bad[:10]]} want={want[bad[:10]]}")
print("recomputed", _native.lib().sfftb_hash_roll_recomputed(1))
