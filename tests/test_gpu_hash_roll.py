"""K3 on the tensor cores, rolling kernel (csrc/hash_roll.cu) against exact
integer hashing.

Hit counts and the detected bitmask must equal the reference's gather
(_core.pyx:185-197) bit for bit: rows inside the limb range [-2^13, 2^13)
through the tcgen05 kind::i8 MMA (A operand in tensor memory), rows outside it
through the exact recompute path.  The expected values are computed here in
numpy int64 (exact: d (M-1)^2 < 2^63 at every shape below) and, independently,
by the CUDA-core kernels.
"""

import os

import numpy as np
import pytest

from test_gpu_hash_tc import _bitmaps, _exact_hits, _mask_of

pytestmark = pytest.mark.gpu


def _run(rows, z, M, words, min_hits, roll):
    import torch

    from paper_2006_13053_b200 import _dev, _native

    n, d = rows.shape
    L = z.shape[0]
    hits = _dev.empty((n,), torch.int64)
    mask = _dev.empty(((n + 31) // 32,), torch.int32)
    env = {"SFFTB_HASH_ROLL": "1" if roll else "0", "SFFTB_HASH_ROLL_MINROWS": "1",
           "SFFTB_HASH_TC": "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        keep = [_dev.upload(rows), _dev.upload(z), _dev.upload(words.view(np.int32))]
        _native.call("sfftb_hash_hits", _dev.ptr(keep[0]), n, d, _dev.ptr(keep[1]), 1, L, M,
                     _dev.ptr(keep[2]), -1, min_hits, _dev.ptr(hits), _dev.ptr(mask),
                     _dev.stream())
        h, m = _dev.download(hits), _dev.download(mask).view(np.uint32)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return h, m


@pytest.mark.parametrize("d,M,L,span,n", [
    (10, 103307, 47, 4096, 300_001),     # config-4 shape: 10 groups of 5 lattices
    (10, 103307, 47, 4096, 2_000_003),   # every CTA rolls through several births
    (4, 2069, 31, 32, 200_000),          # small M, 7 groups
    (14, 20663, 41, 64, 131_072),        # d = 14, exact multiple of the tile
    (6, 10331, 61, 8191, 140_000),       # 13 groups, the whole limb range
    (8, 211, 5, 16, 70_000),             # one group: born and retired in one step
    (10, 103307, 47, 4096, 1000),        # fewer tiles than CTAs
    (12, 65537, 12, 100, 50_000),        # last group partly filled
])
def test_roll_hash_bitexact(cuda, d, M, L, span, n):
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(d * 7919 + L + n)
    rows = rng.integers(-span, span + 1, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.45)
    min_hits = (L + 1) // 2
    want = _exact_hits(rows, z, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    h, m = _run(rows, z, M, words, min_hits, roll=True)
    assert lib.sfftb_hash_roll_recomputed(1) == 0
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, min_hits))
    h_cc, m_cc = _run(rows, z, M, words, min_hits, roll=False)
    assert np.array_equal(h_cc, want) and np.array_equal(m_cc, m)


def test_roll_hash_rows_outside_limb_range(cuda):
    """|k| up to 2^62, the range edges -2^13 and 2^13 - 1, negative generators:
    the flag column catches rows outside the limb range and the exact path
    takes exactly those."""
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(5)
    n, d, M, L = 200_000, 10, 103307, 47
    rows = rng.integers(-8192, 8192, size=(n, d), dtype=np.int64)
    big = rng.choice(np.arange(10, n), size=777, replace=False)
    rows[big, rng.integers(0, d, size=777)] = rng.integers(1 << 20, 1 << 62, size=777) * \
        rng.choice([-1, 1], size=777)
    rows[3, :] = np.iinfo(np.int64).min + 1
    rows[4, :] = np.iinfo(np.int64).max
    rows[5, :] = -8192
    rows[6, :] = 8191
    rows[7, 0] = 8192
    rows[8, 9] = -8193
    z = rng.integers(-(1 << 40), 1 << 40, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.5)
    want = _exact_hits(rows % M, z % M, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    h, m = _run(rows, z, M, words, 24, roll=True)
    nrec = lib.sfftb_hash_roll_recomputed(1)
    outside = np.any((rows < -8192) | (rows > 8191), axis=1).sum()
    assert nrec == outside == 777 + 4
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, 24))


def test_roll_hash_mask_only(cuda):
    """hits64 == NULL: only the detected bitmask is written."""
    import torch

    from paper_2006_13053_b200 import _dev, _native

    rng = np.random.default_rng(11)
    n, d, M, L = 150_001, 10, 103307, 47
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.5)
    want = _exact_hits(rows, z, M, bits)
    mask = _dev.empty(((n + 31) // 32,), torch.int32)
    env = {"SFFTB_HASH_ROLL": "1", "SFFTB_HASH_ROLL_MINROWS": "1"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        keep = [_dev.upload(rows), _dev.upload(z), _dev.upload(words.view(np.int32))]
        _native.call("sfftb_hash_hits", _dev.ptr(keep[0]), n, d, _dev.ptr(keep[1]), 1, L, M,
                     _dev.ptr(keep[2]), -1, 25, 0, _dev.ptr(mask), _dev.stream())
        m = _dev.download(mask).view(np.uint32)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert np.array_equal(m, _mask_of(want, 25))


def test_roll_hash_concurrent_threads(cuda):
    """Three host threads, each on its own stream, one of them with rows outside
    the limb range: every call repairs exactly its own rows (the out-of-range
    flag and the scratch bitmaps are private to a call)."""
    import threading

    import torch

    from paper_2006_13053_b200 import _dev, _native

    rng = np.random.default_rng(23)
    d, M, L = 10, 103307, 47
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.4)
    cases = []
    for t in range(3):
        n = 180_000 + 1000 * t
        rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
        if t == 1:
            rows[rng.choice(n, size=500, replace=False), 3] = 1 << 40
        cases.append((rows, _exact_hits(rows % M, z, M, bits)))
    env = {"SFFTB_HASH_ROLL": "1", "SFFTB_HASH_ROLL_MINROWS": "1", "SFFTB_HASH_TC": "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    out = [None] * 3
    zdev, wdev = _dev.upload(z), _dev.upload(words.view(np.int32))
    torch.cuda.synchronize()

    def work(t):
        rows, _ = cases[t]
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(4):
                rdev = torch.as_tensor(rows, device="cuda")
                hits = torch.empty((rows.shape[0],), dtype=torch.int64, device="cuda")
                mask = torch.empty(((rows.shape[0] + 31) // 32,), dtype=torch.int32, device="cuda")
                _native.call("sfftb_hash_hits", rdev.data_ptr(), rows.shape[0], d, zdev.data_ptr(),
                             1, L, M, wdev.data_ptr(), -1, 24, hits.data_ptr(), mask.data_ptr(),
                             st.cuda_stream)
            st.synchronize()
            out[t] = (hits.cpu().numpy(), mask.cpu().numpy().view(np.uint32))

    try:
        th = [threading.Thread(target=work, args=(t,)) for t in range(3)]
        for x in th:
            x.start()
        for x in th:
            x.join()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for t in range(3):
        assert out[t] is not None
        assert np.array_equal(out[t][0], cases[t][1])
        assert np.array_equal(out[t][1], _mask_of(cases[t][1], 24))
