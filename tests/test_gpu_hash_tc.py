"""K3 on the tensor cores (csrc/hash_tc.cu) against exact integer hashing.

The byte-GEMM path must give the hit counts and detected bitmask of the
reference's gather (_core.pyx:185-197) bit for bit, for any int64 rows: rows
inside the GEMM range through the tcgen05 kind::i8 MMA, rows outside it
(|k| >= 2^(8P)) through the exact recompute path.  The expected values are
computed here in numpy int64 (exact: d (M-1)^2 < 2^63 at every shape below)
and, independently, by the CUDA-core kernels (SFFTB_HASH_TC=0).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _bitmaps(rng, L, M, density):
    W = ((M + 31) // 32 + 3) & ~3
    bits = np.zeros((L, W * 32), dtype=bool)
    bits[:, :M] = rng.random((L, M)) < density
    words = np.packbits(bits.reshape(L, W, 32)[:, :, ::-1], axis=2, bitorder="big")
    return bits[:, :M], words.view(">u4").astype(np.uint32).reshape(L, W)


def _exact_hits(rows, z, M, bits):
    r = ((rows % M) @ (z % M).T) % M  # (n, L), exact in int64 here
    return bits[np.arange(z.shape[0])[None, :], r].sum(axis=1).astype(np.int64)


def _run(rows, z, M, words, min_hits, tc):
    import torch

    from paper_2006_13053_b200 import _dev, _native

    n, d = rows.shape
    L = z.shape[0]
    hits = _dev.empty((n,), torch.int64)
    mask = _dev.empty(((n + 31) // 32,), torch.int32)
    old = os.environ.get("SFFTB_HASH_TC")
    os.environ["SFFTB_HASH_TC"] = "1" if tc else "0"
    try:
        keep = [_dev.upload(rows), _dev.upload(z), _dev.upload(words.view(np.int32))]
        _native.call("sfftb_hash_hits", _dev.ptr(keep[0]), n, d, _dev.ptr(keep[1]), 1, L, M,
                     _dev.ptr(keep[2]), -1, min_hits, _dev.ptr(hits), _dev.ptr(mask),
                     _dev.stream())
        h, m = _dev.download(hits), _dev.download(mask).view(np.uint32)
    finally:
        if old is None:
            os.environ.pop("SFFTB_HASH_TC", None)
        else:
            os.environ["SFFTB_HASH_TC"] = old
    return h, m


def _mask_of(hits, min_hits):
    det = hits >= min_hits
    pad = np.zeros(((len(det) + 31) // 32) * 32, dtype=bool)
    pad[: len(det)] = det
    return np.packbits(pad.reshape(-1, 32)[:, ::-1], axis=1).view(">u4").astype(
        np.uint32).ravel()


@pytest.mark.parametrize("d,M,L,span,n", [
    (10, 103307, 47, 4096, 300_001),     # config-4 shape (C = 4 CTAs x 12 lattices)
    (4, 2069, 31, 32, 200_000),          # small M: 2 coefficient limbs would do
    (16, 20663, 41, 64, 131_072),        # d = 16, exact multiple of the tile
    (6, 10331, 61, 1 << 20, 140_000),    # 8 CTAs per cluster, wide coordinates
    (2, 211, 5, 16, 70_000),             # tiny L, 2-coordinate rows
])
def test_tc_hash_bitexact(cuda, d, M, L, span, n):
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(d * 7919 + L)
    rows = rng.integers(-span, span + 1, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.45)
    min_hits = (L + 1) // 2
    want = _exact_hits(rows, z, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_tc_recomputed(1)
    h_tc, m_tc = _run(rows, z, M, words, min_hits, tc=True)
    assert lib.sfftb_hash_tc_recomputed(1) == 0
    assert np.array_equal(h_tc, want)
    assert np.array_equal(m_tc, _mask_of(want, min_hits))
    h_cc, m_cc = _run(rows, z, M, words, min_hits, tc=False)
    assert np.array_equal(h_cc, want) and np.array_equal(m_cc, m_tc)


def test_tc_hash_rows_outside_gemm_range(cuda):
    """|k| up to 2^62 and negative generators: the validity columns catch the
    rows whose bytes are not a sign extension and the exact path takes them."""
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(5)
    n, d, M, L = 200_000, 10, 103307, 47
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    big = rng.choice(n, size=777, replace=False)
    rows[big, rng.integers(0, d, size=777)] = rng.integers(-(1 << 62), 1 << 62, size=777)
    rows[3, :] = np.iinfo(np.int64).min + 1
    rows[4, :] = np.iinfo(np.int64).max
    z = rng.integers(-(1 << 40), 1 << 40, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.5)
    # exact reference with Python ints for the wide rows
    rmod = rows % M
    want = _exact_hits(rmod, z % M, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_tc_recomputed(1)
    h_tc, m_tc = _run(rows, z, M, words, 24, tc=True)
    nrec = lib.sfftb_hash_tc_recomputed(1)
    outside = np.any((rows < -(1 << 56)) | (rows >= (1 << 56)), axis=1).sum()
    assert nrec == outside > 700
    assert np.array_equal(h_tc, want)
    assert np.array_equal(m_tc, _mask_of(want, 24))
