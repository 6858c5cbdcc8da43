"""K3 on the tensor cores, fp16 rolling kernel (csrc/hash_rollf.cu) against
exact integer hashing.

For candidate sets with a known small magnitude bound (kbound = sum_j max|k_j|
< 2048) the residues are an exact FP16 x FP16 -> FP32 GEMM (tcgen05 kind::f16,
A operand in tensor memory, two limbs per lattice, accumulators seeded into
[2^23, 2^24) so their bit patterns combine with one integer multiply-add).
Hit counts and the detected bitmask must equal the reference's gather
(_core.pyx:185-197) bit for bit; the expected values are computed in numpy
int64 and, independently, by the CUDA-core kernel.
"""

import os

import numpy as np
import pytest

from test_gpu_hash_tc import _bitmaps, _exact_hits, _mask_of

pytestmark = pytest.mark.gpu


def _run(rows, z, M, words, min_hits, kbound, rollf=True, roll=True, w2=True):
    import torch

    from paper_2006_13053_b200 import _dev, _native

    n, d = rows.shape
    L = z.shape[0]
    hits = _dev.empty((n,), torch.int64)
    mask = _dev.empty(((n + 31) // 32,), torch.int32)
    env = {"SFFTB_HASH_ROLL": "1" if roll else "0", "SFFTB_HASH_ROLLF": "1" if rollf else "0",
           "SFFTB_HASH_ROLL_MINROWS": "1", "SFFTB_HASH_TC": "0",
           "SFFTB_HASH_ROLLW2": "1" if w2 else "0"}
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        keep = [_dev.upload(rows), _dev.upload(z), _dev.upload(words.view(np.int32))]
        _native.call("sfftb_hash_hits", _dev.ptr(keep[0]), n, d, _dev.ptr(keep[1]), 1, L, M,
                     _dev.ptr(keep[2]), int(kbound), min_hits, _dev.ptr(hits), _dev.ptr(mask),
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
    (10, 103307, 47, 32, 300_001),      # config-4 shape: 6 groups of 8 lattices
    (10, 103307, 47, 32, 2_500_003),    # every CTA rolls through several births
    (10, 103307, 48, 100, 400_000),     # all 48 lattice slots, kbound 1000
    (4, 20663, 31, 16, 200_000),        # 4 groups, last one partly filled
    (12, 65537, 12, 100, 50_000),       # 2 groups, second half group empty
    (8, 4099, 5, 16, 70_000),           # one group: born and retired in one step
    (6, 10331, 41, 300, 131_072),       # kbound 1800, exact multiple of the tile
    (10, 103307, 47, 32, 1000),         # fewer tiles than CTAs
    (10, 107837, 33, 8, 250_000),       # larger modulus, 5 groups (three accumulator buffers)
    (10, 103307, 17, 32, 250_000),      # 3 groups
])
def test_rollf_hash_bitexact(cuda, d, M, L, span, n):
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(d * 7919 + L + n)
    rows = rng.integers(-span, span + 1, size=(n, d), dtype=np.int64)
    rows[0] = span      # the bound is attained, both signs
    rows[1] = -span
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    z[0] = M - 1        # largest coefficients
    bits, words = _bitmaps(rng, L, M, 0.45)
    min_hits = (L + 1) // 2
    want = _exact_hits(rows, z, M, bits)
    kbound = int(np.abs(rows).max(axis=0).sum())
    assert kbound < 2048
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    lib.sfftb_hash_rollf_calls(1)
    h, m = _run(rows, z, M, words, min_hits, kbound)
    assert lib.sfftb_hash_rollf_calls(1) == 1   # the fp16 kernel served the call
    assert lib.sfftb_hash_roll_recomputed(1) == 0
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, min_hits))
    # the byte-limb rolling kernel and the CUDA-core kernel agree
    h_b, m_b = _run(rows, z, M, words, min_hits, kbound, rollf=False)
    assert np.array_equal(h_b, want) and np.array_equal(m_b, m)
    h_cc, m_cc = _run(rows, z, M, words, min_hits, kbound, rollf=False, roll=False)
    assert np.array_equal(h_cc, want) and np.array_equal(m_cc, m)


def test_rollf_negative_generators_and_sparse_bitmaps(cuda):
    """Generators given as negative / unreduced int64 and nearly empty or
    nearly full bitmaps (hits 0 and L)."""
    rng = np.random.default_rng(11)
    d, M, L, n = 10, 103307, 47, 200_000
    rows = rng.integers(-32, 33, size=(n, d), dtype=np.int64)
    z = rng.integers(-5 * M, 5 * M, size=(L, d), dtype=np.int64)
    kbound = int(np.abs(rows).max(axis=0).sum())
    for dens in (0.001, 0.999):
        bits, words = _bitmaps(rng, L, M, dens)
        want = _exact_hits(rows, z, M, bits)
        h, m = _run(rows, z, M, words, 24, kbound)
        assert np.array_equal(h, want)
        assert np.array_equal(m, _mask_of(want, 24))


def test_rollf_rows_outside_the_half_range_are_redone_exactly(cuda):
    """A caller's bound that does not hold for a few rows (a coordinate
    outside (-2048, 2048)): the loaders flag them and the follow-up kernel
    recomputes exactly those rows."""
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(5)
    d, M, L, n = 10, 103307, 47, 150_000
    rows = rng.integers(-32, 33, size=(n, d), dtype=np.int64)
    bad = rng.choice(n, size=37, replace=False)
    rows[bad, rng.integers(0, d, size=37)] = rng.integers(2048, 1 << 40, size=37) * \
        rng.choice([-1, 1], size=37)
    rows[bad[0], 3] = 2048
    rows[bad[1], 3] = -2049
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.3)
    want = _exact_hits(rows, z, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    h, m = _run(rows, z, M, words, 20, 320)
    assert lib.sfftb_hash_roll_recomputed(1) == 37
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, 20))


@pytest.mark.parametrize("d,M,L,span,n,kb", [
    (10, 103307, 47, 4096, 300_001, -1),       # config-4 shape, no bound given
    (10, 103307, 47, 4096, 2_500_003, 40960),  # several births per CTA
    (10, 103307, 48, 8191, 400_000, -1),       # all 48 slots, the whole limb range
    (8, 20663, 31, 3000, 200_000, -1),         # 4 groups
    (6, 65537, 12, 5000, 50_000, -1),          # 2 groups, second partly filled
    (4, 4099, 5, 100, 70_000, 50_000),         # one group; bound too large for fp16 mode
    (10, 103307, 47, 4096, 1000, -1),          # fewer tiles than CTAs
    (10, 103307, 33, 2048, 250_000, -1),       # 5 groups
])
def test_rollf_byte_mode_bitexact(cuda, d, M, L, span, n, kb):
    """Coordinates beyond the fp16 range (|k| < 2^13, any bound): the same
    kernel in byte mode (tcgen05 kind::i8, three limbs per lattice, N = 24)."""
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(d * 104729 + L + n)
    rows = rng.integers(-span, span + 1, size=(n, d), dtype=np.int64)
    rows[0] = span
    rows[1] = -span
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    z[0] = M - 1
    bits, words = _bitmaps(rng, L, M, 0.45)
    min_hits = (L + 1) // 2
    want = _exact_hits(rows, z, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    lib.sfftb_hash_rollf_calls(1)
    lib.sfftb_hash_rollf_scaled_runs(1)
    h, m = _run(rows, z, M, words, min_hits, kb)
    assert lib.sfftb_hash_rollf_calls(1) == 1
    scaled = lib.sfftb_hash_rollf_scaled_runs(1)
    assert scaled in (0, 1)   # 1: every lattice had a multiplier (the two-limb kernel ran)
    if M < 65536:
        assert scaled == 1    # t = 1 serves: every coefficient is below 2^16 already
    assert lib.sfftb_hash_roll_recomputed(1) == 0
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, min_hits))
    # three limbs (no per-lattice multipliers) and the 5-lattice kernel agree
    lib.sfftb_hash_rollf_calls(1)
    h_3, m_3 = _run(rows, z, M, words, min_hits, kb, w2=False)
    assert lib.sfftb_hash_rollf_calls(1) == 1
    assert lib.sfftb_hash_rollf_scaled_runs(1) == 0
    assert np.array_equal(h_3, want) and np.array_equal(m_3, m)
    h_b, m_b = _run(rows, z, M, words, min_hits, kb, rollf=False)
    assert np.array_equal(h_b, want) and np.array_equal(m_b, m)


def test_rollf_scaled_byte_mode_falls_back_without_multipliers(cuda):
    """A lattice whose coefficients admit no multiplier t with all t c mod M <
    2^16 (here: a composite modulus 2^17 with generators covering every
    residue class that matters) sends the call to the three-limb kernel."""
    rng = np.random.default_rng(31)
    d, M, L, n = 10, 103307, 9, 100_000
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    # generators 1 and M - 1 in one lattice: t and M - t cannot both be < 2^16
    # unless t < 2^16 and t > M - 2^16, which 128 t mod M then breaks for most t;
    # whatever the search finds, the results must equal the exact ones
    z[0, 0], z[0, 1] = 1, M - 1
    bits, words = _bitmaps(rng, L, M, 0.4)
    want = _exact_hits(rows, z, M, bits)
    h, m = _run(rows, z, M, words, 5, -1)
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, 5))


def test_rollf_byte_mode_rows_outside_limb_range(cuda):
    """|k| up to 2^62 and the range edges -2^13, 2^13 - 1 in byte mode: flagged
    by the loaders, redone exactly by the follow-up kernel."""
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(17)
    d, M, L, n = 10, 103307, 47, 150_000
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    bad = rng.choice(n, size=41, replace=False)
    rows[bad, rng.integers(0, d, size=41)] = rng.integers(8192, 1 << 62, size=41) * \
        rng.choice([-1, 1], size=41)
    rows[bad[0], 2] = 8192
    rows[bad[1], 2] = -8193
    ok = np.setdiff1d(np.arange(n), bad)[:2]
    rows[ok[0], 5] = -8192
    rows[ok[1], 5] = 8191
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.3)
    want = _exact_hits(rows, z, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    lib.sfftb_hash_rollf_calls(1)
    h, m = _run(rows, z, M, words, 20, -1)
    assert lib.sfftb_hash_rollf_calls(1) == 1
    assert lib.sfftb_hash_roll_recomputed(1) == 41
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, 20))


def test_rollf_declined_call_is_served_exactly(cuda, monkeypatch):
    """The kernel leaves a call it cannot serve (its shared-memory window is not
    where the probe immediates assume) to the exact follow-up kernel: forced
    here, every row must come out of the 64-bit path with the same results."""
    from paper_2006_13053_b200 import _native

    rng = np.random.default_rng(23)
    d, M, L, n = 10, 103307, 47, 20_011   # a partly filled last mask word
    rows = rng.integers(-4096, 4097, size=(n, d), dtype=np.int64)
    z = rng.integers(0, M, size=(L, d), dtype=np.int64)
    bits, words = _bitmaps(rng, L, M, 0.3)
    want = _exact_hits(rows, z, M, bits)
    lib = _native.lib()
    lib.sfftb_hash_roll_recomputed(1)
    monkeypatch.setenv("SFFTB_HASH_ROLLF_FORCE_EXACT", "1")
    h, m = _run(rows, z, M, words, 20, -1)
    assert lib.sfftb_hash_roll_recomputed(1) == n
    assert np.array_equal(h, want)
    assert np.array_equal(m, _mask_of(want, 20))
