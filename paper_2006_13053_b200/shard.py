"""Multi-GPU fixed-candidate-set detection: rows sharded across ranks.

SURVEY.md section 8(e): every candidate row is independent, so Gamma is cut
into contiguous row shards, one per rank (one process per GPU).  Each rank
computes the L prime-length DFTs of the shared samples itself (cheaper than
shipping 16*L*M bytes) and hashes only its shard -- no collective on the data
path.  The only communication is assembling the (small) result: an
all-gather of the per-rank detected counts, then of the detected indices and
coefficients, concatenated in rank order.  Because shards are contiguous and
each shard's detections are ascending, the concatenation is the globally
ascending ``detected_idx`` of the single-GPU run (detect.py:167) -- the
merge is exact, not approximate.

The sfft driver is sequential across coordinates and runs as independent
replicas (bench.py --gpus N), see DESIGN.md.
"""

from __future__ import annotations

import numpy as np


def shard_bounds(n, world, rank):
    """[lo, hi) rows of `rank`: contiguous, sizes differ by at most one."""
    base, extra = divmod(int(n), int(world))
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def merge_detections(local_idx, local_coeffs, offset, group=None):
    """All-gather per-rank detections (ascending local indices of a
    contiguous shard starting at `offset`) into the global result, identical
    on every rank.  Works with any torch.distributed backend (nccl on the
    GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist

    idx = np.asarray(local_idx, dtype=np.int64) + int(offset)
    co = np.asarray(local_coeffs, dtype=np.complex128) if local_coeffs is not None else None
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else \
        torch.device("cpu")
    cnt = torch.tensor([idx.size], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    cap = max(max(counts), 1)

    def gather(arr, dtype):
        buf = torch.zeros(cap, dtype=dtype, device=dev)
        if arr.size:
            buf[:arr.size] = torch.as_tensor(arr, device=dev)
        parts = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(parts, buf, group=group)
        return np.concatenate([p[:c].cpu().numpy() for p, c in zip(parts, counts)])

    gidx = gather(idx, torch.int64)
    gco = None
    if co is not None:
        re = gather(co.real.copy(), torch.float64)
        im = gather(co.imag.copy(), torch.float64)
        gco = re + 1j * im
    return gidx, gco


def detect_and_compute_sharded(samples, config, gamma_shard, offset, group=None, zero=None):
    """detect_and_compute on this rank's contiguous shard of Gamma, merged.

    `zero` should be the global zero test (it depends only on the samples,
    which every rank holds), so every rank classifies with the same theta0.
    Returns (detected_idx, coeffs, local DetectionResult)."""
    from .detect import default_zero_test, detect_and_compute

    if zero is None:
        zero = default_zero_test(samples)
    res = detect_and_compute(samples, config, gamma_shard, zero=zero)
    gidx, gco = merge_detections(res.detected_idx, res.coeffs, offset, group)
    return gidx, gco, res
