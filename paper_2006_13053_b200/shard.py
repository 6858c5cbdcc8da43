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
        # the float64 pairs are gathered as they are and written back into
        # the complex128 layout (re + 1j*im would turn -0.0 into +0.0 and an
        # infinite imaginary part into a NaN real part)
        parts = gather(np.ascontiguousarray(co).view(np.float64).reshape(-1, 2)[:, 0].copy(),
                       torch.float64), \
            gather(np.ascontiguousarray(co).view(np.float64).reshape(-1, 2)[:, 1].copy(),
                   torch.float64)
        gco = np.empty(parts[0].size, np.complex128)
        gco.real = parts[0]
        gco.imag = parts[1]
    return gidx, gco


def _collective_device(group):
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _all_gather_padded(local, per, world, group, async_op=False):
    """All-gather equal-sized (padded to `per` leading rows) device blocks
    into one (world * per, ...) device tensor.  NCCL gathers in HBM (async:
    returns the pending work); gloo stages through host memory."""
    import torch
    import torch.distributed as dist

    cdev = _collective_device(group)
    shape = (per,) + tuple(local.shape[1:])
    if cdev.type == "cuda":
        send = local if local.shape[0] == per else torch.cat(
            [local, local.new_zeros((per - local.shape[0],) + shape[1:])])
        out = torch.empty((world * per,) + shape[1:], dtype=local.dtype, device=local.device)
        # NCCL moves real words: complex blocks travel as their float64 pairs
        src, dst = send.contiguous(), out
        if src.is_complex():
            src, dst = torch.view_as_real(src), torch.view_as_real(out)
        work = dist.all_gather_into_tensor(dst, src, group=group, async_op=async_op)
        return out, work
    send = torch.zeros(shape, dtype=local.dtype)
    send[:local.shape[0]] = local.cpu()
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send, group=group)
    return torch.cat(parts).to(local.device), None


def detect_and_compute_sharded(samples, config, gamma_shard, offset, group=None, zero=None):
    """detect_and_compute (detect.py:158-169) over G ranks: this rank holds
    the contiguous row shard `gamma_shard` of Gamma starting at row `offset`.

    Work split:
      * theta0 from all L sample norms, on every rank (the samples are
        shared; (L, M) norms cost one HBM read), so every rank classifies
        with the same zero test (detect.py:42-53);
      * the L DFTs are sharded: rank r transforms lattices
        shard_bounds(L, G, r) and builds their nonzero bitmaps;
      * all-gather of the bitmaps (L * W * 4 bytes, 607 KB at config 4),
        then every rank hashes its rows against all L lattices
        (_core.pyx:185-197) -- hits, compaction;
      * the spectra themselves (L * M * 16 bytes) are all-gathered
        asynchronously while the rows hash; the medians of the detected rows
        (_core.pyx:198-200) wait for them;
      * merge: all-gather of detected counts, indices and coefficients.
    Every kernel is the single-GPU one on a row or lattice subset, so the
    merged result is identical to detect_and_compute on all of Gamma.
    Returns (detected_idx, coeffs, local DetectionResult with this shard's
    hits)."""
    import torch
    import torch.distributed as dist

    from . import _dev, _engine, _native
    from .detect import (DetectionResult, ParameterError, _kbound, _stack_samples,
                         _theta_tensor, _zero_from_device)

    if config.nu != 0.5:
        raise ParameterError("coefficient computation requires nu = 1/2")
    if config.L % 2 == 0:
        raise ParameterError("coefficient computation requires odd L")
    M = config.shared_M
    if M is None:
        raise ParameterError("the sharded path needs one shared lattice size M")
    if not gamma_shard.dim * (M - 1) ** 2 < 2**62:
        raise ParameterError("lattice size too large for int64 residues")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    with _dev.stream_scope():
        t = _stack_samples(samples, config)
        if zero is None:
            zero = _zero_from_device(t)
        theta0 = _theta_tensor(zero.theta_zero)
        L = config.L
        W = int(_native.lib().sfftb_bitmap_words(M))
        per = (L + world - 1) // world
        l0, l1 = min(rank * per, L), min((rank + 1) * per, L)
        if l1 > l0:
            ghat_loc, _, bits_loc = _engine.spectra(t[l0:l1], M, 1, l1 - l0, theta0)
        else:
            ghat_loc = _dev.empty((0, M), torch.complex128)
            bits_loc = _dev.empty((0,), torch.int32)
        bits, _ = _all_gather_padded(bits_loc.view(-1, W), per, world, group)
        ghat, ghat_work = _all_gather_padded(ghat_loc, per, world, group, async_op=True)
        bits = bits[:L].reshape(-1)
        rows = gamma_shard.device()
        n, d = len(gamma_shard), gamma_shard.dim
        zmat = config.zmat_device()
        st = _dev.stream()
        nwords = (n + 31) // 32
        detmask = _dev.empty((max(nwords, 1),), torch.int32)
        hits = _dev.empty((max(n, 1),), torch.int64)
        idx = _dev.empty((max(n, 1),), torch.int64)
        counts = _dev.zeros((1,), torch.int64)
        coeffs = _dev.empty((max(n, 1),), torch.complex128)
        if n:
            _native.call("sfftb_hash_hits", _dev.ptr(rows), n, d, _dev.ptr(zmat), 1, L, M,
                         _dev.ptr(bits), int(_kbound(gamma_shard)),
                         _engine.min_hits_for(config.nu, L), _dev.ptr(hits), _dev.ptr(detmask),
                         st)
            ws = _dev.workspace(_native.lib().sfftb_compact_workspace_bytes(1, n))
            _native.call("sfftb_compact_mask", _dev.ptr(detmask), 1, n, _dev.ptr(idx),
                         _dev.ptr(counts), _dev.ptr(ws), st)
        if ghat_work is not None:
            ghat_work.wait()  # the medians read every lattice's spectrum
        ghat = ghat[:L]
        if n:
            _native.call("sfftb_medians", _dev.ptr(rows), d, _dev.ptr(zmat), 1, L, M,
                         _dev.ptr(ghat), _dev.ptr(idx), _dev.ptr(counts), n, _dev.ptr(coeffs),
                         st)
        k = int(_dev.download(counts)[0])
        res = DetectionResult(gamma_shard, hits[:n], idx[:k], coeffs[:k], zero.theta_zero)
        gidx, gco = merge_detections(res.detected_idx, res.coeffs, offset, group)
    return gidx, gco, res
