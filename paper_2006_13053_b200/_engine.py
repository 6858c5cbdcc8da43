"""Device pipeline of one detection batch (G groups x L lattices, shared M).

The chain that replaces detect._gather + the compiled gather
(detect.py:122-169, _core.pyx:164-202) when the samples, generators and
candidate rows are already in HBM:

  samples (G*L, M)  --sumsq/zero test-->  theta0 (G)          [detect.py:42-53]
                    --Bluestein DFT----->  ghat (G*L, M)       [detect.py:98-109]
  ghat, theta0      --bitmap------------>  bits (G*L, W)       [_core.pyx:195]
  rows J, z, bits   --hash + hits------->  hits, detmask       [_core.pyx:185-197]
  detmask           --compaction-------->  idx (ascending)     [detect.py:167]
  idx, ghat         --medians----------->  coeffs              [_core.pyx:198-200]
  idx, coeffs       --top-s (optional)-->  kept idx, coeffs    [detect.py:184-193]

Nothing here synchronises with the host; callers read counts when they need
them (one sync per driver stage).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _dev, _native
from .dft import dft_batch


@dataclass
class Batch:
    G: int
    L: int
    M: int
    n: int
    ghat: torch.Tensor
    theta0: torch.Tensor
    hits: torch.Tensor | None
    idx: torch.Tensor | None
    counts: torch.Tensor | None
    coeffs: torch.Tensor | None


def zero_thresholds(samples, G, L, M):
    """theta0 per group from the sample RMS (detect.py:42-53) -> (G,) f64."""
    sumsq = _dev.empty((G * L,), torch.float64)
    _native.call("sfftb_sumsq", _dev.ptr(samples), M, G * L, M, _dev.ptr(sumsq), _dev.stream())
    theta = _dev.empty((G,), torch.float64)
    _native.call("sfftb_zero_thresholds", _dev.ptr(sumsq), G, L, M, _dev.ptr(theta),
                 _dev.stream())
    return theta


def min_hits_for(nu, L):
    """detected iff hits >= nu*L (a float) <=> hits >= ceil(nu*L)."""
    return int(math.ceil(nu * L))


def spectra(samples, M, G, L, theta0=None):
    """Zero test, DFT and nonzero bitmaps of (G*L, M) samples."""
    st = _dev.stream()
    if theta0 is None:
        theta0 = zero_thresholds(samples, G, L, M)
    ghat = dft_batch(samples, M)
    W = int(_native.lib().sfftb_bitmap_words(M))
    bits = _dev.empty((G * L * W,), torch.int32)
    _native.call("sfftb_nonzero_bitmap", _dev.ptr(ghat), G, L, M, _dev.ptr(theta0),
                 _dev.ptr(bits), st)
    return ghat, theta0, bits


def fused_ok(M):
    """The fused sampler->detection transforms cover M with N1, N2 in {128, 256}."""
    return 4097 <= M <= 32768


def sample_spectra_fused(bins, M, G, L, noise_seed, call0, sigma):
    """samples = M*ifft(bins) (+noise) kept on chip -> theta, ghat, bitmaps."""
    W = int(_native.lib().sfftb_bitmap_words(M))
    ghat = _dev.empty((G * L, M), torch.complex128)
    theta = _dev.empty((G,), torch.float64)
    bits = _dev.empty((G * L * W,), torch.int32)
    ws = _dev.workspace(_native.lib().sfftb_sample_detect_workspace_bytes(G * L, M))
    _native.call("sfftb_sample_detect_dft", _dev.ptr(bins), G, L, M,
                 int(noise_seed) & 0xFFFFFFFFFFFFFFFF, int(call0), float(sigma),
                 _dev.ptr(ghat), _dev.ptr(theta), _dev.ptr(bits), _dev.ptr(ws), _dev.stream())
    return ghat, theta, bits


def gather(ghat, theta0, bits, M, zmat, G, L, rows, kbound, nu, want_medians=True,
           want_hits=False):
    """Hash, hit counts, compaction and medians from the spectra."""
    n, d = int(rows.shape[0]), int(rows.shape[1])
    st = _dev.stream()
    nwords = (n + 31) // 32
    detmask = _dev.empty((G * max(nwords, 1),), torch.int32)
    hits = _dev.empty((G * n,), torch.int64) if want_hits else None
    min_hits = min_hits_for(nu, L)
    if n:
        _native.call("sfftb_hash_hits", _dev.ptr(rows), n, d, _dev.ptr(zmat), G, L, M,
                     _dev.ptr(bits), int(kbound), min_hits, _dev.ptr(hits), _dev.ptr(detmask),
                     st)
    idx = _dev.empty((G * max(n, 1),), torch.int64)
    counts = _dev.zeros((G,), torch.int64)
    if n:
        ws = _dev.workspace(_native.lib().sfftb_compact_workspace_bytes(G, n))
        _native.call("sfftb_compact_mask", _dev.ptr(detmask), G, n, _dev.ptr(idx),
                     _dev.ptr(counts), _dev.ptr(ws), st)
    coeffs = None
    if want_medians:
        coeffs = _dev.empty((G * max(n, 1),), torch.complex128)
        if n:
            _native.call("sfftb_medians", _dev.ptr(rows), d, _dev.ptr(zmat), G, L, M,
                         _dev.ptr(ghat), _dev.ptr(idx), _dev.ptr(counts), n, _dev.ptr(coeffs),
                         st)
    return Batch(G, L, M, n, ghat, theta0, hits, idx, counts, coeffs)


class PendingHost:
    """A host array being filled by asynchronous device-to-host copies: the
    numpy view is handed out once its event has completed."""

    __slots__ = ("array", "event", "_keep")

    def __init__(self, array, event, keep):
        self.array, self.event, self._keep = array, event, keep

    def result(self):
        self.event.synchronize()
        self._keep = None
        return self.array


def gather_streamed(ghat, theta0, bits, M, zmat, L, host_rows, kbound, nu, want_medians=True,
                    want_hits=False, chunk_rows=1 << 22):
    """gather() for one group whose candidate rows are still on the host:
    the rows go up in chunks on a copy stream while each landed chunk is
    hashed on the compute stream (PCIe and hashing overlap); compaction and
    medians follow on the whole set.  With want_hits the hit counts of each
    hashed chunk go down on a third stream while later chunks go up (PCIe is
    full duplex), and Batch.hits is a PendingHost.  Returns (Batch, device
    rows)."""
    n, d = int(host_rows.shape[0]), int(host_rows.shape[1])
    st = _dev.stream()
    dev = _dev.device()
    rows = torch.empty((max(n, 1), d), dtype=torch.int64, device=dev)
    src = torch.from_numpy(host_rows)
    nwords = (n + 31) // 32
    detmask = _dev.empty((max(nwords, 1),), torch.int32)
    hits = _dev.empty((max(n, 1),), torch.int64) if want_hits else None
    min_hits = min_hits_for(nu, L)
    copy = torch.cuda.Stream(device=dev)
    main = torch.cuda.current_stream(dev)
    copy.wait_stream(main)  # the buffers above were allocated on the main stream
    if hits is not None:
        down = torch.cuda.Stream(device=dev)
        hits_host = torch.empty((max(n, 1),), dtype=torch.int64, pin_memory=True)
    for c0 in range(0, n, chunk_rows):
        c1 = min(n, c0 + chunk_rows)
        with torch.cuda.stream(copy):
            rows[c0:c1].copy_(src[c0:c1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        main.wait_event(ev)
        _native.call("sfftb_hash_hits", rows[c0:c1].data_ptr(), c1 - c0, d, _dev.ptr(zmat), 1, L,
                     M, _dev.ptr(bits), int(kbound), min_hits,
                     None if hits is None else hits[c0:c1].data_ptr(),
                     detmask[c0 // 32:].data_ptr(), st)
        if hits is not None:
            hashed = torch.cuda.Event()
            hashed.record(main)
            down.wait_event(hashed)
            with torch.cuda.stream(down):
                hits_host[c0:c1].copy_(hits[c0:c1], non_blocking=True)
    rows.record_stream(copy)
    src_keep = src  # the host rows must outlive the async copies: synchronise below
    idx = _dev.empty((max(n, 1),), torch.int64)
    counts = _dev.zeros((1,), torch.int64)
    if n:
        ws = _dev.workspace(_native.lib().sfftb_compact_workspace_bytes(1, n))
        _native.call("sfftb_compact_mask", _dev.ptr(detmask), 1, n, _dev.ptr(idx),
                     _dev.ptr(counts), _dev.ptr(ws), st)
    coeffs = None
    if want_medians:
        coeffs = _dev.empty((max(n, 1),), torch.complex128)
        if n:
            _native.call("sfftb_medians", _dev.ptr(rows), d, _dev.ptr(zmat), 1, L, M,
                         _dev.ptr(ghat), _dev.ptr(idx), _dev.ptr(counts), n, _dev.ptr(coeffs),
                         st)
    copy.synchronize()
    del src_keep
    if hits is not None:
        done = torch.cuda.Event()
        done.record(down)
        hits = PendingHost(hits_host.numpy()[:n], done, (hits, hits_host, down))
    return Batch(1, L, M, n, ghat, theta0, hits, idx, counts, coeffs), rows[:n]


def detect_batch(samples, M, zmat, G, L, rows, kbound, nu, theta0=None,
                 want_medians=True, want_hits=False):
    """Run the full detection chain on device tensors.

    samples (G*L, M) c128; zmat (G*L, d) i64; rows (n, d) i64 (any signs);
    theta0: (G,) f64 tensor or None (default zero test per group).
    """
    ghat, theta0, bits = spectra(samples, M, G, L, theta0)
    return gather(ghat, theta0, bits, M, zmat, G, L, rows, kbound, nu, want_medians, want_hits)


def topk(idx, coeffs, counts, G, cap, theta, s_tilde, grid=False):
    """Threshold + top-s per group (detect.py:184-193) on device; ``grid``
    spreads each group over the whole GPU (large detected sets)."""
    cap = max(int(cap), 1)
    kidx = _dev.empty((G * cap,), torch.int64)
    kco = _dev.empty((G * cap,), torch.complex128)
    kcounts = _dev.empty((G,), torch.int64)
    ws = _dev.workspace(_native.lib().sfftb_topk_workspace_bytes(G, cap))
    _native.call("sfftb_topk_grid" if grid else "sfftb_topk", _dev.ptr(idx), _dev.ptr(coeffs),
                 _dev.ptr(counts), G, cap,
                 float(theta), int(s_tilde), _dev.ptr(kidx), _dev.ptr(kco), _dev.ptr(kcounts),
                 _dev.ptr(ws), _dev.stream())
    return kidx, kco, kcounts


def union_indices(kidx, kcounts, G, cap, n):
    """Ascending union of the kept indices of all groups (dimincr.py:239-240).

    Returns (idx (n,) i64 tensor, count (1,) i64 tensor)."""
    nwords = max((n + 31) // 32, 1)
    mask = _dev.zeros((nwords,), torch.int32)
    _native.call("sfftb_mark_indices", _dev.ptr(kidx), _dev.ptr(kcounts), G, max(cap, 1),
                 _dev.ptr(mask), n, _dev.stream())
    idx = _dev.empty((max(n, 1),), torch.int64)
    count = _dev.zeros((1,), torch.int64)
    if n:
        ws = _dev.workspace(_native.lib().sfftb_compact_workspace_bytes(1, n))
        _native.call("sfftb_compact_mask", _dev.ptr(mask), 1, n, _dev.ptr(idx), _dev.ptr(count),
                     _dev.ptr(ws), _dev.stream())
    return idx, count


def gather_rows(src, rows_idx, count_dev, cap):
    """dst[k] = src[rows_idx[k]] for k < count (device count)."""
    d = int(src.shape[1])
    dst = _dev.empty((max(int(cap), 1), d), torch.int64)
    _native.call("sfftb_gather_rows", _dev.ptr(src), d, _dev.ptr(rows_idx), _dev.ptr(count_dev),
                 int(cap), _dev.ptr(dst), _dev.stream())
    return dst


def pair_product(prev, vals):
    """J = prev x vals in lexicographic order (dimincr.py:155-175)."""
    n1, t = int(prev.shape[0]), int(prev.shape[1])
    n2 = int(vals.shape[0])
    out = _dev.empty((n1 * n2, t + 1), torch.int64)
    if n1 * n2:
        _native.call("sfftb_pair_product", _dev.ptr(prev), n1, t, _dev.ptr(vals), n2,
                     _dev.ptr(out), _dev.stream())
    return out
