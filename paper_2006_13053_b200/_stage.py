"""One dimension-incremental detection stage per host call (sfftb_sfft_stage).

The structured-oracle path of the driver (dimincr.py) hands a whole stage --
candidate pairing, sampler, fused transforms, hashing, compaction, medians,
top-s and the union -- to csrc/stage.cu in one ctypes call.  Buffers come from
a per-reconstruction ``Arena`` that grows to the largest stage and is reused
(stream order makes reuse safe; J/union buffers alternate between stages
because stage t+1 gathers its prefix from stage t's J).
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _dev, _native

_p = ctypes.c_void_p
_i64 = ctypes.c_int64


class StageDesc(ctypes.Structure):
    """Mirror of sfftb_stage_t (include/sfft_b200.h), field for field."""

    _fields_ = [
        ("prev_J", _p), ("prev_uidx", _p), ("prev_ucount", _p), ("prefix", _p),
        ("vals", _p), ("n1", _i64), ("n2", _i64), ("t", _i64), ("J", _p), ("n", _i64),
        ("tdim", _i64),
        ("support", _p), ("coeffs", _p), ("s", _i64), ("d", _i64),
        ("G", _i64), ("L", _i64), ("M", _i64), ("zmat_host", _p), ("tails_host", _p),
        ("tail_w", _i64), ("zmat", _p), ("tails", _p), ("noise_seed", ctypes.c_uint64),
        ("call0", _i64), ("sigma", ctypes.c_double), ("fused", ctypes.c_int),
        ("kbound", _i64), ("min_hits", _i64), ("s_tilde", _i64), ("theta", ctypes.c_double),
        ("anchored", _p), ("bins", _p), ("samples", _p), ("ghat", _p), ("theta0", _p),
        ("sumsq", _p), ("bits", _p), ("ws_dft", _p), ("detmask", _p), ("idx", _p),
        ("counts", _p), ("med", _p), ("ws_compact", _p), ("kidx", _p), ("kco", _p),
        ("kcounts", _p), ("ws_topk", _p), ("umask", _p), ("uidx", _p), ("ucount", _p),
        ("host_counts", _p), ("events", _p), ("zmat_host_ld", _i64), ("ptab", _p),
        ("vtab", _p), ("topk_grid", _i64), ("phase", _i64),
    ]


PHASES = ("candidates", "sampler", "transforms", "hashing", "compaction+medians",
          "top-s+union")
# (first, last) event of each phase (sfftb_stage_t.events), and the phases a
# call of each stage phase (0 whole, 1 spectra, 2 detection) records
_SPANS = {"candidates": (0, 1), "sampler": (2, 3), "transforms": (3, 4), "hashing": (5, 6),
          "compaction+medians": (6, 7), "top-s+union": (7, 8)}
_CALL = {0: (PHASES, (0, 8)), 1: (("sampler", "transforms"), (2, 4)),
         2: (("candidates", "hashing", "compaction+medians", "top-s+union"), (0, 8)),
         3: (("sampler",), (2, 3)), 4: (("transforms",), (3, 4))}


class Arena:
    """Named, growing device (and pinned host) buffers for one reconstruction."""

    def __init__(self):
        self._bufs = {}
        self.epoch = 0  # bumped on every (re)allocation: cached pointers stay valid until then
        # replaced buffers stay alive until settle(): a stage enqueued ahead
        # (spectra of t+1, planned buffers of t+1) may grow a buffer whose old
        # address an earlier descriptor still holds for pending device work
        self._old = []

    def settle(self):
        """Free replaced buffers -- only when no enqueued work can use them
        (the start of a reconstruction; an early return may have left spectra
        enqueued, so the stream is drained first)."""
        if self._old:
            torch.cuda.current_stream().synchronize()
            side_stream().synchronize()
            samp_stream().synchronize()
            det_stream().synchronize()
            self._old.clear()

    def get(self, name, numel, dtype=torch.int64, pinned=False):
        numel = max(int(numel), 1)
        ent = self._bufs.get(name)
        # a name is one buffer kind: never reinterpret another dtype / memory
        buf = ent[0] if ent is not None and ent[1] == dtype and ent[2] == pinned else None
        if buf is None or buf.numel() < numel:
            if ent is not None:
                self._old.append(ent[0])
            grow = numel if buf is None else max(numel, buf.numel() * 5 // 4)
            if pinned:
                buf = torch.empty(grow, dtype=dtype, pin_memory=True)
            else:
                buf = torch.empty(grow, dtype=dtype, device=_dev.device())
            self._bufs[name] = (buf, dtype, pinned)
            self.epoch += 1
        return buf[:numel]

    def ptr(self, name, numel, dtype=torch.int64):
        """Device address of a buffer of >= numel elements (no view built)."""
        ent = self._bufs.get(name)
        if ent is None or ent[1] != dtype or ent[2] or ent[0].numel() < numel:
            return self.get(name, numel, dtype).data_ptr()
        return ent[0].data_ptr()

    def bytes(self, name, nbytes):
        return self.ptr(name, (int(nbytes) + 7) // 8)


_LOCAL = threading.local()


def arena():
    """The calling thread's stage arena, kept across reconstructions (like a
    cached FFT plan): a repeated sfft allocates nothing.  Nothing returned to
    the caller aliases it -- results are copied to the host before sfft
    returns.  ``release()`` frees it."""
    a = getattr(_LOCAL, "arena", None)
    if a is None:
        a = _LOCAL.arena = Arena()
    return a


def release():
    """Drop the thread's arena.  Work an early return left queued (spectra
    of the next stage on the side / sampler streams, detection on det_stream)
    may still write into its buffers, which were allocated on the caller's
    stream: drain every stream of this thread before the caching allocator
    can hand that memory out again."""
    if getattr(_LOCAL, "arena", None) is not None:
        torch.cuda.current_stream().synchronize()
        for kind in ("side", "samp", "det"):
            st = (getattr(_LOCAL, kind, None) or {}).get(torch.cuda.current_device())
            if st is not None:
                st.synchronize()
    _LOCAL.arena = None


def _stream(kind, priority):
    dev = torch.cuda.current_device()
    cache = getattr(_LOCAL, kind, None)
    if cache is None:
        cache = {}
        setattr(_LOCAL, kind, cache)
    st = cache.get(dev)
    if st is None:
        st = cache[dev] = torch.cuda.Stream(device=dev, priority=priority)
    return st


def side_stream():
    """The calling thread's spectra stream (non-blocking, normal priority):
    stage t+1's sampler + transforms run there while stage t's detection
    runs on det_stream()."""
    return _stream("side", 0)


def samp_stream():
    """The calling thread's sampler stream (non-blocking): the short sampler
    kernels of stage t+1 interleave with stage t's transforms (normal
    priority measured marginally ahead of high: 4.01-4.03 vs 4.04 ms)."""
    return _stream("samp", int(os.environ.get("SFFTB_SAMP_PRIORITY", "0")))


def det_stream():
    """The calling thread's detection stream (non-blocking, high priority:
    its short, latency-bound kernels get SMs ahead of the transforms that
    overlap them, and the host waits on their counts)."""
    return _stream("det", int(os.environ.get("SFFTB_DET_PRIORITY", "-1")))


def run(desc, stream=None):
    """One stage call (desc.phase: 0 whole stage, 1 spectra, 2 detection);
    under a _native.Timeline the phase boundaries are recorded (CUDA events
    on the launch stream) as 'stage:<phase>' entries."""
    lib = _native.lib()
    tl = _native._TIMELINE
    evs = None
    if tl is not None:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
        for e in evs:
            e.record()  # materialise the cudaEvent_t; the stage re-records it
        arr = (ctypes.c_void_p * len(evs))(*[e.cuda_event for e in evs])
        desc.events = ctypes.addressof(arr)
    else:
        desc.events = None
    rc = lib.sfftb_sfft_stage(ctypes.addressof(desc),
                              _dev.stream() if stream is None else stream)
    if evs is not None:
        phases, (a, b) = _CALL[int(desc.phase)]
        for ph in phases:
            i, j = _SPANS[ph]
            tl.records.append((f"stage:{ph}", evs[i], evs[j]))
        tl.records.append(("sfftb_sfft_stage", evs[a], evs[b]))
        desc.events = None
    _native.check(rc, "sfftb_sfft_stage")


def buffers(A, desc, G, L, M, n, s, fused, slot):
    """Point desc's work buffers at arena storage sized for this stage;
    returns the tensors the driver reads afterwards.  A repeat with the same
    sizes and no arena (re)allocation since is a no-op (the pointers in desc
    are still current)."""
    key = (A.epoch, G, L, M, n, s, fused, slot)
    cached = getattr(desc, "_buf_cache", None)
    if cached is not None and cached[0] == key:
        return cached[1]
    out = _buffers(A, desc, G, L, M, n, s, fused, slot)
    desc._buf_cache = ((A.epoch, G, L, M, n, s, fused, slot), out)
    return out


def _buffers(A, desc, G, L, M, n, s, fused, slot):
    lib = _native.lib()
    f64 = torch.float64
    rows = G * L
    W = int(lib.sfftb_bitmap_words(M))
    nw = max((n + 31) // 32, 1)
    cap = max(n, 1)
    P = A.ptr
    # per slot: the sampler of a later stage may run while this one's bins are
    # still being transformed
    desc.anchored = P(f"anchored{slot}", 2 * G * max(s, 1), f64)
    desc.bins = P(f"bins{slot}", 2 * rows * M, f64)
    # the spectra of stage t+1 may be enqueued before stage t's detection:
    # what the detection reads (ghat, theta0, bits) is per slot
    desc.ghat = P(f"ghat{slot}", 2 * rows * M, f64)
    desc.theta0 = P(f"theta0{slot}", G, f64)
    desc.bits = P(f"bits{slot}", rows * W, torch.int32)
    if fused:
        desc.samples = desc.sumsq = None
        # + slack for per-group 256-B aligned regions (stage.cu)
        desc.ws_dft = A.bytes("ws_dft",
                              lib.sfftb_sample_detect_workspace_bytes(rows, M) + 256 * G + 256)
    else:
        desc.samples = P("samples", 2 * rows * M, f64)
        desc.sumsq = P("sumsq", rows, f64)
        desc.ws_dft = A.bytes("ws_dft", lib.sfftb_dft_workspace_bytes(min(rows, 65535), M))
    desc.detmask = P("detmask", G * nw, torch.int32)
    desc.idx = P("idx", G * cap)
    desc.counts = P("counts", G)
    desc.med = P("med", 2 * G * cap, f64)
    desc.ws_compact = A.bytes("ws_compact", max(lib.sfftb_compact_workspace_bytes(G, n),
                                                lib.sfftb_compact_workspace_bytes(1, n)))
    kidx = A.get("kidx", G * cap)
    kco = A.get("kco", 2 * G * cap, f64)
    desc.kidx, desc.kco = kidx.data_ptr(), kco.data_ptr()
    desc.kcounts = A.get("kcounts", G).data_ptr()
    desc.ws_topk = A.bytes("ws_topk", lib.sfftb_topk_workspace_bytes(G, cap))
    desc.umask = P("umask", nw, torch.int32)
    uidx = A.get(f"uidx{slot}", cap)
    ucount = A.get(f"ucount{slot}", 1)
    desc.uidx, desc.ucount = uidx.data_ptr(), ucount.data_ptr()
    hc = A.get(f"host_counts{slot}", G + 1, torch.int64, pinned=True)
    desc.host_counts = hc.data_ptr()
    kcounts = A.get("kcounts", G)
    return kidx, kco, uidx, ucount, hc, kcounts


def host_inputs(A, zs, tails, tail_w, slot=0):
    """Copy generators/tails into pinned staging buffers (one pair per slot,
    so the next stage's draws never overwrite a pending copy)."""
    G, L, tdim = zs.shape
    zh = A.get(f"zmat_host{slot}", G * L * tdim, torch.int64, pinned=True)
    zh.numpy()[:] = zs.reshape(-1)
    th = A.get(f"tails_host{slot}", G * tail_w, torch.float64, pinned=True)
    tn = th.numpy().reshape(G, tail_w)
    tn[:] = 0.0
    for g, tl in enumerate(tails):
        tn[g, :len(tl)] = tl
    return zh, th

