"""Device-buffer plumbing: PyTorch is used only for CUDA memory and streams.

All kernels are launched by libsfftb200 on the caller's current torch stream;
tensors handed to the C ABI are contiguous and their lifetimes are owned by
the Python side.
"""

from __future__ import annotations

import os
import threading
import warnings

import numpy as np
import torch

from . import _native

_PINNED_SMALL = os.environ.get("SFFTB_PINNED_SMALL", "1") == "1"
_CHECKED = False
# (device, stream handle) pinned by stream_scope(), per calling thread: the
# reference's kernels are reentrant and called from worker threads
# (analysis.py:271-274), so each thread keeps its own current stream.
_TLS = threading.local()


def device():
    """The CUDA device; raises if there is none (no CPU fallback exists)."""
    global _CHECKED
    sc = getattr(_TLS, "scope", None)
    if sc is not None:
        return sc[0]
    if not _CHECKED:
        if not torch.cuda.is_available():
            raise RuntimeError(
                "paper_2006_13053_b200 needs a CUDA device (sm_100a); "
                "there is no CPU fallback")
        _native.lib()
        _CHECKED = True
    return torch.device("cuda", torch.cuda.current_device())


def stream():
    """cudaStream_t of the current torch stream, as an int for ctypes."""
    sc = getattr(_TLS, "scope", None)
    if sc is not None:
        return sc[1]
    return torch.cuda.current_stream().cuda_stream


class stream_scope:
    """Pin the current device and stream for the duration of one API call
    (saves a torch query per launch on the driver's hot loop)."""

    def __enter__(self):
        self._prev = getattr(_TLS, "scope", None)
        if self._prev is None:
            dev = device()
            _TLS.scope = (dev, torch.cuda.current_stream(dev).cuda_stream)
        return self

    def __exit__(self, *exc):
        _TLS.scope = self._prev
        return False


def ptr(t):
    return None if t is None else t.data_ptr()


def upload(arr, dtype=None):
    """numpy -> contiguous CUDA tensor (int64 / float64 / complex128)."""
    a = np.ascontiguousarray(arr if dtype is None else np.asarray(arr, dtype=dtype))
    with warnings.catch_warnings():  # read-only FreqSet rows: torch only reads them
        warnings.simplefilter("ignore", UserWarning)
        t = torch.from_numpy(a)
    if t.numel() >= (1 << 20):
        if not t.is_pinned():
            t = t.pin_memory()
        return t.to(device(), non_blocking=True)
    if _PINNED_SMALL:
        # small arrays staged through torch's caching pinned-host allocator: the
        # copy is stream-ordered and asynchronous (no host sync per upload)
        staged = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        staged.copy_(t)
        return staged.to(device(), non_blocking=True)
    return t.to(device())


def download(t):
    """Device tensor -> numpy.  Large results go through a pinned staging
    buffer (the numpy array views it): a pageable D2H copy runs at ~2 GB/s on
    the B200 boxes, a pinned one at ~55 GB/s (tools/micro/h2d_bw.py)."""
    t = t.detach()
    if t.is_cuda and t.numel() * t.element_size() >= (1 << 20):
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t)
        return out.numpy()
    return t.cpu().numpy()


def empty(shape, dtype):
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch.zeros(shape, dtype=dtype, device=device())


def workspace(nbytes):
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device())


def as_i64(t):
    if isinstance(t, torch.Tensor):
        if t.device.type != "cuda":
            t = t.to(device())
        return t.to(torch.int64).contiguous()
    return upload(np.asarray(t, dtype=np.int64))


def as_c128(t):
    if isinstance(t, torch.Tensor):
        if t.device.type != "cuda":
            t = t.to(device())
        return t.to(torch.complex128).contiguous()
    return upload(np.asarray(t, dtype=np.complex128))
