"""Normalised prime-length DFT on the device (Bluestein, FP64).

Public contract of latfft/dft.py:18-27: coefficient h equals
(1/M) sum_j samples[j] exp(-2 pi i j h / M); non-finite, empty or
non-1-d input raises ParameterError.  The transform itself runs in
libsfftb200 (csrc/fft.cu); ``dft_batch`` is the device-resident form the
drivers use for all L (or r*L) lattices at once.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _native
from .errors import ParameterError


def dft_batch(x, M, inverse=False, scale=None, out=None):
    """Row-wise DFT of a (B, M) complex128 CUDA tensor.

    forward (default): scale defaults to 1/M (dft_forward_normalized);
    inverse: y[h] = scale * sum_j x[j] e^{+2 pi i jh/M}, scale default 1
    (the sampler's M * ifft, polyeval.py:87).
    """
    B = x.shape[0]
    if scale is None:
        scale = 1.0 if inverse else 1.0 / M
    if out is None:
        out = _dev.empty((B, M), torch.complex128)
    step = 65535
    ws = _dev.workspace(_native.lib().sfftb_dft_workspace_bytes(min(B, step), M))
    for b0 in range(0, B, step):
        b1 = min(B, b0 + step)
        xs = x[b0:b1]
        _native.call("sfftb_dft", _dev.ptr(xs), M, _dev.ptr(out[b0:b1]), M, b1 - b0, M,
                     int(bool(inverse)), float(scale), _dev.ptr(ws), _dev.stream())
    return out


def dft_forward_normalized(samples):
    """Length-M forward DFT with 1/M normalisation (dft.py:18-27)."""
    x = np.asarray(samples, dtype=np.complex128)
    if x.ndim != 1:
        raise ParameterError("samples must be a 1-d vector")
    if x.size == 0:
        raise ParameterError("samples must be nonempty")
    if not np.all(np.isfinite(x.view(np.float64))):
        raise ParameterError("samples contain NaN or Inf")
    dev = _dev.upload(x).reshape(1, -1)
    return _dev.download(dft_batch(dev, x.size)[0])
