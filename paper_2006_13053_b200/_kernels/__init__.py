"""The drop-in kernel plugin API (mirrors latfft/_kernels/__init__.py).

Same four functions with the same argument order, dtypes, return shapes and
exceptions as the reference's dispatcher (_kernels/__init__.py:29-70); one
backend, ``BACKEND == "cuda"``.  There is no ``LATFFT_PURE_PYTHON`` switch and
no numpy fallback: every call goes through libsfftb200's C ABI (host buffers
in and out, device work inside).
"""

from __future__ import annotations

import ctypes

import numpy as np

from .. import _native

BACKEND = "cuda"


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def hc_count(d, bound, weights):
    """|weighted hyperbolic cross| (_kernels/__init__.py:29-33)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    out = ctypes.c_int64(0)
    _native.check(_native.lib().sfftb_hc_count(int(d), float(bound), _p(w), ctypes.byref(out)),
                  "hc_count")
    return int(out.value)


def hc_enumerate(d, bound, weights):
    """Lexicographic enumeration of the cross (_kernels/__init__.py:36-42)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    n = hc_count(d, bound, w)
    out = np.empty((n, int(d)), dtype=np.int64)
    _native.check(_native.lib().sfftb_hc_enumerate(int(d), float(bound), _p(w), _p(out), n),
                  "hc_enumerate")
    return out


def rows_injective_mod(elems, p):
    """True iff elems reduced componentwise mod p stay distinct
    (_kernels/__init__.py:45-51)."""
    e = np.ascontiguousarray(elems, dtype=np.int64)
    if e.ndim == 1:
        e = e.reshape(-1, 1)
    out = ctypes.c_int(0)
    _native.check(_native.lib().sfftb_rows_injective_mod(_p(e), e.shape[0], e.shape[1], int(p),
                                                         ctypes.byref(out)),
                  "rows_injective_mod")
    return bool(out.value)


def detect_gather(elems, zmat, M, ghat, theta, hit_threshold, want_medians):
    """Hit counts and (odd-L) medians per candidate row
    (_kernels/__init__.py:54-70; elems pre-reduced mod M)."""
    elems = np.ascontiguousarray(elems, dtype=np.int64)
    zmat = np.ascontiguousarray(zmat, dtype=np.int64)
    ghat = np.ascontiguousarray(ghat, dtype=np.complex128)
    L = zmat.shape[0]
    if want_medians and L % 2 == 0:
        raise ValueError("medians require an odd lattice count")
    n = elems.shape[0]
    d = elems.shape[1] if elems.ndim == 2 else 0
    hits = np.zeros(n, dtype=np.int64)
    medians = np.zeros(n, dtype=np.complex128)
    _native.check(_native.lib().sfftb_detect_gather(
        _p(elems), n, d, _p(zmat), L, int(M), _p(ghat), float(theta), float(hit_threshold),
        int(bool(want_medians)), _p(hits), _p(medians)), "detect_gather")
    return hits, medians
