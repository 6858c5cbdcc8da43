"""Frequency detection from samples along a multi-lattice configuration.

Public entry points of latfft/detect.py (detect_frequencies :149-155,
detect_and_compute :158-169, detect_topk :172-195, postprocess_r1l :198-228,
per_lattice_coefficients :112-119, default_zero_test :42-53, DetectionResult
:56-95, format_detection :231-240) with their argument and return
conventions.  The work runs on the device (_engine.detect_batch); results are
held as device tensors and materialised as numpy arrays on first access.

``samples`` may be the reference's list of L host vectors, or (B200 path) a
(L, M) complex128 CUDA tensor already in HBM.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _dev, _engine, _native
from .dft import dft_batch
from .errors import ParameterError
from .freqset import FreqSet


class ZeroTest:
    """Absolute magnitude threshold for the approximate zero test."""

    __slots__ = ("theta_zero",)

    def __init__(self, theta_zero):
        if theta_zero < 0:
            raise ParameterError("theta_zero must be >= 0")
        self.theta_zero = float(theta_zero)

    def __repr__(self):
        return f"ZeroTest({self.theta_zero!r})"


def _lazy_np(v):
    if isinstance(v, torch.Tensor):
        return _dev.download(v)
    if isinstance(v, _engine.PendingHost):
        return v.result()
    return v


class DetectionResult:
    """Detected frequencies, coefficients and per-candidate hit counts.

    ``hits`` aligns with ``candidates``; ``detected_idx`` indexes the
    candidate set; ``coeffs`` (if present) aligns with ``detected``.
    """

    __slots__ = ("candidates", "_hits", "_idx", "_coeffs", "theta_zero", "_detected")

    def __init__(self, candidates, hits, detected_idx, coeffs, theta_zero):
        self.candidates = candidates
        self._hits = hits
        self._idx = detected_idx
        self._coeffs = coeffs
        self.theta_zero = float(theta_zero)
        self._detected = None

    @property
    def hits(self):
        self._hits = _lazy_np(self._hits)
        return self._hits

    @property
    def detected_idx(self):
        self._idx = _lazy_np(self._idx)
        return self._idx

    @property
    def coeffs(self):
        self._coeffs = _lazy_np(self._coeffs)
        return self._coeffs

    def device_arrays(self):
        """(detected_idx, coeffs) as CUDA tensors when still resident."""
        return self._idx, self._coeffs

    @property
    def detected(self):
        if self._detected is None:
            idx = self._idx
            if isinstance(idx, torch.Tensor):
                self._detected = self.candidates.take(idx)
            else:
                self._detected = self.candidates.take(np.asarray(idx, dtype=np.int64))
        return self._detected

    def __repr__(self):
        return (f"DetectionResult(candidates={len(self.candidates)}, "
                f"detected={len(self.detected)})")

    @property
    def per_lattice_hits(self):
        return {k: int(h) for k, h in zip(self.candidates, self.hits)}

    def hit_count(self, k):
        row = np.asarray(k, dtype=np.int64)
        where = np.flatnonzero(np.all(self.candidates.elems == row, axis=1))
        if where.size == 0:
            raise KeyError(k)
        return int(self.hits[where[0]])

    def coeffs_dict(self):
        if self._coeffs is None:
            return {}
        return {k: complex(c) for k, c in zip(self.detected, self.coeffs)}


# ---------------------------------------------------------------------------

def _stack_samples(samples, config, deferred=False, check=True):
    """Validated (L, M) complex128 CUDA tensor (detect.py:98-109 checks).
    With ``deferred`` the finiteness check is returned as a device flag
    instead of being read here: (tensor, flag or None)."""
    L = config.L
    if isinstance(samples, torch.Tensor):
        if samples.ndim != 2 or samples.shape[0] != L:
            raise ParameterError(f"expected {L} sample vectors, got {tuple(samples.shape)}")
        M = config.shared_M
        if M is None or samples.shape[1] != M:
            raise ParameterError("sample tensor does not match the lattice sizes")
        t = _dev.as_c128(samples)
    else:
        if len(samples) != L:
            raise ParameterError(f"expected {L} sample vectors, got {len(samples)}")
        rows = []
        for s, lat in zip(samples, config.lattices):
            s = np.asarray(s, dtype=np.complex128)
            if s.shape != (lat.M,):
                raise ParameterError(
                    f"sample vector of length {s.shape} does not match M={lat.M}")
            rows.append(s)
        if config.shared_M is None:
            t = [_dev.upload(r).reshape(1, -1) for r in rows]
            return (t, None) if deferred else t
        t = _dev.upload(np.vstack(rows))
    if deferred:
        return t, (torch.isfinite(torch.view_as_real(t)).all() if check else None)
    if not bool(torch.isfinite(torch.view_as_real(t)).all()):
        raise ParameterError("samples contain NaN or Inf")
    return t


def _zero_from_device(t):
    """default_zero_test on staged device samples (one value per config)."""
    if isinstance(t, list):  # distinct lattice sizes: per-lattice RMS on device
        rms = []
        for s in t:
            M = int(s.shape[1])
            sq = _dev.empty((1,), torch.float64)
            _native.call("sfftb_sumsq", _dev.ptr(s), M, 1, M, _dev.ptr(sq), _dev.stream())
            rms.append(sq)
        vals = sorted(math.sqrt(float(v[0]) / int(s.shape[1])) for v, s in zip(rms, t))
        h = len(vals) // 2
        mid = vals[h] if len(vals) % 2 == 1 else 0.5 * (vals[h - 1] + vals[h])
        return ZeroTest(max(1e-12, 1e-10 * mid))
    L, M = int(t.shape[0]), int(t.shape[1])
    return ZeroTest(float(_engine.zero_thresholds(t, 1, L, M)[0]))


def default_zero_test(samples):
    """max(1e-12, 1e-10 * median per-lattice RMS) (detect.py:42-53), on device."""
    if isinstance(samples, torch.Tensor):
        return _zero_from_device(_dev.as_c128(samples))
    rows = [np.asarray(s, dtype=np.complex128).reshape(-1) for s in samples]
    if len({r.size for r in rows}) == 1:
        return _zero_from_device(_dev.upload(np.vstack(rows)))
    return _zero_from_device([_dev.upload(r).reshape(1, -1) for r in rows])


# host-resident candidate sets at least this large are uploaded in chunks
# overlapped with hashing (_engine.gather_streamed)
STREAM_UPLOAD_BYTES = 256 << 20


# candidate sets at least this large hash without a host bound (-1): the hash
# kernel checks the rows warp by warp on the device and takes the 32-bit
# residue chain where it is exact, the 64-bit chain elsewhere (csrc/hash.cu
# AUTO), so no host pass over the rows (a min/max over 5.4 GB at config 4)
AUTO_BOUND_ROWS = 1 << 16


def _kbound(gamma):
    kb = gamma.memo_get("kbound")
    if kb is not None:
        return kb
    if len(gamma) >= AUTO_BOUND_ROWS and gamma.memo_get("bounds") is None:
        return -1
    return gamma.memo("kbound", gamma.kbound)


def _theta_tensor(theta):
    return torch.full((1,), float(theta), dtype=torch.float64, device=_dev.device())


# the reference dispatcher serves L <= 128 with its compiled gather and larger
# L with the numpy fallback (_kernels/__init__.py:26,62): |v| by hypot, np.median
MAX_COMPILED_L = 128


def _gather(samples, config, gamma, zero, want_medians, want_hits=True):
    """Device detection for one configuration -> engine Batch (G = 1)."""
    M = config.shared_M
    if M is None or config.L > MAX_COMPILED_L:
        # distinct lattice sizes, or more lattices than the reference's
        # compiled gather serves: the reference's numpy semantics
        return _gather_mixed(samples, config, gamma, zero, want_medians)
    if not gamma.dim * (M - 1) ** 2 < 2**62:
        raise ParameterError("lattice size too large for int64 residues")
    if config.dim != gamma.dim:
        raise ParameterError("candidate set/lattice dimension mismatch")
    host = gamma._host if gamma._dev is None else None
    if host is not None and host.nbytes >= STREAM_UPLOAD_BYTES:
        # large host-resident candidate set: upload in chunks, overlapped with
        # the hashing of the chunks already on the device
        ghat, theta0, bits = _engine.spectra(samples, M, 1, config.L,
                                             _theta_tensor(zero.theta_zero))
        b, rows = _engine.gather_streamed(ghat, theta0, bits, M, config.zmat_device(),
                                          config.L, host, _kbound(gamma), config.nu,
                                          want_medians=want_medians, want_hits=want_hits)
        gamma._dev = rows  # cached like FreqSet.device()
        return b
    return _engine.detect_batch(samples, M, config.zmat_device(), 1, config.L,
                                gamma.device(), _kbound(gamma), config.nu,
                                theta0=_theta_tensor(zero.theta_zero),
                                want_medians=want_medians, want_hits=want_hits)


def _gather_mixed(samples, config, gamma, zero, want_medians):
    """Distinct lattice sizes (detect.py:134-145): each lattice's spectrum and
    per-row values on the device, then hits by |v| > theta with np.abs's
    hypot and np.median per row (csrc/hash.cu rows_hits_medians)."""
    rows = gamma.device()
    n = len(gamma)
    L = config.L
    theta = float(zero.theta_zero)
    allrows = torch.arange(max(n, 1), dtype=torch.int64, device=_dev.device())
    vals = torch.empty((max(n, 1), L), dtype=torch.complex128, device=_dev.device())
    col_buf = torch.empty((max(n, 1),), dtype=torch.complex128, device=_dev.device())
    for col, (s, lat) in enumerate(zip(samples, config.lattices)):  # staged per lattice
        g = dft_batch(s.reshape(1, -1), lat.M)
        z = _dev.upload(lat.z.reshape(1, -1))
        if n:
            _native.call("sfftb_lattice_values", _dev.ptr(rows), gamma.dim, _dev.ptr(z), 1,
                         lat.M, _dev.ptr(g), _dev.ptr(allrows), n, _dev.ptr(col_buf),
                         _dev.stream())
            vals[:n, col] = col_buf[:n]
    thr = config.nu * L
    hits = _dev.empty((max(n, 1),), torch.int64)
    med = _dev.zeros((max(n, 1),), torch.complex128)
    if n:
        _native.call("sfftb_rows_hits_medians", _dev.ptr(vals), n, L, theta, float(thr),
                     int(bool(want_medians)), _dev.ptr(hits), _dev.ptr(med), _dev.stream())
    hits = hits[:n]
    mask = _dev.empty((max((n + 31) // 32, 1),), torch.int32)
    idx = _dev.empty((max(n, 1),), torch.int64)
    cnt = _dev.zeros((1,), torch.int64)
    if n:
        _native.call("sfftb_threshold_mask", _dev.ptr(hits), n, float(thr), _dev.ptr(mask),
                     _dev.stream())
        ws = _dev.workspace(_native.lib().sfftb_compact_workspace_bytes(1, n))
        _native.call("sfftb_compact_mask", _dev.ptr(mask), 1, n, _dev.ptr(idx), _dev.ptr(cnt),
                     _dev.ptr(ws), _dev.stream())
    k = int(_dev.download(cnt)[0])
    idx = idx[:k]
    coeffs = None
    if want_medians:
        coeffs = _dev.empty((max(k, 1),), torch.complex128)
        if k:
            _native.call("sfftb_gather_rows", _dev.ptr(med.view(torch.int64).view(-1, 2)), 2,
                         _dev.ptr(idx), _dev.ptr(cnt), k, _dev.ptr(coeffs), _dev.stream())
        coeffs = coeffs[:k]
    return _engine.Batch(1, L, 0, n, None, _theta_tensor(theta), hits, idx, cnt, coeffs)


def _result_from_batch(gamma, b, theta0, with_coeffs):
    cnt = int(b.counts[0]) if b.counts is not None else 0
    idx = b.idx[:cnt]
    coeffs = b.coeffs[:cnt] if (with_coeffs and b.coeffs is not None) else None
    return DetectionResult(gamma, b.hits, idx, coeffs, theta0)


def _detect_async(samples, config, gamma, zero, want_medians):
    """The shared-M detection with ONE host synchronisation: the finiteness
    check, the zero test and the whole chain are enqueued back to back, then
    (finite flag, theta0, detected count) come back in one read.  None when
    the call takes another path (distinct lattice sizes, L > 128, a large
    host-resident candidate set that streams its upload)."""
    M = config.shared_M
    if M is None or config.L > MAX_COMPILED_L:
        return None
    host = gamma._host if gamma._dev is None else None
    if host is not None and host.nbytes >= STREAM_UPLOAD_BYTES:
        return None
    t = _stack_samples(samples, config, deferred=True, check=False)[0]
    if not gamma.dim * (M - 1) ** 2 < 2**62:
        raise ParameterError("lattice size too large for int64 residues")
    if config.dim != gamma.dim:
        raise ParameterError("candidate set/lattice dimension mismatch")
    L, n, d = config.L, len(gamma), gamma.dim
    rows = gamma.device()
    lib = _native.lib()
    ws = _dev.workspace(lib.sfftb_detect_dev_workspace_bytes(L, M, n))
    hits = _dev.empty((max(n, 1),), torch.int64)
    idx = _dev.empty((max(n, 1),), torch.int64)
    coeffs = _dev.empty((max(n, 1),), torch.complex128) if want_medians else None
    small = _dev.empty((3,), torch.int64)  # count | theta0 (f64) | non-finite flag (i32)
    theta_in = None if zero is None else _theta_tensor(zero.theta_zero)
    # the whole chain in one C call (csrc/detect_dev.cu), one read-back
    _native.call("sfftb_detect_dev", _dev.ptr(t), L, M, _dev.ptr(rows), n, d,
                 _dev.ptr(config.zmat_device()), _dev.ptr(theta_in), int(_kbound(gamma)),
                 _engine.min_hits_for(config.nu, L), int(bool(want_medians)), _dev.ptr(hits),
                 _dev.ptr(idx), small.data_ptr(), _dev.ptr(coeffs), small[1:].data_ptr(),
                 small[2:].data_ptr(), _dev.ptr(ws), _dev.stream())
    host = _dev.download(small)
    if int(host[2]) & 0xFFFFFFFF:
        raise ParameterError("samples contain NaN or Inf")
    cnt = int(host[0])
    th = float(host[1:2].view(np.float64)[0])
    return DetectionResult(gamma, hits[:n], idx[:cnt],
                           coeffs[:cnt] if want_medians else None, th)


def detect_frequencies(samples, config, gamma, zero=None):
    """Alg. 1: keep k when its nonzero count reaches nu*L (detect.py:149-155)."""
    res = _detect_async(samples, config, gamma, zero, False)
    if res is not None:
        return res
    t = _stack_samples(samples, config)
    if zero is None:
        zero = _zero_from_device(t)
    b = _gather(t, config, gamma, zero, False)
    return _result_from_batch(gamma, b, zero.theta_zero, False)


def detect_and_compute(samples, config, gamma, zero=None):
    """Alg. 2: classification + coefficient medians (detect.py:158-169)."""
    if config.nu != 0.5:
        raise ParameterError("coefficient computation requires nu = 1/2")
    if config.L % 2 == 0:
        raise ParameterError("coefficient computation requires odd L")
    res = _detect_async(samples, config, gamma, zero, True)
    if res is not None:
        return res
    t = _stack_samples(samples, config)
    if zero is None:
        zero = _zero_from_device(t)
    b = _gather(t, config, gamma, zero, True)
    return _result_from_batch(gamma, b, zero.theta_zero, True)


def detect_topk(samples, config, gamma, s_tilde, theta, zero=None):
    """Alg. 4: detect_and_compute, |coeff| >= theta, s_tilde largest
    (ties: ascending lexicographic frequency), candidate order (detect.py:172-195)."""
    s_tilde = int(s_tilde)
    if s_tilde < 0:
        raise ParameterError("s_tilde must be >= 0")
    if theta < 0:
        raise ParameterError("theta must be >= 0")
    res = detect_and_compute(samples, config, gamma, zero=zero)
    idx, coeffs = res.device_arrays()
    if not isinstance(idx, torch.Tensor):
        idx = _dev.as_i64(idx)
        coeffs = _dev.as_c128(coeffs)
    n = int(idx.numel())
    counts = torch.tensor([n], dtype=torch.int64, device=_dev.device())
    kidx, kco, kcounts = _engine.topk(idx, coeffs, counts, 1, n, theta, s_tilde)
    k = int(kcounts[0])
    return DetectionResult(res.candidates, res._hits, kidx[:k], kco[:k], res.theta_zero)


def _per_lattice_values_dev(samples, config, gamma):
    """(L, n) complex128 device tensor of ghat_l[r_l(k)] (detect.py:112-119)."""
    t = _stack_samples(samples, config)
    n, L = len(gamma), config.L
    out = _dev.empty((L, max(n, 1)), torch.complex128)
    rows = gamma.device()
    if isinstance(t, list):
        for col, (s, lat) in enumerate(zip(t, config.lattices)):
            g = dft_batch(s, lat.M)
            z = _dev.upload(lat.z.reshape(1, -1))
            if n:
                _native.call("sfftb_lattice_values", _dev.ptr(rows), gamma.dim, _dev.ptr(z), 1,
                             lat.M, _dev.ptr(g), None, n, _dev.ptr(out[col]), _dev.stream())
        return out
    M = config.shared_M
    g = dft_batch(t, M)
    z = config.zmat_device()
    for col in range(L):
        if n:
            _native.call("sfftb_lattice_values", _dev.ptr(rows), gamma.dim, _dev.ptr(z[col]), 1,
                         M, _dev.ptr(g[col]), None, n, _dev.ptr(out[col]), _dev.stream())
    return out


def per_lattice_coefficients(samples, config, gamma):
    """(n, L) per-lattice estimates ghat_l[r_l(k)] (detect.py:112-119)."""
    n = len(gamma)
    return _dev.download(_per_lattice_values_dev(samples, config, gamma)[:, :n].T.contiguous())


def postprocess_r1l(result, samples, config, zero=None):
    """Average the estimates of lattices on which a detected frequency's
    residue is unique within the detected set; keep the median otherwise;
    drop |value| <= theta_zero (detect.py:198-228).  One K9 call
    (csrc/postprocess.cu) plus the compaction of the kept rows."""
    if zero is None:
        zero = ZeroTest(result.theta_zero)
    n = len(result.detected)
    if n == 0:
        return result
    L = config.L
    vals = _per_lattice_values_dev(samples, config, result.detected)
    if vals.shape[1] != n:
        vals = vals[:, :n].contiguous()
    rows = result.detected.device()
    Ms = np.array([lat.M for lat in config.lattices], dtype=np.int64)
    offs_h = np.concatenate([[0], np.cumsum(Ms)]).astype(np.int64)
    offs = _dev.upload(offs_h)
    med = _dev.as_c128(result.coeffs).contiguous()
    refined = _dev.empty((n,), torch.complex128)
    keep = _dev.empty(((n + 31) // 32,), torch.int32)
    lib = _native.lib()
    ws = _dev.workspace(lib.sfftb_r1l_workspace_bytes(n, L, int(offs_h[-1])))
    _native.call("sfftb_postprocess_r1l", _dev.ptr(rows), n, result.detected.dim,
                 _dev.ptr(config.zmat_device()), _dev.ptr(offs), L, int(offs_h[-1]),
                 _dev.ptr(vals), _dev.ptr(med), float(zero.theta_zero), _dev.ptr(refined),
                 _dev.ptr(keep), _dev.ptr(ws), _dev.stream())
    pos = _dev.empty((n,), torch.int64)
    cnt = _dev.zeros((1,), torch.int64)
    cws = _dev.workspace(lib.sfftb_compact_workspace_bytes(1, n))
    _native.call("sfftb_compact_mask", _dev.ptr(keep), 1, n, _dev.ptr(pos), _dev.ptr(cnt),
                 _dev.ptr(cws), _dev.stream())
    k = int(_dev.download(cnt)[0])
    det = _dev.as_i64(result.detected_idx).contiguous()
    idx = _dev.empty((max(k, 1),), torch.int64)
    co = _dev.empty((max(k, 1),), torch.complex128)
    if k:
        _native.call("sfftb_gather_rows", _dev.ptr(det), 1, _dev.ptr(pos), _dev.ptr(cnt), k,
                     _dev.ptr(idx), _dev.stream())
        _native.call("sfftb_gather_rows", _dev.ptr(refined.view(torch.int64).view(n, 2)), 2,
                     _dev.ptr(pos), _dev.ptr(cnt), k, _dev.ptr(co), _dev.stream())
    return DetectionResult(result.candidates, result._hits, idx[:k], co[:k], result.theta_zero)


def format_detection(result):
    """Text form: components, Re, Im, hit count (detect.py:231-240)."""
    lines = []
    has = result.coeffs is not None
    for i, idx in enumerate(result.detected_idx):
        row = result.candidates.elems[idx]
        c = complex(result.coeffs[i]) if has else 0j
        comps = " ".join(str(int(v)) for v in row)
        lines.append(f"{comps} {float(c.real)!r} {float(c.imag)!r} {int(result.hits[idx])}")
    return "\n".join(lines) + ("\n" if lines else "")

