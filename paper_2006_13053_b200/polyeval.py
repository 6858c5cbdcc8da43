"""Sparse trigonometric polynomials and sampling oracles.

Public surface of latfft/polyeval.py:22-143 for the hot path: ``SparsePoly``,
``evaluate``/``evaluate_many`` (dense), ``evaluate_on_lattice`` (structured),
``SamplingOracle`` with its evaluation counter, ``oracle_from_poly``,
``sample_on_lattice``, ``random_poly``.  Every evaluation runs on the device
(csrc/sample.cu + csrc/fft.cu).

``oracle_from_poly`` returns a :class:`PolyOracle`: a SamplingOracle whose
lattice samplings -- including the fixed-tail lattices of the
dimension-incremental driver -- take the structured path (anchor-phase
scatter into residue bins + inverse Bluestein DFT), batched over all lattices
of a detection stage.  Black-box oracles (any ``fn``) are evaluated on the
host by their own ``fn`` and uploaded.

Noise (config 5): ``oracle_from_poly(p, noise_sigma=s, noise_seed=k)`` adds
s*(N(0,1) + i N(0,1)) to every sample, drawn per oracle call from the
Philox4x32-10 stream keyed by k with counter (sample index, call index) --
the harness noise model (the reference has none), restated in
oracle/port.py:noise_for_call.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _dev, _native
from .dft import dft_batch
from .errors import ParameterError
from .freqset import FreqSet


class SparsePoly:
    """Support (FreqSet) plus aligned nonzero complex coefficients."""

    __slots__ = ("support", "coeffs", "_dev")

    def __init__(self, support, coeffs):
        if not isinstance(support, FreqSet):
            raise ParameterError("support must be a FreqSet")
        coeffs = np.asarray(coeffs, dtype=np.complex128)
        if coeffs.shape != (len(support),):
            raise ParameterError("need exactly one coefficient per support frequency")
        if len(support) and np.any(coeffs == 0):
            raise ParameterError("coefficients must be nonzero")
        coeffs.setflags(write=False)
        self.support, self.coeffs = support, coeffs
        self._dev = None

    @classmethod
    def from_dict(cls, dim, mapping):
        support = FreqSet(dim, list(mapping.keys()))
        return cls(support, np.array([mapping[k] for k in support], dtype=np.complex128))

    def as_dict(self):
        return {k: complex(c) for k, c in zip(self.support, self.coeffs)}

    @property
    def dim(self):
        return self.support.dim

    def __len__(self):
        return len(self.support)

    def device(self):
        """(support int64 (s, d), coeffs complex128 (s,)) on the device."""
        if self._dev is None:
            sup = self.support
            if sup._dev is not None:
                self._dev = (sup.device(), _dev.upload(self.coeffs))
            else:
                # host support: rows and coefficients travel as ONE staged
                # buffer and one host-to-device copy (the polynomial upload
                # opens every end-to-end reconstruction)
                s, d = len(self), self.dim
                rows = np.ascontiguousarray(sup.elems, dtype=np.int64).reshape(s, d)
                co = np.ascontiguousarray(self.coeffs, dtype=np.complex128)
                off = s * d + (s * d) % 2  # coefficients 16-byte aligned
                buf = np.zeros(off + 2 * s, dtype=np.int64)
                buf[:s * d] = rows.reshape(-1)
                buf[off:] = co.view(np.int64)
                dev = _dev.upload(buf)
                sup._dev = dev[:s * d].view(s, d)
                self._dev = (sup._dev, dev[off:].view(torch.complex128))
        return self._dev


def _eval_points_dev(p, X_dev):
    sup, c = p.device()
    m = X_dev.shape[0]
    out = _dev.empty((m,), torch.complex128)
    if len(p) == 0:
        out.zero_()
        return out
    _native.call("sfftb_eval_dense", _dev.ptr(sup), len(p), p.dim, _dev.ptr(c),
                 _dev.ptr(X_dev), m, _dev.ptr(out), _dev.stream())
    return out


def evaluate(p, x):
    """p(x) at one point by direct summation (polyeval.py:57-63)."""
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (p.dim,):
        raise ParameterError("point/polynomial dimension mismatch")
    return complex(_dev.download(_eval_points_dev(p, _dev.upload(x.reshape(1, -1))))[0])


def evaluate_many(p, X):
    """p at the rows of an (m, d) point array (polyeval.py:66-75)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != p.dim:
        raise ParameterError("points must be an (m, d) array")
    return _dev.download(_eval_points_dev(p, _dev.upload(X)))


def lattice_bins_device(p, zmat_dev, M, tails_dev, G, L, t_dim):
    """Residue bins B (G*L, M) of the anchored coefficients (polyeval.py:85-86)."""
    sup, c = p.device()
    s = len(p)
    anchored = _dev.empty((G, max(s, 1)), torch.complex128)
    if s:
        _native.call("sfftb_anchor_coeffs", _dev.ptr(sup), s, p.dim, t_dim, _dev.ptr(c),
                     _dev.ptr(tails_dev), G, _dev.ptr(anchored), _dev.stream())
    bins = _dev.empty((G * L, M), torch.complex128)
    _native.call("sfftb_scatter_bins", _dev.ptr(sup), s, p.dim, t_dim, _dev.ptr(anchored),
                 _dev.ptr(zmat_dev), G, L, M, _dev.ptr(bins), None, _dev.stream())
    return bins


def sample_lattices_device(p, zmat_dev, M, tails_dev, G, L, t_dim):
    """Structured samples of G*L lattices (G tails, L generators each).

    zmat_dev: (G*L, t_dim) int64; tails_dev: (G, d - t_dim) float64.
    Returns (G*L, M) complex128 = values at [j z/M mod 1 | tail_g], j < M.
    """
    sup, c = p.device()
    s = len(p)
    anchored = _dev.empty((G, max(s, 1)), torch.complex128)
    if s:
        _native.call("sfftb_anchor_coeffs", _dev.ptr(sup), s, p.dim, t_dim, _dev.ptr(c),
                     _dev.ptr(tails_dev), G, _dev.ptr(anchored), _dev.stream())
    bins = _dev.empty((G * L, M), torch.complex128)
    _native.call("sfftb_scatter_bins", _dev.ptr(sup), s, p.dim, t_dim, _dev.ptr(anchored),
                 _dev.ptr(zmat_dev), G, L, M, _dev.ptr(bins), None, _dev.stream())
    return dft_batch(bins, M, inverse=True, scale=1.0)


def evaluate_on_lattice(p, lat):
    """p at all M nodes of one lattice (polyeval.py:78-87), structured."""
    if lat.dim != p.dim:
        raise ParameterError("lattice/polynomial dimension mismatch")
    z = _dev.upload(lat.z.reshape(1, -1))
    tails = _dev.empty((1, 1), torch.float64)
    return _dev.download(sample_lattices_device(p, z, lat.M, tails, 1, 1, p.dim)[0])


class SamplingOracle:
    """Black-box evaluator with a cumulative sample counter (polyeval.py:90-130)."""

    __slots__ = ("fn", "dim", "lattice_fn", "count")

    def __init__(self, fn, dim, lattice_fn=None):
        self.fn = fn
        self.dim = int(dim)
        self.lattice_fn = lattice_fn
        self.count = 0

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        if x.shape != (self.dim,):
            raise ParameterError("point/oracle dimension mismatch")
        self.count += 1
        return complex(self.fn(x[None, :])[0])

    def sample_many(self, X):
        X = np.asarray(X, dtype=np.float64)
        if X.ndim != 2 or X.shape[1] != self.dim:
            raise ParameterError("points must be an (m, d) array")
        self.count += X.shape[0]
        return np.asarray(self.fn(X), dtype=np.complex128)

    def sample_lattice(self, lat):
        if lat.dim != self.dim:
            raise ParameterError("lattice/oracle dimension mismatch")
        if self.lattice_fn is not None:
            self.count += lat.M
            return np.asarray(self.lattice_fn(lat), dtype=np.complex128)
        from .lattice import lattice_nodes

        return self.sample_many(lattice_nodes(lat))


class PolyOracle(SamplingOracle):
    """SamplingOracle over a SparsePoly with device sampling paths.

    ``calls`` counts oracle calls (one per sample_many / lattice); it indexes
    the optional noise stream.
    """

    __slots__ = ("poly", "noise_sigma", "noise_seed", "calls", "fast_lattice")

    def __init__(self, p, fast_lattice=True, noise_sigma=0.0, noise_seed=0):
        super().__init__(self._dense, p.dim,
                         lattice_fn=self._lattice if fast_lattice else None)
        self.poly = p
        self.fast_lattice = bool(fast_lattice)
        self.noise_sigma = float(noise_sigma)
        self.noise_seed = int(noise_seed)
        self.calls = 0

    def add_noise_device(self, vals, rows, M):
        """Noise for `rows` consecutive calls of M samples each (in place)."""
        if self.noise_sigma > 0:
            _native.call("sfftb_add_noise", _dev.ptr(vals), rows, M,
                         self.noise_seed & 0xFFFFFFFFFFFFFFFF, self.calls,
                         self.noise_sigma, _dev.stream())
        self.calls += rows

    def eval_points_device(self, X_dev):
        out = _eval_points_dev(self.poly, X_dev)
        self.add_noise_device(out, 1, out.shape[0])
        return out

    def _dense(self, X):
        return _dev.download(self.eval_points_device(_dev.upload(np.asarray(X, np.float64))))

    def _lattice(self, lat):
        z = _dev.upload(lat.z.reshape(1, -1))
        tails = _dev.empty((1, 1), torch.float64)
        vals = sample_lattices_device(self.poly, z, lat.M, tails, 1, 1, self.dim)
        self.add_noise_device(vals, 1, lat.M)
        return _dev.download(vals[0])

    def sample_spectra_device(self, zmat_dev, M, tails_dev, G, L, t_dim):
        """Fused sampling + detection transforms (samples stay on chip):
        returns (ghat, theta0 per group, bitmaps) or None when M is outside
        the fused path.  Counts and calls advance as G*L sample_many calls."""
        from . import _engine

        if not _engine.fused_ok(M):
            return None
        bins = lattice_bins_device(self.poly, zmat_dev, M, tails_dev, G, L, t_dim)
        out = _engine.sample_spectra_fused(bins, M, G, L, self.noise_seed, self.calls,
                                           self.noise_sigma)
        self.calls += G * L
        self.count += G * L * M
        return out

    def sample_lattices_device(self, zmat_dev, M, tails_dev, G, L, t_dim):
        """Batched fixed-tail lattice sampling; advances count and calls
        exactly as G*L separate sample_many calls would (dimincr.py:186-191)."""
        vals = sample_lattices_device(self.poly, zmat_dev, M, tails_dev, G, L, t_dim)
        self.add_noise_device(vals, G * L, M)
        self.count += G * L * M
        return vals


def oracle_from_poly(p, fast_lattice=True, *, noise_sigma=0.0, noise_seed=0):
    """Oracle over a SparsePoly (polyeval.py:133-136) + optional harness noise."""
    return PolyOracle(p, fast_lattice=fast_lattice, noise_sigma=noise_sigma,
                      noise_seed=noise_seed)


def sample_on_lattice(oracle, lat, d=None):
    """Node values of one lattice through an oracle (polyeval.py:139-143)."""
    if d is not None and d != lat.dim:
        raise ParameterError("dimension mismatch")
    return oracle.sample_lattice(lat)


def random_poly(I, rng, min_mag=1e-6):
    """Coefficients uniform on [-1,1)+[-1,1)i, rejected below min_mag
    (polyeval.py:146-158; same RNG calls)."""
    if min_mag >= 1:
        raise ParameterError("min_mag must be < 1")
    n = len(I)
    coeffs = np.zeros(n, dtype=np.complex128)
    todo = np.arange(n)
    while todo.size:
        draw = rng.uniform(-1, 1, size=(todo.size, 2))
        vals = draw[:, 0] + 1j * draw[:, 1]
        coeffs[todo] = vals
        todo = todo[np.abs(vals) < min_mag]
    return SparsePoly(I, coeffs)


# ---------------------------------------------------------------------------
# periodised B-splines and the ten-variate test function f10
# (polyeval.py:160-350).  Function values are computed on the device
# (csrc/analysis.cu, sfftb_spline_sum_*); the closed-form Fourier
# coefficients and norms below are scalar host formulas of the error metric.
# ---------------------------------------------------------------------------

import math as _math

_BSPLINE_NORM_CACHE = {}

#: (axes, spline order) of the three tensor-product summands (0-based axes)
F10_GROUPS = (((0, 2, 7), 2), ((1, 4, 5, 9), 4), ((3, 6, 8), 6))
F10_DIM = 10


def _sinc(t):
    out = np.ones_like(t)
    nz = t != 0
    out[nz] = np.sin(t[nz]) / t[nz]
    return out


def bspline_norm_constant(m):
    """C_m = (sum_k sinc(pi k / m)^(2m))^(-1/2), truncated at |k| <=
    max(1e5, 1000 m) and summed smallest-first (polyeval.py:175-190)."""
    m = int(m)
    if m < 1:
        raise ParameterError("spline order must be >= 1")
    if m not in _BSPLINE_NORM_CACHE:
        horizon = max(100_000, 1000 * m)
        k = np.arange(1, horizon + 1, dtype=np.float64)
        s = _sinc(np.pi * k / m) ** (2 * m)
        total = 1.0 + 2.0 * float(np.sum(s[::-1]))
        _BSPLINE_NORM_CACHE[m] = total ** -0.5
    return _BSPLINE_NORM_CACHE[m]


def bspline_coeffs(m, ks):
    """Fourier coefficients C_m sinc(pi k / m)^m (-1)^k (polyeval.py:198-203)."""
    ks = np.asarray(ks, dtype=np.int64)
    c = bspline_norm_constant(m)
    vals = c * _sinc(np.pi * ks / m) ** m
    vals[ks % 2 == 1] *= -1.0
    return vals


def bspline_coeff(m, k):
    return float(bspline_coeffs(m, np.asarray([k]))[0])


class SplineSum:
    """sum over groups of tensor products of periodised unit-norm B-splines,
    evaluated on the device (one kernel over all points / lattice nodes)."""

    __slots__ = ("dim", "groups", "_axis", "_order", "_scale")

    def __init__(self, dim, groups):
        self.dim = int(dim)
        self.groups = tuple((tuple(int(a) for a in axes), int(m)) for axes, m in groups)
        axis = np.full(self.dim, -1, dtype=np.int32)
        for g, (axes, _) in enumerate(self.groups):
            for a in axes:
                if not 0 <= a < self.dim or axis[a] != -1:
                    raise ParameterError("spline groups must be disjoint axes of the domain")
                axis[a] = g
            if list(axes) != sorted(axes):
                raise ParameterError("spline group axes must be ascending")
        self._axis = axis
        self._order = np.array([m for _, m in self.groups], dtype=np.int32)
        self._scale = np.array([bspline_norm_constant(m) * m for _, m in self.groups],
                               dtype=np.float64)

    def _args(self):
        return (self.dim, self._axis.ctypes.data, len(self.groups), self._order.ctypes.data,
                self._scale.ctypes.data)

    def points_device(self, X_dev):
        """(m,) complex128 device values at the rows of a (m, dim) device tensor."""
        X_dev = X_dev.to(torch.float64).contiguous()
        m = int(X_dev.shape[0])
        out = _dev.empty((max(m, 1),), torch.complex128)
        _native.call("sfftb_spline_sum_points", *self._args(), _dev.ptr(X_dev), m,
                     _dev.ptr(out), _dev.stream())
        return out[:m]

    def lattice_device(self, zmat_dev, M, tails_dev, G, L, t_dim):
        """(G*L, M) complex128 values at [(j z mod M)/M | tail_g] (dimincr.py:186-191)."""
        out = _dev.empty((G * L, M), torch.complex128)
        _native.call("sfftb_spline_sum_lattice", *self._args(), _dev.ptr(zmat_dev), G, L, M,
                     t_dim, _dev.ptr(tails_dev), _dev.ptr(out), _dev.stream())
        return out


def bspline_values(m, x):
    """N_m at torus points x (polyeval.py:216-225), on the device."""
    x = np.asarray(x, dtype=np.float64)
    f = SplineSum(1, (((0,), int(m)),))
    vals = _dev.download(f.points_device(_dev.upload(x.reshape(-1, 1))))
    return vals.real.reshape(x.shape)


_F10 = None


def _f10():
    global _F10
    if _F10 is None:
        _F10 = SplineSum(F10_DIM, F10_GROUPS)
    return _F10


def f10_values(X):
    """Test-function values at an (m, 10) array of torus points (polyeval.py:261-272)."""
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2 or X.shape[1] != F10_DIM:
        raise ParameterError("points must be an (m, 10) array")
    return _dev.download(_f10().points_device(_dev.upload(X))).real


class SplineOracle(SamplingOracle):
    """Black-box oracle of a SplineSum whose evaluations run on the device:
    sample_many / sample_lattice evaluate at the given points, and the sfft
    driver's batched fixed-tail lattice samplings (sample_lattices_device)
    never leave the GPU.  Counts advance like the reference's
    SamplingOracle (polyeval.py:107-130)."""

    __slots__ = ("spline",)

    def __init__(self, spline):
        super().__init__(self._host_fn, spline.dim)
        self.spline = spline

    def _host_fn(self, X):
        return _dev.download(self.spline.points_device(_dev.upload(np.asarray(X, np.float64))))

    def sample_lattices_device(self, zmat_dev, M, tails_dev, G, L, t_dim):
        vals = self.spline.lattice_device(zmat_dev, M, tails_dev, G, L, t_dim)
        self.count += G * L * M
        return vals


def f10_oracle():
    """SamplingOracle of f10 (polyeval.py:275-277), sampled on the device."""
    return SplineOracle(_f10())


def _summand_coeffs(elems, axes, m):
    """Coefficients of one tensor-product summand: the product of its axes'
    spline coefficients where every other component is zero, else 0."""
    vals = np.zeros(elems.shape[0])
    on = ~np.delete(elems, list(axes), axis=1).any(axis=1)
    if on.any():
        cols = np.stack([bspline_coeffs(m, elems[on, a]) for a in axes], axis=1)
        vals[on] = np.multiply.reduce(cols, axis=1)
    return vals


def f10_coeffs(elems):
    """Exact Fourier coefficients of f10 at (n, 10) indices (polyeval.py:280-300):
    the groups use disjoint axes, so only k = 0 collects more than one summand."""
    elems = np.asarray(elems, dtype=np.int64)
    if elems.ndim != 2 or elems.shape[1] != F10_DIM:
        raise ParameterError("indices must be an (n, 10) array")
    total = np.zeros(elems.shape[0])
    for axes, m in F10_GROUPS:
        total = total + _summand_coeffs(elems, axes, m)
    return total


def f10_coeff(k):
    k = np.asarray(k, dtype=np.int64)
    if k.shape != (F10_DIM,):
        raise ParameterError("index must have 10 components")
    return float(f10_coeffs(k.reshape(1, F10_DIM))[0])


def f10_sq_norm():
    """||f10||^2 (polyeval.py:310-322): each summand has unit norm and two
    summands overlap only in their k = 0 coefficient C_m^|axes|."""
    from itertools import combinations

    zero_coeff = [bspline_norm_constant(m) ** len(axes) for axes, m in F10_GROUPS]
    total = float(len(zero_coeff))
    for a, b in combinations(zero_coeff, 2):
        total += 2.0 * a * b
    return total


def rel_l2_error(I, coeffs, f_sq_norm, f_coeff_fn):
    """||f - sum_{k in I} c_k e_k|| / ||f|| by Parseval (polyeval.py:325-347):
    ||f||^2 - sum_I |f_k|^2 + sum_I |c_k - f_k|^2, clamped at 0 for roundoff,
    ParameterError when it is clearly negative."""
    if f_sq_norm <= 0:
        raise ParameterError("f_sq_norm must be positive")
    if isinstance(coeffs, dict):
        coeffs = [coeffs[k] for k in I]
    c = np.asarray(coeffs, dtype=np.complex128)
    if c.shape != (len(I),):
        raise ParameterError("need one coefficient per frequency")
    rad = f_sq_norm
    if len(I):
        fk = np.asarray(f_coeff_fn(I.elems), dtype=np.complex128)
        rad = f_sq_norm - float(np.sum(np.abs(fk) ** 2)) + float(np.sum(np.abs(c - fk) ** 2))
    if rad < -1e-12 * f_sq_norm:
        raise ParameterError(f"negative radicand {rad} in error formula")
    return _math.sqrt(max(rad, 0.0) / f_sq_norm)
