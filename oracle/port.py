"""numpy restatement of the reference's hot path (TEST INFRASTRUCTURE ONLY).

Every function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/latfft/).  Candidate sets are plain ``(n, d)`` int64
arrays in canonical (lexicographic, duplicate-free) order; a lattice
configuration is ``(M, zmat)`` with one shared prime M (lattice.py:221-229).

The per-candidate gather runs in C: either the reference's own compiled
kernel (oracle/_ref, ``gather_backend="reference"``) or the plain-C
restatement in oracle/gather.c (``gather_backend="port"``).
"""

from __future__ import annotations

import ctypes
import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_LIB_LOCK = threading.Lock()


class OracleParameterError(ValueError):
    """Mirror of latfft.errors.ParameterError (errors.py:7-8)."""


class OracleCapacityError(Exception):
    """Mirror of latfft.errors.CapacityError (errors.py:11-12)."""


# ---------------------------------------------------------------------------
# native helpers
# ---------------------------------------------------------------------------

def lib():
    """oracle/liboracle.so (built by ``make -C oracle``)."""
    global _LIB
    with _LIB_LOCK:
        if _LIB is None:
            path = os.path.join(HERE, "liboracle.so")
            if not os.path.exists(path):
                raise RuntimeError("oracle/liboracle.so missing: run make -C oracle")
            so = ctypes.CDLL(path)
            i64, p = ctypes.c_int64, ctypes.c_void_p
            so.oracle_detect_gather.argtypes = [p, i64, i64, p, i64, i64, p,
                                                ctypes.c_double, ctypes.c_double,
                                                ctypes.c_int, p, p]
            so.oracle_detect_gather.restype = ctypes.c_int
            so.oracle_rows_injective_mod.argtypes = [p, i64, i64, i64]
            so.oracle_rows_injective_mod.restype = ctypes.c_int
            _LIB = so
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def gather_c(elems_mod, zmat, M, ghat, theta, thr, want_medians, workers=1):
    """_core.pyx:164-202 restated in oracle/gather.c (elems pre-reduced).

    ``workers > 1`` runs contiguous row chunks on a thread pool (ctypes
    releases the GIL); rows are independent, so results are identical.
    """
    e = np.ascontiguousarray(elems_mod, dtype=np.int64)
    z = np.ascontiguousarray(zmat, dtype=np.int64)
    g = np.ascontiguousarray(ghat, dtype=np.complex128)
    n, d = e.shape
    L = z.shape[0]
    hits = np.zeros(n, dtype=np.int64)
    med = np.zeros(n, dtype=np.complex128)
    so = lib()

    def run(lo, hi):
        rc = so.oracle_detect_gather(_ptr(e[lo:hi]), hi - lo, d, _ptr(z), L,
                                     int(M), _ptr(g), float(theta), float(thr),
                                     int(bool(want_medians)), _ptr(hits[lo:hi]),
                                     _ptr(med[lo:hi]))
        if rc != 0:
            raise MemoryError("oracle gather allocation failed")

    if workers <= 1 or n < 4096:
        run(0, n)
    else:
        b = np.linspace(0, n, workers + 1).astype(np.int64)
        with ThreadPoolExecutor(workers) as ex:
            list(ex.map(lambda k: run(int(b[k]), int(b[k + 1])), range(workers)))
    return hits, med


def gather_ref(elems_mod, zmat, M, ghat, theta, thr, want_medians, workers=1):
    """The reference's own compiled kernel (oracle/_ref/_core*.so).

    ``workers > 1`` splits the rows into contiguous chunks run on a thread
    pool -- the kernel releases the GIL (_core.pyx:184) and rows are
    independent, so results are identical to one call.
    """
    from .refload import load_ref_core

    core = load_ref_core()
    if core is None:
        raise RuntimeError("oracle/_ref missing: run make -C oracle ref")
    e = np.ascontiguousarray(elems_mod, dtype=np.int64)
    z = np.ascontiguousarray(zmat, dtype=np.int64)
    g = np.ascontiguousarray(ghat, dtype=np.complex128)
    if workers <= 1 or e.shape[0] < 4096:
        return core.detect_gather(e, z, int(M), g, float(theta), float(thr),
                                  bool(want_medians))
    bounds = np.linspace(0, e.shape[0], workers + 1).astype(np.int64)

    def run(k):
        return core.detect_gather(np.ascontiguousarray(e[bounds[k]:bounds[k + 1]]),
                                  z, int(M), g, float(theta), float(thr),
                                  bool(want_medians))

    with ThreadPoolExecutor(workers) as ex:
        parts = list(ex.map(run, range(workers)))
    return (np.concatenate([p[0] for p in parts]),
            np.concatenate([p[1] for p in parts]))


def rows_injective_mod(elems, p):
    """Reduction mod p keeps rows distinct (fallback.py:78-103 semantics)."""
    e = np.ascontiguousarray(elems, dtype=np.int64)
    if e.ndim != 2:
        raise OracleParameterError("elems must be 2-d")
    rc = lib().oracle_rows_injective_mod(_ptr(e), e.shape[0], e.shape[1], int(p))
    if rc < 0:
        raise MemoryError("oracle injectivity allocation failed")
    return bool(rc)


# ---------------------------------------------------------------------------
# frequency sets (freqset.py)
# ---------------------------------------------------------------------------

def canonical_rows(arr):
    """Lexicographically sorted unique rows (freqset.py:48-67)."""
    arr = np.asarray(arr, dtype=np.int64)
    if arr.shape[0] == 0:
        return arr.reshape(0, arr.shape[1] if arr.ndim == 2 else 0)
    order = np.lexsort(arr.T[::-1])
    s = arr[order]
    keep = np.ones(s.shape[0], dtype=bool)
    keep[1:] = np.any(s[1:] != s[:-1], axis=1)
    return np.ascontiguousarray(s[keep])


def random_rows_from_box(d, lo, hi, count, rng):
    """Distinct uniform rows of [lo, hi]^d; RNG calls of freqset.py:266-280."""
    rows = np.empty((0, d), dtype=np.int64)
    need = count
    while need > 0:
        batch = rng.integers(lo, hi + 1, size=(int(need * 1.05) + 16, d),
                             dtype=np.int64)
        rows = canonical_rows(np.vstack([rows, batch]))
        if len(rows) > count:
            rows = rows[np.sort(rng.choice(len(rows), size=count, replace=False))]
        need = count - len(rows)
    return rows


def random_rows_from_set(elems, count, rng):
    """random_subset of a FreqSet (freqset.py:257-260)."""
    idx = rng.choice(elems.shape[0], size=count, replace=False)
    return elems[np.sort(idx)]


def rows_in(rows, pool):
    """Membership mask of rows in pool (freqset.py:70-82 semantics)."""
    if rows.shape[0] == 0 or pool.shape[0] == 0:
        return np.zeros(rows.shape[0], dtype=bool)
    dt = np.dtype((np.void, 8 * rows.shape[1]))
    a = np.ascontiguousarray(rows, dtype=np.int64).view(dt).ravel()
    b = np.ascontiguousarray(pool, dtype=np.int64).view(dt).ravel()
    return np.isin(a, b)


# ---------------------------------------------------------------------------
# host lattice construction (lattice.py)
# ---------------------------------------------------------------------------

def is_prime(n):
    """Exact primality for 64-bit n (lattice.py:24-47 answers the same)."""
    n = int(n)
    if n < 2:
        return False
    small = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)
    for q in small:
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x == 1 or x == n - 1:
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def next_prime_above(x):
    """lattice.py:50-59."""
    n = int(math.floor(x)) + 1
    if n <= 2:
        return 2
    n += (n % 2 == 0)
    while not is_prime(n):
        n += 2
    return n


def next_valid_prime(elems, lower):
    """lattice.py:114-125."""
    if elems.shape[0] == 0:
        raise OracleParameterError("need a nonempty frequency set")
    p = next_prime_above(lower)
    while not rows_injective_mod(elems, p):
        p = next_prime_above(p)
    return p


def required_L(gamma_size, delta, nu=0.5, c=10.33, force_odd=True, L_scale=1.0):
    """lattice.py:128-153 (same floating-point expression)."""
    pref = c * (c - 2.0) / ((c * nu - 1.0) ** 2 * math.log(c - 1.0))
    value = L_scale * pref * (math.log(int(gamma_size)) - math.log(delta))
    n = max(1, math.ceil(value))
    if force_odd and n % 2 == 0:
        n += 1
    return n


def draw_config(elems, sparsity, delta, rng, nu=0.5, c=10.33, L_scale=1.0, L=None):
    """lattice.py:210-230 -> (M, zmat (L, d) int64)."""
    M = next_valid_prime(elems, c * sparsity)
    if L is None:
        L = required_L(elems.shape[0], delta, nu=nu, c=c,
                       force_odd=(nu == 0.5), L_scale=L_scale)
    zmat = rng.integers(0, M, size=(int(L), elems.shape[1]), dtype=np.int64)
    return M, zmat


def residues(elems, z, M):
    """lattice.py:108-111."""
    return (np.asarray(elems, dtype=np.int64) % M) @ np.asarray(z, np.int64) % M


def lattice_nodes(z, M):
    """lattice.py:91-97."""
    j = np.arange(M, dtype=np.int64)[:, None]
    return (j * np.asarray(z, np.int64)[None, :] % M) / M


# ---------------------------------------------------------------------------
# signal model and sampling (polyeval.py, dft.py)
# ---------------------------------------------------------------------------

def dft_normalized(x):
    """dft.py:18-27."""
    x = np.asarray(x, dtype=np.complex128)
    if x.ndim != 1 or x.size == 0:
        raise OracleParameterError("samples must be a nonempty 1-d vector")
    if not np.all(np.isfinite(x.view(np.float64))):
        raise OracleParameterError("samples contain NaN or Inf")
    return np.fft.fft(x) / x.size


def evaluate_dense(support, coeffs, X, chunk=4096):
    """polyeval.py:66-75 (dense: exp(2 pi i X K^T) @ c, 4096-row chunks)."""
    X = np.asarray(X, dtype=np.float64)
    out = np.empty(X.shape[0], dtype=np.complex128)
    K = np.asarray(support, np.int64).T
    for lo in range(0, X.shape[0], chunk):
        hi = min(lo + chunk, X.shape[0])
        out[lo:hi] = np.exp(2j * np.pi * (X[lo:hi] @ K)) @ coeffs
    return out


def sample_lattice_structured(support, coeffs, z, M, tail=None):
    """polyeval.py:78-87, generalised with the anchor phase of a fixed tail.

    p(j z/M | tail) = sum_h B[h] e^{2 pi i jh/M},
    B[h] = sum_{k: k_{<=t}.z = h} c_k e^{2 pi i k_{>t}.tail}.
    """
    support = np.asarray(support, np.int64)
    t_dim = len(z)
    c = np.asarray(coeffs, np.complex128)
    if tail is not None and len(tail):
        c = c * np.exp(2j * np.pi * (support[:, t_dim:] @ np.asarray(tail)))
    r = residues(support[:, :t_dim], z, M)
    b = np.bincount(r, weights=c.real, minlength=M) + 1j * np.bincount(
        r, weights=c.imag, minlength=M)
    return M * np.fft.ifft(b)


# Philox4x32-10 counter-based noise (the harness noise model of SURVEY
# Appendix B "Config 5"; the reference has no noise model).
_PH_M0, _PH_M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
_PH_W0, _PH_W1 = 0x9E3779B9, 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit words."""
    c0, c1, c2, c3 = (np.asarray(v, np.uint64) & _MASK32 for v in (c0, c1, c2, c3))
    k0, k1 = int(k0) & 0xFFFFFFFF, int(k1) & 0xFFFFFFFF
    for rnd in range(10):
        p0 = _PH_M0 * c0
        p1 = _PH_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
        if rnd < 9:
            k0 = (k0 + _PH_W0) & 0xFFFFFFFF
            k1 = (k1 + _PH_W1) & 0xFFFFFFFF
    return c0, c1, c2, c3


def noise_for_call(seed, call, m, sigma):
    """sigma*(N(0,1) + i N(0,1)) for samples 0..m-1 of oracle call ``call``.

    counter = (m_lo, m_hi, call_lo, call_hi), key = (seed_lo, seed_hi);
    u1 = (x0>>5 * 2^26 + x1>>6 + 1) / 2^53 in (0, 1],
    u2 = (x2>>5 * 2^26 + x3>>6) / 2^53 in [0, 1); Box-Muller.
    """
    idx = np.arange(m, dtype=np.uint64)
    x0, x1, x2, x3 = philox4x32(idx & _MASK32, idx >> np.uint64(32),
                                np.uint64(call & 0xFFFFFFFF),
                                np.uint64((call >> 32) & 0xFFFFFFFF),
                                seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    a = ((x0 >> np.uint64(5)) << np.uint64(26)) + (x1 >> np.uint64(6))
    b = ((x2 >> np.uint64(5)) << np.uint64(26)) + (x3 >> np.uint64(6))
    u1 = (a.astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = b.astype(np.float64) * 2.0 ** -53
    rad = sigma * np.sqrt(-2.0 * np.log(u1))
    ang = 2.0 * np.pi * u2
    return rad * np.cos(ang) + 1j * (rad * np.sin(ang))


class PolyOracle:
    """SamplingOracle over a sparse polynomial (polyeval.py:90-136).

    ``mode="dense"`` evaluates point sets like ``evaluate_many`` (the
    reference as shipped); ``mode="structured"`` evaluates whole lattices with
    the scatter + inverse FFT restatement.  Optional harness noise is added
    per call.  ``count`` advances by the number of points (polyeval.py:118).
    """

    def __init__(self, support, coeffs, mode="dense", sigma=0.0, noise_seed=0):
        self.support = np.ascontiguousarray(support, np.int64)
        self.coeffs = np.ascontiguousarray(coeffs, np.complex128)
        self.dim = self.support.shape[1]
        self.mode = mode
        self.sigma = float(sigma)
        self.noise_seed = int(noise_seed)
        self.count = 0
        self.calls = 0

    def _noise(self, vals):
        if self.sigma > 0:
            vals = vals + noise_for_call(self.noise_seed, self.calls, vals.size,
                                         self.sigma)
        self.calls += 1
        return vals

    def sample_points(self, X):
        X = np.asarray(X, dtype=np.float64)
        self.count += X.shape[0]
        return self._noise(evaluate_dense(self.support, self.coeffs, X))

    def sample_lattices_tail(self, zmat, M, tail, workers=1):
        """sample_lattice_tail for every row of zmat, in order; the structured
        noise-free evaluations run on `workers` threads (the noise stream and
        the counter still advance lattice by lattice)."""
        if self.mode == "dense" or workers <= 1:
            return [self.sample_lattice_tail(z, M, tail) for z in zmat]
        vals = _pmap(lambda z: sample_lattice_structured(self.support, self.coeffs, z, M, tail),
                     list(zmat), workers)
        out = []
        for v in vals:
            self.count += M
            out.append(self._noise(v))
        return out

    def sample_lattice_tail(self, z, M, tail):
        """Samples at [j z/M mod 1 | tail], j < M (dimincr.py:186-191)."""
        if self.mode == "dense":
            nodes = np.empty((M, self.dim))
            nodes[:, :len(z)] = lattice_nodes(z, M)
            nodes[:, len(z):] = tail
            return self.sample_points(nodes)
        self.count += M
        return self._noise(sample_lattice_structured(self.support, self.coeffs,
                                                     z, M, tail))


# ---------------------------------------------------------------------------
# detection (detect.py)
# ---------------------------------------------------------------------------

def zero_threshold(samples):
    """default_zero_test (detect.py:42-53)."""
    rms = sorted(float(np.sqrt(np.mean(np.abs(np.asarray(s)) ** 2)))
                 for s in samples)
    h = len(rms) // 2
    mid = rms[h] if len(rms) % 2 else 0.5 * (rms[h - 1] + rms[h])
    return max(1e-12, 1e-10 * mid)


def _pmap(fn, items, workers):
    """list(map(fn, items)), on a thread pool when workers > 1 (numpy's FFT
    and bincount release the GIL; results keep the input order)."""
    items = list(items)
    if workers <= 1 or len(items) < 2:
        return [fn(x) for x in items]
    from concurrent.futures import ThreadPoolExecutor

    with ThreadPoolExecutor(min(workers, len(items))) as ex:
        return list(ex.map(fn, items))


def ghat_matrix(samples, M, workers=1):
    """_ghat_list + np.vstack (detect.py:98-109, :132)."""
    def one(s):
        s = np.asarray(s, dtype=np.complex128)
        if s.shape != (M,):
            raise OracleParameterError("sample vector length does not match M")
        return dft_normalized(s)

    return np.vstack(_pmap(one, samples, workers))


def gather(samples, M, zmat, elems, theta0, nu, want_medians,
           gather_backend="port", workers=1):
    """_gather with a shared M (detect.py:122-133)."""
    L, d = zmat.shape
    if len(samples) != L:
        raise OracleParameterError("sample count does not match L")
    if not d * (M - 1) ** 2 < 2 ** 62:
        raise OracleParameterError("lattice size too large for int64 residues")
    g = ghat_matrix(samples, M, workers)
    thr = nu * L
    em = np.asarray(elems, np.int64) % M
    if gather_backend == "reference":
        hits, med = gather_ref(em, zmat, M, g, theta0, thr, want_medians, workers)
    else:
        hits, med = gather_c(em, zmat, M, g, theta0, thr, want_medians, workers)
    return hits, med, thr


def gather_mixed(samples, Ms, zmat, elems, theta0, nu, want_medians):
    """_gather for distinct lattice sizes (detect.py:134-145): hits by np.abs
    (hypot) > theta, np.median of the real and imaginary parts."""
    L = len(Ms)
    vals = np.empty((elems.shape[0], L), dtype=np.complex128)
    for col, (s, M) in enumerate(zip(samples, Ms)):
        g = dft_normalized(np.asarray(s, dtype=np.complex128))
        vals[:, col] = g[residues(elems, zmat[col], M)]
    hits = np.sum(np.abs(vals) > theta0, axis=1).astype(np.int64)
    thr = nu * L
    med = np.zeros(elems.shape[0], dtype=np.complex128)
    det = hits >= thr
    if want_medians and np.any(det):
        sel = vals[det]
        med[det] = np.median(sel.real, axis=1) + 1j * np.median(sel.imag, axis=1)
    return hits, med, thr


def detect_and_compute(samples, M, zmat, elems, theta0=None, nu=0.5, **kw):
    """Alg. 2 (detect.py:158-169) -> (hits, detected_idx, coeffs, theta0)."""
    if nu != 0.5:
        raise OracleParameterError("coefficient computation requires nu = 1/2")
    if zmat.shape[0] % 2 == 0:
        raise OracleParameterError("coefficient computation requires odd L")
    if theta0 is None:
        theta0 = zero_threshold(samples)
    hits, med, thr = gather(samples, M, zmat, elems, theta0, nu, True, **kw)
    idx = np.flatnonzero(hits >= thr)
    return hits, idx, med[idx], theta0


def detect_frequencies(samples, M, zmat, elems, theta0=None, nu=0.5, **kw):
    """Alg. 1 (detect.py:149-155) -> (hits, detected_idx, theta0)."""
    if theta0 is None:
        theta0 = zero_threshold(samples)
    hits, _, thr = gather(samples, M, zmat, elems, theta0, nu, False, **kw)
    return hits, np.flatnonzero(hits >= thr), theta0


def topk_filter(idx, coeffs, s_tilde, theta):
    """detect_topk's selection (detect.py:184-193).

    candidate rows are lexicographically sorted, so the reference's
    lexicographic tie key equals the ascending candidate index.
    """
    keep = np.abs(coeffs) >= theta
    idx, coeffs = idx[keep], coeffs[keep]
    if idx.size > s_tilde:
        order = np.sort(np.lexsort((idx, -np.abs(coeffs)))[:s_tilde])
        idx, coeffs = idx[order], coeffs[order]
    return idx, coeffs


def detect_topk(samples, M, zmat, elems, s_tilde, theta, theta0=None, **kw):
    """Alg. 4 (detect.py:172-195)."""
    if int(s_tilde) < 0 or theta < 0:
        raise OracleParameterError("s_tilde and theta must be >= 0")
    hits, idx, coeffs, theta0 = detect_and_compute(samples, M, zmat, elems,
                                                   theta0, **kw)
    idx, coeffs = topk_filter(idx, coeffs, int(s_tilde), theta)
    return hits, idx, coeffs, theta0


def postprocess_r1l(det_rows, coeffs, det_idx, samples, M, zmat, theta0):
    """R1L refinement (detect.py:198-228) -> (kept det_idx, refined coeffs)."""
    n = det_rows.shape[0]
    if n == 0:
        return det_idx, coeffs
    g = ghat_matrix(samples, M)
    refined = np.array(coeffs, dtype=np.complex128)
    cnt = np.zeros(n, dtype=np.int64)
    acc = np.zeros(n, dtype=np.complex128)
    for l in range(zmat.shape[0]):
        r = residues(det_rows, zmat[l], M)
        uniq = np.bincount(r, minlength=M)[r] == 1
        cnt += uniq
        acc[uniq] += g[l, r[uniq]]
    has = cnt > 0
    refined[has] = acc[has] / cnt[has]
    keep = np.abs(refined) > theta0
    return det_idx[keep], refined[keep]


# ---------------------------------------------------------------------------
# dimension-incremental driver (dimincr.py)
# ---------------------------------------------------------------------------

def rng_for(master, tag, t, i):
    """dimincr.py:99-100."""
    return np.random.default_rng(np.random.SeedSequence((master, tag, t, i)))


def choose_r(s, d, delta):
    """r of choose_params (dimincr.py:87-96)."""
    return math.ceil(2 * s * math.log(3 * d * s / delta))


class Box:
    """Implicit cube [lo, hi]^d (freqset.py:158-197), len() clamped."""

    def __init__(self, d, lo, hi):
        self.dim, self.lo, self.hi = int(d), int(lo), int(hi)


def axis_values(gamma, axis):
    """dimincr.py:109-112."""
    if isinstance(gamma, Box):
        return np.arange(gamma.lo, gamma.hi + 1, dtype=np.int64)
    return np.unique(gamma[:, axis])


def sfft(oracle, gamma, s, delta, seed, s_local=None, theta=1e-12, r=None,
         c=10.33, L_scale=1.0, pair_cap=10_000_000, gather_backend="port",
         workers=1, on_stage=None):
    """Alg. 3 driver (dimincr.py:195-256) -> (support, coeffs, count, log).

    ``gamma`` is a Box or a canonical (n, d) int64 array.  ``on_stage`` is
    called after each detect call (used to bound the CPU-baseline sample).
    """
    d = oracle.dim
    s_local = 2 * s if s_local is None else int(s_local)
    master = int(seed)
    if r is None:
        r = choose_r(s, d, delta)
    gamma_A = delta / (3 * d * r)
    gamma_fin = delta / (3 * d)
    log = []
    count0 = oracle.count
    kw = dict(gather_backend=gather_backend, workers=workers)

    def empty():
        return (np.zeros((0, d), np.int64), np.zeros(0, np.complex128),
                oracle.count - count0, log)

    # step 1 (dimincr.py:122-152)
    comp = []
    for t in range(d):
        vals = axis_values(gamma, t)
        if vals.size == 0:
            raise OracleParameterError(f"candidate set has no values on axis {t}")
        K = int(vals.max() - vals.min() + 1)
        kept = np.zeros(0, dtype=np.int64)
        for i in range(r):
            rng = rng_for(master, 0, t, i)
            nodes = np.broadcast_to(rng.uniform(size=d), (K, d)).copy()
            nodes[:, t] = np.arange(K) / K
            est = dft_normalized(oracle.sample_points(nodes))
            mags = np.abs(est[vals % K])
            order = np.lexsort((vals, -mags))[:s_local]
            order = order[mags[order] >= theta]
            kept = np.union1d(kept, vals[order])
            log.append({"stage": "step1", "t": t, "i": i, "candidates": K,
                        "kept": int(order.size), "samples": K})
        comp.append(kept)
    if any(v.size == 0 for v in comp):
        return empty()

    def detect_on(J, sparsity, s_tilde, budget, tail, rng, ls):
        M, zmat = draw_config(J, sparsity, budget, rng, c=c, L_scale=ls)
        if hasattr(oracle, "sample_lattices_tail"):
            samples = oracle.sample_lattices_tail(zmat, M, tail, workers)
        else:
            samples = [oracle.sample_lattice_tail(z, M, tail) for z in zmat]
        _, idx, coeffs, _ = detect_topk(samples, M, zmat, J, s_tilde, theta, **kw)
        return idx, coeffs, M, zmat.shape[0]

    prefix = comp[0].reshape(-1, 1)
    for t in range(1, d):
        last = t == d - 1
        r_t = 1 if last else r
        s_tilde = s if last else s_local
        # pairing (dimincr.py:155-175)
        vals = np.unique(comp[t])
        n1, n2 = prefix.shape[0], vals.size
        if n1 * n2 > pair_cap:
            raise OracleCapacityError("candidate product exceeds the cap")
        J = np.column_stack([np.repeat(prefix, n2, axis=0), np.tile(vals, n1)])
        if not isinstance(gamma, Box):
            J = J[rows_in(J, canonical_rows(gamma[:, :t + 1]))]
        if J.shape[0] == 0:
            return empty()
        union = None
        for i in range(r_t):
            rng = rng_for(master, 1, t, i)
            tail = rng.uniform(size=d - t - 1)
            idx, _, M, L = detect_on(J, min(s_local, J.shape[0]), s_tilde,
                                     gamma_A, tail, rng, L_scale)
            log.append({"stage": "pair", "t": t, "i": i,
                        "candidates": int(J.shape[0]), "kept": int(idx.size),
                        "samples": L * M})
            union = idx if union is None else np.union1d(union, idx)
            if on_stage is not None:
                on_stage(log)
        if union.size == 0:
            return empty()
        prefix = J[union]

    rng = rng_for(master, 2, 0, 0)
    idx, coeffs, M, L = detect_on(prefix, s, s, gamma_fin, np.zeros(0), rng, 1.0)
    log.append({"stage": "final", "t": d - 1, "i": 0,
                "candidates": int(prefix.shape[0]), "kept": int(idx.size),
                "samples": L * M})
    return prefix[idx], coeffs, oracle.count - count0, log
