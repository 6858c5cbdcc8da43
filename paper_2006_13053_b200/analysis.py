"""Worst-case alias accounting and the experiment harness (latfft/analysis.py).

Running the detector on the all-ones polynomial over a support I turns every
median into an exact alias count (analysis.py:1-11): an active frequency whose
median reaches 2 is a potential false negative, an inactive one reaching 1 a
potential false positive.  ``run_success_experiment`` sweeps the lattice count
L over seeded trials (analysis.py:218-297).

B200 design: under the "lattices" redraw protocol every trial of one L shares
the candidate set, the support and M, and differs only in its L generating
vectors.  All T trials of one L therefore run as ONE batched device chain with
G = T groups -- fused sampler->detection transforms for all T*L lattices,
one hashing launch over the resident candidate set with G bitmap groups, a
capped per-group compaction, medians of the detected rows, and the alias
classification (csrc/analysis.cu, K12) that reduces each trial to the five
counts its record needs.  Only trials that need the R1L postprocess touch
their detected rows again (K9, per group).  The "both" protocol redraws the
candidate set per trial on the host with the reference's RNG call sequence
and runs the same chain with G = 1.  Records equal the reference's
``as_jsonable()`` output (wall time aside) -- tests/test_gpu_analysis.py
pins them against tests/golden/analysis_*.json, produced by the reference.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _engine, _native, hostrng
from .detect import _kbound, detect_and_compute
from .dimincr import SfftParams, sfft
from .errors import ParameterError
from .freqset import Box, FreqSet, hyperbolic_cross, random_subset
from .lattice import next_valid_prime
from .polyeval import (
    PolyOracle,
    SparsePoly,
    f10_coeffs,
    f10_oracle,
    f10_sq_norm,
    oracle_from_poly,
    rel_l2_error,
)

# tallies written by sfftb_alias_classify, per group
_T_DET_IN, _T_NONINT, _T_LT1, _T_PFN, _T_PFP = range(5)
_CLS_PFN, _CLS_PFP = 3, 4


def theoretical_failure_bound(gamma_size, L, c):
    """|Gamma| (c-1)^(-L(c-2)/(4c)): failure bound at nu = 1/2 (analysis.py:38-42)."""
    if c <= 2:
        raise ParameterError("bound requires c > 2")
    return float(gamma_size) * (c - 1.0) ** (-L * (c - 2.0) / (4.0 * c))


def sample_budget(config):
    """Sum of the lattice sizes of a configuration (analysis.py:45-47)."""
    return int(sum(config.sizes))


def guaranteed_sample_budget(sparsity, gamma_size, delta):
    """37 |I| (ln |Gamma| - ln delta) samples (analysis.py:50-52)."""
    return 37.0 * sparsity * (math.log(gamma_size) - math.log(delta))


class PfpPfnOutcome:
    """Classification of one auxiliary-polynomial run (analysis.py:55-65)."""

    __slots__ = ("pfn", "pfp", "anomalies", "detection", "samples")

    def __init__(self, pfn, pfp, anomalies, detection, samples):
        self.pfn = pfn
        self.pfp = pfp
        self.anomalies = anomalies
        self.detection = detection
        self.samples = samples


# ---------------------------------------------------------------------------
# device helpers

def _membership_mask(rows_dev, pool):
    """Bit per row of rows_dev: is it a row of the FreqSet pool?"""
    n, d = int(rows_dev.shape[0]), int(rows_dev.shape[1])
    mask = _dev.empty((max((n + 31) // 32, 1),), torch.int32)
    if n:
        _native.call("sfftb_rows_in_sorted", _dev.ptr(rows_dev), n, d, _dev.ptr(pool.device()),
                     len(pool), _dev.ptr(mask), _dev.stream())
    return mask


def _support_in_gamma(I, gamma):
    """|I intersect Gamma| (the reference's in_I.sum()), on the device."""
    if len(I) == 0 or len(gamma) == 0:
        return 0
    bits = _dev.download(_membership_mask(I.device(), gamma)).view(np.uint32)
    return int(np.unpackbits(bits.view(np.uint8)).sum())


def _check_support(I, gamma):
    if len(I) == 0:
        raise ParameterError("support must be nonempty")
    if I.dim != gamma.dim:
        raise ParameterError("support/candidate dimension mismatch")


def _aux_poly(I):
    return SparsePoly(I, np.ones(len(I)))


# ---------------------------------------------------------------------------
# single configuration (public API)

def pfp_pfn_count(I, gamma, config, tol=1e-6, zero=None):
    """Potential false negatives / positives of a configuration for support I
    (analysis.py:67-104): the median detector on the all-ones polynomial over
    I; medians farther than ``tol`` from an integer count as anomalies.

    ``samples`` of the outcome is the (L, M) device tensor of the lattice
    samples when the lattices share M (a list of host arrays otherwise); both
    forms are accepted by detect_* and postprocess_r1l."""
    _check_support(I, gamma)
    oracle = oracle_from_poly(_aux_poly(I))
    M = config.shared_M
    if M is not None and config.dim == I.dim:
        zdev = config.zmat_device()
        tails = _dev.zeros((1, 1), torch.float64)
        samples = oracle.sample_lattices_device(zdev, M, tails, 1, config.L, I.dim)
    else:
        samples = [oracle.sample_lattice(lat) for lat in config.lattices]
    det = detect_and_compute(samples, config, gamma, zero=zero)

    idx, med = det.device_arrays()
    if not isinstance(idx, torch.Tensor):
        idx, med = _dev.as_i64(idx), _dev.as_c128(med)
    k = int(idx.numel())
    in_mask = _membership_mask(gamma.device(), I) if len(gamma) else None
    tallies = np.zeros(5, dtype=np.int64)
    cls = np.zeros(0, dtype=np.uint8)
    if k:
        counts = torch.tensor([k], dtype=torch.int64, device=_dev.device())
        cls_dev = _dev.empty((k,), torch.uint8)
        tal_dev = _dev.empty((5,), torch.int64)
        _native.call("sfftb_alias_classify", _dev.ptr(idx.contiguous()),
                     _dev.ptr(med.contiguous()), _dev.ptr(counts), 1, k, _dev.ptr(in_mask),
                     float(tol), _dev.ptr(cls_dev), _dev.ptr(tal_dev), _dev.stream())
        cls, tallies = _dev.download(cls_dev), _dev.download(tal_dev)
    n_in = _support_in_gamma(I, gamma)
    anomalies = (n_in - int(tallies[_T_DET_IN])) + int(tallies[_T_NONINT]) \
        + int(tallies[_T_LT1])
    det_idx = det.detected_idx
    code = cls >> 1
    pfn = gamma.take(np.ascontiguousarray(det_idx[code == _CLS_PFN]))
    pfp = gamma.take(np.ascontiguousarray(det_idx[code == _CLS_PFP]))
    return PfpPfnOutcome(pfn, pfp, anomalies, det, samples)


# ---------------------------------------------------------------------------
# experiment specification and records

@dataclass
class TrialRecord:
    seed: int
    L: int
    M: int
    pfn_count: int
    pfp_count: int
    success_plain: bool
    success_pfp_budget: dict
    success_postprocessed: bool
    sample_count: int
    wall_time: float
    anomalies: int = 0

    def as_jsonable(self):
        """Deterministic JSON-lines record, wall time excluded (analysis.py:120-134)."""
        return {
            "seed": self.seed,
            "L": self.L,
            "M": self.M,
            "pfn": self.pfn_count,
            "pfp": self.pfp_count,
            "success_plain": self.success_plain,
            "success_pfp_budget": {str(k): v for k, v in self.success_pfp_budget.items()},
            "success_postprocessed": self.success_postprocessed,
            "samples": self.sample_count,
            "anomalies": self.anomalies,
        }


@dataclass
class ExperimentSpec:
    """Declarative worst-case experiment (analysis.py:137-182): set generators,
    L sweep, trials; ``redraw`` = "both" (candidate set, support and lattices
    per trial) or "lattices" (fixed sets, fresh generating vectors)."""

    name: str
    candidates: dict
    support: dict
    L_values: list
    trials: int
    master_seed: int
    c: float = 10.33
    nu: float = 0.5
    delta: float = 0.5
    redraw: str = "both"
    pfp_budgets: tuple = (10, 100)
    postprocess: bool = True

    def as_dict(self):
        return {
            "name": self.name,
            "candidates": self.candidates,
            "support": self.support,
            "L_values": list(self.L_values),
            "trials": self.trials,
            "master_seed": self.master_seed,
            "c": self.c,
            "nu": self.nu,
            "delta": self.delta,
            "redraw": self.redraw,
            "pfp_budgets": list(self.pfp_budgets),
            "postprocess": self.postprocess,
        }

    @classmethod
    def from_dict(cls, data):
        data = dict(data)
        data["pfp_budgets"] = tuple(data.get("pfp_budgets", (10, 100)))
        return cls(**data)


def _resolve_weights(spec, d):
    w = spec.get("weights")
    if w is None:
        return None
    if isinstance(w, str):
        if w != "t^1.08":
            raise ParameterError(f"unknown weight rule {w!r}")
        return np.arange(1, d + 1, dtype=np.float64) ** 1.08
    return np.asarray(w, dtype=np.float64)


def _make_candidates(spec, rng):
    """Candidate-set generators (analysis.py:196-206), same RNG calls."""
    kind = spec["kind"]
    if kind == "random-box":
        return random_subset(Box(spec["d"], spec["lo"], spec["hi"]), spec["count"], rng)
    if kind == "hyperbolic":
        return hyperbolic_cross(spec["d"], spec["N"], _resolve_weights(spec, spec["d"]))
    if kind == "grid":
        return Box(spec["d"], -spec["N"], spec["N"]).materialize()
    raise ParameterError(f"unknown candidate generator {kind!r}")


def _make_support(spec, gamma, rng):
    """Support generators (analysis.py:209-215), same RNG calls."""
    kind = spec["kind"]
    if kind == "random-subset":
        return random_subset(gamma, spec["count"], rng)
    if kind == "hyperbolic":
        return hyperbolic_cross(gamma.dim, spec["N"], _resolve_weights(spec, gamma.dim))
    raise ParameterError(f"unknown support generator {kind!r}")


# ---------------------------------------------------------------------------
# batched trials: T trials of one L against one (Gamma, I, M)

# trial groups per device batch are bounded by the spectra (T*L*M*16 B) and
# the capped index lists (T*cap*8 B)
_BATCH_BYTES = 3 << 30
_MIN_CAP = 1 << 16
_CAP_PER_SUPPORT = 8  # detected rows kept per trial: max(_MIN_CAP, 8 |I|)


class _Shared:
    """Per-(Gamma, I) device state reused by every batch."""

    def __init__(self, gamma, I):
        self.gamma = gamma
        self.I = I
        self.rows = gamma.device()
        self.n = len(gamma)
        self.in_mask = _membership_mask(self.rows, I)
        self.n_in = _support_in_gamma(I, gamma)
        self.kbound = _kbound(gamma)
        self.oracle = PolyOracle(_aux_poly(I))


def _postprocess_group(sh, b, g, cap, zdev, L, M, theta0, count, cls):
    """R1L postprocess of trial g (K9); True iff the kept set is I with every
    refined coefficient within 1e-6 of 1 (analysis.py:241-243)."""
    d = sh.gamma.dim
    st = _dev.stream()
    idx_g = b.idx[g * cap:g * cap + count]
    med_g = b.coeffs[g * cap:g * cap + count]
    cnt_dev = torch.tensor([count], dtype=torch.int64, device=_dev.device())
    rows_det = _dev.empty((count, d), torch.int64)
    _native.call("sfftb_gather_rows", _dev.ptr(sh.rows), d, _dev.ptr(idx_g), _dev.ptr(cnt_dev),
                 count, _dev.ptr(rows_det), st)
    vals = _dev.empty((L, count), torch.complex128)
    for l in range(L):
        gl = g * L + l
        _native.call("sfftb_lattice_values", _dev.ptr(rows_det), d, _dev.ptr(zdev[gl]), 1, M,
                     _dev.ptr(b.ghat[gl]), None, count, _dev.ptr(vals[l]), st)
    offs = torch.arange(0, (L + 1) * M, M, dtype=torch.int64, device=_dev.device())
    refined = _dev.empty((count,), torch.complex128)
    keep = _dev.empty(((count + 31) // 32,), torch.int32)
    ws = _dev.workspace(_native.lib().sfftb_r1l_workspace_bytes(count, L, L * M))
    _native.call("sfftb_postprocess_r1l", _dev.ptr(rows_det), count, d,
                 _dev.ptr(zdev[g * L:(g + 1) * L].contiguous()), _dev.ptr(offs), L, L * M,
                 _dev.ptr(vals), _dev.ptr(med_g), float(theta0), _dev.ptr(refined),
                 _dev.ptr(keep), _dev.ptr(ws), st)
    kept = np.unpackbits(_dev.download(keep).view(np.uint8), bitorder="little")[:count]
    kept = kept.astype(bool)
    if int(kept.sum()) != len(sh.I):
        return False
    if not np.all(cls[kept] & 1):  # a kept row outside I
        return False
    co = _dev.download(refined)[kept]
    return bool(np.all(np.abs(co - 1.0) <= 1e-6))


def _run_batch(sh, M, L, zs, seeds, spec, tol, cap):
    """Trials with generators zs (T, L, d) -> list of TrialRecord."""
    T, d = zs.shape[0], sh.gamma.dim
    t0 = time.perf_counter()
    zdev = _dev.upload(zs.reshape(T * L, d))
    tails = _dev.zeros((T, 1), torch.float64)
    oracle = sh.oracle
    spec_dev = oracle.sample_spectra_device(zdev, M, tails, T, L, d)
    if spec_dev is not None:
        ghat, theta0, bits = spec_dev
    else:
        samples = oracle.sample_lattices_device(zdev, M, tails, T, L, d)
        ghat, theta0, bits = _engine.spectra(samples, M, T, L)
    st = _dev.stream()
    n = sh.n
    nwords = (n + 31) // 32
    detmask = _dev.empty((T * max(nwords, 1),), torch.int32)
    _native.call("sfftb_hash_hits", _dev.ptr(sh.rows), n, d, _dev.ptr(zdev), T, L, M,
                 _dev.ptr(bits), int(sh.kbound), _engine.min_hits_for(spec.nu, L), None,
                 _dev.ptr(detmask), st)
    idx = _dev.empty((T * max(cap, 1),), torch.int64)
    counts = _dev.empty((T,), torch.int64)
    totals = _dev.empty((T,), torch.int64)
    ws = _dev.workspace(_native.lib().sfftb_compact_workspace_bytes(T, n))
    _native.call("sfftb_compact_mask_cap", _dev.ptr(detmask), T, n, cap, _dev.ptr(idx),
                 _dev.ptr(counts), _dev.ptr(totals), _dev.ptr(ws), st)
    coeffs = _dev.empty((T * max(cap, 1),), torch.complex128)
    _native.call("sfftb_medians", _dev.ptr(sh.rows), d, _dev.ptr(zdev), T, L, M, _dev.ptr(ghat),
                 _dev.ptr(idx), _dev.ptr(counts), cap, _dev.ptr(coeffs), st)
    cls_dev = _dev.empty((T * max(cap, 1),), torch.uint8)
    tal_dev = _dev.empty((T, 5), torch.int64)
    _native.call("sfftb_alias_classify", _dev.ptr(idx), _dev.ptr(coeffs), _dev.ptr(counts), T,
                 cap, _dev.ptr(sh.in_mask), float(tol), _dev.ptr(cls_dev), _dev.ptr(tal_dev), st)
    tallies = _dev.download(tal_dev)
    cnt = _dev.download(counts)
    tot = _dev.download(totals)
    b = _engine.Batch(T, L, M, n, ghat, theta0, None, idx, counts, coeffs)

    overflow = [g for g in range(T) if tot[g] > cnt[g]]
    out = []
    theta_h = None
    cls_h = None
    for g in range(T):
        if g in overflow:  # more detections than the cap: this trial alone, uncapped
            out.append(_run_batch(sh, M, L, zs[g:g + 1], seeds[g:g + 1], spec, tol,
                                  max(n, 1))[0])
            continue
        t = tallies[g]
        pfn, pfp = int(t[_T_PFN]), int(t[_T_PFP])
        anomalies = (sh.n_in - int(t[_T_DET_IN])) + int(t[_T_NONINT]) + int(t[_T_LT1])
        clean = anomalies == 0
        plain = clean and pfn == 0 and pfp == 0
        budgets = {bb: clean and pfn == 0 and pfp <= bb for bb in spec.pfp_budgets}
        post = plain
        if spec.postprocess and clean and pfn == 0 and not plain:
            if theta_h is None:
                theta_h = _dev.download(theta0)
                cls_h = _dev.download(cls_dev)
            c = int(cnt[g])
            post = _postprocess_group(sh, b, g, cap, zdev, L, M, theta_h[g], c,
                                      cls_h[g * cap:g * cap + c])
        out.append(TrialRecord(seed=int(seeds[g]), L=L, M=M, pfn_count=pfn, pfp_count=pfp,
                               success_plain=plain, success_pfp_budget=budgets,
                               success_postprocessed=bool(post), sample_count=L * M,
                               wall_time=0.0, anomalies=anomalies))
    dt = (time.perf_counter() - t0) / max(T, 1)
    for r in out:
        if r.wall_time == 0.0:
            r.wall_time = dt
    return out


def _cap_for(gamma, I):
    return min(max(len(gamma), 1), max(_MIN_CAP, _CAP_PER_SUPPORT * len(I)))


def _trials_per_batch(n, L, M, cap):
    per_trial = L * M * 16 * 2 + cap * 17 + ((n + 31) // 32) * 4
    return max(1, min(1024, _BATCH_BYTES // per_trial))


def _check_spec(spec, L):
    if spec.nu != 0.5:
        raise ParameterError("coefficient computation requires nu = 1/2")
    if L % 2 == 0:
        raise ParameterError("coefficient computation requires odd L")


def run_success_experiment(spec, threads=1):
    """All (L, trial) runs of a spec plus one aggregate row per L
    (analysis.py:253-297).  Records come out in the reference's task order
    ((L, trial) for L in L_values for trial in range(trials)) and do not depend
    on ``threads`` (kept for signature parity; batching replaces the thread
    pool)."""
    with _dev.stream_scope():
        return _run_success_experiment(spec)


def _run_success_experiment(spec):
    records = []
    if spec.redraw == "lattices":
        rng = np.random.default_rng(np.random.SeedSequence((spec.master_seed, 0xFACE)))
        gamma = _make_candidates(spec.candidates, rng)
        I = _make_support(spec.support, gamma, rng)
        M = next_valid_prime(gamma, spec.c * len(I))
        _check_support(I, gamma)
        sh = _Shared(gamma, I)
        d = gamma.dim
        cap = _cap_for(gamma, I)
        for L in spec.L_values:
            if spec.trials == 0:
                continue
            _check_spec(spec, L)
            streams = hostrng.Streams([(spec.master_seed, L, t) for t in range(spec.trials)])
            zs = streams.integers_each(0, M, (L, d))
            per = _trials_per_batch(len(gamma), L, M, cap)
            for a in range(0, spec.trials, per):
                b = min(spec.trials, a + per)
                records += _run_batch(sh, M, L, zs[a:b], np.arange(a, b), spec, 1e-6, cap)
        gamma_size = len(gamma)
    elif spec.redraw == "both":
        for L in spec.L_values:
            for trial in range(spec.trials):
                _check_spec(spec, L)
                t0 = time.perf_counter()
                rng = np.random.default_rng(np.random.SeedSequence((spec.master_seed, L, trial)))
                gamma = _make_candidates(spec.candidates, rng)
                I = _make_support(spec.support, gamma, rng)
                M = next_valid_prime(gamma, spec.c * len(I))
                zs = rng.integers(0, M, size=(L, gamma.dim), dtype=np.int64)
                _check_support(I, gamma)
                sh = _Shared(gamma, I)
                cap = _cap_for(gamma, I)
                rec = _run_batch(sh, M, L, zs[None], np.array([trial]), spec, 1e-6, cap)[0]
                rec.wall_time = time.perf_counter() - t0
                records.append(rec)
        gamma_size = spec.candidates["count"]
    else:
        raise ParameterError(f"unknown redraw policy {spec.redraw!r}")

    aggregate = []
    for L in spec.L_values:
        recs = [r for r in records if r.L == L]
        n = len(recs)
        aggregate.append({
            "L": L,
            "trials": n,
            "fail_rate": (1.0 - sum(r.success_plain for r in recs) / n) if n else 0.0,
            "fail_rate_postprocessed": (1.0 - sum(r.success_postprocessed for r in recs) / n)
            if n else 0.0,
            "max_pfn": max((r.pfn_count for r in recs), default=0),
            "max_pfp": max((r.pfp_count for r in recs), default=0),
            "theo_bound": theoretical_failure_bound(gamma_size, L, spec.c),
            "samples": max((r.sample_count for r in recs), default=0),
        })
    return records, aggregate


def run_bspline_experiment(N, s, runs, master_seed, r=5, delta=0.999, L_scale=0.25,
                           theta=1e-12, s_local=None):
    """Approximation study of the ten-variate B-spline test function
    (analysis.py:300-316): sfft over [-N, N]^10 with f10 sampled on the
    device, relative L2 error from the closed-form coefficients."""
    rows = []
    sq_norm = f10_sq_norm()
    for run in range(runs):
        oracle = f10_oracle()
        params = SfftParams(s, delta, s_local=s_local, theta=theta, r=r, L_scale=L_scale)
        seed = int(np.random.SeedSequence((master_seed, run)).generate_state(1)[0])
        result = sfft(oracle, Box(10, -N, N), params, seed)
        err = rel_l2_error(result.support, result.coeffs, sq_norm, f10_coeffs)
        rows.append({"run": run, "N": N, "s": s, "samples": result.sample_count,
                     "rel_l2_error": err})
    return rows
