"""Seeded synthetic workloads for BASELINE.json's five configs (harness only).

Shared by bench.py, tests/ and tests/golden/make_golden.py.  Host numpy RNG,
drawn in the order SURVEY.md Appendix C records, so the same seed yields the
same candidate sets / polynomials here, in the oracle and in the reference.
BASELINE.json's "threshold delta" is the reference's coefficient threshold
``theta``; the failure probability ``delta`` stays at
the reference CLI defaults (0.1 fixed-Gamma, 0.9 sfft).

The paper's benchmarks are synthetic (random frequencies, random
coefficients); nothing here reproduces a public dataset.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np


def _canon(arr):
    order = np.lexsort(arr.T[::-1])
    s = arr[order]
    keep = np.ones(s.shape[0], dtype=bool)
    keep[1:] = np.any(s[1:] != s[:-1], axis=1)
    return np.ascontiguousarray(s[keep])


def rows_from_box(d, lo, hi, count, rng):
    """Distinct uniform rows of [lo, hi]^d (RNG call order of the reference's
    freqset._random_from_box, freqset.py:266-280)."""
    rows = np.empty((0, d), dtype=np.int64)
    need = count
    while need > 0:
        batch = rng.integers(lo, hi + 1, size=(int(need * 1.05) + 16, d),
                             dtype=np.int64)
        rows = _canon(np.vstack([rows, batch]))
        if len(rows) > count:
            rows = rows[np.sort(rng.choice(len(rows), size=count, replace=False))]
        need = count - len(rows)
    return rows


def rows_from_set(elems, count, rng):
    """random_subset of a materialised set (freqset.py:257-260)."""
    return elems[np.sort(rng.choice(elems.shape[0], size=count, replace=False))]


def mag_phase_coeffs(n, rng):
    """|c| ~ U[1, 10], arg c ~ U[0, 2 pi) (BASELINE.json configs 1-4)."""
    mags = rng.uniform(1.0, 10.0, size=n)
    phases = rng.uniform(0.0, 2 * np.pi, size=n)
    return mags * np.exp(1j * phases)


@dataclass
class FixedGammaWorkload:
    """Configs 1 and 4: Gamma, true support (rows of Gamma), coefficients."""
    name: str
    d: int
    gamma: np.ndarray
    support_idx: np.ndarray
    coeffs: np.ndarray
    s: int
    delta: float = 0.1
    seed: int = 0
    rng: object = None          # generator positioned for draw_config


@dataclass
class SfftWorkload:
    """Configs 2, 3, 5 and the metric instance: box, polynomial, params."""
    name: str
    d: int
    lo: int
    hi: int
    support: np.ndarray
    coeffs: np.ndarray
    s: int
    r: int
    theta: float
    delta: float = 0.9
    seed: int = 7
    sigma: float = 0.0
    noise_seed: int = 0
    extra: dict = field(default_factory=dict)


def config1(seed=2026, n=10_000, d=5, N=16, s=20):
    """Config 1: |Gamma| = 1e4 in [-16,16]^5, s = 20."""
    rng = np.random.default_rng(seed)
    gamma = rows_from_box(d, -N, N, n, rng)
    idx = np.sort(rng.choice(gamma.shape[0], size=s, replace=False))
    coeffs = mag_phase_coeffs(s, rng)
    return FixedGammaWorkload("cfg1", d, gamma, idx, coeffs, s, 0.1, seed, rng)


def config4_host(seed=2026, n=1 << 26, d=10, N=4096, s=10_000):
    """Config 4 generated on the host (slow at full size: minutes)."""
    rng = np.random.default_rng(seed)
    gamma = rows_from_box(d, -N, N, n, rng)
    idx = np.sort(rng.choice(gamma.shape[0], size=s, replace=False))
    coeffs = mag_phase_coeffs(s, rng)
    return FixedGammaWorkload("cfg4", d, gamma, idx, coeffs, s, 0.1, seed, rng)


def _box_poly(seed, d, N, s):
    rng = np.random.default_rng(seed)
    support = rows_from_box(d, -N, N, s, rng)
    return support, mag_phase_coeffs(s, rng)


def config2(seed=12345):
    """Config 2: d=10, [-32,32]^10, s=100, r=5, theta=1e-12."""
    sup, c = _box_poly(seed, 10, 32, 100)
    return SfftWorkload("cfg2", 10, -32, 32, sup, c, 100, 5, 1e-12)


def metric_config(seed=2006):
    """The metric's literal instance "(d=10, s=1000)": config-2 generator
    with s = 1000 (paper Table 4 row, PAPER.md:1737 uses the same box)."""
    sup, c = _box_poly(seed, 10, 32, 1000)
    return SfftWorkload("d10_s1000", 10, -32, 32, sup, c, 1000, 5, 1e-12)


def config3(seed=777):
    """Config 3: d=20, [-64,64]^20, s=1000, r=5, theta=1e-12."""
    sup, c = _box_poly(seed, 20, 64, 1000)
    return SfftWorkload("cfg3", 20, -64, 64, sup, c, 1000, 5, 1e-12)


def config5(seed=99, sigma=1e-3):
    """Config 5: d=9, [-32,32]^9, 5000 decaying coefficients
    c_k = (1+|k|_2)^-2 e^{i phi}, sigma=1e-3 complex noise, s=1000, r=5,
    theta=1e-6."""
    rng = np.random.default_rng(seed)
    sup = rows_from_box(9, -32, 32, 5000, rng)
    phi = rng.uniform(0.0, 2 * np.pi, size=sup.shape[0])
    c = (1.0 + np.sqrt(np.sum(sup.astype(np.float64) ** 2, axis=1))) ** -2.0
    c = c * np.exp(1j * phi)
    return SfftWorkload("cfg5", 9, -32, 32, sup, c, 1000, 5, 1e-6,
                        sigma=sigma, noise_seed=seed)


def small_sfft(seed, d, N, n, s=None, r=1, theta=1e-12, delta=0.9, sfft_seed=7,
               sigma=0.0, decaying=False):
    """Reduced-scale sfft instance used by parity tests."""
    rng = np.random.default_rng(seed)
    sup = rows_from_box(d, -N, N, n, rng)
    if decaying:
        phi = rng.uniform(0.0, 2 * np.pi, size=n)
        c = (1.0 + np.sqrt(np.sum(sup.astype(np.float64) ** 2, axis=1))) ** -2.0
        c = c * np.exp(1j * phi)
    else:
        c = mag_phase_coeffs(n, rng)
    return SfftWorkload(f"small_{seed}", d, -N, N, sup, c, s or n, r, theta,
                        delta, sfft_seed, sigma, seed if sigma else 0)


def rel_l2(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = math.sqrt(float(np.sum(np.abs(b) ** 2))) or 1.0
    return math.sqrt(float(np.sum(np.abs(a - b) ** 2))) / den
