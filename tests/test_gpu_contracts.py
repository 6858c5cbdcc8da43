"""Error contracts of the public entry points, mirroring the reference's own
tests (tests/test_detect.py:88-127, test_dft.py:28-42, test_dimincr.py:25-47,
120-135 of latfft): the same exception types for the same bad inputs, on the
device path."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(pkg, M, L, d, nu=0.5, seed=0):
    rng = np.random.default_rng(seed)
    lats = [pkg.Rank1Lattice(rng.integers(0, M, d), M) for _ in range(L)]
    return pkg.MultiLatticeConfig(lats, nu, 10.33, 0.5)


def test_sample_length_mismatch(cuda):
    pkg = cuda
    lat = pkg.Rank1Lattice([1, 2], 11)
    config = pkg.MultiLatticeConfig([lat], 0.5, 10.33, 0.5)
    with pytest.raises(pkg.ParameterError):
        pkg.detect_frequencies([np.zeros(10)], config, pkg.FreqSet(2, [(0, 0)]))


def test_detect_and_compute_requires_odd_L_and_half_nu(cuda):
    pkg = cuda
    G = pkg.FreqSet(1, [(0,)])
    with pytest.raises(pkg.ParameterError):
        pkg.detect_and_compute([np.zeros(11, dtype=complex)] * 4, _cfg(pkg, 11, 4, 1), G)
    with pytest.raises(pkg.ParameterError):
        pkg.detect_and_compute([np.zeros(11, dtype=complex)] * 3, _cfg(pkg, 11, 3, 1, nu=0.25),
                               G)


@pytest.mark.parametrize("where", ["host", "device"])
@pytest.mark.parametrize("bad", [np.nan, np.inf])
def test_nonfinite_samples_rejected(cuda, where, bad):
    """The finiteness check of the single-sync detection path is read back
    with the counts; the call must still raise before returning."""
    import torch

    pkg = cuda
    M, L = 31, 5
    cfg = _cfg(pkg, M, L, 2, seed=3)
    G = pkg.FreqSet(2, [(0, 0), (1, 2), (3, -1)])
    smp = np.ones((L, M), dtype=np.complex128)
    smp[2, 7] = bad
    arg = [r for r in smp] if where == "host" else torch.as_tensor(smp, device="cuda")
    for fn in (pkg.detect_and_compute, pkg.detect_frequencies):
        with pytest.raises(pkg.ParameterError):
            fn(arg, cfg, G)
    with pytest.raises(pkg.ParameterError):
        pkg.detect_topk(arg, cfg, G, 2, 0.1)


def test_dft_contracts(cuda):
    pkg = cuda
    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized([1.0, np.nan])
    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized([np.inf + 0j, 1.0])
    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized([])
    with pytest.raises(pkg.ParameterError):
        pkg.dft_forward_normalized(np.zeros((2, 2)))


@pytest.mark.parametrize("M", [211, 1039, 2069, 4099])
def test_dft_mixed_small_lengths_vs_numpy(cuda, M):
    """The single-CTA Bluestein at 9 * 2^k lengths (M = 1039 -> 2304, 2069 ->
    4608) and at powers of two, against numpy's pocketfft (dft.py:27)."""
    pkg = cuda
    rng = np.random.default_rng(M)
    x = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    got = pkg.dft_forward_normalized(x)
    want = np.fft.fft(x) / M
    assert np.max(np.abs(got - want)) < 1e-15 * max(1.0, np.sqrt(M))


def test_sfft_params_validation(cuda):
    pkg = cuda
    p = pkg.SfftParams(10, 0.9)
    assert p.s_local == 20 and p.theta == 1e-12 and p.c == 10.33
    with pytest.raises(pkg.ParameterError):
        pkg.SfftParams(10, 0.9, s_local=5)
    with pytest.raises(pkg.ParameterError):
        pkg.SfftParams(0, 0.9)
    with pytest.raises(pkg.ParameterError):
        pkg.SfftParams(3, 0.9, theta=-1)


def test_pair_candidates_capacity_and_restriction(cuda):
    pkg = cuda
    prev = pkg.FreqSet(1, [(k,) for k in range(100)])
    with pytest.raises(pkg.CapacityError):
        pkg.pair_candidates(prev, np.arange(200), pkg.Box(2, -200, 200), 1, cap=10_000)
    # restriction to the prefix projection of a FreqSet Gamma (device filter)
    rng = np.random.default_rng(5)
    gamma = np.unique(rng.integers(-6, 7, size=(400, 3)), axis=0)
    G = pkg.FreqSet(3, gamma, _sorted=True)
    prev = pkg.FreqSet(1, np.unique(gamma[:, :1], axis=0), _sorted=True)
    vals = np.arange(-6, 7)
    J = pkg.pair_candidates(prev, vals, G, 1)
    rows = np.column_stack([np.repeat(prev.elems, len(vals), axis=0),
                            np.tile(vals, len(prev))])
    pool = {tuple(r) for r in np.unique(gamma[:, :2], axis=0)}
    want = rows[[tuple(r) in pool for r in rows]]
    assert np.array_equal(J.elems, want)
    assert len(J) < len(prev) * len(vals)


@pytest.mark.parametrize("n", [0, 1, 33])
def test_tiny_and_empty_candidate_sets(cuda, oracle_lib, n):
    """Empty and tiny candidate sets through the single-sync detection path:
    the same hits / detections as the oracle (detect.py:158-169)."""
    pkg, port = cuda, oracle_lib
    rng = np.random.default_rng(40 + n)
    d, M, L = 3, 101, 7
    gamma = np.unique(rng.integers(-20, 21, size=(n, d)), axis=0) if n else \
        np.zeros((0, d), np.int64)
    cfg = _cfg(pkg, M, L, d, seed=n)
    smp = [rng.standard_normal(M) + 1j * rng.standard_normal(M) for _ in range(L)]
    G = pkg.FreqSet(d, gamma, _sorted=True)
    res = pkg.detect_and_compute(smp, cfg, G)
    hits, idx, co, th = port.detect_and_compute(smp, M, cfg.zmat(), gamma)
    assert res.theta_zero == pytest.approx(th, rel=1e-14)
    assert np.array_equal(res.hits, hits)
    assert np.array_equal(res.detected_idx, idx)
    assert len(res.coeffs) == len(co)
    if len(co):
        assert np.max(np.abs(res.coeffs - co)) <= 1e-10 * max(1.0, np.max(np.abs(co)))
