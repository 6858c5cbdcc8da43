"""Experiment harness on the B200 against the reference's outputs
(tests/golden/analysis_cases.json, pfp_pfn_cases.npz, f10_cases.json):
trial records bit-identical (wall time aside), alias classifications exact,
device B-spline values within 1e-12 absolute of numpy's (O(1) values)."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

SPECS = ("desk", "hc_small", "hc_fused", "box_fused")


@pytest.mark.parametrize("key", SPECS)
def test_success_experiment_records_match_reference(cuda, key):
    from paper_2006_13053_b200 import analysis

    case = golden("analysis_cases.json")[key]
    spec = analysis.ExperimentSpec.from_dict(case["spec"])
    recs, agg = analysis.run_success_experiment(spec)
    assert [r.as_jsonable() for r in recs] == case["records"]
    assert agg == case["aggregate"]
    assert all(r.wall_time >= 0 for r in recs)


def test_batching_and_capacity_overflow_do_not_change_records(cuda, monkeypatch):
    """Tiny device batches and a detection cap far below the detected counts
    (every trial re-run uncapped) give the same records."""
    from paper_2006_13053_b200 import analysis

    case = golden("analysis_cases.json")["hc_fused"]
    spec = analysis.ExperimentSpec.from_dict(case["spec"])
    spec.L_values = [5, 9]
    spec.trials = 7
    want = [r for r in case["records"] if r["L"] in (5, 9) and r["seed"] < 7]
    monkeypatch.setattr(analysis, "_BATCH_BYTES", 3 * 5 * 7681 * 40)
    monkeypatch.setattr(analysis, "_MIN_CAP", 64)
    monkeypatch.setattr(analysis, "_CAP_PER_SUPPORT", 0)
    recs, _ = analysis.run_success_experiment(spec)
    assert [r.as_jsonable() for r in recs] == want


def test_zero_trials(cuda):
    from paper_2006_13053_b200 import analysis

    spec = analysis.ExperimentSpec.from_dict(golden("analysis_cases.json")["desk"]["spec"])
    spec.trials = 0
    recs, agg = analysis.run_success_experiment(spec)
    assert recs == [] and all(row["trials"] == 0 for row in agg)


def test_pfp_pfn_count_matches_reference(cuda):
    from paper_2006_13053_b200 import FreqSet, MultiLatticeConfig, Rank1Lattice, analysis

    z = golden("pfp_pfn_cases.npz")
    for k in range(int(z["ncases"])):
        G = FreqSet.from_array(z[f"gamma_{k}"], _sorted=True)
        I = FreqSet.from_array(z[f"I_{k}"], _sorted=True)
        lats = [Rank1Lattice(zz, int(M)) for zz, M in zip(z[f"z_{k}"], z[f"M_{k}"])]
        cfg = MultiLatticeConfig(lats, 0.5, 10.33, 0.5)
        out = analysis.pfp_pfn_count(I, G, cfg)
        assert np.array_equal(out.pfn.elems, z[f"pfn_{k}"].reshape(-1, G.dim)), k
        assert np.array_equal(out.pfp.elems, z[f"pfp_{k}"].reshape(-1, G.dim)), k
        assert out.anomalies == int(z[f"anomalies_{k}"]), k
        assert np.all(I.contains_rows(out.pfn.elems))
        assert not np.any(I.contains_rows(out.pfp.elems))


def test_pfp_pfn_count_rejects_empty_support(cuda):
    from paper_2006_13053_b200 import Box, FreqSet, ParameterError, analysis, draw_config
    from paper_2006_13053_b200 import random_subset

    rng = np.random.default_rng(5)
    G = random_subset(Box(2, -20, 20), 60, rng)
    cfg = draw_config(G, 1, 0.5, rng=rng, L=5)
    with pytest.raises(ParameterError):
        analysis.pfp_pfn_count(FreqSet(2, np.zeros((0, 2), dtype=np.int64)), G, cfg)


def test_device_bspline_and_f10_values(cuda):
    from paper_2006_13053_b200 import polyeval

    f = golden("f10_cases.json")
    x = np.array(f["x"])
    for m, want in f["bspline"].items():
        got = polyeval.bspline_values(int(m), x)
        # the alternating cardinal sum (terms up to C(6,3) 3^5 / 5! ~ 40) cancels
        # to O(1): both evaluations carry ~1e-13 absolute rounding, so the bound
        # is absolute at the spline's scale
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-12)
    X = np.array(f["X"])
    np.testing.assert_allclose(polyeval.f10_values(X), f["f10"], rtol=1e-13, atol=1e-12)


def test_f10_lattice_sampler_equals_points(cuda):
    """Fixed-tail lattice nodes sampled in-kernel == the same nodes evaluated
    as explicit points (dimincr.py:186-191 node construction)."""
    import torch

    from paper_2006_13053_b200 import Rank1Lattice, _dev, lattice_nodes, polyeval

    rng = np.random.default_rng(3)
    orc = polyeval.f10_oracle()
    M, L, t_dim = 1031, 3, 4
    z = rng.integers(0, M, size=(L, t_dim))
    tail = rng.uniform(size=10 - t_dim)
    vals = _dev.download(orc.sample_lattices_device(
        _dev.upload(z), M, _dev.upload(tail.reshape(1, -1)), 1, L, t_dim))
    assert orc.count == L * M
    for l in range(L):
        nodes = np.empty((M, 10))
        nodes[:, :t_dim] = lattice_nodes(Rank1Lattice(z[l], M))
        nodes[:, t_dim:] = tail
        np.testing.assert_array_equal(vals[l], orc.sample_many(nodes))
    assert torch.is_tensor(orc.spline.points_device(_dev.upload(np.zeros((1, 10)))))


def test_bspline_study_matches_reference(cuda):
    """run_bspline_experiment: sfft on f10 sampled on the device.  The sample
    count is exact; the error agrees to 1e-6 relative (FFT rounding may reorder
    equal-magnitude coefficients of the symmetric test function)."""
    from paper_2006_13053_b200 import analysis

    st = golden("f10_cases.json")["study"]
    N, s, runs, seed, r, delta, Ls = st["args"]
    rows = analysis.run_bspline_experiment(N, s, runs=runs, master_seed=seed, r=r, delta=delta,
                                           L_scale=Ls)
    for got, want in zip(rows, st["rows"]):
        assert got["samples"] == want["samples"]
        assert got["rel_l2_error"] == pytest.approx(want["rel_l2_error"], rel=1e-6)


@pytest.mark.parametrize("which", [0, 1])
def test_bspline_paper_setting_matches_reference(cuda, which):
    """f10, N = 16, s = 200 / 1000, r = 2 / 5 (the paper's B-spline study):
    the same sample count as the reference and the same error to 1e-6."""
    from paper_2006_13053_b200 import analysis

    st = golden("f10_cases.json")["studies_paper"][which]
    N, s, runs, seed, r, delta, Ls = st["args"]
    rows = analysis.run_bspline_experiment(N, s, runs=runs, master_seed=seed, r=r, delta=delta,
                                           L_scale=Ls)
    for got, want in zip(rows, st["rows"]):
        assert got["samples"] == want["samples"]
        assert got["rel_l2_error"] == pytest.approx(want["rel_l2_error"], rel=1e-6)


def test_fullscale_hyperbolic_trials_match_reference(cuda):
    """Paper scale: |Gamma| = 10.7M (hyperbolic cross, d = 8), |I| = 1069,
    M = 11047; three trials each at L = 9 (about 6300 potential false
    positives per trial) and L = 37, against the reference's records."""
    from paper_2006_13053_b200 import analysis

    case = golden("analysis_fullscale.json")
    spec = analysis.ExperimentSpec.from_dict(case["spec"])
    recs, _ = analysis.run_success_experiment(spec)
    assert [r.as_jsonable() for r in recs] == case["records"]
