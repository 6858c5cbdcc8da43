"""Experiment-harness host logic (no GPU): specs, budgets, bounds, the
closed-form B-spline / f10 formulas and the trial seed streams, pinned to
tests/golden/{analysis,f10}_cases.json (made by the reference)."""

import json
import math

import numpy as np
import pytest

from conftest import golden
from paper_2006_13053_b200 import analysis, hostrng, polyeval
from paper_2006_13053_b200.errors import ParameterError


def test_bounds_and_budgets_match_reference():
    ba = golden("analysis_cases.json")["budgets"]
    for L, want in zip((0, 9, 37, 41), ba["bound"]):
        assert analysis.theoretical_failure_bound(1e7, L, 10.33) == want
    assert analysis.guaranteed_sample_budget(1000, 10**7, 0.5) == ba["guaranteed"]
    assert analysis.theoretical_failure_bound(1e7, 37, 10.33) == pytest.approx(0.583, abs=1e-3)
    with pytest.raises(ParameterError):
        analysis.theoretical_failure_bound(10.0, 5, 2.0)


def test_spec_round_trip_and_golden_specs():
    cases = golden("analysis_cases.json")
    for key in ("desk", "hc_small", "hc_fused", "box_fused"):
        spec = analysis.ExperimentSpec.from_dict(cases[key]["spec"])
        again = analysis.ExperimentSpec.from_dict(json.loads(json.dumps(spec.as_dict())))
        assert again.as_dict() == spec.as_dict() == cases[key]["spec"]


def test_paper_fullscale_spec_parses():
    # the paper's hyperbolic-cross sweep (Sec. 5 worst-case study), as a spec
    spec = analysis.ExperimentSpec.from_dict({
        "name": "hyperbolic-fullscale", "candidates": {"kind": "hyperbolic", "d": 8, "N": 32,
                                                       "weights": None},
        "support": {"kind": "hyperbolic", "N": 32, "weights": "t^1.08"},
        "L_values": list(range(9, 38, 2)), "trials": 1000, "master_seed": 2023,
        "redraw": "lattices", "pfp_budgets": [10, 100]})
    assert spec.trials == 1000 and spec.pfp_budgets == (10, 100)


def test_trial_records_serialise_without_wall_time():
    r = analysis.TrialRecord(seed=3, L=5, M=53, pfn_count=0, pfp_count=2, success_plain=False,
                             success_pfp_budget={0: False, 10: True},
                             success_postprocessed=True, sample_count=265, wall_time=0.25)
    blob = r.as_jsonable()
    json.dumps(blob)
    assert "wall_time" not in blob and blob["success_pfp_budget"] == {"0": False, "10": True}


def test_trial_generator_streams_match_numpy():
    """The batched runner draws every trial's generators natively
    (SeedSequence((master, L, trial)), analysis.py:219-229)."""
    for master, L, M, d in ((2023, 9, 7681, 4), (99, 3, 113, 2), (2**40 + 7, 37, 11057, 8)):
        zs = hostrng.Streams([(master, L, t) for t in range(5)]).integers_each(0, M, (L, d))
        for t in range(5):
            rng = np.random.default_rng(np.random.SeedSequence((master, L, t)))
            assert np.array_equal(zs[t], rng.integers(0, M, size=(L, d), dtype=np.int64))


def test_bspline_constants_and_f10_coefficients_match_reference():
    f = golden("f10_cases.json")
    for m, want in f["norm"].items():
        assert polyeval.bspline_norm_constant(int(m)) == want
    K = np.array(f["K"], dtype=np.int64)
    assert np.array_equal(polyeval.f10_coeffs(K), np.array(f["f10_coeffs"]))
    assert polyeval.f10_sq_norm() == f["sq_norm"]
    assert polyeval.f10_coeff(np.zeros(10, dtype=np.int64)) == f["f10_coeffs"][5]
    c = {m: polyeval.bspline_norm_constant(m) for m in (2, 4, 6)}
    assert polyeval.f10_sq_norm() == pytest.approx(
        3 + 2 * (c[2] ** 3 * c[4] ** 4 + c[2] ** 3 * c[6] ** 3 + c[4] ** 4 * c[6] ** 3))
    assert polyeval.bspline_coeff(2, 2) == pytest.approx(0.0, abs=1e-15)


def test_rel_l2_error_formula():
    from paper_2006_13053_b200 import FreqSet

    I = FreqSet(10, [[0] * 10])
    f0 = polyeval.f10_coeff(np.zeros(10, dtype=np.int64))
    sq = polyeval.f10_sq_norm()
    assert polyeval.rel_l2_error(I, [f0], sq, polyeval.f10_coeffs) == pytest.approx(
        math.sqrt((sq - f0 ** 2) / sq))
    empty = FreqSet(10, np.zeros((0, 10), dtype=np.int64))
    assert polyeval.rel_l2_error(empty, [], sq, polyeval.f10_coeffs) == 1.0
    with pytest.raises(ParameterError):
        polyeval.rel_l2_error(I, [1, 2], sq, polyeval.f10_coeffs)
