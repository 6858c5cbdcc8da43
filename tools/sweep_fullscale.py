"""Time the paper-scale worst-case sweep on one B200.

The reference's hyperbolic-cross study (|Gamma| = 10,665,297 in d = 8,
|I| = 1069, M = 11047, L = 9..37 odd, 1000 trials per L): every trial of one
L runs as one batched device chain (paper_2006_13053_b200/analysis.py).
The reference needs 4.6-11.9 s per trial on one core
(tests/golden/analysis_fullscale.json), about 29 h for the sweep.

    python tools/sweep_fullscale.py [trials] [L ...]   # default 1000, all 15 L

Prints one JSON line per L and a summary line.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2006_13053_b200 import analysis  # noqa: E402


def main():
    trials = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    Ls = [int(v) for v in sys.argv[2:]] or list(range(9, 38, 2))
    base = {"name": "hyperbolic-fullscale",
            "candidates": {"kind": "hyperbolic", "d": 8, "N": 32, "weights": None},
            "support": {"kind": "hyperbolic", "N": 32, "weights": "t^1.08"},
            "trials": trials, "master_seed": 2023, "redraw": "lattices",
            "pfp_budgets": [10, 100]}
    ref = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                      "analysis_fullscale.json")))
    # warm-up: sets, M, kernels (one trial at the smallest L)
    t0 = time.perf_counter()
    analysis.run_success_experiment(analysis.ExperimentSpec.from_dict(
        dict(base, L_values=[Ls[0]], trials=1)))
    torch.cuda.synchronize()
    warm = time.perf_counter() - t0
    spec = analysis.ExperimentSpec.from_dict(dict(base, L_values=Ls))
    torch.cuda.synchronize()
    t = time.perf_counter()
    recs, agg = analysis.run_success_experiment(spec)  # the whole sweep, one call
    torch.cuda.synchronize()
    total = time.perf_counter() - t
    for row in agg:
        secs = sum(r.wall_time for r in recs if r.L == row["L"])
        print(json.dumps(dict(row, seconds=round(secs, 3),
                              ms_per_trial=round(1e3 * secs / trials, 3))), flush=True)
    ref_s = ref["ref_seconds_per_trial"]
    ref9, ref37 = np.mean(ref_s[:3]), np.mean(ref_s[3:])
    # reference seconds per trial grow linearly in L (hashing + medians of L lattices)
    ref_total = sum(trials * (ref9 + (ref37 - ref9) * (L - 9) / 28.0) for L in Ls)
    print(json.dumps({"summary": "hyperbolic-fullscale sweep", "trials_per_L": trials,
                      "L_values": Ls, "gpu_seconds": round(total, 2),
                      "first_call_setup_seconds": round(warm, 2),
                      "reference_seconds_estimate": round(ref_total, 1),
                      "reference_basis": "mean of 3 measured trials at L=9 and L=37, "
                                         "linear in L (tests/golden/analysis_fullscale.json)",
                      "speedup": round(ref_total / total, 1)}), flush=True)


if __name__ == "__main__":
    main()
