"""Spectra-ahead hit/miss counts per config (phase-2 detections reuse the
enqueued spectra; phase-0 calls are whole-stage fallbacks) and the predicted
vs used lattice counts."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _stage  # noqa: E402
import workloads  # noqa: E402

orig = _stage.run
calls = []


def run(desc, stream=None):
    calls.append((int(desc.phase), int(desc.t), int(desc.L), int(desc.n), int(desc.call0)))
    return orig(desc, stream)


_stage.run = run
for name in ("metric_config", "config3", "config5", "config2"):
    w = getattr(workloads, name)()
    poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
    calls.clear()
    pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed),
             pkg.Box(w.d, w.lo, w.hi), pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r),
             seed=w.seed)
    torch.cuda.synchronize()
    ph = [c[0] for c in calls]
    print(name, "spectra", ph.count(1) + ph.count(4), "reused", ph.count(2), "fallback", ph.count(0))
    print("   ", [(c[0], c[2], c[3]) for c in calls])
