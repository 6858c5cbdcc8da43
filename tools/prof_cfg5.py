"""One config-5 reconstruction (profiling helper for its medians/top-s)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

w = workloads.config5()
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
for _ in range(2):
    pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed),
             pkg.Box(w.d, w.lo, w.hi), pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r),
             seed=w.seed)
