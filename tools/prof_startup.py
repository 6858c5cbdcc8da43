"""Host timeline of the start of one metric-size sfft (before stage 1's
spectra are enqueued): wall time at entry/exit of the driver's setup steps."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import dimincr, hostrng, polyeval, _stage  # noqa: E402
import workloads  # noqa: E402

w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
marks = []
T0 = [0.0]


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        t = time.perf_counter()
        out = f(*a, **k)
        marks.append((name, (t - T0[0]) * 1e3, (time.perf_counter() - T0[0]) * 1e3))
        return out
    setattr(mod, name, g)


for mod, name in ((dimincr, "_step1_box_launch"), (dimincr, "_step1_box_finish"),
                  (dimincr, "_sfft_stages"), (polyeval, "_eval_points_dev"),
                  (dimincr, "dft_batch"), (_stage, "run"), (_stage, "buffers"),
                  (_stage, "host_inputs"), (hostrng, "streams"), (hostrng, "grid"),
                  (dimincr, "_master_seed")):
    wrap(mod, name)
for _ in range(5):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
for rep in range(2):
    marks.clear()
    orc = pkg.oracle_from_poly(poly)
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    pkg.sfft(orc, box, params, seed=w.seed)
    tot = (time.perf_counter() - T0[0]) * 1e3
    print(f"rep {rep}: total {tot:.3f} ms")
    for name, a, b in sorted(marks, key=lambda m: m[1])[:24]:
        print(f"  {a:7.3f} -> {b:7.3f}  {name}")
