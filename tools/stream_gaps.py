"""Idle time of the spectra (transforms) stream during one reconstruction of
the metric instance: union of the 'stage:transforms' intervals vs the step.
    python tools/stream_gaps.py"""
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _native  # noqa: E402
import workloads  # noqa: E402

w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
for _ in range(3):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
start = torch.cuda.Event(enable_timing=True)
end = torch.cuda.Event(enable_timing=True)
start.record()
with _native.Timeline() as tl:
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
end.record()
torch.cuda.synchronize()
total = start.elapsed_time(end)
rec = [(n, start.elapsed_time(a), start.elapsed_time(b)) for (n, a, b) in tl.records]
tr = sorted((a, b) for n, a, b in rec if n == "stage:transforms")
busy, last, gaps = 0.0, 0.0, []
for a, b in tr:
    if a > last:
        gaps.append((last, a))
    busy += max(0.0, b - max(a, last))
    last = max(last, b)
print(f"step {total:.3f} ms; transforms busy {busy:.3f} ms over {len(tr)} calls; "
      f"first start {tr[0][0]:.3f}, last end {last:.3f}, tail {total - last:.3f}")
for a, b in gaps:
    if b - a > 0.01:
        print(f"  gap {a:7.3f} -> {b:7.3f}  ({(b - a) * 1e3:.0f} us)")
for n, a, b in sorted(rec, key=lambda x: x[1]):
    if not n.startswith("stage:") or n in ("stage:transforms",):
        continue
    if a > last - 0.3:
        print(f"  {a:7.3f} {b:7.3f} {n}")
