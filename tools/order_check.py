import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg
from paper_2006_13053_b200 import _native
import workloads
w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
for _ in range(3):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
start = torch.cuda.Event(enable_timing=True); start.record()
with _native.Timeline() as tl:
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
tr = [(n, start.elapsed_time(a), start.elapsed_time(b)) for (n, a, b) in tl.records if n.startswith("stage:transforms") or n.startswith("stage:hashing") or n.startswith("stage:candidates")]
for n, a, b in tr:
    print(f"{a:7.3f} {b:7.3f} {n}")
