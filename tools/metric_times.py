import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg
import workloads
w = workloads.metric_config()
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
def run():
    return pkg.sfft(pkg.oracle_from_poly(poly), pkg.Box(w.d, w.lo, w.hi), pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r), seed=w.seed)
for _ in range(3): run()
torch.cuda.synchronize()
ts=[]
for _ in range(20):
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record(); run(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
ts.sort(); print(os.environ.get("SFFTB_MEDIANS2"), "min %.3f med %.3f" % (ts[0], ts[10]))
