import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2006_13053_b200 as pkg
import workloads
w = workloads.metric_config()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
for _ in range(5):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    pkg.sfft(pkg.oracle_from_poly(poly), box, params, seed=w.seed)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(35)
