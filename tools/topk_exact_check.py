import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np
import paper_2006_13053_b200 as pkg
import workloads
from conftest import golden
g = golden("fixed_noisy.npz")
rng = np.random.default_rng(4242)
gamma = workloads.rows_from_box(5, -20, 20, 20_000, rng)
G = pkg.FreqSet(5, gamma, _sorted=True)
lats = [pkg.Rank1Lattice(z, int(g["M"])) for z in g["zmat"]]
cfg = pkg.MultiLatticeConfig(lats, 0.5, 10.33, 0.5)
smp = list(g["samples"])
top = pkg.detect_topk(smp, cfg, G, 40, 0.5)
print("topk exact:", np.array_equal(top.detected_idx, g["topk_idx"]), np.max(np.abs(top.coeffs - g["topk_coeffs"])))
t = golden("tiny_detect.npz")
bad = 0
for k in range(int(t["n"])):
    p = f"t{k}_"
    S = pkg.FreqSet(t[p + "gamma"].shape[1], t[p + "gamma"], _sorted=True)
    c = pkg.MultiLatticeConfig([pkg.Rank1Lattice(z, int(t[p + "M"])) for z in t[p + "zmat"]], 0.5, 10.33, 0.5)
    tp = pkg.detect_topk(list(t[p + "samples"]), c, S, 2, 0.1)
    if not np.array_equal(tp.detected_idx, t[p + "topk_idx"]): bad += 1; print("tiny mismatch", k)
print("tiny mismatches", bad, "of", int(t["n"]))
