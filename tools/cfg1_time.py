import sys, os, time, torch
sys.path.insert(0, os.getcwd())
import bench, workloads
import paper_2006_13053_b200 as pkg
w = workloads.config1()
G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
cfg = pkg.draw_config(G, w.s, 0.1, rng=w.rng)
orc = pkg.oracle_from_poly(pkg.SparsePoly(G.take(w.support_idx), w.coeffs))
smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M, torch.zeros((1, 1), dtype=torch.float64, device="cuda"), 1, cfg.L, w.d).contiguous()
for _ in range(3):
    ms, det = bench._timed(lambda: pkg.detect_and_compute(smp, cfg, G).detected_idx, reps=20)
    print("cfg1 us", ms * 1e3)
