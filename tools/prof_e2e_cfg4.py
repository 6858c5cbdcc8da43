"""Where the cfg4 end-to-end time goes (host rows in, results out)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402

n, d, N = 1 << 26, 10, 4096
G = pkg.random_box_device(pkg.Box(d, -N, N), n, 5)
rows = G.device()
rng = np.random.default_rng(1)
sup = np.sort(rng.choice(n, size=10_000, replace=False))
poly = pkg.SparsePoly(G.take(sup), rng.normal(size=10_000) + 1j * rng.normal(size=10_000) + 3)
cfg = pkg.draw_config(G, 10_000, 0.1, rng=rng)
smp = pkg.oracle_from_poly(poly).sample_lattices_device(
    cfg.zmat_device(), cfg.shared_M, torch.zeros((1, 1), dtype=torch.float64, device="cuda"), 1,
    cfg.L, d).contiguous()
host = torch.empty((n, d), dtype=torch.int64, pin_memory=True)
host.copy_(rows)
hnp = host.numpy()
for rep in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    Gh = pkg.FreqSet(d, hnp, _sorted=True)
    Gh.memo("bounds", lambda: np.array([[-N, N]] * d, dtype=np.int64))
    t1 = time.perf_counter()
    r2 = pkg.detect_and_compute(smp, cfg, Gh)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    h = r2.hits
    t3 = time.perf_counter()
    i, c = r2.detected_idx, r2.coeffs
    t4 = time.perf_counter()
    print(f"rep {rep}: freqset {1e3*(t1-t0):.1f}  detect {1e3*(t2-t1):.1f}  hits D2H {1e3*(t3-t2):.1f}"
          f"  idx/coeffs {1e3*(t4-t3):.1f}  total {1e3*(t4-t0):.1f} ms")
    del Gh, r2, h
