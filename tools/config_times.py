"""Device time of the public entry point on every BASELINE config (one B200).

    python tools/config_times.py [reps]

sfft configs (2, 3, 5, the metric instance): CUDA events around sfft(...)
(after warm-up).  Config 1: detect_and_compute on device-resident samples.
Prints one JSON object per config."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
import workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts), out


for name in ("config2", "metric_config", "config3", "config5"):
    w = getattr(workloads, name)()
    poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
    box = pkg.Box(w.d, w.lo, w.hi)
    params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)

    def run():
        return pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma,
                                             noise_seed=w.noise_seed), box, params, seed=w.seed)

    ms, res = timed(run)
    exact = (np.array_equal(res.support.elems, w.support[np.lexsort(w.support.T[::-1])])
             if w.sigma == 0 else None)
    print(json.dumps({"config": w.name, "d": w.d, "s": w.s, "ms": round(ms, 3),
                      "samples": res.sample_count, "stages": len(res.stage_log),
                      "support_size": len(res.support), "exact_support": exact}))

w = workloads.config1()
G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
p = pkg.SparsePoly(G.take(w.support_idx), w.coeffs)
cfg = pkg.draw_config(G, w.s, 0.1, rng=w.rng)
orc = pkg.oracle_from_poly(p)
smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M,
                                 torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                 1, cfg.L, w.d).contiguous()
ms, res = timed(lambda: pkg.detect_and_compute(smp, cfg, G).detected_idx)
print(json.dumps({"config": "cfg1", "entry": "detect_and_compute", "ms": round(ms, 3),
                  "n": len(G), "L": cfg.L, "M": cfg.shared_M,
                  "detected_equals_support": bool(np.array_equal(res, np.sort(w.support_idx)))}))
