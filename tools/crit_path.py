"""Critical-path probe of the metric reconstruction: insert a spin of X us on
the detection stream (before every phase-2 call) or on the spectra stream
(before every phase-4 call) and report how the step time moves.  A slope
near the number of stages means that chain is critical; near 0, slack.
    python tools/crit_path.py [workload name, default metric_config]"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.getcwd())
import paper_2006_13053_b200 as pkg  # noqa: E402
from paper_2006_13053_b200 import _stage  # noqa: E402
import workloads  # noqa: E402

w = getattr(workloads, sys.argv[1] if len(sys.argv) > 1 else "metric_config")()
box = pkg.Box(w.d, w.lo, w.hi)
params = pkg.SfftParams(w.s, w.delta, theta=w.theta, r=w.r)
poly = pkg.SparsePoly(pkg.FreqSet(w.d, w.support, _sorted=True), w.coeffs)
poly.device()
orig = _stage.run
CYC_PER_US = 1965
calls = {}


def make(phase_target, us):
    def run(desc, stream=None):
        if desc.phase == phase_target and us > 0:
            st = torch.cuda.ExternalStream(stream) if stream is not None else \
                torch.cuda.current_stream()
            with torch.cuda.stream(st):
                torch.cuda._sleep(int(us * CYC_PER_US))
        calls[desc.phase] = calls.get(desc.phase, 0) + 1
        return orig(desc, stream)
    return run


def step():
    return pkg.sfft(pkg.oracle_from_poly(poly, noise_sigma=w.sigma, noise_seed=w.noise_seed),
                    box, params, seed=w.seed)


def timeit(reps=7):
    for _ in range(2):
        step()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


base = timeit()
print(f"base {base:.3f} ms")
for phase, name in ((2, "detection"), (4, "transforms"), (3, "sampler")):
    for us in (20, 50, 100):
        _stage.run = make(phase, us)
        calls.clear()
        t = timeit()
        n = calls.get(phase, 0) / 9  # 2 warm-up + 7 timed
        _stage.run = orig
        print(f"{name:10s} +{us:3d} us x {n:.1f} calls/step: {t:.3f} ms "
              f"(+{t - base:.3f}, slope {(t - base) * 1e3 / us:.2f} per stage-spin)")
