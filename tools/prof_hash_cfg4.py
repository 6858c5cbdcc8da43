"""sfftb_hash_hits on the bench's own cfg4 instance (the reference's seeded
Gamma, its lattices and the spectra's nonzero bitmaps), timed per call with a
synchronisation in between, next to a row-shuffled copy of the same Gamma."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2006_13053_b200 as pkg  # noqa: E402
from bench import CFG4_SEED, cfg4_instance  # noqa: E402
from paper_2006_13053_b200 import _dev, _engine, _native  # noqa: E402

n, d, N, s = 1 << 26, 10, 4096, 10_000
G, I, pick, coeffs, cfg, gen_ms = cfg4_instance(n, d, N, s, CFG4_SEED)
M, L = cfg.shared_M, cfg.L
orc = pkg.oracle_from_poly(pkg.SparsePoly(I, coeffs))
samples = orc.sample_lattices_device(cfg.zmat_device(), M,
                                     torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                     1, L, d).contiguous()
_g, th, bits = _engine.spectra(samples, M, 1, L)
del _g
rows = G.device()
zdev = cfg.zmat_device()
hits = torch.empty((n,), dtype=torch.int64, device="cuda")
mask = torch.empty(((n + 31) // 32,), dtype=torch.int32, device="cuda")
W = int(_native.lib().sfftb_bitmap_words(M))
dens = float(sum(bin(int(x) & 0xFFFFFFFF).count("1") for x in bits[:W].cpu().tolist())) / M
print(f"M={M} L={L} bitmap density of lattice 0: {dens:.4f}")


def run(r, label):
    ms = []
    for _ in range(6):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        _native.call("sfftb_hash_hits", r.data_ptr(), n, d, zdev.data_ptr(), 1, L, M,
                     bits.data_ptr(), -1, 24, hits.data_ptr(), mask.data_ptr(), _dev.stream())
        b.record()
        torch.cuda.synchronize()
        ms.append(round(a.elapsed_time(b), 4))
    print(label, ms, "mean hits", float(hits.float().mean()))


run(rows, "sorted Gamma  ")
perm = torch.randperm(n, device="cuda")
shuf = rows[perm].contiguous()
del perm
run(shuf, "shuffled rows ")
