"""Multi-rank fixed-Gamma detection on the product path, and reentrancy.

* Two ranks (gloo for the collectives, both on the one GPU of a gpurun box)
  run shard.detect_and_compute_sharded -- lattice-sharded DFTs, bitmap and
  spectra all-gathers, row-sharded hashing -- and the merged result must
  equal the single-process detect_and_compute bit for bit
  (detect.py:158-169 semantics).
* Four host threads, each on its own torch stream, call detect_and_compute
  and sfft concurrently; every result must be bitwise the serial one (the
  reference's kernels are reentrant and run from worker threads,
  analysis.py:271-274).
"""

import os
import socket
import threading

import numpy as np
import pytest

import workloads

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _instance(pkg, n, seed):
    import torch

    w = workloads.config1(seed=seed, n=n, d=6, N=40, s=25)
    G = pkg.FreqSet(w.d, w.gamma, _sorted=True)
    cfg = pkg.draw_config(G, w.s, 0.1, rng=w.rng)
    orc = pkg.oracle_from_poly(pkg.SparsePoly(G.take(w.support_idx), w.coeffs))
    smp = orc.sample_lattices_device(cfg.zmat_device(), cfg.shared_M,
                                     torch.zeros((1, 1), dtype=torch.float64, device="cuda"),
                                     1, cfg.L, w.d).contiguous()
    return w, G, cfg, smp


def _rank(rank, world, port, n, seed, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2006_13053_b200 as pkg
    from paper_2006_13053_b200.shard import detect_and_compute_sharded, shard_bounds

    w, G, cfg, smp = _instance(pkg, n, seed)
    lo, hi = shard_bounds(len(G), world, rank)
    shard = pkg.FreqSet(w.d, w.gamma[lo:hi], _sorted=True)
    gidx, gco, loc = detect_and_compute_sharded(smp, cfg, shard, lo)
    ref = pkg.detect_and_compute(smp, cfg, G)
    ok = {
        "idx": bool(np.array_equal(gidx, ref.detected_idx)),
        "coeffs_bitwise": bool(np.array_equal(gco.view(np.int64), ref.coeffs.view(np.int64))),
        "local_hits": bool(np.array_equal(loc.hits, ref.hits[lo:hi])),
        "support": bool(np.array_equal(gidx, np.sort(w.support_idx))),
        "theta0": loc.theta_zero == ref.theta_zero,
    }
    out[rank] = ok
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 40_000), (3, 100_001)])
def test_sharded_detection_bitwise_equals_single_gpu(cuda, world, n):
    import torch.multiprocessing as mp

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_rank, args=(world, _free_port(), n, 5 + world, out), nprocs=world, join=True)
    want = {"idx": True, "coeffs_bitwise": True, "local_hits": True, "support": True,
            "theta0": True}
    assert dict(out) == {r: want for r in range(world)}


def test_concurrent_threads_bitwise_equal_serial(cuda):
    import torch

    pkg = cuda
    w, G, cfg, smp = _instance(pkg, 30_000, 3)
    sw = workloads.small_sfft(21, 5, 8, 12, r=2)
    sp = pkg.SparsePoly(pkg.FreqSet(sw.d, sw.support, _sorted=True), sw.coeffs)
    box = pkg.Box(sw.d, sw.lo, sw.hi)
    params = pkg.SfftParams(sw.s, 0.9, r=sw.r)

    def job():
        r = pkg.detect_and_compute(smp, cfg, G)
        s = pkg.sfft(pkg.oracle_from_poly(sp), box, params, seed=sw.seed)
        return (r.hits.copy(), r.detected_idx.copy(), r.coeffs.copy(),
                s.support.elems.copy(), s.coeffs.copy(), s.sample_count)

    serial = job()
    results, errors = {}, []

    def worker(k):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                for rep in range(3):
                    results[(k, rep)] = job()
                st.synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
    assert len(results) == 12
    for got in results.values():
        for a, b in zip(got[:5], serial[:5]):
            assert a.dtype == b.dtype and np.array_equal(a.view(np.uint8), b.view(np.uint8))
        assert got[5] == serial[5]
