"""Multi-rank fixed-Gamma MERGE logic on CPU: world_size 2 over gloo.

The product path (lattice-sharded DFTs, bitmap and spectra all-gathers,
row-sharded hashing on the device) is tested on the GPU in
tests/test_gpu_shard_threads.py.  Here, with no GPU, each rank runs the CPU
oracle on its contiguous shard (standing in for its device) and merges with
paper_2006_13053_b200.shard.merge_detections; the merged result must equal
the single-process detection exactly (indices) and bitwise (coefficients).
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import port as orc
    from paper_2006_13053_b200.shard import merge_detections, shard_bounds

    w = workloads.config1(seed=11, n=6000, s=15)
    M, z = orc.draw_config(w.gamma, w.s, 0.1, w.rng)
    smp = [orc.sample_lattice_structured(w.gamma[w.support_idx], w.coeffs, zl, M) for zl in z]
    theta0 = orc.zero_threshold(smp)
    lo, hi = shard_bounds(w.gamma.shape[0], world, rank)
    _, idx, co, _ = orc.detect_and_compute(smp, M, z, w.gamma[lo:hi], theta0=theta0)
    gidx, gco = merge_detections(idx, co, lo)
    _, ridx, rco, _ = orc.detect_and_compute(smp, M, z, w.gamma, theta0=theta0)
    out[rank] = (np.array_equal(gidx, ridx) and np.array_equal(gco, rco)
                 and np.array_equal(ridx, w.support_idx))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_detection_equals_single_process(world, oracle_lib):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert dict(out) == {r: True for r in range(world)}


def test_shard_bounds_cover_exactly():
    from paper_2006_13053_b200.shard import shard_bounds

    for n in (0, 1, 7, 1 << 26):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1
