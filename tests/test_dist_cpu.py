"""Multi-process (world_size 2, gloo, CPU) tests of the batch-sharding path.

The GPU kernels are not involved: each rank runs the CPU oracle on its shard,
which checks the plumbing the multi-GPU bench relies on -- disjoint shards
covering the global batch, the max-over-ranks time, and that sharded results
equal the single-process results item for item (no cross-item dependence).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2406_05128_b200 import data
from paper_2406_05128_b200 import dist as pdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, B, T, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    d = pdist.init("gloo")
    lo, hi = pdist.shard(B, rank)
    e, A, g = data.d1_batch(lo, hi - lo, T, 22)
    s, ge, gA = oracle.batch_fwd_bwd("tv", e, A, g, nthreads=1)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), lo=lo, hi=hi, s=s, ge=ge, gA=gA)
    t = pdist.max_over_ranks(1.0 + rank, d)
    n = pdist.sum_over_ranks(hi - lo, d)
    np.savez(os.path.join(outdir, f"t{rank}.npz"), t=t, n=n)
    d.barrier()
    d.destroy_process_group()


def test_world2_batch_sharding(tmp_path):
    world, B, T = 2, 3, 960
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, B, T, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    e, A, g = data.d1_batch(0, world * B, T, 22)
    s, ge, gA = oracle.batch_fwd_bwd("tv", e, A, g, nthreads=1)
    covered = []
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        lo, hi = int(z["lo"]), int(z["hi"])
        covered += list(range(lo, hi))
        np.testing.assert_array_equal(z["s"], s[lo:hi])
        np.testing.assert_array_equal(z["ge"], ge[lo:hi])
        np.testing.assert_array_equal(z["gA"], gA[lo:hi])
        tz = np.load(tmp_path / f"t{r}.npz")
        assert float(tz["t"]) == 2.0  # max over ranks
        assert float(tz["n"]) == world * B
    assert covered == list(range(world * B))


def test_strong_shard_partition():
    for B in (1, 7, 64, 256):
        for world in (1, 2, 4, 8):
            parts = [pdist.strong_shard(B, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == B
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
