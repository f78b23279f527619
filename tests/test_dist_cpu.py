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


def test_bench_shard_plans():
    """bench.py's split: config 3 strong (global 64 over 1/2/4/8 ranks, disjoint
    and covering, B_global = 64 on every rank), the one-GPU --shard-of probe
    (rank 0's share, reported as its own global batch), weak (64 per rank)."""
    for world in (1, 2, 4, 8):
        got = [pdist.bench_shard(64, "strong", r, world) for r in range(world)]
        assert [lo for lo, _, _ in got] == [64 * r // world for r in range(world)]
        assert sum(n for _, n, _ in got) == 64 and all(g == 64 for _, _, g in got)
        weak = [pdist.bench_shard(64, "weak", r, world) for r in range(world)]
        assert [(lo, n, g) for lo, n, g in weak] == [(64 * r, 64, 64 * world)
                                                      for r in range(world)]
    for s in (2, 4, 8):
        assert pdist.bench_shard(64, "strong", 0, 1, shard_of=s) == (0, 64 // s, 64 // s)


def _allreduce_worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    d = pdist.init("gloo")
    grad = torch.full((1 << 20,), float(rank + 1))
    e, A, g = data.d1_batch(10 + rank, 1, 2000, 22)

    def work():  # the rank's LP backward stands in as the overlapped work
        s = oracle.lp_forward_tv(e[0].astype(np.float64), A[0].astype(np.float64))
        return oracle.lp_backward_tv(g[0].astype(np.float64), A[0].astype(np.float64), s)

    ge, gA = pdist.overlapped_allreduce(grad, d, work)
    s = oracle.lp_forward_tv(e[0].astype(np.float64), A[0].astype(np.float64))
    ge2, gA2 = oracle.lp_backward_tv(g[0].astype(np.float64), A[0].astype(np.float64), s)
    np.savez(os.path.join(outdir, f"a{rank}.npz"), grad=grad[:8].numpy(),
             same=np.array_equal(ge, ge2) and np.array_equal(gA, gA2))
    d.barrier()
    d.destroy_process_group()


def test_world2_hpn_allreduce_overlap(tmp_path):
    """The HpN step's encoder all-reduce (bench hpn config) runs asynchronously
    around the rank's backward: the reduced gradient is the sum over ranks and
    the overlapped work's result is unchanged."""
    world = 2
    port = _free_port()
    mp.start_processes(_allreduce_worker, args=(world, port, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    for r in range(world):
        z = np.load(tmp_path / f"a{r}.npz")
        assert np.all(z["grad"] == 3.0)  # 1 + 2
        assert bool(z["same"])
    assert pdist.overlapped_allreduce(None, None, lambda: 7) == 7


# ---------------------------------------------------------------- one sequence split in time
class _NumpySegments:
    """Segment primitives of longseq.py restated in numpy on the oracle (CPU),
    so the exchange and its fold can run on a gloo world without a GPU."""

    def forward(self, e, A, zi, tape=None):
        s = np.stack([oracle.lp_forward_tv(e[b].numpy(), A[b].numpy(),
                                           None if zi is None else zi[b].numpy())
                      for b in range(e.shape[0])])
        return torch.from_numpy(s), (A, e)

    def transition(self, tape, B, T, M, dtype, device):
        A, _ = tape
        Phi = np.zeros((B, M, M))
        for b in range(B):
            for k in range(M):
                zi = np.zeros(M)
                zi[k] = 1.0
                s = oracle.lp_forward_tv(np.zeros(T), A[b].numpy(), zi)
                Phi[b, :, k] = s[::-1][:M]
        return torch.from_numpy(Phi)

    def backward(self, g, A, s, zi, tape, mu_in):
        B, T = g.shape
        M = A.shape[-1]
        ge = np.zeros((B, T))
        gA = np.zeros((B, T, M))
        nu = np.zeros((B, M))
        for b in range(B):
            a = A[b].numpy()
            lam = np.zeros(M) if mu_in is None else mu_in[b].numpy().copy()
            for t in range(T - 1, -1, -1):  # transposed-state adjoint (k_adjoint)
                l0 = lam[0] + g[b, t].item()
                ge[b, t] = l0
                new = np.empty(M)
                new[:-1] = -a[t, :-1] * l0 + lam[1:]
                new[-1] = -a[t, -1] * l0
                lam = new
            nu[b] = lam
            sb = s[b].numpy()
            z = np.zeros(M) if zi is None else zi[b].numpy()
            for t in range(T):
                for c in range(M):
                    u = t - 1 - c
                    gA[b, t, c] = -ge[b, t] * (sb[u] if u >= 0 else z[-u - 1])
        return torch.from_numpy(ge), torch.from_numpy(gA), torch.from_numpy(nu)


def _split_worker(rank, world, port, outdir):
    from paper_2406_05128_b200 import longseq

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo")
    e, A, g = data.d1_batch(77, 2, 3 * 40, 3, hop=17, dtype=np.float64)
    zi = np.array([[0.3, -0.2, 0.1], [0.0, 0.5, -0.4]])
    seg = slice(rank * 40, (rank + 1) * 40)
    eng = _NumpySegments()
    s, ctx = longseq.lp_tv_forward_split(torch.from_numpy(e[:, seg].copy()),
                                         torch.from_numpy(A[:, seg].copy()),
                                         torch.from_numpy(zi), engine=eng)
    ge, gA = longseq.lp_tv_backward_split(torch.from_numpy(g[:, seg].copy()),
                                          torch.from_numpy(A[:, seg].copy()), s, ctx, engine=eng)
    np.savez(os.path.join(outdir, f"split{rank}.npz"), s=s.numpy(), ge=ge.numpy(), gA=gA.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_world3_time_split_exchange(tmp_path):
    """SURVEY.md §8(e) exchange step on a gloo world of 3: one all_gather of
    (Phi, end state) forward and of the boundary adjoints backward gives every
    rank its exact segment of the whole-sequence result."""
    world = 3
    port = _free_port()
    mp.start_processes(_split_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    e, A, g = data.d1_batch(77, 2, 3 * 40, 3, hop=17, dtype=np.float64)
    zi = np.array([[0.3, -0.2, 0.1], [0.0, 0.5, -0.4]])
    parts = [np.load(tmp_path / f"split{r}.npz") for r in range(world)]
    s = np.concatenate([p["s"] for p in parts], 1)
    ge = np.concatenate([p["ge"] for p in parts], 1)
    gA = np.concatenate([p["gA"] for p in parts], 1)
    for b in range(2):
        rs = oracle.lp_forward_tv(e[b], A[b], zi[b])
        rge, rgA = oracle.lp_backward_tv(g[b], A[b], rs, zi[b])
        np.testing.assert_allclose(s[b], rs, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(ge[b], rge, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(gA[b], rgA, rtol=1e-10, atol=1e-12)
