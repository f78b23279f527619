"""Multi-GPU plumbing for the LP path: one process per GPU, batch sharding.

The LP filter has no cross-item dependence (items are independent
sequences), so N GPUs each filter their own shard of the batch with no
collective in the filter itself.  torch.distributed (NCCL on
GPUs, gloo in the CPU tests) carries only the barrier around the timed region,
the max-over-ranks reduction of the measured time, and -- for the HpN config
-- the encoder-gradient all-reduce stand-in.
"""
from __future__ import annotations

import os

import torch


def env_rank_world():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def init(backend=None):
    """Initialise the default process group from torchrun's environment."""
    import torch.distributed as dist

    rank, world = env_rank_world()
    if world <= 1:
        return None
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if not dist.is_initialized():
        dist.init_process_group(backend)
    return dist


def shard(B_per_rank, rank):
    """Weak scaling: rank r owns global items [r*B, (r+1)*B); item i uses seed i."""
    return rank * B_per_rank, (rank + 1) * B_per_rank


def strong_shard(B_total, rank, world):
    """Strong scaling: a fixed global batch split as evenly as possible."""
    lo = B_total * rank // world
    hi = B_total * (rank + 1) // world
    return lo, hi


def bench_shard(B_cfg, scaling, rank, world, shard_of=0):
    """The bench's batch split (bench.py): returns (lo, B_local, B_global).
    strong -- a fixed global batch B_cfg over the ranks (BASELINE.json config 3:
    64 items over 1/2/4/8 GPUs); with world == 1 and shard_of > 1, rank 0's
    share of a shard_of-way split (a one-GPU probe of the per-GPU regime:
    B_global is then that share).  weak -- B_cfg items per rank."""
    if scaling == "strong":
        parts = shard_of if (world == 1 and shard_of > 1) else world
        lo, hi = strong_shard(B_cfg, rank, parts)
        return lo, hi - lo, (B_cfg if parts == world else hi - lo)
    lo, hi = shard(B_cfg, rank)
    return lo, B_cfg, B_cfg * world


def overlapped_allreduce(grad, dist, work):
    """The HpN step's encoder-gradient all-reduce issued
    asynchronously, ``work()`` (the LP backward) run while it is in flight,
    then joined; returns work()'s result.  dist None: just work()."""
    if dist is None:
        return work()
    handle = dist.all_reduce(grad, async_op=True)
    out = work()
    handle.wait()
    return out


def max_over_ranks(value, dist, device=None):
    """The timed value of a multi-rank run is the slowest rank's."""
    if dist is None:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value, dist, device=None):
    if dist is None:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())
