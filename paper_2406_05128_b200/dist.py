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
