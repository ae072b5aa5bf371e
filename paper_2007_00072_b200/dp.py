"""Data parallelism over the batch ("a mini-batch of samples is partitioned
among many GPUs").

Rank r of N owns global batch rows [r*B_local, (r+1)*B_local) and runs the layer with
batch_offset = r*B_local, so its Philox dropout masks are exactly the slice of the
single-GPU global-batch masks.  The one exchange step is a SUM all-reduce of the
parameter gradients (two contiguous fp32 buckets, FFN first), issued through
torch.distributed (NCCL over NVLink/NVSwitch on the GPU box; gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """(batch_offset, local_batch) of `rank`.  Requires world | global_batch."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    if global_batch % world:
        raise ValueError(f"global batch {global_batch} not divisible by {world} ranks")
    b = global_batch // world
    return rank * b, b


def allreduce_buckets(buckets, group=None, async_op: bool = False):
    """SUM all-reduce of each gradient bucket (a list of flat tensors), in order.
    Returns the work handles when async_op."""
    works = []
    for t in buckets:
        works.append(dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group, async_op=async_op))
    return works if async_op else None


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (used for device timings: the slowest rank)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
