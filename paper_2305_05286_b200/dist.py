"""Multi-GPU BER simulation: frames shard by global frame range, one
all-reduce of the 8 int64 counters per Eb/N0 point.

The channel is keyed by (seed, global frame index), so the summed counters are
identical for every world size (weak or strong scaling alike).  The collective
is torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist


def shard_range(frames: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of global frames owned by `rank` (contiguous, sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or frames < 0:
        raise ValueError("bad shard arguments")
    q, r = divmod(frames, world)
    begin = rank * q + min(rank, r)
    return begin, begin + q + (1 if rank < r else 0)


def allreduce_counts(counts: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the int64[8] counters over all ranks in place (one collective).

    The collective is issued whenever a process group exists -- at world size 1 too, so
    every single-GPU bench run executes the NCCL all-reduce of the multi-GPU path."""
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def ber_sim_sharded(run_shard: Callable[[int, int, torch.Tensor], None], frames: int, frame_offset: int,
                    counts: torch.Tensor, group=None) -> torch.Tensor:
    """Run this rank's slice of [frame_offset, frame_offset + frames) through
    `run_shard(begin, count, counts)` (which accumulates into `counts`), then
    all-reduce.  `counts` lives where the process group's backend expects it."""
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    b, e = shard_range(frames, rank, world)
    if e > b:
        run_shard(frame_offset + b, e - b, counts)
    return allreduce_counts(counts, group)
