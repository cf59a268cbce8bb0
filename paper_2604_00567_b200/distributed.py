"""Batch partitioner: independent transforms sharded over GPUs, no collectives.

SURVEY.md 8(e): a batched FFT exchanges nothing between transforms, so each
device (one process per GPU under torchrun, or one host thread per device in
``dsfft_execute_multi``) takes a contiguous range of the batch,
[rank*B/W, (rank+1)*B/W), with its own replicated plan.  The only
communication is control-plane: a barrier around the timed region and a MAX
of the per-rank CUDA-event times (the job's step time is its slowest rank).
"""
from __future__ import annotations

import os
from typing import Tuple


def shard_range(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) of `batch` transforms owned by `rank`.

    Shards differ in size by at most one transform; for fp16 pair-packed
    kernels an even split keeps whole pairs on each device when possible."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    if batch < 0:
        raise ValueError("batch must be >= 0")
    return batch * rank // world, batch * (rank + 1) // world


def env_rank() -> Tuple[int, int, int]:
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device=None) -> float:
    """Control-plane MAX over ranks (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sharded_forward(plan, x_global, rank: int, world: int, inverse: bool = False):
    """Transform this rank's shard of a global batch held on this rank's GPU
    (x_global[start:stop] is a view; nothing crosses devices)."""
    from . import execute
    start, stop = shard_range(x_global.shape[0], rank, world)
    if stop == start:
        return x_global[start:stop]
    return execute(plan, 1 if inverse else 0, x_global[start:stop].contiguous())
