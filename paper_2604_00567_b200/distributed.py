"""Batch partitioner: independent transforms sharded over GPUs, no collectives.

SURVEY.md 8(e): a batched FFT exchanges nothing between transforms, so each
device (one process per GPU under torchrun, or one host thread per device in
``dsfft_execute_multi``) takes a contiguous range of the batch,
[rank*B/W, (rank+1)*B/W), with its own replicated plan (plans are immutable
and shareable, fft.hpp:14-16).  The only communication is control-plane: a
barrier around the timed region and a MAX of the per-rank CUDA-event times
(the job's step time is its slowest rank).

Two ways to grow the job with the GPU count (bench.py):
  * strong scaling -- one global batch (BASELINE configs[3]: 2^20 transforms)
    split by ``shard_range``;
  * weak scaling -- a fixed per-GPU batch; rank r owns global transforms
    [r*B, (r+1)*B).
Either way a rank generates its inputs on its own GPU from the global
transform index (``dsfft_fill_uniform``), so every shard is bit-identical to
the same rows of a 1-GPU run.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Tuple


def shard_range(batch: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, stop) of `batch` transforms owned by `rank`.

    Shards differ in size by at most one transform."""
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
    """Control-plane MAX over ranks (identity when not distributed).  NCCL
    reduces device tensors: pass the rank's device; gloo uses the CPU."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64,
                     device=device if device is not None else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


@dataclass
class Shard:
    """This rank's part of a sharded batched transform."""
    start: int          # first global transform index
    stop: int
    x: object           # [stop-start, n, 2] input on the rank's GPU
    y: object           # output buffer of the same shape

    @property
    def count(self) -> int:
        return self.stop - self.start


def make_shard(plan, rank: int, world: int, seed: int, global_batch: int = None,
               per_rank_batch: int = None) -> Shard:
    """Allocate and fill this rank's shard on the plan's device.

    Exactly one of `global_batch` (strong scaling: shard_range of it) and
    `per_rank_batch` (weak scaling: rank r owns [r*B, (r+1)*B)) is given."""
    import torch

    from . import synthetic_batch
    if (global_batch is None) == (per_rank_batch is None):
        raise ValueError("give exactly one of global_batch / per_rank_batch")
    if global_batch is not None:
        start, stop = shard_range(global_batch, rank, world)
    else:
        start, stop = rank * per_rank_batch, (rank + 1) * per_rank_batch
    x = synthetic_batch(plan.n, start, stop - start, seed, plan.precision, device=plan.device)
    return Shard(start, stop, x, torch.empty_like(x))


def sharded_forward(plan, shard: Shard, stream=None, inverse: bool = False) -> Shard:
    """Transform this rank's shard in place of its output buffer (nothing
    crosses devices)."""
    from . import execute
    if shard.count:
        execute(plan, 1 if inverse else 0, shard.x, out=shard.y, stream=stream)
    return shard
