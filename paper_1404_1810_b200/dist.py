"""Multi-GPU plumbing (one process per GPU, torch.distributed).

Batched AM-QFT workloads shard by rows with no data-path collective: rank r
owns rows [start, start + count) of the global batch, runs its own plan on
its own device, and only the timing (max over ranks) and optional result
gathering use the process group.  The fused single-transform four-step
over NCCL is not part of round 1.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import FunctionId, Order, Plan


def shard_rows(total_rows: int, world: int, rank: int):
    """Contiguous, balanced row range of `rank` (first ranks take the
    remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(int(total_rows), int(world))
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank scalar (timing)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, total_rows: int):
    """Gather every rank's shard (rows) into the full batch on every rank
    (shards are padded to the largest one for the collective)."""
    world = dist.get_world_size()
    counts = [shard_rows(total_rows, world, r)[1] for r in range(world)]
    cmax = max(counts)
    pad = torch.zeros((cmax,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: counts[r]] for r in range(world)], dim=0)


class ShardedPlan:
    """One Plan per rank over its row shard (weak or strong scaling is the
    caller's choice of total_rows)."""

    def __init__(self, variant: int, n: int, total_rows: int, *, dtype="f32", order=Order.Fast,
                 device: int = 0):
        world = dist.get_world_size() if dist.is_initialized() else 1
        rank = dist.get_rank() if dist.is_initialized() else 0
        self.start, self.rows = shard_rows(total_rows, world, rank)
        self.plan = Plan(variant, FunctionId.Cdft, n, max(1, self.rows), dtype=dtype, order=order,
                         device=device)

    def forward(self, local_in, local_out, stream=None):
        if self.rows:
            self.plan.forward(local_in, local_out, rows=self.rows, stream=stream)
