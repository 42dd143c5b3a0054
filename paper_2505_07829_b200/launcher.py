"""Row/head-sharded multi-GPU launcher (one process per GPU, torch.distributed plumbing).

The fused programs shard without any exchange step: token
rows are independent for K1/K2 (statistics are per row) and heads are
independent for K3. Each rank runs the same C-ABI entry point on its own
contiguous shard; NCCL is used only for barriers, the max-over-ranks timing
reduction and an optional all-gather of the row-sharded output.
"""
from __future__ import annotations

import os
from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int
    stop: int

    @property
    def size(self) -> int:
        return self.stop - self.start


def shard(total: int, rank: int, world: int, align: int = 1) -> Shard:
    """Contiguous shard of `total` units for `rank`; shard boundaries are multiples of
    `align` (e.g. 128-row tiles) except the last, and sizes differ by at most one align unit."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    units = (total + align - 1) // align
    lo = units * rank // world
    hi = units * (rank + 1) // world
    return Shard(rank, world, min(total, lo * align), min(total, hi * align))


def env_rank() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (device time) across the process group."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local, shards: list[Shard]):
    """All-gather row-sharded outputs (optional; not on the kernel data path)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return local
    width = local.shape[1:]
    biggest = max(s.size for s in shards)
    padded = torch.zeros((biggest, *width), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in shards]
    dist.all_gather(parts, padded)
    return torch.cat([p[: s.size] for p, s in zip(parts, shards)], dim=0)
