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


PATTERNS = {"rms_ffn_swiglu": 0, "layernorm_matmul": 1, "attention": 2}


def shard_range(pattern: str, units: int, world: int, rank: int) -> tuple[int, int]:
    """The C-ABI's shard boundaries (bf_shard_range): 128-row aligned rows, whole heads."""
    import ctypes

    from . import _lib

    a, b = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(_lib.lib().bf_shard_range(PATTERNS[pattern], units, world, rank, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def launch_sharded(pattern: str, shards: list[dict], dims, eps_or_scale: float = 0.0, schedule: str = "fused",
                   gather: bool = False) -> None:
    """One host thread, N devices: bf_launch_sharded over per-device shards.

    Each shard is {"device": int, "inputs": [tensors on that device], "out": tensor,
    "out_full": tensor or None}; `dims` are the whole problem's (rms_ffn_swiglu: M, D, F, N;
    layernorm_matmul: M, K, N; attention: BH, Sq, Skv, D, Dv). With gather=True every
    out_full receives the whole output (NCCL all-gather-v over NVLink, or peer copies).
    Streams are each device's current torch stream."""
    import ctypes

    import torch

    from . import _lib
    from .ops import _dtype_code

    L = _lib.lib()
    pid = PATTERNS[pattern]
    ios = (_lib.ShardIO * len(shards))()
    keep = []
    dtype = _dtype_code(shards[0]["inputs"][0])
    for g, sh in enumerate(shards):
        dev = torch.device("cuda", sh["device"])
        lo, hi = shard_range(pattern, int(dims[0]), len(shards), g)
        n = hi - lo
        io = ios[g]
        io.device = sh["device"]
        for i, t in enumerate(sh["inputs"]):
            io.in_[i] = t.data_ptr()
        io.out = sh["out"].data_ptr()
        io.out_full = sh["out_full"].data_ptr() if sh.get("out_full") is not None else None
        if pid == 0:
            ws_bytes = L.bf_rms_ffn_swiglu_workspace_bytes(max(n, 1), dims[1], dims[2], dims[3], dtype,
                                                           0 if schedule == "fused" else 1)
        elif pid == 1:
            ws_bytes = L.bf_layernorm_matmul_workspace_bytes(max(n, 1), dims[1], dims[2], dtype)
        else:
            ws_bytes = 256
        ws = torch.empty(max(int(ws_bytes), 256), dtype=torch.uint8, device=dev)
        keep.append(ws)
        io.workspace = ws.data_ptr()
        io.workspace_bytes = ws.numel()
        io.stream = torch.cuda.current_stream(dev).cuda_stream
    arr = (ctypes.c_int64 * len(dims))(*[int(d) for d in dims])
    _lib.check(L.bf_launch_sharded(pid, len(shards), ios, arr, len(dims), dtype, 0 if schedule == "fused" else 1,
                                   float(eps_or_scale), 1 if gather else 0))
    # the workspaces must outlive the kernels: tie them to each device's stream
    for sh, ws in zip(shards, keep):
        ws.record_stream(torch.cuda.current_stream(torch.device("cuda", sh["device"])))
