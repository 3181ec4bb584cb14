"""Host-side logic of the M-sharded multi-GPU path (one process per GPU).

The GEMM needs no collective: rank r owns rows [row_start[r], row_start[r+1]) of A and C,
B is replicated.  torch.distributed is plumbing only: the barrier and max-over-ranks of the
timed region, and an optional gather of the row-major C shards (a pure concatenation).
These helpers are shared by bench.py and the world-size-2 gloo tests (tests/test_multi_cpu.py).
"""
from __future__ import annotations

from . import api


def row_block(m: int, rank: int, world: int, align: int = 128):
    """Contiguous, tile-aligned row block of this rank (C-ABI ngemm_cuda_shard_rows)."""
    rs = api.shard_rows(m, world, align)
    return rs[rank], rs[rank + 1]


def reduce_max(x: float, world: int, device=None) -> float:
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(x: float, world: int, device=None) -> float:
    if world == 1:
        return float(x)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_rows(c_local, m: int, world: int, align: int = 128):
    """Assemble the full row-major C [m x n] on every rank from the ragged row shards
    (padded all_gather of equal-size blocks, then trimmed and concatenated)."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return c_local
    rs = api.shard_rows(m, world, align)
    rows = max(rs[i + 1] - rs[i] for i in range(world))
    n = c_local.shape[1]
    pad = torch.zeros((rows, n), dtype=c_local.dtype, device=c_local.device)
    pad[: c_local.shape[0]] = c_local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([bufs[i][: rs[i + 1] - rs[i]] for i in range(world)], dim=0)
