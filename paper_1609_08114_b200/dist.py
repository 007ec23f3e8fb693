"""Batch partitioning over the GPUs of one box (one process per GPU, torch.distributed).

The LPs of a batch are independent (one LP per block), so the
batch is split into contiguous shards, one per rank, and each rank solves its shard with
its own lpb context on its own GPU.  There is NO collective on the data path: the only
communication is (1) an all_reduce(MAX) of the per-rank device time, so the reported time is
the slowest rank's, and (2) an optional gather of the results to rank 0 after the solve.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard of rank r: [floor(r*B/W), floor((r+1)*B/W))."""
    return (B * rank) // world, (B * (rank + 1)) // world


def max_over_ranks(value: float, device=None) -> float:
    """all_reduce(MAX) of a per-rank scalar (e.g. device-timed milliseconds)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_rows(local: torch.Tensor, B: int, dst: int = 0):
    """Gather each rank's contiguous shard (rows [lo, hi) of a length-B batch) to rank `dst`,
    in batch order.  Uneven shards are padded to the largest shard for the collective.
    Returns the full [B, ...] tensor on `dst` and None elsewhere."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [shard_range(B, r, world) for r in range(world)]
    cap = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    if rank != dst:
        return None
    return torch.cat([bufs[r][: hi - lo] for r, (lo, hi) in enumerate(sizes)], dim=0)


def solve_sharded(A, b, c, B: int, *, gather: bool = True, **opts):
    """Solve this rank's shard (device tensors A [b_r, m, n], b [b_r, m], c [b_r, n] holding
    rows shard_range(B, rank, world) of the batch) on the current CUDA device.
    Returns (results_on_rank0_or_local, max_over_ranks_ms)."""
    from . import lpb
    Bl, m, n = A.shape
    world = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank() if world > 1 else 0
    # LP indices of the whole batch key the RPC rule: a sharded run follows the same pivot
    # paths as an unsharded one
    opts.setdefault("lp_index_base", shard_range(B, rank, world)[0])
    s = lpb.Solver(Bl, m, n, lpb.GENERAL, **opts)
    s.solve_device(A, b, c, sync=True)
    ms = max_over_ranks(s.timing()[0], device=A.device)
    res = {k: v.clone() for k, v in s.device_results().items()}
    s.close()
    if gather:
        res = {k: gather_rows(v, B) for k, v in res.items()}
    return res, ms
