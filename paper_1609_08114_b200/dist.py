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


def world_rank() -> tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


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
    lo, hi = sizes[rank]
    if local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} holds {local.shape[0]} rows, its shard is {hi - lo}")
    cap = max(h - l for l, h in sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    if rank != dst:
        return None
    return torch.cat([bufs[r][: h - l] for r, (l, h) in enumerate(sizes)], dim=0)


def _lpb_solve(A, b, c, *, hyperbox, shared, lp_index_base, **opts):
    """This rank's shard through the C ABI (device pointers); returns (results, device ms)."""
    from . import lpb
    Bl, n = c.shape
    if hyperbox:
        s = lpb.Solver(Bl, 2 * n, n, lpb.HYPERBOX, **opts)
        s.solve_device(None, b, c, shared_box=True, sync=True)
    else:
        m = A.shape[-2]
        s = lpb.Solver(Bl, m, n, lpb.GENERAL, lp_index_base=lp_index_base, **opts)
        s.solve_device(A, b, c, shared_ab=shared, sync=True)
    ms = s.timing()[0]
    res = {k: v.clone() for k, v in s.device_results().items()
           if not (hyperbox and k == "iters")}
    s.close()
    return res, ms


def solve_sharded(A, b, c, B: int, *, hyperbox: bool = False, gather: bool = True,
                  solve_fn=None, **opts):
    """Solve this rank's shard and (optionally) gather the batch's results to rank 0.

    A, b, c hold rows shard_range(B, rank, world) of a B-LP batch on the current device:
    general LPs A [b_r, m, n] (or one shared A [m, n] with b [m]), b [b_r, m], c [b_r, n];
    hyperbox: A None, b the shared box [hi; -lo] (2n), c the directions [b_r, n].
    The RPC rule keys on each LP's index in the whole batch (lp_index_base = the shard's
    first index), so a sharded run follows exactly the pivot paths of an unsharded one.
    ``solve_fn(A, b, c, hyperbox=, shared=, lp_index_base=, **opts) -> (results, ms)``
    replaces the C-ABI solve (CPU tests of the partition / gather logic only).
    Returns (results: dict of [B, ...] tensors on rank 0 -- None elsewhere -- or this rank's
    shard when gather=False, max-over-ranks device milliseconds)."""
    world, rank = world_rank()
    lo, hi = shard_range(B, rank, world)
    if c.shape[0] != hi - lo:
        raise ValueError(f"rank {rank}: c has {c.shape[0]} rows, shard [{lo}, {hi}) expected")
    shared = (not hyperbox) and A is not None and A.dim() == 2
    fn = solve_fn or _lpb_solve
    res, ms = fn(A, b, c, hyperbox=hyperbox, shared=shared, lp_index_base=lo, **opts)
    ms = max_over_ranks(ms, device=c.device if c.is_cuda else None)
    if gather:
        out = {k: gather_rows(v, B) for k, v in res.items()}
        res = out if rank == 0 else None
    return res, ms
