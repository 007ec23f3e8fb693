"""Multi-process host logic of the batch partitioning (gloo, world size 2, CPU): shards cover
the batch exactly once and in order, the MAX timing reduction, and the padded gather that
reassembles uneven shards in batch order."""
import os
import socket

import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, B, q):
    import torch.distributed as dist

    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "lpb_dist", os.path.join(root, "paper_1609_08114_b200", "dist.py"))
    d = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(d)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = d.shard_range(B, rank, world)
    local = torch.arange(lo, hi, dtype=torch.float64)[:, None].repeat(1, 3)
    full = d.gather_rows(local, B)
    mx = d.max_over_ranks(10.0 + rank)
    if rank == 0:
        q.put((full.tolist(), mx))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("B", [7, 10, 1])
def test_gather_and_max_world2(B):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    full, mx = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert mx == 11.0
    assert [row[0] for row in full] == list(range(B))


def test_shard_range_partitions():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "lpb_dist", os.path.join(root, "paper_1609_08114_b200", "dist.py"))
    d = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(d)
    for B in (1, 7, 50000, 6003000):
        for W in (1, 2, 3, 4, 8):
            rs = [d.shard_range(B, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))
            assert max(h - l for l, h in rs) - min(h - l for l, h in rs) <= 1


# ---- solve_sharded end to end on CPU: shard -> per-rank solve -> gather == one N=1 solve ----

def _oracle_solve_fn(A, b, c, *, hyperbox, shared, lp_index_base, **opts):
    """Stands in for the C-ABI solve in the CPU test (the oracle on this rank's shard)."""
    import numpy as np

    import oracle
    if hyperbox:
        n = c.shape[1]
        box = b.numpy()
        r = oracle.hyperbox(-box[n:], box[:n], c.numpy())
        return {k: torch.from_numpy(np.ascontiguousarray(r[k])) for k in ("status", "obj", "x")}, 1.0
    An, bn = A.numpy(), b.numpy()
    if shared:
        B = c.shape[0]
        An = np.ascontiguousarray(np.broadcast_to(An, (B,) + An.shape))
        bn = np.ascontiguousarray(np.broadcast_to(bn, (B,) + bn.shape))
    r = oracle.solve(An, bn, c.numpy(), lp_index_base=lp_index_base, **opts)
    return {k: torch.from_numpy(r[k]) for k in ("status", "obj", "x", "iters")}, 1.0 + lp_index_base


def _sharded_worker(rank, world, port, case, q):
    import importlib.util

    import torch.distributed as dist

    import lpgen
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location(
        "lpb_dist", os.path.join(root, "paper_1609_08114_b200", "dist.py"))
    d = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(d)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name, B, opts = case
    lo, hi = d.shard_range(B, rank, world)
    hyper = lpgen.CONFIGS[name]["kind"] == "hyperbox"
    if hyper:
        lo_b, hi_b, dirs = lpgen.make_config_shard(name, B, lo, hi)
        import numpy as np
        A, b, c = None, torch.from_numpy(np.concatenate([hi_b, -lo_b])), torch.from_numpy(dirs)
    else:
        A, b, c = (torch.from_numpy(v) for v in lpgen.make_config_shard(name, B, lo, hi))
    res, ms = d.solve_sharded(A, b, c, B, hyperbox=hyper, solve_fn=_oracle_solve_fn, **opts)
    if rank == 0:
        q.put(({k: v.numpy() for k, v in res.items()}, ms))
    else:
        assert res is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", [
    ("cfg2", 37, {}),                                   # G1 type-1, uneven shards
    ("cfg3", 5, {}),                                    # G2 two-phase, 200x200
    ("cfg2r", 21, {"pivot_rule": "RPC", "rpc_seed": 2}),  # RPC keyed on the batch index
    ("cfg2s", 30, {}),                                  # shared A/b (NEXT-1)
    ("cfg4", 1001, {}),                                 # hyperbox
])
def test_solve_sharded_equals_unsharded_world2(case):
    """shard + per-rank solve + gather reproduces the N=1 results
    bit for bit (status, obj, x, iters) and the reported time is the MAX over ranks."""
    import numpy as np

    import lpgen
    import oracle
    name, B, opts = case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, ms = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if lpgen.CONFIGS[name]["kind"] == "hyperbox":
        lo, hi, dirs = lpgen.make_config(name, B)
        ref = oracle.hyperbox(lo, hi, dirs)
        keys = ("status", "obj", "x")
        assert ms == 1.0
    else:
        A, b, c = lpgen.make_config(name, B)
        if A.ndim == 2:
            A = np.ascontiguousarray(np.broadcast_to(A, (B,) + A.shape))
            b = np.ascontiguousarray(np.broadcast_to(b, (B,) + b.shape))
        ref = oracle.solve(A, b, c, **opts)
        keys = ("status", "obj", "x", "iters")
        assert ms == 1.0 + B // 2  # rank 1's "time" (1 + its lp_index_base) is the max
    for k in keys:
        assert got[k].shape == ref[k].shape, k
        assert np.array_equal(got[k], ref[k], equal_nan=True), k
