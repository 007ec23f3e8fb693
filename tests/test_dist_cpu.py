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
