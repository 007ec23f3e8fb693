"""torchrun worker for tests/test_gpu_dist.py::test_two_rank_sharded_parity.

Every rank generates only its shard of a seeded config batch (lpgen.make_config_shard),
solves it through the C ABI on the GPU (dist.solve_sharded: contiguous shards, RPC keyed on
the batch index), and rank 0 receives the gathered results.  Rank 0 then solves the WHOLE
batch once more at N=1 (one context, same launch path) and checks the gathered results
against it bit for bit (status, obj, x, iters), and against the oracle on a sample.
Prints one line "PARITY-OK <case>" on success; any mismatch raises.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import lpgen  # noqa: E402
from paper_1609_08114_b200 import dist as lpdist  # noqa: E402
from paper_1609_08114_b200 import lpb  # noqa: E402

CASES = {  # name -> (config, batch, options)
    "G1": ("cfg2", 3001, {}),
    "G2": ("cfg3", 61, {}),
    "cfg2r": ("cfg2r", 1201, {"pivot_rule": "RPC", "rpc_seed": 2}),
    "cfg5": ("cfg5", 200003, {}),
}


def main():
    case = sys.argv[1]
    name, B, opts = CASES[case]
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist.init_process_group(os.environ.get("LPB_DIST_BACKEND", "gloo"))
    world, rank = lpdist.world_rank()
    lo, hi = lpdist.shard_range(B, rank, world)
    hyper = lpgen.CONFIGS[name]["kind"] == "hyperbox"
    if hyper:
        lo_b, hi_b, dirs = lpgen.make_config_shard(name, B, lo, hi)
        A = None
        b = torch.from_numpy(np.concatenate([hi_b, -lo_b])).cuda()
        c = torch.from_numpy(dirs).cuda()
    else:
        A, b, c = (torch.from_numpy(v).cuda() for v in lpgen.make_config_shard(name, B, lo, hi))
    res, ms = lpdist.solve_sharded(A, b, c, B, hyperbox=hyper, **opts)
    assert ms > 0
    if rank == 0:
        got = {k: v.cpu().numpy() for k, v in res.items()}
        # the N = 1 run of the same batch
        if hyper:
            lo_f, hi_f, dirs_f = lpgen.make_config(name, B)
            one = lpb.hyperbox(lo_f, hi_f, torch.from_numpy(dirs_f).cuda())
            keys = ("status", "obj", "x")
        else:
            Af, bf, cf = lpgen.make_config(name, B)
            one = lpb.solve(*(torch.from_numpy(v).cuda() for v in (Af, bf, cf)), **opts)
            keys = ("status", "obj", "x", "iters")
        one = {k: v.cpu().numpy() for k, v in one.items()}
        for k in keys:
            assert got[k].shape == one[k].shape, (k, got[k].shape, one[k].shape)
            assert np.array_equal(got[k], one[k], equal_nan=True), f"{case}: {k} differs from N=1"
        # and the gathered batch against the oracle on a sample (first, last, random)
        import oracle
        from gpu_util import compare
        idx = np.unique(np.concatenate([[0, B - 1, hi - 1, hi],
                                        lpgen.rng(7).integers(0, B, 64)]))
        if hyper:
            o = oracle.hyperbox(lo_f, hi_f, dirs_f[idx])
            assert np.array_equal(got["obj"][idx], o["obj"])
            assert np.array_equal(got["x"][idx], o["x"])
        else:
            rs = [oracle.solve(Af[k:k + 1], bf[k:k + 1], cf[k:k + 1], lp_index_base=int(k), **opts)
                  for k in idx]
            o = {k: np.concatenate([r[k] for r in rs]) for k in ("status", "obj", "x", "iters")}
            compare(Af, bf, cf, got, o, sample=idx)
        print(f"PARITY-OK {case} B={B} world={world}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
