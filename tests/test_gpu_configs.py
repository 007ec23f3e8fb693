"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (device
pointers, auto size class): the whole batch runs on the GPU; the oracle checks a sample of
LPs one by one (cfg2, cfg3), or the whole batch where it is cheap (cfg1, cfg4, cfg5)."""
import numpy as np
import pytest

import lpgen
import oracle
from gpu_util import compare, gpu_solve

pytestmark = pytest.mark.gpu


def test_cfg1_full():
    A, b, c = lpgen.make_config("cfg1")
    o = oracle.solve(A, b, c)
    g = gpu_solve(A, b, c)
    compare(A, b, c, g, o)


@pytest.mark.parametrize("name,sample", [("cfg2", 600), ("cfg3", 12)])
def test_general_full_size_sampled(name, sample):
    A, b, c = lpgen.make_config(name)
    g = gpu_solve(A, b, c)
    B = A.shape[0]
    idx = np.unique(np.concatenate([[0, B - 1], lpgen.rng(99).integers(0, B, sample)]))
    o = oracle.solve(A[idx], b[idx], c[idx])
    compare(A, b, c, g, o, sample=idx)
    assert np.all(g["status"] == 0)  # G1 / G2 are feasible and bounded by construction


@pytest.mark.parametrize("name", ["cfg4", "cfg5"])
def test_hyperbox_full_size(name):
    import torch

    from paper_1609_08114_b200 import lpb
    lo, hi, dirs = lpgen.make_config(name)
    o = oracle.hyperbox(lo, hi, dirs)
    g = lpb.hyperbox(lo, hi, torch.from_numpy(dirs).cuda())
    assert np.array_equal(g["status"].cpu().numpy(), o["status"])
    assert np.array_equal(g["obj"].cpu().numpy(), o["obj"])
    assert np.array_equal(g["x"].cpu().numpy(), o["x"])


@pytest.mark.parametrize("name,sample", [("cfg2r", 300), ("cfg2s", 300), ("cfg3s", 8),
                                         ("cfg6", 24), ("cfg7", 4), ("cfg8", 4),
                                         ("cfg9", 600), ("cfg10", 300),
                                         ("cfg1m", 3000)])
def test_next_rows_full_size_sampled(name, sample):
    """The §8(f) rows' bench configs at full size in bench.py's launch configuration (device
    pointers, auto size class, the config's entering rule; shared configs use LPB_SHARED_AB
    and, for two-phase, the phase-I warm start), checked against the oracle on a sample."""
    import bench
    cfg = lpgen.CONFIGS[name]
    A, b, c = lpgen.make_config(name)
    opts = bench.rule_opts(name)
    g = gpu_solve(A, b, c, **opts)
    B = c.shape[0]
    idx = np.unique(np.concatenate([[0, B - 1], lpgen.rng(98).integers(0, B, sample)]))
    if A.ndim == 2:  # shared constraints: broadcast the sample's A and b
        As = np.ascontiguousarray(np.broadcast_to(A, (len(idx),) + A.shape))
        bs = np.ascontiguousarray(np.broadcast_to(b, (len(idx),) + b.shape))
        Af = np.broadcast_to(A, (B,) + A.shape)
        bf = np.broadcast_to(b, (B,) + b.shape)
    else:
        As, bs, Af, bf = A[idx], b[idx], A, b
    if opts:  # RPC keys on the LP's batch index: the oracle solves each sample at its index
        rs = [oracle.solve(As[t:t + 1], bs[t:t + 1], c[k:k + 1], lp_index_base=int(k), **opts)
              for t, k in enumerate(idx)]
        o = {key: np.concatenate([r[key] for r in rs]) for key in ("status", "obj", "x", "iters")}
    else:
        o = oracle.solve(As, bs, c[idx])
    compare(Af, bf, c, g, o, sample=idx)
    assert np.all(g["status"] == 0)
    assert cfg["B"] == B

