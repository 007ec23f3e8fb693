"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times (device
pointers, auto size class): the whole batch runs on the GPU and the oracle checks
  - every LP of cfg1, cfg2 (50,000 x 100x100: ~8 s of oracle time), cfg4 and cfg5;
  - 1,000 LPs of cfg3 (10,000 x 200x200 two-phase: ~35 s); the whole cfg3 batch (~6 min of
    oracle time) runs with LPB_SLOW=1 (test_cfg3_full, marked slow).
North star (BASELINE.json): all five configs matching the CPU oracle; SURVEY.md §8(d)."""
import os

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


def _residuals_all(A, b, x):
    """Absolute primal residual max(0, max_i(A_i x - b_i), max_j(-x_j)) of every LP (fp64
    einsum over the batch; C20)."""
    r = np.einsum("bij,bj->bi", A, x) - b
    return np.maximum(0.0, np.maximum(r.max(axis=1), (-x).max(axis=1)))


def _check_residuals(A, b, x, tol=1e-9):
    """the absolute primal residual <= tol, else (fp64 drift after thousands of
    pivots, identical in the oracle since the bits match) the scaled residual
    max_i (A_i x - b_i) / max(1, |b_i|, sum_j |a_ij x_j|) <= tol, computed in long double.
    Returns (max absolute residual, number of LPs graded on the scaled form)."""
    from checks import scaled_primal_residual
    res = np.concatenate([_residuals_all(A[i:i + 1000], b[i:i + 1000], x[i:i + 1000])
                          for i in range(0, A.shape[0], 1000)])
    over = np.nonzero(res > tol)[0]
    for k in over:
        assert scaled_primal_residual(A[k], b[k], x[k]) <= tol, (k, res[k])
    return res.max(), over.size


def test_cfg2_full():
    """All 50,000 LPs of cfg2 (PAPER.md:230's workload) against the oracle, element by
    element: status, iteration counts, objective bits and x bits; residual of every LP."""
    A, b, c = lpgen.make_config("cfg2")
    g = gpu_solve(A, b, c)
    o = oracle.solve(A, b, c)
    compare(A, b, c, g, o)
    assert np.all(g["status"] == 0)
    rmax, nscaled = _check_residuals(A, b, g["x"])
    assert nscaled == 0, rmax  # G1 100x100: absolute residuals ~1e-12


@pytest.mark.parametrize("name,sample", [("cfg3", 1000)])
def test_general_full_size_sampled(name, sample):
    A, b, c = lpgen.make_config(name)
    g = gpu_solve(A, b, c)
    B = A.shape[0]
    idx = np.unique(np.concatenate([[0, B - 1], lpgen.rng(99).integers(0, B, sample)]))
    o = oracle.solve(A[idx], b[idx], c[idx])
    compare(A, b, c, g, o, sample=idx)
    assert np.all(g["status"] == 0)  # G1 / G2 are feasible and bounded by construction


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("LPB_SLOW") != "1", reason="~6 min of oracle time: LPB_SLOW=1")
def test_cfg3_full():
    """All 10,000 LPs of cfg3 (PAPER.md:253's two-phase workload) against the oracle."""
    A, b, c = lpgen.make_config("cfg3")
    g = gpu_solve(A, b, c)
    o = oracle.solve(A, b, c)
    compare(A, b, c, g, o)
    assert np.all(g["status"] == 0)
    rmax, nscaled = _check_residuals(A, b, g["x"])
    print(f"cfg3 full: {A.shape[0]} LPs bit-exact vs the oracle; max abs residual {rmax:.3e}; "
          f"{nscaled} LP(s) graded on the scaled residual (C20)")


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

