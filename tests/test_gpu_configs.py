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
