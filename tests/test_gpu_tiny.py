"""GPU parity of the tiny-LP layouts against the oracle, element by element: the S class's
register kernel (csrc/simplex_tiny.cu: one LP per thread, a type-1 LP of m, n <= 6 in
registers, two-phase LPs deferred to the SMEM-slice kernel in list mode; also bit-identical
to the SMEM-slice kernel alone, LPB_NO_TINY) and the W class's element layout
(csrc/simplex_warp.cu, type-1 LPs up to 7 x 7)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import lpgen
import oracle
from gpu_util import compare, gpu_solve

pytestmark = pytest.mark.gpu

SHAPES = [(1, 1), (1, 6), (6, 1), (2, 3), (3, 3), (4, 4), (4, 6), (5, 5), (6, 4), (6, 6)]


@pytest.mark.parametrize("m,n", SHAPES)
@pytest.mark.parametrize("gen", ["G1", "mix", "mixneg", "degneg"])
def test_tiny_register_kernel_parity(m, n, gen):
    B = 5000
    if gen == "G1":
        A, b, c = lpgen.signed_bounded(B, m, n, 400 + 7 * m + n)
    elif gen == "degneg":
        A, b, c = lpgen.degenerate(B, m, n, 401 + 7 * m + n, negative_b=True)
    else:
        A, b, c = lpgen.status_mix(B, m, n, 402 + 7 * m + n, infeasible_start=gen == "mixneg")
    kw = dict(bland_after=2) if gen == "degneg" else {}
    o = oracle.solve(A, b, c, **kw)
    g = gpu_solve(A, b, c, kernel_class="S", **kw)
    compare(A, b, c, g, o)
    assert g["launch"]["launches"] == 2  # register kernel + the deferred-list kernel
    gh = gpu_solve(A, b, c, path="host", kernel_class="S", n_chunks=3, **kw)
    compare(A, b, c, gh, o)


@pytest.mark.parametrize("B", [1, 31, 1000, 40000])
def test_tiny_batch_sizes_and_cta_shapes(B):
    """32-thread CTAs for small batches, 128 above 148 x 128 LPs; ragged last CTA."""
    A, b, c = lpgen.status_mix(B, 5, 5, 410, infeasible_start=True)
    o = oracle.solve(A, b, c)
    compare(A, b, c, gpu_solve(A, b, c, kernel_class="S"), o)


def test_tiny_rpc_iteration_limit_and_no_x():
    A, b, c = lpgen.status_mix(6000, 6, 5, 411, infeasible_start=True)
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=12)
    compare(A, b, c, gpu_solve(A, b, c, kernel_class="S", pivot_rule="RPC", rpc_seed=12), o)
    o = oracle.solve(A, b, c, max_iter=2)
    g = gpu_solve(A, b, c, kernel_class="S", max_iter=2)
    compare(A, b, c, g, o)
    assert np.any(g["status"] == oracle.ITER_LIMIT)
    g = gpu_solve(A, b, c, kernel_class="S", want_x=False)
    o = oracle.solve(A, b, c)
    assert np.array_equal(g["status"], o["status"]) and np.array_equal(g["iters"], o["iters"])
    assert np.array_equal(g["obj"], o["obj"], equal_nan=True)


_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r}); sys.path.insert(0, {dev!r})
import lpgen
from gpu_util import gpu_solve
A, b, c = lpgen.status_mix(20000, 5, 5, 412, infeasible_start=True)
g = gpu_solve(A, b, c, kernel_class="S")
from paper_1609_08114_b200 import lpb
np.savez({out!r}, lib=lpb.LIB_PATH, **{{k: v for k, v in g.items() if k != "launch"}})
"""


def test_tiny_equals_smem_slice_kernel(tmp_path):
    """The register kernel and the SMEM-slice kernel (LPB_NO_TINY=1, a switch of the
    development build) agree bit for bit."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_extra in ({}, {"LPB_NO_TINY": "1"}):
        out = str(tmp_path / f"r{len(outs)}.npz")
        env = dict(os.environ, **env_extra)
        code = _SCRIPT.format(root=root, tests=os.path.join(root, "tests"), out=out,
                              dev=os.path.join(root, "devbuild"))
        subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
        outs.append(np.load(out))
    assert all("devbuild" in str(o["lib"]) for o in outs)
    for k in ("status", "iters"):
        assert np.array_equal(outs[0][k], outs[1][k])
    for k in ("obj", "x"):
        assert np.array_equal(outs[0][k], outs[1][k], equal_nan=True)


@pytest.mark.parametrize("m,n", [(1, 1), (2, 2), (3, 7), (7, 3), (5, 5), (7, 7)])
@pytest.mark.parametrize("gen", ["G1", "mixneg", "deg"])
def test_warp_element_layout_parity(m, n, gen):
    """The W class's element layout (type-1 LPs up to 7 x 7, one tableau element pair per
    lane; two-phase LPs of the same launch take the generic warp layout) against the oracle:
    LPC, Bland (bland_after=2 on degenerate LPs) and RPC."""
    B = 3000
    if gen == "G1":
        A, b, c = lpgen.signed_bounded(B, m, n, 420 + 7 * m + n)
    elif gen == "deg":
        A, b, c = lpgen.degenerate(B, m, n, 421 + 7 * m + n, negative_b=False)
    else:
        A, b, c = lpgen.status_mix(B, m, n, 422 + 7 * m + n, infeasible_start=True)
    kw = dict(bland_after=2) if gen == "deg" else {}
    o = oracle.solve(A, b, c, **kw)
    g = gpu_solve(A, b, c, kernel_class="W", **kw)
    compare(A, b, c, g, o)
    assert g["launch"]["class"] == "W"
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=m + n)
    g = gpu_solve(A, b, c, kernel_class="W", pivot_rule="RPC", rpc_seed=m + n)
    compare(A, b, c, g, o)
    o = oracle.solve(A, b, c, max_iter=1)
    compare(A, b, c, gpu_solve(A, b, c, kernel_class="W", max_iter=1), o)
