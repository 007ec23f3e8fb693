"""GPU parity of the L class's TMR variants (constraint rows in tensor memory during the pivot
loop; csrc/simplex_block.cu pivot_local_tm): clusters of >= 4 CTAs whose
CTAs run one per SM (SMEM tableaux above half the SM) take them.  Against the oracle element by
element (status, iterations, objective and x bits), over the row-slot shapes (one, two, three
row slots of 128 TMEM lanes; a last slot holding a single row), both phases with the phase
switch's TMEM <-> SMEM copies and drive-outs, Bland pivots on degenerate LPs, the RPC rule,
and the phase-I record + warm start of shared-constraint batches; and bit for bit against the
SMEM-row kernel of the development build (LPB_NO_TMEM=1)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import lpgen
import oracle
from gpu_util import compare, gpu_solve

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gen,m,n,B,cl", [
    ("G1", 300, 300, 12, 4),   # three row slots (128, 128, 44), cfg6's shape
    ("G1", 256, 300, 12, 4),   # two full row slots
    ("G1", 129, 500, 12, 4),   # the second slot holds one row; 16 chunks per row
    ("G2", 250, 250, 10, 4),   # two-phase: phase switch, compaction, copies back to TMEM
    ("G2", 340, 340, 4, 8),    # the paper's two-phase limit on 8-CTA (PULL) clusters
])
def test_tmr_parity(gen, m, n, B, cl):
    f = lpgen.signed_bounded if gen == "G1" else lpgen.twophase_signed
    A, b, c = f(B, m, n, 700 + m + cl)
    o = oracle.solve(A, b, c)
    g = gpu_solve(A, b, c, kernel_class="L", cluster_ctas=cl)
    compare(A, b, c, g, o)
    assert g["launch"]["class"] == "L" and g["launch"]["cluster"] == cl
    assert np.all(g["status"] == oracle.OPTIMAL)


def test_tmr_bland_degenerate():
    """Degenerate two-phase LPs (drive-outs, redundant rows) with Bland pivots after 2 stalls."""
    A, b, c = lpgen.degenerate(8, 250, 250, 731, negative_b=True)
    o = oracle.solve(A, b, c, bland_after=2)
    g = gpu_solve(A, b, c, kernel_class="L", cluster_ctas=4, bland_after=2)
    compare(A, b, c, g, o)


def test_tmr_rpc():
    A, b, c = lpgen.signed_bounded(8, 300, 300, 733)
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=5)
    g = gpu_solve(A, b, c, kernel_class="L", cluster_ctas=4, pivot_rule="RPC", rpc_seed=5)
    compare(A, b, c, g, o)


def test_tmr_warm_start_shared():
    """Shared-constraint two-phase batch: phase I recorded once (mode 1), every LP warm-started
    from the record (mode 2), both on the TMR kernel."""
    A, b, c = lpgen.shared_polytope(6, 250, 250, 735, "G2")
    Ab = np.broadcast_to(A, (c.shape[0],) + A.shape)
    bb = np.broadcast_to(b, (c.shape[0],) + b.shape)
    o = oracle.solve(np.ascontiguousarray(Ab), np.ascontiguousarray(bb), c)
    g = gpu_solve(A, b, c, kernel_class="L", cluster_ctas=4)
    compare(np.ascontiguousarray(Ab), np.ascontiguousarray(bb), c, g, o)


_SCRIPT = r"""
import sys
sys.path.insert(0, {dev!r}); sys.path.insert(1, {root!r}); sys.path.insert(2, {tests!r})
import numpy as np
import lpgen
from gpu_util import gpu_solve
from paper_1609_08114_b200 import lpb
A, b, c = lpgen.twophase_signed(6, 250, 250, 741)
g = gpu_solve(A, b, c, kernel_class="L", cluster_ctas=4)
np.savez({out!r}, lib=lpb.LIB_PATH, **{{k: v for k, v in g.items() if k != "launch"}})
"""


def test_tmr_equals_smem_rows(tmp_path):
    """The TMR kernel and the SMEM-row kernel (LPB_NO_TMEM=1, a switch of the development
    build) agree bit for bit on a two-phase batch."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for env_extra in ({}, {"LPB_NO_TMEM": "1"}):
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
