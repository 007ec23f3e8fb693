"""GPU parity for the SURVEY §8(f) "next" rows, against the oracle element by element:
  NEXT-2  larger LPs (the paper's fig:TimeLPplotting dims 300/500 and its limits 511 type-1 /
          340 type-2) on 4-, 8- and 16-CTA clusters (L class), plus the
          8/16-CTA PULL column exchange forced on small LPs;
  NEXT-3  the RPC entering rule (include/lpb.h LPB_RULE_RPC, reading R15) in
          every size class, on the device and the chunked host path.
Bit-exact as everywhere else: status, iterations, objective and x identical."""
import numpy as np
import pytest

import lpgen
import oracle
from gpu_util import compare, gpu_solve

pytestmark = pytest.mark.gpu

CLASSES = ["S", "W", "R", "M", "L"]


@pytest.mark.parametrize("gen,m,n,B,cl", [
    ("G1", 300, 300, 8, 4), ("G2", 340, 340, 4, 8), ("G1", 511, 511, 4, 16),
    ("G1", 500, 500, 3, 16), ("G2", 300, 300, 3, 8),
])
def test_large_sizes(gen, m, n, B, cl):
    A, b, c = (lpgen.signed_bounded if gen == "G1" else lpgen.twophase_signed)(B, m, n, 11 + m)
    o = oracle.solve(A, b, c)
    g = gpu_solve(A, b, c)  # auto size class
    compare(A, b, c, g, o)
    assert g["launch"]["class"] == "L" and g["launch"]["cluster"] == cl, g["launch"]


@pytest.mark.parametrize("cl", [2, 4, 8, 16])
@pytest.mark.parametrize("gen,m,n,B", [("G1", 100, 100, 60), ("G2", 50, 50, 80),
                                       ("mixneg", 20, 20, 400), ("deg", 8, 8, 600)])
def test_forced_cluster_sizes(cl, gen, m, n, B):
    if gen == "G1":
        A, b, c = lpgen.signed_bounded(B, m, n, 21 + cl)
    elif gen == "G2":
        A, b, c = lpgen.twophase_signed(B, m, n, 22 + cl)
    elif gen == "deg":
        A, b, c = lpgen.degenerate(B, m, n, 23 + cl, negative_b=True)
    else:
        A, b, c = lpgen.status_mix(B, m, n, 24 + cl, infeasible_start=True)
    kw = dict(bland_after=2) if gen == "deg" else {}
    o = oracle.solve(A, b, c, **kw)
    g = gpu_solve(A, b, c, kernel_class="L", cluster_ctas=cl, **kw)
    compare(A, b, c, g, o)
    assert g["launch"]["cluster"] == cl


@pytest.mark.parametrize("klass", CLASSES)
@pytest.mark.parametrize("gen,m,n,B", [
    ("G1", 5, 5, 3000), ("G1", 28, 28, 400), ("G1", 100, 100, 100), ("mixneg", 6, 6, 3000),
    ("G2", 8, 8, 2000), ("G2", 50, 50, 60), ("deg", 8, 8, 2000), ("mix", 7, 60, 300),
])
def test_rpc_parity(klass, gen, m, n, B):
    if gen == "G1":
        A, b, c = lpgen.signed_bounded(B, m, n, 31 + m)
    elif gen == "G2":
        A, b, c = lpgen.twophase_signed(B, m, n, 32 + m)
    elif gen == "deg":
        A, b, c = lpgen.degenerate(B, m, n, 33 + m, negative_b=True)
    else:
        A, b, c = lpgen.status_mix(B, m, n, 34 + m, infeasible_start=gen.endswith("neg"))
    k = int((b < 0).sum(axis=1).max())
    if klass == "S" and (m > 8 or n > 8):
        pytest.skip("the thread-per-LP class holds m, n <= 8")
    if klass == "W" and (m > 32 or n + k > 32):
        pytest.skip("the warp-per-LP class holds m <= 32, n + k <= 32")
    if klass == "R" and not (m <= 112 and n + k <= 112):
        pytest.skip("no register layout for this size")
    seed = 0xC0FFEE + m
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=seed)
    try:
        g = gpu_solve(A, b, c, kernel_class=klass, pivot_rule="RPC", rpc_seed=seed)
    except Exception as ex:  # a class without a layout for (m, n + k) reports ETOOBIG
        if "size class" in str(ex):
            pytest.skip(str(ex))
        raise
    compare(A, b, c, g, o)
    if gen == "G1" and m >= 28:  # RPC takes more pivots than LPC on average
        assert o["iters"][:, 1].mean() > oracle.solve(A, b, c)["iters"][:, 1].mean()


def test_rpc_host_path_chunks_keep_batch_indices():
    """The RPC draw is keyed on the LP's index in the whole call: chunked host pipelines
    (lp_base per chunk) and the device path give identical pivot paths."""
    A, b, c = lpgen.status_mix(1999, 9, 9, 41, infeasible_start=True)
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=5)
    for nch in (1, 7):
        g = gpu_solve(A, b, c, path="host", n_chunks=nch, pivot_rule="RPC", rpc_seed=5)
        compare(A, b, c, g, o)


def test_rpc_large_cluster():
    A, b, c = lpgen.twophase_signed(3, 200, 200, 43)
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=9)
    g = gpu_solve(A, b, c, pivot_rule="RPC", rpc_seed=9)
    compare(A, b, c, g, o)


def test_rpc_lp_index_base_reproduces_unsharded_paths():
    """A rank solving LPs [lo, hi) of a sharded batch passes lp_index_base = lo and follows
    the pivot paths of the unsharded run (dist.solve_sharded / bench.py do this)."""
    A, b, c = lpgen.signed_bounded(900, 20, 20, 45)
    o = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=77)
    for lo, hi in ((0, 300), (300, 900), (451, 452)):
        g = gpu_solve(A[lo:hi], b[lo:hi], c[lo:hi], pivot_rule="RPC", rpc_seed=77,
                      lp_index_base=lo)
        sl = {k: v[lo:hi] for k, v in o.items() if isinstance(v, np.ndarray)}
        compare(A[lo:hi], b[lo:hi], c[lo:hi], g, sl)


# ---------------- NEXT-1: phase-I warm start of shared-constraint two-phase batches ----------

def _shared(kind, B, m, n, seed):
    g = lpgen.rng(seed)
    if kind == "G2":
        A, b, _ = lpgen.twophase_signed(1, m, n, seed)
    elif kind == "deg":  # degenerate pivots, Bland mode, artificial drive-outs
        A, b, _ = lpgen.degenerate(1, m, n, seed, negative_b=True)
    elif kind == "infeasible":  # x1 <= -1 style rows: phase I ends with w* > 0
        A, b, _ = lpgen.status_mix(1, m, n, seed, infeasible_start=True)
        A[0, 0, :] = np.abs(A[0, 0, :])
        b[0, 0] = -5.0
    else:
        A, b, _ = lpgen.status_mix(1, m, n, seed, infeasible_start=True)
    c = g.uniform(-10.0, 10.0, size=(B, n))
    return A[0], b[0], c


@pytest.mark.parametrize("klass,cl", [("M", 0), ("L", 0), ("L", 8)])
@pytest.mark.parametrize("kind,m,n,B", [("G2", 60, 60, 300), ("deg", 12, 12, 800),
                                        ("mix", 20, 20, 500), ("infeasible", 10, 10, 200),
                                        ("G2", 200, 200, 20)])
def test_warm_start_shared_two_phase(klass, cl, kind, m, n, B):
    A, b, c = _shared(kind, B, m, n, 7 + m)
    if not np.any(b < 0):
        pytest.skip("no infeasible row drawn")
    if klass == "M" and m >= 200:
        pytest.skip("200x200 two-phase needs the cluster class")
    Ab = np.ascontiguousarray(np.broadcast_to(A, (B, m, n)))
    bb = np.ascontiguousarray(np.broadcast_to(b, (B, m)))
    kw = dict(bland_after=2) if kind == "deg" else {}
    o = oracle.solve(Ab, bb, c, **kw)
    opts = dict(kernel_class=klass, **kw)
    if cl:
        opts["cluster_ctas"] = cl
    warm = gpu_solve(A, b, c, **opts)
    assert warm["launch"]["launches"] >= 2  # the phase-I record pass ran
    compare(Ab, bb, c, warm, o)
    cold = gpu_solve(A, b, c, warm_start=-1, **opts)
    for key in ("status", "iters"):
        assert np.array_equal(warm[key], cold[key])
    assert np.array_equal(warm["obj"], cold["obj"], equal_nan=True)
    assert np.array_equal(warm["x"], cold["x"], equal_nan=True)
    gh = gpu_solve(A, b, c, path="host", n_chunks=3, **opts)  # record once, chunks reuse it
    compare(Ab, bb, c, gh, o)
    if kind == "infeasible":
        assert np.all(o["status"] == oracle.INFEASIBLE)


def test_warm_start_iteration_limit_in_phase_one():
    A, b, c = _shared("G2", 300, 40, 40, 3)
    Ab = np.ascontiguousarray(np.broadcast_to(A, (300, 40, 40)))
    bb = np.ascontiguousarray(np.broadcast_to(b, (300, 40)))
    o = oracle.solve(Ab, bb, c, max_iter=5)
    g = gpu_solve(A, b, c, kernel_class="M", max_iter=5)
    compare(Ab, bb, c, g, o)
    assert np.all(g["status"] == oracle.ITER_LIMIT)


@pytest.mark.parametrize("klass", ["M", "L", "R"])
def test_rpc_shared_two_phase_cold_path(klass):
    """Under RPC the phase-I path depends on the LP index, so shared-constraint two-phase
    batches are solved from scratch (no warm start) -- still the oracle's, bit for bit."""
    A, b, c = _shared("G2", 300, 40, 40, 19)
    Ab = np.ascontiguousarray(np.broadcast_to(A, (300, 40, 40)))
    bb = np.ascontiguousarray(np.broadcast_to(b, (300, 40)))
    o = oracle.solve(Ab, bb, c, pivot_rule="RPC", rpc_seed=4)
    g = gpu_solve(A, b, c, kernel_class=klass, pivot_rule="RPC", rpc_seed=4)
    compare(Ab, bb, c, g, o)
    assert len(np.unique(o["iters"][:, 0])) > 1  # phase I differs across the batch under RPC
