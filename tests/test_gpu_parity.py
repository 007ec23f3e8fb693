"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element,
on the same seeded inputs.  Pass bar (BASELINE.json north_star): status bit-exact,
objective within 1e-9*max(1,|obj|), primal residual <= 1e-9; in addition the iteration
counts and fp64 values are required to be identical (the kernels reproduce the oracle's
arithmetic; a mismatch is a bug, not a tolerance question -- SURVEY §8(c) C-P18)."""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle
from gpu_util import compare, gpu_solve

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lp_fixtures.json")))
CLASSES = ["S", "W", "R", "M", "L"]


def _skip_class(klass, m, n, k):
    if klass == "R" and not _reg_fits(m, n, k):
        pytest.skip("no register layout for this size")
    if klass == "S" and (m > 8 or n > 8):
        pytest.skip("the thread-per-LP class holds m, n <= 8")
    if klass == "W" and (m > 32 or n + k > 32):
        pytest.skip("the warp-per-LP class holds m <= 32, n + k <= 32")


def _reg_fits(m, n, k):
    # mirrors the instantiated register layouts in csrc/simplex_reg.cu (capacity m x (n+k))
    caps = [(8, 12, 1), (16, 24, 1), (32, 32, 1), (56, 56, 0), (56, 56, 1), (64, 64, 0),
            (64, 64, 1),
            (104, 112, 0), (112, 112, 0), (112, 112, 1)]
    return any(m <= r and n + k <= c and (k == 0 or two) for r, c, two in caps)


@pytest.mark.parametrize("klass", CLASSES)
def test_golden_fixtures(klass):
    for fx in GOLD["fixtures"]:
        A = np.array([fx["A"]], float)
        b = np.array([fx["b"]], float)
        c = np.array([fx["c"]], float)
        o = oracle.solve(A, b, c)
        g = gpu_solve(A, b, c, kernel_class=klass)
        compare(A, b, c, g, o)
        assert g["status"][0] == fx["status"], fx["name"]


@pytest.mark.parametrize("klass", CLASSES)
def test_klee_minty_and_chvatal(klass):
    for n in range(2, 9 if klass == "S" else 10):
        A, b, c = lpgen.klee_minty(n)
        A, b, c = A[None], b[None], c[None]
        g = gpu_solve(A, b, c, kernel_class=klass)
        assert g["status"][0] == 0 and g["obj"][0] == 100.0 ** (n - 1)
        assert list(g["iters"][0]) == [0, 2 ** n - 1]
    ch = GOLD["chvatal_cycling"]
    A, b, c = (np.array([ch[k]], float) for k in ("A", "b", "c"))
    for K, piv in ch["pivots_by_K"].items():
        g = gpu_solve(A, b, c, kernel_class=klass, bland_after=int(K))
        assert g["status"][0] == 0 and g["obj"][0] == 1.0 and g["iters"][0][1] == piv
    g = gpu_solve(A, b, c, kernel_class=klass, bland_after=-1, max_iter=300)
    assert g["status"][0] == oracle.ITER_LIMIT


CASES = [
    ("G1", 5, 5, 3000), ("G1", 28, 28, 600), ("G1", 100, 100, 200), ("G1", 60, 13, 300),
    ("G1", 7, 64, 300), ("G1", 1, 1, 50), ("G1", 1, 9, 50), ("G1", 9, 1, 50),
    ("mix", 6, 6, 3000), ("mixneg", 6, 6, 3000), ("mixneg", 20, 20, 500),
    ("mix", 100, 100, 60), ("G2", 8, 8, 2000), ("G2", 50, 50, 100), ("G2light", 60, 60, 60),
    ("deg", 8, 8, 3000), ("degneg", 8, 8, 3000), ("degneg", 20, 20, 1000),
    ("G1", 50, 50, 300), ("G2", 40, 40, 150), ("mixneg", 48, 40, 300),
    ("G1", 64, 60, 200), ("G2", 56, 48, 100),
]


def _gen(gen, B, m, n, seed):
    if gen == "G1":
        return lpgen.signed_bounded(B, m, n, seed)
    if gen == "G2":
        return lpgen.twophase_signed(B, m, n, seed)
    if gen == "G2light":
        return lpgen.twophase_light(B, m, n, seed)
    if gen.startswith("mix"):
        return lpgen.status_mix(B, m, n, seed, infeasible_start=gen.endswith("neg"))
    return lpgen.degenerate(B, m, n, seed, negative_b=gen.endswith("neg"))


@pytest.mark.parametrize("klass", CLASSES)
@pytest.mark.parametrize("gen,m,n,B", CASES, ids=[f"{g}-{m}x{n}" for g, m, n, _ in CASES])
def test_random_batches(klass, gen, m, n, B):
    A, b, c = _gen(gen, B, m, n, 1000 + 7 * m + n)
    _skip_class(klass, m, n, int((b < 0).sum(axis=1).max()))
    o = oracle.solve(A, b, c)
    g = gpu_solve(A, b, c, kernel_class=klass)
    compare(A, b, c, g, o)


SHARED_CASES = [("G1", 5, 5, 3000), ("G1", 100, 100, 300), ("G2", 8, 8, 2000),
                ("G2", 60, 60, 200), ("G2", 200, 200, 12)]


@pytest.mark.parametrize("klass", CLASSES)
@pytest.mark.parametrize("gen,m,n,B", SHARED_CASES,
                         ids=[f"{g}-{m}x{n}" for g, m, n, _ in SHARED_CASES])
def test_shared_constraints(klass, gen, m, n, B):
    """NEXT-1: many objectives over one polytope, A and b read with stride 0
    (LPB_SHARED_AB), device and host paths, against the oracle on the broadcast batch."""
    A, b, c = lpgen.shared_polytope(B, m, n, 900 + m, gen)
    k = int((b < 0).sum())
    _skip_class(klass, m, n, k)
    if klass != "L" and m >= 200:
        pytest.skip("200x200 two-phase needs the cluster class")
    Ab = np.ascontiguousarray(np.broadcast_to(A, (B, m, n)))
    bb = np.ascontiguousarray(np.broadcast_to(b, (B, m)))
    o = oracle.solve(Ab, bb, c)
    g = gpu_solve(A, b, c, kernel_class=klass)
    compare(Ab, bb, c, g, o)
    gh = gpu_solve(A, b, c, path="host", kernel_class=klass, n_chunks=3)
    compare(Ab, bb, c, gh, o)


@pytest.mark.parametrize("K", [1, 3])
def test_bland_coverage_degenerate(K):
    """G-deg with small Bland thresholds: exercises Bland mode and artificial drive-outs."""
    for neg in (False, True):
        A, b, c = lpgen.degenerate(4000, 8, 8, 50 + K + neg, negative_b=neg)
        o = oracle.solve(A, b, c, bland_after=K)
        for klass in CLASSES:
            g = gpu_solve(A, b, c, kernel_class=klass, bland_after=K)
            compare(A, b, c, g, o)


def test_iteration_limit_status():
    A, b, c = lpgen.signed_bounded(200, 30, 30, 77)
    o = oracle.solve(A, b, c, max_iter=5)
    g = gpu_solve(A, b, c, max_iter=5)
    compare(A, b, c, g, o)
    assert np.any(g["status"] == oracle.ITER_LIMIT)


def test_host_path_equals_device_path_and_chunking():
    A, b, c = lpgen.status_mix(997, 10, 12, 5, infeasible_start=True)
    gd = gpu_solve(A, b, c)
    for nch in (1, 3, 10):
        gh = gpu_solve(A, b, c, path="host", n_chunks=nch)
        for k in ("status", "iters"):
            assert np.array_equal(gd[k], gh[k])
        assert np.array_equal(gd["obj"], gh["obj"], equal_nan=True)
        assert np.array_equal(gd["x"], gh["x"], equal_nan=True)


def test_scheduling_invariance_grid_and_class():
    A, b, c = lpgen.status_mix(1500, 16, 16, 6, infeasible_start=True)
    ref = gpu_solve(A, b, c, kernel_class="M")
    for kw in (dict(kernel_class="M", grid_ctas=1), dict(kernel_class="M", grid_ctas=37),
               dict(kernel_class="R"), dict(kernel_class="R", grid_ctas=5),
               dict(kernel_class="L"), dict(kernel_class="L", grid_ctas=3)):
        g = gpu_solve(A, b, c, **kw)
        for k in ("status", "iters"):
            assert np.array_equal(ref[k], g[k]), kw
        assert np.array_equal(ref["obj"], g["obj"], equal_nan=True), kw


def test_batch_of_one_and_repeat_solves():
    import torch

    from paper_1609_08114_b200 import lpb
    A, b, c = lpgen.signed_bounded(1, 12, 9, 3)
    o = oracle.solve(A, b, c)
    s = lpb.Solver(1, 12, 9)
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    for _ in range(3):
        s.solve_device(At, bt, ct, sync=True)
        r = {k: v.cpu().numpy() for k, v in s.device_results().items()}
        compare(A, b, c, r, o)
    s.close()


def test_abi_errors_on_gpu():
    import ctypes

    from paper_1609_08114_b200 import lpb
    s = lpb.Solver(4, 3, 3)
    st = np.empty(4, np.int32)
    assert lpb._lib.lpb_results(s._ctx, st.ctypes.data_as(ctypes.c_void_p), None, None, None) == lpb.ESTATE
    assert lpb._lib.lpb_solve_batch(s._ctx, None, None, None, 0) == lpb.EINVAL
    s.close()


# ---------------- hyperbox (type 3) ----------------

@pytest.mark.parametrize("n,B", [(1, 1000), (2, 5000), (5, 200000), (7, 10001), (28, 60000),
                                 (33, 3001)])
def test_hyperbox_bit_exact(n, B):
    import torch

    from paper_1609_08114_b200 import lpb
    lo, hi, dirs = lpgen.hyperbox(B, n, 60 + n)
    dirs = dirs.copy()
    dirs[: min(B, 7), 0] = -0.0  # the l_i = -0.0 branch takes hi (C15)
    o = oracle.hyperbox(lo, hi, dirs)
    g = lpb.hyperbox(lo, hi, torch.from_numpy(dirs).cuda())
    assert np.array_equal(g["status"].cpu().numpy(), o["status"])
    assert np.array_equal(g["obj"].cpu().numpy(), o["obj"])
    assert np.array_equal(g["x"].cpu().numpy(), o["x"])
    gh = lpb.hyperbox(lo, hi, dirs)  # host pipeline path
    assert np.array_equal(gh["obj"], o["obj"]) and np.array_equal(gh["x"], o["x"])


def test_hyperbox_per_lp_box_and_empty():
    import torch

    from paper_1609_08114_b200 import lpb
    B, n = 3000, 6
    g0 = lpgen.rng(9)
    lo = g0.uniform(-1, 1, (B, n))
    hi = lo + g0.uniform(-0.1, 1, (B, n))  # some boxes empty
    dirs = g0.standard_normal((B, n))
    o = oracle.hyperbox(lo, hi, dirs)
    box = torch.from_numpy(np.ascontiguousarray(np.concatenate([hi, -lo], axis=1))).cuda()
    s = lpb.Solver(B, 2 * n, n, lpb.HYPERBOX)
    s.solve_device(None, box, torch.from_numpy(dirs).cuda(), sync=True)
    r = {k: v.cpu().numpy() for k, v in s.device_results().items()}
    assert np.array_equal(r["status"], o["status"])
    assert np.array_equal(r["obj"], o["obj"])
    assert np.array_equal(r["x"], o["x"], equal_nan=True)
    assert np.any(o["status"] == oracle.INFEASIBLE)
    s.close()


@pytest.mark.parametrize("n,B", [(4, 70001), (5, 4099), (28, 9000), (3, 100000)])
def test_hyperbox_no_x_empty_shared_box_and_misaligned_chunks(n, B):
    """Shared-box kernel paths: NO_X (no x stores), an empty shared box (all INFEASIBLE, x NaN),
    and host-pipeline chunks whose x slices are not 16-byte aligned (per-thread store path)."""
    import torch

    from paper_1609_08114_b200 import lpb
    lo, hi, dirs = lpgen.hyperbox(B, n, 70 + n)
    o = oracle.hyperbox(lo, hi, dirs)
    s = lpb.Solver(B, 2 * n, n, lpb.HYPERBOX)
    box = torch.from_numpy(np.concatenate([hi, -lo])).cuda()
    s.solve_device(None, box, torch.from_numpy(dirs).cuda(), shared_box=True, want_x=False,
                   sync=True)
    r = s.device_results(want_x=False)
    assert np.array_equal(r["obj"].cpu().numpy(), o["obj"])
    assert np.array_equal(r["status"].cpu().numpy(), o["status"])
    s.close()
    hi_e = hi.copy()
    hi_e[n // 2] = lo[n // 2] - 0.5  # empty box
    oe = oracle.hyperbox(lo, hi_e, dirs)
    ge = lpb.hyperbox(lo, hi_e, torch.from_numpy(dirs).cuda())
    assert np.all(oe["status"] == oracle.INFEASIBLE)
    assert np.array_equal(ge["status"].cpu().numpy(), oe["status"])
    assert np.array_equal(ge["obj"].cpu().numpy(), oe["obj"])
    assert np.array_equal(ge["x"].cpu().numpy(), oe["x"], equal_nan=True)
    gh = lpb.hyperbox(lo, hi, dirs, n_chunks=7)  # odd chunk boundaries
    assert np.array_equal(gh["obj"], o["obj"]) and np.array_equal(gh["x"], o["x"])


@pytest.mark.parametrize("klass", CLASSES)
@pytest.mark.parametrize("scale_a,scale_b", [(1e-300, 1.0), (1.0, 1e-310), (1e300, 1e-300),
                                             (2.0 ** -1060, 2.0 ** 1000)])
def test_extreme_magnitudes(klass, scale_a, scale_b):
    """Quotients outside the branch-free division's fast range (subnormal / huge ratios and
    pivot elements) take the IEEE fallback (ddiv_slow) in the ratio test and the pivot row;
    the result must still be the oracle's bit for bit.  Magnitudes also move the eps tests,
    so statuses differ from the unscaled LPs -- only parity is asserted."""
    A, b, c = lpgen.status_mix(400, 6, 6, 77, infeasible_start=True)
    A = A * scale_a
    b = b * scale_b
    o = oracle.solve(A, b, c)
    g = gpu_solve(A, b, c, kernel_class=klass)
    compare(A, b, c, g, o, check_x=False)
    ok = o["status"] == oracle.OPTIMAL
    assert np.array_equal(g["x"][ok], o["x"][ok])


def test_concurrent_host_threads_share_the_library():
    """Host threads driving their own contexts at once (ctypes drops the GIL inside the C
    ABI): the launchers' memoised attribute / occupancy queries are thread-safe and every
    thread's results equal a solo run's."""
    import threading

    cases = [("G1", 5, 5, 3000, "S"), ("G1", 28, 28, 400, "W"), ("G1", 60, 60, 200, "R"),
             ("G2", 40, 40, 120, "M"), ("G2", 60, 60, 60, "L"), ("mixneg", 20, 20, 500, "R")]
    inputs = [_gen(g, B, m, n, 500 + m) for g, m, n, B, _ in cases]
    solo = [gpu_solve(*inp, kernel_class=k) for inp, (*_, k) in zip(inputs, cases)]
    out = [None] * len(cases)
    errs = []

    def run(t):
        try:
            for _ in range(3):
                out[t] = gpu_solve(*inputs[t], kernel_class=cases[t][-1])
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=run, args=(t,)) for t in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a_, b_ in zip(solo, out):
        for k in ("status", "iters"):
            assert np.array_equal(a_[k], b_[k])
        assert np.array_equal(a_["obj"], b_["obj"], equal_nan=True)


def test_concurrent_same_class_different_smem():
    """host threads launching the SAME kernel instantiation with DIFFERENT dynamic
    SMEM sizes at once (M class at 24x24 .. 90x90) -- the launch memo only ever raises the
    function's SMEM attribute, so no launch sees a limit lowered by another thread."""
    import threading

    sizes = [24, 90, 40, 80, 56, 70]
    inputs = [_gen("G2", 40, m, m, 700 + m) for m in sizes]
    solo = [gpu_solve(*inp, kernel_class="M") for inp in inputs]
    out = [None] * len(sizes)
    errs = []

    def run(t):
        try:
            for _ in range(6):
                out[t] = gpu_solve(*inputs[t], kernel_class="M")
        except Exception as ex:  # surfaced below
            errs.append(ex)

    th = [threading.Thread(target=run, args=(t,)) for t in range(len(sizes))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for a_, b_ in zip(solo, out):
        assert b_["launch"]["class"] == "M"
        for k in ("status", "iters"):
            assert np.array_equal(a_[k], b_[k])
        assert np.array_equal(a_["obj"], b_["obj"], equal_nan=True)


@pytest.mark.parametrize("klass,m,n,B,hint", [("S", 5, 5, 20000, 0), ("S", 6, 6, 3000, 0),
                                             ("W", 12, 12, 2000, 0), ("R", 40, 40, 600, 0),
                                             ("R", 60, 60, 300, 3), ("M", 40, 40, 200, 2),
                                             ("L", 60, 60, 100, 4)])
def test_kmax_hint_contract(klass, m, n, B, hint):
    """lpb_options.kmax_hint (include/lpb.h): the solve is one launch sized for the promised
    k; every LP that keeps the promise (#{b_i < 0} <= hint) is solved exactly as without the
    hint (oracle parity), every LP that breaks it reports LPB_BAD_HINT (obj NaN, x NaN,
    iters 0) instead of a wrong answer."""
    A, b, c = lpgen.status_mix(B, m, n, 900 + m + hint)
    g0 = lpgen.rng(77 + m)
    want = g0.integers(0, hint + 3, size=B)  # per-LP count of negated rows: 0 .. hint + 2
    for t in range(B):
        rows = g0.permutation(m)[:want[t]]
        b[t, rows] = -b[t, rows]
    k = (b < 0).sum(axis=1)
    ok = k <= hint
    assert ok.any() and (~ok).any()
    g = gpu_solve(A, b, c, kernel_class=klass, kmax_hint=hint)
    assert g["launch"]["class"] == klass
    assert np.all(g["status"][~ok] == 5)
    assert np.all(np.isnan(g["obj"][~ok])) and np.all(g["iters"][~ok] == 0)
    assert np.all(np.isnan(g["x"][~ok]))
    idx = np.nonzero(ok)[0]
    o = oracle.solve(A[idx], b[idx], c[idx])
    compare(A, b, c, g, o, sample=idx)
    if hint == 0 or klass in ("R", "W", "M", "L"):
        assert g["launch"]["launches"] == 1  # no prepass, no deferred list


@pytest.mark.parametrize("seed,K", [(40, 3), (43, 3), (43, 2), (47, 3)])
@pytest.mark.parametrize("klass", ["M", "L", "auto"])
def test_numerical_status_parity(seed, K, klass):
    """LPB_NUMERICAL (phase I without a ratio candidate: a rounding artifact, pinned in
    tests/test_oracle_pins.py) is reproduced LP for LP on degenerate 100x100 batches with
    small Bland thresholds, together with every other status, iteration count and bit."""
    A, b, c = lpgen.degenerate(300, 100, 100, seed, negative_b=True)
    o = oracle.solve(A, b, c, bland_after=K)
    assert (o["status"] == oracle.NUMERICAL).any()
    g = gpu_solve(A, b, c, kernel_class=klass, bland_after=K)
    compare(A, b, c, g, o)
