"""Pins for the CPU oracle (oracle/), all CPU-only.

The oracle is checked against things other than itself:
worked examples from SPEC.md (tests/golden, cited), closed forms (Klee-Minty, fractional
knapsack, diagonal, hyperbox), Chvatal's cycling LP, LP certificates from the original data,
exact-rational brute force on m,n <= 4, and scipy's HiGHS with presolve off.
"""
import json
import math
import os
from fractions import Fraction
from itertools import product

import numpy as np
import pytest

import lpgen
import oracle
from checks import check_infeasible, check_optimal, check_unbounded, primal_residual
from exact_brute import brute_force

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lp_fixtures.json")))


def _solve1(A, b, c, **kw):
    r = oracle.solve(np.array(A, float), np.array(b, float), np.array(c, float), certs=True,
                     threads=1, **kw)
    return {k: (v[0] if isinstance(v, np.ndarray) else v) for k, v in r.items()}


@pytest.mark.parametrize("fx", GOLD["fixtures"], ids=[f["name"] for f in GOLD["fixtures"]])
def test_golden_fixture(fx):
    r = _solve1(fx["A"], fx["b"], fx["c"])
    assert r["status"] == fx["status"], fx["cite"]
    if "obj" in fx:
        assert abs(r["obj"] - fx["obj"]) <= 1e-9 * max(1, abs(fx["obj"]))
    if "x" in fx:
        np.testing.assert_allclose(r["x"], fx["x"], atol=1e-12)
    if "iters" in fx:
        assert list(r["iters"]) == fx["iters"]
    if "y" in fx:
        np.testing.assert_allclose(r["y"], fx["y"], atol=1e-12)
    if "ray" in fx:
        np.testing.assert_allclose(r["ray"], fx["ray"], atol=1e-12)


@pytest.mark.parametrize("fx", GOLD["fixtures"], ids=[f["name"] for f in GOLD["fixtures"]])
def test_golden_fixture_brute_force(fx):
    """The fixture's expected status/objective agree with exact vertex enumeration."""
    st, obj = brute_force(fx["A"], fx["b"], fx["c"])
    assert st == {0: "optimal", 1: "unbounded", 2: "infeasible"}[fx["status"]]
    if st == "optimal":
        assert obj == Fraction(fx["obj"]).limit_denominator(1000)


@pytest.mark.parametrize("n", range(2, 10))
def test_klee_minty_closed_form(n):
    """Dantzig's rule on the Klee-Minty cube: 2^n - 1 pivots, optimum 100^(n-1) (C-P9)."""
    A, b, c = lpgen.klee_minty(n)
    r = _solve1(A, b, c)
    assert r["status"] == oracle.OPTIMAL
    assert r["obj"] == 100.0 ** (n - 1)
    assert list(r["iters"]) == [0, 2 ** n - 1]
    expect_x = np.zeros(n)
    expect_x[-1] = 100.0 ** (n - 1)
    np.testing.assert_array_equal(r["x"], expect_x)


def test_chvatal_cycling_pure_dantzig_cycles():
    ch = GOLD["chvatal_cycling"]
    r = _solve1(ch["A"], ch["b"], ch["c"], bland_after=-1, max_iter=300)
    assert r["status"] == ch["pure_dantzig_status"] == oracle.ITER_LIMIT


@pytest.mark.parametrize("K", list(GOLD["chvatal_cycling"]["pivots_by_K"]))
def test_chvatal_cycling_bland_fallback(K):
    ch = GOLD["chvatal_cycling"]
    r = _solve1(ch["A"], ch["b"], ch["c"], bland_after=int(K))
    assert r["status"] == oracle.OPTIMAL
    assert r["obj"] == ch["obj"]
    np.testing.assert_array_equal(r["x"], ch["x"])
    np.testing.assert_allclose(r["y"], ch["y"], atol=1e-12)
    assert r["iters"][1] == ch["pivots_by_K"][K]


def test_chvatal_default_K_is_n_plus_m():
    ch = GOLD["chvatal_cycling"]
    r = _solve1(ch["A"], ch["b"], ch["c"])  # default K = n + m = 7
    assert r["iters"][1] == ch["pivots_by_K"]["7"]


def test_fractional_knapsack_closed_form():
    """m = 1, a > 0: obj = b * max_j (c_j / a_j)^+  (C-P12)."""
    g = lpgen.rng(12)
    for _ in range(300):
        n = int(g.integers(1, 7))
        a = g.uniform(0.5, 5.0, n)
        c = g.uniform(-3.0, 3.0, n)
        bb = g.uniform(0.5, 20.0)
        r = _solve1(a[None, :], [bb], c)
        expect = bb * max(0.0, float(np.max(c / a)))
        assert r["status"] == oracle.OPTIMAL
        assert abs(r["obj"] - expect) <= 4e-16 * max(1.0, abs(expect)) * 4


def test_diagonal_closed_form():
    """A = diag(a), a > 0: obj = sum_j max(c_j, 0) b_j / a_j  (C-P13)."""
    g = lpgen.rng(13)
    for _ in range(300):
        n = int(g.integers(1, 9))
        a = g.uniform(0.5, 5.0, n)
        c = g.uniform(-3.0, 3.0, n)
        bb = g.uniform(0.0, 20.0, n)
        r = _solve1(np.diag(a), bb, c)
        expect = math.fsum(max(cj, 0.0) * bj / aj for cj, bj, aj in zip(c, bb, a))
        assert r["status"] == oracle.OPTIMAL
        assert abs(r["obj"] - expect) <= 1e-14 * max(1.0, abs(expect))


def _int_lp(g, m, n):
    A = g.integers(-5, 7, size=(m, n)).astype(float)
    b = g.integers(-5, 7, size=m).astype(float)
    c = g.integers(-5, 7, size=n).astype(float)
    return A, b, c


def test_brute_force_exact_small():
    """Exact-rational vertex enumeration on random integer LPs, m,n <= 4 (C-P16): status must
    match exactly and the objective within the pass tolerance."""
    g = lpgen.rng(16)
    seen = {0: 0, 1: 0, 2: 0}
    for _ in range(600):
        m, n = int(g.integers(1, 5)), int(g.integers(1, 5))
        A, b, c = _int_lp(g, m, n)
        r = _solve1(A, b, c)
        st, obj = brute_force(A.tolist(), b.tolist(), c.tolist())
        code = {"optimal": 0, "unbounded": 1, "infeasible": 2}[st]
        assert r["status"] == code, (A, b, c, r)
        seen[code] += 1
        if st == "optimal":
            assert abs(r["obj"] - float(obj)) <= 1e-9 * max(1.0, abs(float(obj)))
    assert min(seen.values()) > 50, seen


def _certify(A, b, c, r, tol=1e-9):
    st = r["status"]
    if st == oracle.OPTIMAL:
        return check_optimal(A, b, c, r["obj"], r["x"], r["y"], tol)
    if st == oracle.INFEASIBLE:
        return check_infeasible(A, b, r["y"], tol)
    if st == oracle.UNBOUNDED:
        return check_unbounded(A, b, c, r["xb"], r["ray"], tol)
    return [f"status {st}"]


@pytest.mark.parametrize("gen,m,n,B", [
    ("G1", 5, 5, 300), ("G1", 28, 28, 60), ("G1", 60, 60, 10),
    ("G2", 8, 8, 200), ("G2", 40, 40, 10),
    ("mix", 6, 6, 300), ("mixneg", 6, 6, 300), ("mixneg", 20, 20, 40),
    ("G2light", 30, 30, 20),
])
def test_certificates(gen, m, n, B):
    """Every returned status carries a duality certificate computed from the original data
    (C-P15): dual feasibility + zero gap, Farkas, or a ray from a feasible point."""
    if gen == "G1":
        A, b, c = lpgen.signed_bounded(B, m, n, 100 + m)
    elif gen == "G2":
        A, b, c = lpgen.twophase_signed(B, m, n, 200 + m)
    elif gen == "G2light":
        A, b, c = lpgen.twophase_light(B, m, n, 300 + m)
    else:
        A, b, c = lpgen.status_mix(B, m, n, 400 + m, infeasible_start=(gen == "mixneg"))
    r = oracle.solve(A, b, c, certs=True)
    for k in range(B):
        rk = {key: v[k] for key, v in r.items() if isinstance(v, np.ndarray)}
        errs = _certify(A[k], b[k], c[k], rk)
        assert not errs, (gen, k, errs)
    if gen in ("G1", "G2", "G2light"):
        assert np.all(r["status"] == oracle.OPTIMAL)
    if gen == "G1":
        assert np.all(r["iters"][:, 0] == 0)
    if gen in ("G2", "G2light"):
        assert np.all(r["iters"][:, 0] >= 1)


def test_scipy_highs_agreement():
    """scipy.optimize.linprog (HiGHS, presolve off; C-P17) on mid-size instances."""
    linprog = pytest.importorskip("scipy.optimize").linprog
    cases = [lpgen.signed_bounded(6, 40, 40, 17), lpgen.twophase_signed(4, 40, 40, 18),
             lpgen.status_mix(20, 10, 10, 19, infeasible_start=True)]
    for A, b, c in cases:
        r = oracle.solve(A, b, c)
        for k in range(A.shape[0]):
            h = linprog(-c[k], A_ub=A[k], b_ub=b[k], bounds=(0, None), method="highs",
                        options={"presolve": False})
            code = {0: oracle.OPTIMAL, 2: oracle.INFEASIBLE, 3: oracle.UNBOUNDED}[h.status]
            assert r["status"][k] == code
            if code == oracle.OPTIMAL:
                assert abs(r["obj"][k] - (-h.fun)) <= 1e-8 * max(1.0, abs(h.fun))


def test_bland_threshold_independence_degenerate():
    """G-deg (C-P20): status and optimum are properties of the LP, so they must not depend on
    the Bland threshold K (except the documented NUMERICAL breakdown, C6)."""
    for neg in (False, True):
        A, b, c = lpgen.degenerate(3000, 8, 8, 20 + neg, negative_b=neg)
        rs = [oracle.solve(A, b, c, bland_after=K) for K in (0, 1, 3)]
        ok = np.all([r["status"] != oracle.NUMERICAL for r in rs], axis=0)
        for r in rs[1:]:
            assert np.array_equal(r["status"][ok], rs[0]["status"][ok])
            opt = ok & (r["status"] == oracle.OPTIMAL)
            np.testing.assert_allclose(r["obj"][opt], rs[0]["obj"][opt], rtol=1e-9, atol=1e-9)
        # the coverage generator really reaches drive-outs (phase-I pivots > k is impossible
        # without them only if ... ) -- checked via certificates instead:
        r = oracle.solve(A, b, c, certs=True)
        for k in range(0, A.shape[0], 7):
            rk = {key: v[k] for key, v in r.items() if isinstance(v, np.ndarray)}
            if rk["status"] in (oracle.OPTIMAL, oracle.INFEASIBLE, oracle.UNBOUNDED):
                assert not _certify(A[k], b[k], c[k], rk)


def test_degenerate_brute_force():
    """G-deg at m,n <= 4 against exact enumeration: catches a missing drive-out (C9/C-P19)."""
    g_small = [lpgen.degenerate(300, m, n, 30 + 4 * m + n, negative_b=True)
               for m, n in ((2, 2), (3, 3), (4, 3), (3, 4), (4, 4))]
    for A, b, c in g_small:
        r = oracle.solve(A, b, c)
        for k in range(A.shape[0]):
            st, obj = brute_force(A[k].tolist(), b[k].tolist(), c[k].tolist())
            code = {"optimal": 0, "unbounded": 1, "infeasible": 2}[st]
            assert r["status"][k] == code
            if st == "optimal":
                assert abs(r["obj"][k] - float(obj)) <= 1e-9 * max(1.0, abs(float(obj)))


def test_thread_invariance():
    """Scheduling invariance: 1 thread vs many threads, bit-identical."""
    A, b, c = lpgen.status_mix(500, 12, 12, 21, infeasible_start=True)
    r1 = oracle.solve(A, b, c, threads=1)
    r8 = oracle.solve(A, b, c, threads=8)
    for k in ("status", "iters"):
        assert np.array_equal(r1[k], r8[k])
    assert np.array_equal(r1["obj"].view(np.int64), r8["obj"].view(np.int64))


# ---------------- hyperbox (Eq. 6) ----------------

def test_hyperbox_golden():
    for cs in GOLD["hyperbox"]["cases"]:
        r = oracle.hyperbox(np.array(cs["lo"], float), np.array(cs["hi"], float),
                            np.array([cs["l"]], float))
        assert r["status"][0] == oracle.OPTIMAL
        assert r["obj"][0] == cs["obj"]
        np.testing.assert_array_equal(r["x"][0], cs["x"])


def test_hyperbox_spec_batch():
    """box [0,1]^2, directions +-e1, +-e2 -> [1, 0, 1, 0]."""
    r = oracle.hyperbox(np.zeros(2), np.ones(2), lpgen.box_directions(2))
    np.testing.assert_array_equal(r["obj"], [1.0, 0.0, 1.0, 0.0])


def test_hyperbox_vertex_brute_force():
    """max over all 2^n box vertices, exact rationals, equals Eq. 6 (C-P14); the maximiser is
    the vertex Eq. 6 names whenever no l_i is 0."""
    g = lpgen.rng(14)
    for _ in range(120):
        n = int(g.integers(1, 9))
        lo = g.uniform(-2.0, 1.0, n)
        hi = lo + g.uniform(0.0, 2.0, n)
        l = g.standard_normal(n)
        r = oracle.hyperbox(lo, hi, l[None, :])
        best, arg = None, None
        for v in product((0, 1), repeat=n):
            pt = [hi[i] if v[i] else lo[i] for i in range(n)]
            val = sum(Fraction(l[i]) * Fraction(pt[i]) for i in range(n))
            if best is None or val > best:
                best, arg = val, pt
        bound = n * 2.0 ** -52 * float(sum(abs(Fraction(l[i]) * Fraction(arg[i])) for i in range(n)))
        assert abs(r["obj"][0] - float(best)) <= bound + 1e-300
        np.testing.assert_array_equal(r["x"][0], arg)


def test_hyperbox_properties():
    """Positive homogeneity (exact for powers of two) and box monotonicity."""
    lo, hi, dirs = lpgen.hyperbox(5000, 7, 15)
    r = oracle.hyperbox(lo, hi, dirs)
    r4 = oracle.hyperbox(lo, hi, 4.0 * dirs)
    np.testing.assert_array_equal(r4["obj"], 4.0 * r["obj"])
    r_big = oracle.hyperbox(lo - 0.5, hi + 0.25, dirs)
    assert np.all(r_big["obj"] >= r["obj"])
    empty = oracle.hyperbox(hi, lo, dirs[:3])
    assert np.all(empty["status"] == oracle.INFEASIBLE)


def test_hyperbox_equals_simplex_encoding():
    """With lo >= 0 the box LP is also max l.x s.t. x <= hi, -x <= -lo, x >= 0: the two-phase
    simplex oracle must give the same value (C-P14)."""
    g = lpgen.rng(22)
    for n in (2, 5, 9):
        lo = g.uniform(0.0, 1.0, n)
        hi = lo + g.uniform(0.1, 1.0, n)
        dirs = lpgen.oct_directions(n)
        A = np.concatenate([np.eye(n), -np.eye(n)])[None].repeat(len(dirs), 0)
        bb = np.concatenate([hi, -lo])[None].repeat(len(dirs), 0)
        rs = oracle.solve(A, bb, dirs)
        rh = oracle.hyperbox(lo, hi, dirs)
        assert np.all(rs["status"] == oracle.OPTIMAL)
        np.testing.assert_allclose(rs["obj"], rh["obj"], rtol=1e-12, atol=1e-12)


def test_residual_on_config_shapes():
    """Primal residual <= 1e-9 absolute at the cfg1 shape (full batch) and samples of cfg2."""
    A, b, c = lpgen.make_config("cfg1")
    r = oracle.solve(A, b, c)
    assert np.all(r["status"] == oracle.OPTIMAL)
    for k in range(0, 1000, 10):
        assert primal_residual(A[k], b[k], r["x"][k]) <= 1e-9


# LPB_NUMERICAL (reading R2 / C6): phase I reporting "unbounded" is impossible in exact
# arithmetic -- the phase-I objective -sum(artificials) is bounded above by 0 -- so the branch
# fires only when fp64 rounding under an aggressive Bland threshold leaves an improving
# phase-I column without a positive pivot candidate.  Pinned on seeded degenerate LPs where it
# happens: the same LPs under the default threshold end with a certified status, and HiGHS
# (presolve off, C-P17) finds them feasible or proves infeasibility -- never unbounded in
# phase I.
NUMERICAL_CASES = [(40, 3, 207), (43, 3, 147), (43, 2, 154), (47, 3, 81)]


@pytest.mark.parametrize("seed,K,k", NUMERICAL_CASES)
def test_numerical_status_is_a_rounding_artifact(seed, K, k):
    linprog = pytest.importorskip("scipy.optimize").linprog
    A, b, c = lpgen.degenerate(300, 100, 100, seed, negative_b=True)
    A1, b1, c1 = A[k:k + 1], b[k:k + 1], c[k:k + 1]
    o = oracle.solve(A1, b1, c1, bland_after=K)
    assert o["status"][0] == oracle.NUMERICAL and o["iters"][0][1] == 0  # ended in phase I
    assert np.isnan(o["obj"][0]) and np.all(np.isnan(o["x"][0]))
    # another threshold (the default, else Bland after every degenerate pivot) solves the same
    # LP to a certified outcome
    for Kalt in (0, 1):
        od = oracle.solve(A1, b1, c1, bland_after=Kalt, certs=True)
        st = od["status"][0]
        if st != oracle.NUMERICAL:
            break
    assert st in (oracle.OPTIMAL, oracle.INFEASIBLE, oracle.UNBOUNDED)
    if st == oracle.OPTIMAL:
        assert not check_optimal(A1[0], b1[0], c1[0], od["obj"][0], od["x"][0], od["y"][0])
    elif st == oracle.INFEASIBLE:
        assert not check_infeasible(A1[0], b1[0], od["y"][0])
    h = linprog(-c1[0], A_ub=A1[0], b_ub=b1[0], bounds=(0, None), method="highs",
                options={"presolve": False})
    assert h.status in (0, 2, 3)  # optimal / infeasible / unbounded: a real LP status
    assert (h.status == 2) == (st == oracle.INFEASIBLE)
