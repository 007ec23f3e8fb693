"""Pins of the oracle's RPC entering rule ("we choose a
random index having a positive coefficient from the last row"; reading R15 in DESIGN.md).

What the paper fixes, and what these tests check without re-typing the score formula:
  * the optimum is rule-independent: status and objective equal LPC's, and every RPC result
    carries an LP duality certificate computed from the original data (checks.py);
  * the entering column is drawn uniformly from the positive-coefficient columns (an LP whose
    first entering variable is visible in x, tested with a chi-square bound);
  * the draw is a function of (seed, LP index, pivot count) only:
    same seed -> bit-identical results, different seed -> different pivot paths;
  * Bland's fallback still terminates the degenerate cycling example under RPC;
  * the paper's observation that LPC needs fewer iterations on average.
"""
import json
import os

import numpy as np
import pytest

import lpgen
import oracle
from checks import check_infeasible, check_optimal, check_unbounded

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "lp_fixtures.json")))


def _certify(A, b, c, r):
    st = r["status"]
    if st == oracle.OPTIMAL:
        return check_optimal(A, b, c, r["obj"], r["x"], r["y"])
    if st == oracle.INFEASIBLE:
        return check_infeasible(A, b, r["y"])
    if st == oracle.UNBOUNDED:
        return check_unbounded(A, b, c, r["xb"], r["ray"])
    return [f"status {st}"]


@pytest.mark.parametrize("gen,m,n,B", [
    ("G1", 5, 5, 300), ("G1", 28, 28, 60), ("G2", 8, 8, 200), ("G2", 30, 30, 10),
    ("mix", 6, 6, 300), ("mixneg", 6, 6, 300), ("deg", 8, 8, 300),
])
def test_rpc_same_optimum_and_certified(gen, m, n, B):
    if gen == "G1":
        A, b, c = lpgen.signed_bounded(B, m, n, 500 + m)
    elif gen == "G2":
        A, b, c = lpgen.twophase_signed(B, m, n, 600 + m)
    elif gen == "deg":
        A, b, c = lpgen.degenerate(B, m, n, 700 + m)
    else:
        A, b, c = lpgen.status_mix(B, m, n, 800 + m, infeasible_start=(gen == "mixneg"))
    lpc = oracle.solve(A, b, c)
    rpc = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=12345, certs=True)
    assert np.array_equal(lpc["status"], rpc["status"])
    opt = lpc["status"] == oracle.OPTIMAL
    err = np.abs(lpc["obj"][opt] - rpc["obj"][opt]) / np.maximum(1.0, np.abs(lpc["obj"][opt]))
    assert err.size == 0 or err.max() <= 1e-9
    for k in range(B):
        rk = {key: v[k] for key, v in rpc.items() if isinstance(v, np.ndarray)}
        assert not _certify(A[k], b[k], c[k], rk), (gen, k)


def test_rpc_first_choice_is_uniform():
    """max sum_j x_j s.t. sum_j x_j <= 1: every x_j has reduced cost 1 at the slack basis and
    whichever enters first ends the solve (x = e_j).  LPC takes j = 0 (lowest index on ties,
    R5); RPC must pick each of the n columns with probability 1/n."""
    n, B = 6, 6000
    A = np.ones((B, 1, n))
    b = np.ones((B, 1))
    c = np.ones((B, n))
    lpc = oracle.solve(A, b, c)
    assert np.all(lpc["x"][:, 0] == 1.0)
    r = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=2024)
    assert np.all(r["status"] == oracle.OPTIMAL) and np.all(r["obj"] == 1.0)
    assert np.all(r["iters"][:, 1] == 1)
    first = np.argmax(r["x"], axis=1)
    assert np.all(r["x"][np.arange(B), first] == 1.0)
    counts = np.bincount(first, minlength=n)
    expect = B / n
    chi2 = float(((counts - expect) ** 2 / expect).sum())
    assert chi2 < 25.7, counts  # chi-square, 5 dof, p = 1e-4


def test_rpc_second_pivot_uniform():
    """max x0 + 2 x1 + 3 x2 s.t. x0 + x1 + x2 <= 3 (optimum x = (0, 0, 3), obj 9).  All three
    columns start positive.  x2 first ends in 1 pivot; x1 first forces x2 next (2 pivots);
    x0 first leaves {x1, x2} positive and a second uniform draw decides between 2 and 3
    pivots.  Hence P(1, 2, 3 pivots) = (1/3, 1/2, 1/6) -- the pivot counter keys a fresh
    uniform draw at every pivot."""
    B = 6000
    A = np.ones((B, 1, 3))
    b = np.full((B, 1), 3.0)
    c = np.array([[1.0, 2.0, 3.0]]).repeat(B, 0)
    r = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=7)
    assert np.all(r["status"] == oracle.OPTIMAL) and np.all(r["obj"] == 9.0)
    counts = np.bincount(r["iters"][:, 1], minlength=4)[1:]
    assert counts.sum() == B
    expect = B * np.array([1 / 3, 1 / 2, 1 / 6])
    chi2 = float(((counts - expect) ** 2 / expect).sum())
    assert chi2 < 18.4, counts  # chi-square, 2 dof, p = 1e-4
    assert np.all(oracle.solve(A, b, c)["iters"][:, 1] == 1)  # LPC: x2 (largest) enters


def test_rpc_determinism_and_seed_dependence():
    A, b, c = lpgen.signed_bounded(200, 20, 20, 31)
    r1 = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=99)
    r2 = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=99, threads=1)
    for key in ("status", "iters"):
        assert np.array_equal(r1[key], r2[key])
    assert np.array_equal(r1["obj"], r2["obj"]) and np.array_equal(r1["x"], r2["x"])
    r3 = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=100)
    assert np.any(r1["iters"] != r3["iters"])
    # the LP index keys the stream: the same LP at two batch positions takes different paths
    A2, b2, c2 = (np.repeat(v[:1], 64, axis=0) for v in (A, b, c))
    r4 = oracle.solve(A2, b2, c2, pivot_rule="RPC", rpc_seed=99)
    assert len(np.unique(r4["iters"][:, 1])) > 1
    assert np.array_equal(r4["iters"][0], r1["iters"][0])


def test_rpc_bland_fallback_terminates_chvatal():
    ch = GOLD["chvatal_cycling"]
    A, b, c = (np.array([ch[k]], float) for k in ("A", "b", "c"))
    A, b, c = (np.repeat(v, 200, axis=0) for v in (A, b, c))
    r = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=3, bland_after=2)
    assert np.all(r["status"] == oracle.OPTIMAL) and np.all(r["obj"] == 1.0)


def test_lpc_fewer_iterations_than_rpc_on_average():
    """"in most cases, the LPC rule converges to the optimum in less number of
    simplex iterations compared to the RPC rule" -- an average-case statement; at 28x28 G1
    the gap is about 2x, far outside sampling noise over 300 LPs."""
    A, b, c = lpgen.signed_bounded(300, 28, 28, 41)
    lpc = oracle.solve(A, b, c)["iters"][:, 1].mean()
    rpc = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=1)["iters"][:, 1].mean()
    assert rpc > 1.2 * lpc, (lpc, rpc)


def test_rpc_lp_index_base_selects_the_stream():
    """lp_index_base = k makes a one-LP batch follow LP k's draws in a larger batch."""
    A, b, c = lpgen.signed_bounded(40, 12, 12, 51)
    full = oracle.solve(A, b, c, pivot_rule="RPC", rpc_seed=8)
    for k in (0, 7, 39):
        one = oracle.solve(A[k:k + 1], b[k:k + 1], c[k:k + 1], pivot_rule="RPC", rpc_seed=8,
                           lp_index_base=k)
        assert np.array_equal(one["iters"][0], full["iters"][k])
        assert one["obj"][0] == full["obj"][k] and np.array_equal(one["x"][0], full["x"][k])
