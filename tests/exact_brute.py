"""Exact-rational brute force for tiny LPs (test-only pin for the oracle).

max c.x s.t. A x <= b, x >= 0 with m, n <= 4, in Python ``fractions`` (no rounding):
  * feasible iff some vertex of P = {A x <= b, x >= 0} exists (P is pointed because x >= 0);
  * unbounded iff feasible and max{c.d : d >= 0, A d <= 0, 1.d = 1} > 0 (the recession cone
    cut by a normalising plane is a bounded polytope: enumerate its vertices);
  * otherwise the optimum is the max of c.x over the vertices of P.
Everything is linear algebra over Q written out here; nothing is shared with oracle/ or the
CUDA path.
"""
from __future__ import annotations

from fractions import Fraction
from itertools import combinations


def _solve_square(M, r):
    """Gauss-Jordan over Q; returns the unique solution or None if singular."""
    n = len(M)
    a = [list(M[i]) + [r[i]] for i in range(n)]
    for col in range(n):
        piv = next((i for i in range(col, n) if a[i][col] != 0), None)
        if piv is None:
            return None
        a[col], a[piv] = a[piv], a[col]
        p = a[col][col]
        a[col] = [v / p for v in a[col]]
        for i in range(n):
            if i != col and a[i][col] != 0:
                f = a[i][col]
                a[i] = [vi - f * vc for vi, vc in zip(a[i], a[col])]
    return [a[i][n] for i in range(n)]


def _vertices(G, h, eq=None):
    """Vertices of {z : G z <= h} (optionally with one equality row eq = (g, h0))."""
    n = len(G[0])
    need = n - (1 if eq else 0)
    out = []
    for S in combinations(range(len(G)), need):
        M = [G[i] for i in S]
        r = [h[i] for i in S]
        if eq:
            M = M + [eq[0]]
            r = r + [eq[1]]
        z = _solve_square(M, r)
        if z is None:
            continue
        if all(sum(gi * zi for gi, zi in zip(G[k], z)) <= h[k] for k in range(len(G))):
            out.append(z)
    return out


def brute_force(A, b, c):
    """Returns (status, obj) with status in {'optimal','unbounded','infeasible'} and obj an
    exact Fraction (None unless optimal)."""
    m, n = len(A), len(A[0])
    Aq = [[Fraction(v) for v in row] for row in A]
    bq = [Fraction(v) for v in b]
    cq = [Fraction(v) for v in c]
    # P: A x <= b, -x <= 0
    G = Aq + [[Fraction(-1 if j == k else 0) for j in range(n)] for k in range(n)]
    h = bq + [Fraction(0)] * n
    V = _vertices(G, h)
    if not V:
        return "infeasible", None
    # recession cone: A d <= 0, -d <= 0, sum d = 1
    G2 = Aq + [[Fraction(-1 if j == k else 0) for j in range(n)] for k in range(n)]
    h2 = [Fraction(0)] * (m + n)
    R = _vertices(G2, h2, eq=([Fraction(1)] * n, Fraction(1)))
    if any(sum(ci * di for ci, di in zip(cq, d)) > 0 for d in R):
        return "unbounded", None
    return "optimal", max(sum(ci * xi for ci, xi in zip(cq, x)) for x in V)
