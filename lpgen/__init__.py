"""Seeded synthetic LP batch generators (shared input source for the oracle and the CUDA path).

This module holds NO simplex / hyperbox arithmetic: it only draws the input arrays
(A, b, c, box, directions) that both sides consume.  Every generator uses
``numpy.random.Generator(PCG64(seed))`` with batch-vectorised draws in the order stated
in SURVEY.md §8(d), because the paper only says the LPs were "generated randomly"
(D2 "Implementation Strategy"; reading C17 in DESIGN.md).

Layouts (the C-ABI's, include/lpb.h):
  A : float64 [B, m, n]  row-major, LP-contiguous
  b : float64 [B, m]
  c : float64 [B, n]
Hyperbox inputs: ``lo, hi`` float64 [n] (one shared box, "the same LPs ...
with large number of different objective functions") and ``dirs`` float64 [B, n].
"""
from __future__ import annotations

import math

import numpy as np

__all__ = [
    "rng",
    "signed_bounded",
    "twophase_signed",
    "twophase_light",
    "hyperbox",
    "oct_directions",
    "box_directions",
    "status_mix",
    "degenerate",
    "klee_minty",
    "chvatal_cycling",
    "shared_polytope",
    "CONFIGS",
    "make_config",
    "kmax_bound",
]


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def signed_bounded(B: int, m: int, n: int, seed: int):
    """G1 (type-1 workload).  A ~ U[-10,10), row 0 replaced by a positive
    budget row U[1,10) so every LP is bounded, b ~ U[1,100) (> 0: slack basis feasible,
    PAPER.md:76 "initial basic solution ... feasible"), c ~ U[-10,10).  SPEC.md:391 ranges."""
    g = rng(seed)
    A = g.uniform(-10.0, 10.0, size=(B, m, n))
    A[:, 0, :] = g.uniform(1.0, 10.0, size=(B, n))
    b = g.uniform(1.0, 100.0, size=(B, m))
    c = g.uniform(-10.0, 10.0, size=(B, n))
    return A, b, c


def twophase_signed(B: int, m: int, n: int, seed: int):
    """G2 (type-2 workload).  Feasible by construction (x* is feasible) with
    kk = ceil(m/4) covering rows (SPEC.md:357 count) whose b < 0, so the slack basis is
    infeasible and phase I is needed.  Non-cover rows get
    b_i = max(A_i x*, 0) + U[1,100) (>= 1), covering rows b_i = -(Q_i x*) + U[0,1).

    Draw order: A U[-10,10)^{BxMxN}; budget U[1,10)^{BxN}; x* U[0,1)^{BxN};
    slack U[1,100)^{BxM}; keys U[0,1)^{Bx(M-1)}; cover U[1,10)^{BxKKxN};
    cover slack U[0,1)^{BxKK}; c U[-10,10)^{BxN}."""
    g = rng(seed)
    kk = min(int(math.ceil(m / 4)), m - 1)
    A = g.uniform(-10.0, 10.0, size=(B, m, n))
    A[:, 0, :] = g.uniform(1.0, 10.0, size=(B, n))
    xs = g.uniform(0.0, 1.0, size=(B, n))
    slack = g.uniform(1.0, 100.0, size=(B, m))
    keys = g.uniform(0.0, 1.0, size=(B, max(m - 1, 0)))
    cover = g.uniform(1.0, 10.0, size=(B, max(kk, 0), n))
    cover_slack = g.uniform(0.0, 1.0, size=(B, max(kk, 0)))
    c = g.uniform(-10.0, 10.0, size=(B, n))
    # max(., 0) keeps every non-cover b_i >= 1 (x* stays feasible), so exactly kk rows start
    # infeasible, as SPEC.md:357 states ("forces ceil(m/4) entries of b negative")
    b = np.maximum(np.einsum("bij,bj->bi", A, xs), 0.0) + slack
    if kk > 0:
        rows = 1 + np.argsort(keys, axis=1, kind="stable")[:, :kk]
        bi = np.arange(B)[:, None]
        A[bi, rows, :] = -cover
        b[bi, rows] = np.einsum("bkj,bj->bk", -cover, xs) + cover_slack
    return A, b, c


def twophase_light(B: int, m: int, n: int, seed: int):
    """G2' (light type-2 alternative).  m-kk packing rows P ~ U[0,1) with
    b = P x* + U[0,1)*n/8, kk covering rows -Q (Q ~ U[0,1)) with b = -(Q x*) * U[0.5,1),
    c ~ U[0,1); rows permuted per LP."""
    g = rng(seed)
    kk = int(math.ceil(m / 4))
    xs = g.uniform(0.0, 1.0, size=(B, n))
    P = g.uniform(0.0, 1.0, size=(B, m - kk, n))
    bp = np.einsum("bij,bj->bi", P, xs) + g.uniform(0.0, 1.0, size=(B, m - kk)) * (n / 8.0)
    Q = g.uniform(0.0, 1.0, size=(B, kk, n))
    bq = -np.einsum("bij,bj->bi", Q, xs) * g.uniform(0.5, 1.0, size=(B, kk))
    c = g.uniform(0.0, 1.0, size=(B, n))
    A = np.concatenate([P, -Q], axis=1)
    b = np.concatenate([bp, bq], axis=1)
    perm = np.argsort(g.uniform(0.0, 1.0, size=(B, m)), axis=1, kind="stable")
    bi = np.arange(B)[:, None]
    return np.ascontiguousarray(A[bi, perm, :]), np.ascontiguousarray(b[bi, perm]), c


def box_directions(n: int) -> np.ndarray:
    """+e1, -e1, ..., +en, -en  (SPEC.md:364-370 'box' template)."""
    d = np.zeros((2 * n, n))
    for i in range(n):
        d[2 * i, i] = 1.0
        d[2 * i + 1, i] = -1.0
    return d


def oct_directions(n: int) -> np.ndarray:
    """Box template then, for i<j lexicographic, (+,+),(+,-),(-,+),(-,-) times 1/sqrt(2):
    2n^2 unit directions.  Exercises l_i = 0 (C15)."""
    out = [box_directions(n)]
    s = 1.0 / math.sqrt(2.0)
    pairs = []
    for i in range(n):
        for j in range(i + 1, n):
            for si, sj in ((1, 1), (1, -1), (-1, 1), (-1, -1)):
                v = np.zeros(n)
                v[i] = si * s
                v[j] = sj * s
                pairs.append(v)
    if pairs:
        out.append(np.array(pairs))
    return np.concatenate(out, axis=0)


# directions beyond the template come in blocks of HB_BLOCK rows, block q drawn from its own
# stream PCG64([seed, 2, q]): any contiguous shard of a batch is generated without drawing the
# rest (multi-GPU ranks each draw only their slice of a 6M x 28 batch)
HB_BLOCK = 1 << 16


def hyperbox_box(n: int, seed: int):
    """The shared box of G3: n=5 is the five-dimensional benchmark's initial set, a box
    centred at (1,0,0,0,0) with side 0.02 (reading R14); other n:
    lo ~ U[-1,0), hi = lo + U[0.01,1) from PCG64(seed)."""
    if n == 5:
        lo = np.array([0.99, -0.01, -0.01, -0.01, -0.01])
        return lo, lo + 0.02
    g = rng(seed)
    lo = g.uniform(-1.0, 0.0, size=n)
    return lo, lo + g.uniform(0.01, 1.0, size=n)


def hyperbox_dirs(n: int, seed: int, lo: int, hi: int):
    """Rows [lo, hi) of G3's direction list: the oct template (2n^2 rows, SPEC.md:365-367,
    exercising l_i = 0) first, then row-normalised standard normals, HB_BLOCK rows per
    independently seeded block."""
    tmpl = oct_directions(n)
    t = tmpl.shape[0]
    out = np.empty((hi - lo, n))
    if lo < t:
        out[: min(hi, t) - lo] = tmpl[lo:min(hi, t)]
    a, b = max(lo, t), hi
    if a < b:
        for q in range((a - t) // HB_BLOCK, (b - 1 - t) // HB_BLOCK + 1):
            z = np.random.Generator(np.random.PCG64([seed, 2, q])).standard_normal((HB_BLOCK, n))
            z /= np.linalg.norm(z, axis=1, keepdims=True)
            g0 = t + q * HB_BLOCK  # global row of the block's first row
            s0, s1 = max(a, g0), min(b, g0 + HB_BLOCK)
            out[s0 - lo:s1 - lo] = z[s0 - g0:s1 - g0]
    return np.ascontiguousarray(out)


def hyperbox(B: int, n: int, seed: int):
    """G3 (type-3 workload).  One shared box and B
    directions (hyperbox_box, hyperbox_dirs).  Returns (lo, hi, dirs)."""
    lo, hi = hyperbox_box(n, seed)
    return lo, hi, hyperbox_dirs(n, seed, 0, B)


def status_mix(B: int, m: int, n: int, seed: int, infeasible_start: bool = False):
    """SPEC raw generator (correctness only): A, c ~ U[-10,10], b ~ U[1,100];
    with ``infeasible_start`` ceil(m/4) random rows per LP get b_i negated.  Produces a mix
    of optimal / unbounded / infeasible LPs."""
    g = rng(seed)
    A = g.uniform(-10.0, 10.0, size=(B, m, n))
    b = g.uniform(1.0, 100.0, size=(B, m))
    c = g.uniform(-10.0, 10.0, size=(B, n))
    if infeasible_start:
        kk = int(math.ceil(m / 4))
        rows = np.argsort(g.uniform(0.0, 1.0, size=(B, m)), axis=1, kind="stable")[:, :kk]
        bi = np.arange(B)[:, None]
        b[bi, rows] = -b[bi, rows]
    return A, b, c


def degenerate(B: int, m: int, n: int, seed: int, negative_b: bool = False):
    """G-deg: small-integer data that produces degenerate pivots,
    Bland-mode pivots and artificial drive-outs.  A ~ int U[-3,3], b ~ int U[0,3]
    (G5); with ``negative_b`` about 25% of b replaced by int U[-4,-1] (G6);
    c ~ int U[-3,3]."""
    g = rng(seed)
    A = g.integers(-3, 4, size=(B, m, n)).astype(np.float64)
    b = g.integers(0, 4, size=(B, m)).astype(np.float64)
    c = g.integers(-3, 4, size=(B, n)).astype(np.float64)
    if negative_b:
        mask = g.uniform(0.0, 1.0, size=(B, m)) < 0.25
        neg = g.integers(-4, 0, size=(B, m)).astype(np.float64)
        b = np.where(mask, neg, b)
    return A, b, c


def klee_minty(n: int):
    """Klee-Minty cube in Chvatal's form: max sum_j 10^(n-j) x_j s.t.
    2 sum_{j<i} 10^(i-j) x_j + x_i <= 100^(i-1), x >= 0 (1-based i, j).  Dantzig's rule
    takes exactly 2^n - 1 pivots; optimum 100^(n-1)."""
    A = np.zeros((n, n))
    b = np.zeros(n)
    c = np.zeros(n)
    for i in range(1, n + 1):
        for j in range(1, i):
            A[i - 1, j - 1] = 2.0 * 10.0 ** (i - j)
        A[i - 1, i - 1] = 1.0
        b[i - 1] = 100.0 ** (i - 1)
    for j in range(1, n + 1):
        c[j - 1] = 10.0 ** (n - j)
    return A, b, c


def chvatal_cycling():
    """Chvatal's cycling example (Linear Programming, 1983, ch. 3): pure largest-coefficient
    pivoting cycles with period 6."""
    A = np.array([[0.5, -5.5, -2.5, 9.0],
                  [0.5, -1.5, -0.5, 1.0],
                  [1.0, 0.0, 0.0, 0.0]])
    b = np.array([0.0, 0.0, 1.0])
    c = np.array([10.0, -57.0, -9.0, -24.0])
    return A, b, c


def shared_polytope(B: int, m: int, n: int, seed: int, gen: str = "G1"):
    """Many objectives over ONE polytope (the support-function sampling
    of PAPER.md:313,330 for a general polytope): A (m x n) and b (m) are LP 0 of G1 / G2 with
    this seed, and the B objectives are c ~ U[-10,10)^{B x n} drawn from PCG64([seed, 1]).
    Returns (A [m, n], b [m], c [B, n]) -- the LPB_SHARED_AB layout."""
    A, b, _ = {"G1": signed_bounded, "G2": twophase_signed}[gen](1, m, n, seed)
    c = np.random.Generator(np.random.PCG64([seed, 1])).uniform(-10.0, 10.0, size=(B, n))
    return np.ascontiguousarray(A[0]), np.ascontiguousarray(b[0]), c


# BASELINE.json configs (SURVEY §8(d) "Configs as concrete runs"; seeds cfgK -> K).  The
# "s" configs are the NEXT-1 shared-constraint variants (one polytope, B objectives).
CONFIGS = {
    "cfg1": dict(kind="general", gen="G1", B=1000, m=5, n=5, seed=1),
    "cfg2": dict(kind="general", gen="G1", B=50000, m=100, n=100, seed=2),
    "cfg3": dict(kind="general", gen="G2", B=10000, m=200, n=200, seed=3),
    "cfg4": dict(kind="hyperbox", gen="G3", B=4001000, n=5, seed=4),
    "cfg5": dict(kind="hyperbox", gen="G3", B=6003000, n=28, seed=5),
    "cfg2s": dict(kind="general", gen="G1", B=50000, m=100, n=100, seed=2, shared=True),
    "cfg3s": dict(kind="general", gen="G2", B=10000, m=200, n=200, seed=3, shared=True),
    # cfg2's workload under the RPC rule (the paper's 6.74x RPC run,
    # 50k LPs of 100-dim); the rule's seed is the config seed
    "cfg2r": dict(kind="general", gen="G1", B=50000, m=100, n=100, seed=2, rule="RPC"),
    # the paper's larger dims (fig:TimeLPplotting 300/500, PAPER.md:
    # 230-249) and its size limits (511 type-1, 340 type-2)
    "cfg6": dict(kind="general", gen="G1", B=5000, m=300, n=300, seed=6),
    "cfg7": dict(kind="general", gen="G1", B=1000, m=500, n=500, seed=7),
    "cfg8": dict(kind="general", gen="G2", B=1000, m=340, n=340, seed=8),
    # the rest of the paper's type-1 dimension sweep (fig:TimeLPplotting: 5, 28, 50, 100,
    # 300, 500) at its largest batch
    "cfg9": dict(kind="general", gen="G1", B=50000, m=28, n=28, seed=9),
    "cfg10": dict(kind="general", gen="G1", B=50000, m=50, n=50, seed=10),
    # cfg1's generator scaled to 1M LPs, where thread-per-LP (S) runs
    # and the HBM roofline is the relevant bound
    "cfg1m": dict(kind="general", gen="G1", B=1000000, m=5, n=5, seed=1),
}


def kmax_bound(name: str) -> int:
    """The most rows with b_i < 0 any LP of config `name` can have, by construction of its
    generator -- the LP "type" the paper's application knows in advance: G1
    draws b ~ U[1,100) (type 1: 0); G2 draws exactly kk = min(ceil(m/4), m-1) covering rows
    (type 2).  Passed to the solver as lpb_options.kmax_hint."""
    cfg = CONFIGS[name]
    if cfg["kind"] != "general":
        return -1
    if cfg["gen"] == "G1":
        return 0
    m = cfg["m"]
    return min(int(math.ceil(m / 4)), m - 1)


def make_config(name: str, B: int | None = None):
    """Inputs of a BASELINE.json config (optionally with a different batch size B; the
    generator, shapes and seed are kept).  General: (A, b, c); hyperbox: (lo, hi, dirs)."""
    cfg = CONFIGS[name]
    Bv = cfg["B"] if B is None else B
    if cfg["kind"] == "hyperbox":
        return hyperbox(Bv, cfg["n"], cfg["seed"])
    if cfg.get("shared"):
        return shared_polytope(Bv, cfg["m"], cfg["n"], cfg["seed"], cfg["gen"])
    gen = {"G1": signed_bounded, "G2": twophase_signed}[cfg["gen"]]
    return gen(Bv, cfg["m"], cfg["n"], cfg["seed"])


# ---- shards of a seeded batch (multi-GPU: each rank generates only its LPs) ----
# numpy's PCG64 draws exactly one 64-bit output per uniform double, so the draws of LPs
# [lo, hi) of an array drawn for the whole batch are reached with bit_generator.advance().

class _ShardDraw:
    def __init__(self, seed: int, B: int, lo: int, hi: int):
        self.bg = np.random.PCG64(seed)
        self.g = np.random.Generator(self.bg)
        self.B, self.lo, self.hi = B, lo, hi

    def uniform(self, low, high, per_lp: int, shape):
        self.bg.advance(self.lo * per_lp)
        out = self.g.uniform(low, high, size=(self.hi - self.lo,) + tuple(shape))
        self.bg.advance((self.B - self.hi) * per_lp)
        return out


def signed_bounded_shard(B: int, m: int, n: int, seed: int, lo: int, hi: int):
    """LPs [lo, hi) of signed_bounded(B, m, n, seed), bit-identical, without drawing the rest."""
    d = _ShardDraw(seed, B, lo, hi)
    A = d.uniform(-10.0, 10.0, m * n, (m, n))
    A[:, 0, :] = d.uniform(1.0, 10.0, n, (n,))
    b = d.uniform(1.0, 100.0, m, (m,))
    c = d.uniform(-10.0, 10.0, n, (n,))
    return A, b, c


def twophase_signed_shard(B: int, m: int, n: int, seed: int, lo: int, hi: int):
    """LPs [lo, hi) of twophase_signed(B, m, n, seed), bit-identical."""
    d = _ShardDraw(seed, B, lo, hi)
    kk = min(int(math.ceil(m / 4)), m - 1)
    A = d.uniform(-10.0, 10.0, m * n, (m, n))
    A[:, 0, :] = d.uniform(1.0, 10.0, n, (n,))
    xs = d.uniform(0.0, 1.0, n, (n,))
    slack = d.uniform(1.0, 100.0, m, (m,))
    keys = d.uniform(0.0, 1.0, max(m - 1, 0), (max(m - 1, 0),))
    cover = d.uniform(1.0, 10.0, max(kk, 0) * n, (max(kk, 0), n))
    cover_slack = d.uniform(0.0, 1.0, max(kk, 0), (max(kk, 0),))
    c = d.uniform(-10.0, 10.0, n, (n,))
    b = np.maximum(np.einsum("bij,bj->bi", A, xs), 0.0) + slack
    if kk > 0:
        Bs = hi - lo
        rows = 1 + np.argsort(keys, axis=1, kind="stable")[:, :kk]
        bi = np.arange(Bs)[:, None]
        A[bi, rows, :] = -cover
        b[bi, rows] = np.einsum("bkj,bj->bk", -cover, xs) + cover_slack
    return A, b, c


def make_config_shard(name: str, B: int, lo: int, hi: int):
    """LPs [lo, hi) of config `name` drawn for a batch of B (general configs are drawn
    shard-locally, hyperbox directions block by block)."""
    cfg = CONFIGS[name]
    if cfg["kind"] == "hyperbox":
        lo_b, hi_b = hyperbox_box(cfg["n"], cfg["seed"])
        return lo_b, hi_b, hyperbox_dirs(cfg["n"], cfg["seed"], lo, hi)
    if cfg.get("shared"):
        A, b, _ = shared_polytope(1, cfg["m"], cfg["n"], cfg["seed"], cfg["gen"])
        bg = np.random.PCG64([cfg["seed"], 1])
        g = np.random.Generator(bg)
        bg.advance(lo * cfg["n"])
        return A, b, g.uniform(-10.0, 10.0, size=(hi - lo, cfg["n"]))
    f = {"G1": signed_bounded_shard, "G2": twophase_signed_shard}[cfg["gen"]]
    return f(B, cfg["m"], cfg["n"], cfg["seed"], lo, hi)
