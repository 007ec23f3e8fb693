"""Solution checkers computed from the ORIGINAL data (A, b, c) in long double (test-only).

These pin results to LP duality, not to any implementation:
  OPTIMAL    : x >= 0, A x <= b (primal residual), c.x = obj; y >= 0, A^T y >= c, b.y = obj
  INFEASIBLE : Farkas y >= 0, A^T y >= 0, b.y < 0
  UNBOUNDED  : a feasible point xb and a ray d >= 0, A d <= 0, c.d > 0
"""
from __future__ import annotations

import numpy as np

LD = np.longdouble


def primal_residual(A, b, x):
    """max(0, max_i(A_i x - b_i), max_j(-x_j))  (SPEC.md:61-65 evaluate; C20 absolute form)."""
    A = np.asarray(A, LD)
    r = A @ np.asarray(x, LD) - np.asarray(b, LD)
    return float(max(LD(0), np.max(r) if r.size else LD(0), np.max(-np.asarray(x, LD))))


def scaled_primal_residual(A, b, x):
    A = np.asarray(A, LD)
    x = np.asarray(x, LD)
    r = A @ x - np.asarray(b, LD)
    scale = np.maximum(LD(1), np.maximum(np.abs(np.asarray(b, LD)), np.abs(A) @ np.abs(x)))
    return float(max(LD(0), np.max(r / scale), np.max(-x)))


def check_optimal(A, b, c, obj, x, y=None, tol=1e-9):
    A = np.asarray(A, LD)
    b = np.asarray(b, LD)
    c = np.asarray(c, LD)
    x = np.asarray(x, LD)
    errs = []
    if primal_residual(A, b, x) > tol * 10 and scaled_primal_residual(A, b, x) > tol:
        errs.append(f"primal residual {primal_residual(A, b, x):.3e}")
    cx = float(c @ x)
    if abs(cx - obj) > tol * max(1.0, abs(obj)) * 10:
        errs.append(f"c.x={cx!r} obj={obj!r}")
    if y is not None:
        y = np.asarray(y, LD)
        scale = 1.0 + float(np.max(np.abs(A).T @ np.abs(y))) + float(np.max(np.abs(c)))
        if float(np.min(y)) < -tol * scale:
            errs.append(f"dual y min {float(np.min(y)):.3e}")
        dres = float(np.max(c - A.T @ y))
        if dres > tol * scale:
            errs.append(f"dual residual {dres:.3e}")
        by = float(b @ y)
        if abs(by - obj) > tol * max(1.0, abs(obj)) * 100:
            errs.append(f"gap b.y={by!r} obj={obj!r}")
    return errs


def check_infeasible(A, b, y, tol=1e-9):
    A = np.asarray(A, LD)
    b = np.asarray(b, LD)
    y = np.asarray(y, LD)
    scale = 1.0 + float(np.max(np.abs(A).T @ np.abs(y)))
    errs = []
    if float(np.min(y)) < -tol * scale:
        errs.append("farkas y < 0")
    if float(np.min(A.T @ y)) < -tol * scale:
        errs.append(f"farkas A^T y min {float(np.min(A.T @ y)):.3e}")
    if not float(b @ y) < -tol:
        errs.append(f"farkas b.y={float(b @ y)!r}")
    return errs


def check_unbounded(A, b, c, xb, d, tol=1e-9):
    A = np.asarray(A, LD)
    c = np.asarray(c, LD)
    d = np.asarray(d, LD)
    errs = []
    if primal_residual(A, b, xb) > tol * 10 and scaled_primal_residual(A, b, xb) > tol:
        errs.append(f"basic point infeasible {primal_residual(A, b, xb):.3e}")
    scale = 1.0 + float(np.max(np.abs(A) @ np.abs(d)))
    if float(np.min(d)) < -tol * scale:
        errs.append("ray d < 0")
    if float(np.max(A @ d)) > tol * scale:
        errs.append(f"ray A d max {float(np.max(A @ d)):.3e}")
    if not float(c @ d) > tol:
        errs.append(f"ray c.d={float(c @ d)!r}")
    return errs
