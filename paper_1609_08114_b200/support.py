"""Support-function sampling through the batched solver.

The paper's application (§7): "sampling the support function of convex
sets which are convex polytopes, is a linear programming problem" -- one LP per template
direction l, all over the SAME set.  Two engines, both entirely in this package's kernels:

  closed form  (box sets only): Eq. 6, h_B(l) = sum_i l_i * (l_i < 0 ? lo_i : hi_i)
               (PAPER.md:291-300), the hyperbox kernel H with one shared box;
  simplex      any polytope {x : A x <= b}: one general LP per direction with A and b shared
               by the whole batch (LPB_SHARED_AB).  A box is handed to it as a polytope over
               free variables split x = x+ - x-:  [I -I; -I I] [x+; x-] <= [hi; -lo],
               objective (l, -l), so the LP optimum is h_B(l) itself (two-phase whenever some
               lo_i > 0 or hi_i < 0) and no arithmetic happens outside the kernels.

The direction templates (box / oct / random) are lpgen's.
"""
from __future__ import annotations

import numpy as np

from . import lpb

ENGINES = ("closed-form", "simplex")


def _device(a):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def box_as_polytope(lo, hi):
    """(A, b) of the split-variable encoding of the box [lo, hi] (x = x+ - x-, x+- >= 0)."""
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    n = lo.shape[0]
    eye = np.eye(n)
    A = np.block([[eye, -eye], [-eye, eye]])
    b = np.concatenate([hi, -lo])
    return A, b


def support_polytope(A, b, dirs, *, want_x=False, **opts):
    """max l.x s.t. A x <= b, x >= 0 for every direction l (row of dirs), the constraint
    system shared by the batch.  Returns dict(status, obj[, x], iters) as torch CUDA tensors
    (copies), plus the device solve time in ms."""
    d = _device(dirs)
    B, n = d.shape
    At, bt = _device(A), _device(b)
    m = At.shape[0]
    s = lpb.Solver(B, m, n, lpb.GENERAL, **opts)
    s.solve_device(At, bt, d, shared_ab=True, want_x=want_x, sync=True)
    out = {k: v.clone() for k, v in s.device_results(want_x).items()}
    out["ms"] = s.timing()[0]
    s.close()
    return out


def support_box(lo, hi, dirs, engine="closed-form", **opts):
    """Support function of the box [lo, hi] along every row of dirs.
    engine="closed-form": the hyperbox kernel (Eq. 6); engine="simplex": the general simplex
    on the split-variable polytope (box_as_polytope).  Returns dict(status, obj, ms)."""
    if engine == "closed-form":
        import torch
        d = _device(dirs)
        B, n = d.shape
        box = _device(np.concatenate([np.asarray(hi, np.float64), -np.asarray(lo, np.float64)]))
        s = lpb.Solver(B, 2 * n, n, lpb.HYPERBOX, **opts)
        s.solve_device(None, box, d, shared_box=True, want_x=False, sync=True)
        r = s.device_results(want_x=False)
        out = {"status": r["status"].clone(), "obj": r["obj"].clone(), "ms": s.timing()[0]}
        s.close()
        return out
    if engine == "simplex":
        import torch
        A, b = box_as_polytope(lo, hi)
        d = _device(dirs)
        r = support_polytope(A, b, torch.cat([d, -d], dim=1), **opts)
        return {"status": r["status"], "obj": r["obj"], "ms": r["ms"], "iters": r["iters"]}
    raise ValueError(f"engine must be one of {ENGINES}")
