"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and compare it with
the oracle element by element."""
from __future__ import annotations

import numpy as np

import oracle
from checks import primal_residual, scaled_primal_residual

TOL_OBJ = 1e-9  # BASELINE.json north_star: objective within 1e-9 * max(1, |obj|)
TOL_RES = 1e-9  # primal residual (absolute; scaled form as documented fallback, C20)


def dev_lib():
    """The development build of the library (devbuild/, build.py --dev): the product
    liblpb.so plus diagnostic entry points (include/dev/lpb_selftest.h) and the A/B switches
    read from the environment.  Tests use it only for those diagnostics."""
    import ctypes
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "devbuild", "paper_1609_08114_b200", "liblpb.so")
    assert os.path.exists(path), "development build missing: python paper_1609_08114_b200/build.py --dev"
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    lib.lpb_selftest_div.argtypes = [P, P, P, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
    lib.lpb_selftest_div.restype = ctypes.c_int
    return lib


DEV_ROOT = "devbuild"  # sys.path entry (relative to the repo) whose package is the dev build


def gpu_solve(A, b, c, *, path="device", want_x=True, **opts):
    import torch

    from paper_1609_08114_b200 import lpb
    if path == "device":
        At = torch.from_numpy(np.ascontiguousarray(A)).cuda()
        bt = torch.from_numpy(np.ascontiguousarray(b)).cuda()
        ct = torch.from_numpy(np.ascontiguousarray(c)).cuda()
        shared = At.dim() == 2  # one constraint system for the batch (LPB_SHARED_AB)
        B, n = ct.shape
        m = At.shape[-2]
        s = lpb.Solver(B, m, n, lpb.GENERAL, **opts)
        s.solve_device(At, bt, ct, want_x=want_x, sync=True, shared_ab=shared)
        r = {k: v.cpu().numpy() for k, v in s.device_results(want_x).items()}
        nl, klass = s.launch_info()
        cl, grid = s.launch_shape()
        r["launch"] = dict(launches=nl, **{"class": klass}, cluster=cl, grid=grid)
        s.close()
        return r
    r = lpb.solve(A, b, c, want_x=want_x, **opts)
    return r


def compare(A, b, c, g, o, *, bits=True, check_x=True, sample=None):
    """Parity of GPU result g with oracle result o on the same LPs.
    Always: status identical; OPTIMAL objective within TOL_OBJ; x feasible (residual) and
    c.x == obj.  With ``bits``: iteration counts identical and objective/x equal as fp64
    values (the condensed tableau reproduces the oracle's full-tableau arithmetic)."""
    idx = np.arange(len(o["status"])) if sample is None else np.asarray(sample)
    gs, os_ = g["status"][idx], o["status"]
    bad = np.nonzero(gs != os_)[0]
    assert bad.size == 0, f"status mismatch at {idx[bad[:10]]}: gpu {gs[bad[:10]]} oracle {os_[bad[:10]]}"
    opt = os_ == oracle.OPTIMAL
    go, oo = g["obj"][idx], o["obj"]
    err = np.abs(go[opt] - oo[opt]) / np.maximum(1.0, np.abs(oo[opt]))
    assert err.size == 0 or err.max() <= TOL_OBJ, f"obj rel err {err.max():.3e}"
    # non-optimal sentinels
    nonopt = ~opt
    assert np.all(np.isposinf(go[nonopt & (os_ == oracle.UNBOUNDED)]))
    assert np.all(np.isneginf(go[nonopt & (os_ == oracle.INFEASIBLE)]))
    assert np.all(np.isnan(go[nonopt & (os_ >= oracle.ITER_LIMIT)]))
    if check_x and g.get("x") is not None:
        gx = g["x"][idx]
        assert np.all(np.isnan(gx[nonopt]))
        for t in np.nonzero(opt)[0][:400]:
            k = idx[t]
            r = primal_residual(A[k], b[k], gx[t])
            assert r <= TOL_RES or scaled_primal_residual(A[k], b[k], gx[t]) <= TOL_RES, (k, r)
    if bits:
        gi = g["iters"][idx]
        badi = np.nonzero(np.any(gi != o["iters"], axis=1))[0]
        assert badi.size == 0, f"iteration mismatch at {idx[badi[:10]]}: gpu {gi[badi[:5]]} oracle {o['iters'][badi[:5]]}"
        badb = np.nonzero(opt & (go != oo))[0]
        assert badb.size == 0, f"objective bits differ at {idx[badb[:10]]}"
        if check_x and g.get("x") is not None:
            gx = g["x"][idx]
            assert np.array_equal(gx[opt], o["x"][opt]), "x differs"
