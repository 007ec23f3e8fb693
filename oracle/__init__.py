"""ctypes wrapper of the CPU fp64 oracle (oracle/lpb_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs, never by the product package
(paper_1609_08114_b200/), which fails loudly without its CUDA library instead.

Each function mirrors one C entry point; see lpb_oracle.c for the paper passages followed.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lpb_oracle.c")
_LIB = os.path.join(_HERE, "liblpb_oracle.so")
_lock = threading.Lock()
_lib = None

OPTIMAL, UNBOUNDED, INFEASIBLE, ITER_LIMIT, NUMERICAL = range(5)


class OracleOpts(ctypes.Structure):
    _fields_ = [
        ("eps_enter", ctypes.c_double),
        ("eps_piv", ctypes.c_double),
        ("eps_phase1", ctypes.c_double),
        ("max_iter", ctypes.c_int),
        ("bland_after", ctypes.c_int),
        ("pivot_rule", ctypes.c_int),
        ("rpc_seed", ctypes.c_uint64),
        ("lp_base", ctypes.c_int64),
    ]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc: -O2 -ffp-contract=off (no implicit FMA contraction),
    explicit fma() from libm, no -ffast-math."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
            "-shared", "-pthread", "-o", tmp, _SRC, "-lm",
        ])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            lib.oracle_solve_batch.argtypes = [
                ctypes.c_int64, ctypes.c_int, ctypes.c_int, P, P, P,
                ctypes.POINTER(OracleOpts), ctypes.c_int, P, P, P, P, P, P, P]
            lib.oracle_solve_batch.restype = ctypes.c_int
            lib.oracle_hyperbox_batch.argtypes = [
                ctypes.c_int64, ctypes.c_int, P, P, ctypes.c_int64, P, ctypes.c_int, P, P, P]
            lib.oracle_hyperbox_batch.restype = ctypes.c_int
            _lib = lib
    return _lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def default_threads() -> int:
    return max(1, len(os.sched_getaffinity(0)))


RULES = {"LPC": 0, "RPC": 1}  # Step 1 entering rules


def solve(A, b, c, *, eps_enter=1e-9, eps_piv=1e-9, eps_phase1=1e-9, max_iter=0,
          bland_after=0, pivot_rule="LPC", rpc_seed=0, lp_index_base=0, threads=None,
          certs=False):
    """Solve a batch: A [B,m,n], b [B,m], c [B,n] (fp64); LP k of the batch is LP index
    lp_index_base + k of the RPC stream (pivot_rule="RPC", reading R15).  Returns a dict with
    status int32[B], obj f64[B], x f64[B,n], iters int32[B,2] and, with ``certs``,
    y f64[B,m], ray f64[B,n] and the terminal basic point xb f64[B,n],
    plus ``threads`` actually used."""
    lib = _load()
    A = np.ascontiguousarray(A, dtype=np.float64)
    if A.ndim == 2:
        A, b, c = A[None], np.asarray(b)[None], np.asarray(c)[None]
    b = np.ascontiguousarray(b, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    B, m, n = A.shape
    assert b.shape == (B, m) and c.shape == (B, n)
    rule = RULES[pivot_rule.upper()] if isinstance(pivot_rule, str) else int(pivot_rule)
    o = OracleOpts(eps_enter, eps_piv, eps_phase1, int(max_iter), int(bland_after), rule,
                   int(rpc_seed) & 0xFFFFFFFFFFFFFFFF, int(lp_index_base))
    status = np.empty(B, np.int32)
    obj = np.empty(B, np.float64)
    x = np.empty((B, n), np.float64)
    iters = np.empty((B, 2), np.int32)
    y = np.empty((B, m), np.float64) if certs else None
    ray = np.empty((B, n), np.float64) if certs else None
    xb = np.empty((B, n), np.float64) if certs else None
    nt = default_threads() if threads is None else int(threads)
    used = lib.oracle_solve_batch(B, m, n, _ptr(A), _ptr(b), _ptr(c), ctypes.byref(o), nt,
                                  _ptr(status), _ptr(obj), _ptr(x), _ptr(iters), _ptr(y),
                                  _ptr(ray), _ptr(xb))
    out = dict(status=status, obj=obj, x=x, iters=iters, threads=used)
    if certs:
        out.update(y=y, ray=ray, xb=xb)
    return out


def hyperbox(lo, hi, dirs, *, threads=None, want_x=True):
    """Eq. (6) for a batch of directions over one shared box (lo, hi: [n]) or one box per
    LP (lo, hi: [B, n]).  Returns dict(status, obj, x, threads)."""
    lib = _load()
    dirs = np.ascontiguousarray(dirs, dtype=np.float64)
    B, n = dirs.shape
    lo = np.ascontiguousarray(lo, dtype=np.float64)
    hi = np.ascontiguousarray(hi, dtype=np.float64)
    stride = 0 if lo.ndim == 1 else n
    status = np.empty(B, np.int32)
    obj = np.empty(B, np.float64)
    x = np.empty((B, n), np.float64) if want_x else None
    nt = default_threads() if threads is None else int(threads)
    used = lib.oracle_hyperbox_batch(B, n, _ptr(lo), _ptr(hi), stride, _ptr(dirs), nt,
                                     _ptr(status), _ptr(obj), _ptr(x))
    return dict(status=status, obj=obj, x=x, threads=used)
