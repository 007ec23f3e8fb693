"""Thin ctypes binding of liblpb.so (include/lpb.h): argument marshalling only.

Every step of the solve runs in the library's CUDA kernels; this module only converts
arrays to pointers.  It raises ImportError at import time when liblpb.so has not been
built -- there is no CPU fallback anywhere in the product path.

Device path: pass torch CUDA tensors (float64, contiguous); the library reads them in place
on torch's current stream (LPB_DEVICE_PTRS) and results come back as torch CUDA tensors.
Host path: pass numpy arrays (ideally pinned, see ``pinned_empty``); inputs go through the
library's chunked H2D -> kernel -> D2H stream pipeline and results come back as numpy.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblpb.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python paper_1609_08114_b200/build.py` "
                      "(no CPU fallback exists)")
_lib = ctypes.CDLL(LIB_PATH)

GENERAL, HYPERBOX = 0, 1
OPTIMAL, UNBOUNDED, INFEASIBLE, ITER_LIMIT, NUMERICAL, BAD_HINT = range(6)
OK, EINVAL, ENOMEM, ECUDA, ESTATE, ETOOBIG = 0, -1, -2, -3, -4, -5
DEVICE_PTRS, SHARED_BOX, NO_X, ASYNC, SHARED_AB, NO_TIMING = 1, 2, 4, 8, 16, 32
CLASS_NAMES = {0: "auto", 1: "S", 2: "M", 3: "L", 4: "R", 5: "H", 7: "W"}
CLASS_IDS = {v: k for k, v in CLASS_NAMES.items()}
RULE_LPC, RULE_RPC = 0, 1  # lpb_options.pivot_rule
RULE_IDS = {"LPC": RULE_LPC, "RPC": RULE_RPC}


class Options(ctypes.Structure):
    _fields_ = [
        ("struct_size", ctypes.c_int32),
        ("eps_enter", ctypes.c_double),
        ("eps_piv", ctypes.c_double),
        ("eps_phase1", ctypes.c_double),
        ("max_iter", ctypes.c_int32),
        ("bland_after", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("stream", ctypes.c_void_p),
        ("n_chunks", ctypes.c_int32),
        ("kernel_class", ctypes.c_int32),
        ("grid_ctas", ctypes.c_int32),
        ("cluster_ctas", ctypes.c_int32),
        ("pivot_rule", ctypes.c_int32),
        ("rpc_seed", ctypes.c_uint64),
        ("lp_index_base", ctypes.c_int64),
        ("warm_start", ctypes.c_int32),
        ("kmax_hint", ctypes.c_int32),
    ]


P = ctypes.c_void_p
_lib.lpb_default_options.argtypes = [ctypes.POINTER(Options)]
_lib.lpb_create.argtypes = [ctypes.POINTER(P), ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                            ctypes.c_int32, ctypes.POINTER(Options)]
_lib.lpb_solve_batch.argtypes = [P, P, P, P, ctypes.c_uint32]
_lib.lpb_solve_batch_into.argtypes = [P, P, P, P, ctypes.c_uint32, P, P, P, P]
_lib.lpb_results.argtypes = [P, P, P, P, P]
_lib.lpb_result_device_ptrs.argtypes = [P, P, P, P, P]
_lib.lpb_sync.argtypes = [P]
_lib.lpb_last_timing.argtypes = [P, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_double)]
_lib.lpb_last_kernel_timing.argtypes = [P, ctypes.POINTER(ctypes.c_double)]
_lib.lpb_last_kernel_timing.restype = ctypes.c_int
_lib.lpb_last_launch_info.argtypes = [P, ctypes.POINTER(ctypes.c_int32),
                                      ctypes.POINTER(ctypes.c_int32)]
_lib.lpb_last_launch_shape.argtypes = [P, ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_int32)]
_lib.lpb_destroy.argtypes = [P]
_lib.lpb_strerror.argtypes = [ctypes.c_int]
_lib.lpb_strerror.restype = ctypes.c_char_p
_lib.lpb_last_error.argtypes = [P]
_lib.lpb_last_error.restype = ctypes.c_char_p
for _f in ("lpb_default_options", "lpb_create", "lpb_solve_batch", "lpb_solve_batch_into",
           "lpb_results", "lpb_result_device_ptrs", "lpb_sync", "lpb_last_timing",
           "lpb_last_launch_info", "lpb_last_launch_shape", "lpb_destroy"):
    getattr(_lib, _f).restype = ctypes.c_int


class LpbError(RuntimeError):
    def __init__(self, code, detail=""):
        super().__init__(f"lpb error {code} ({_lib.lpb_strerror(code).decode()}) {detail}")
        self.code = code


def _check(rc, ctx=None):
    if rc != OK:
        detail = _lib.lpb_last_error(ctx).decode() if ctx else ""
        raise LpbError(rc, detail)


def default_options(**kw) -> Options:
    o = Options()
    _check(_lib.lpb_default_options(ctypes.byref(o)))
    for k, v in kw.items():
        if v is None:
            continue
        if k == "kernel_class" and isinstance(v, str):
            v = CLASS_IDS[v]
        if k == "pivot_rule" and isinstance(v, str):
            v = RULE_IDS[v.upper()]
        setattr(o, k, v)
    return o


def _is_torch(a):
    try:
        import torch
        return isinstance(a, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def _dptr(t):
    if t is None:
        return None
    import torch
    assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous(), \
        "device inputs must be contiguous float64 CUDA tensors"
    return ctypes.c_void_p(t.data_ptr())


def _hptr(a):
    if a is None:
        return None
    assert a.dtype in (np.float64, np.int32) and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


_PINNED = {}


def pinned_empty(shape, dtype=np.float64) -> np.ndarray:
    """A numpy view of page-locked host memory (torch pin_memory), for the host path.
    The owning torch tensor is kept alive until ``pinned_release(array)``."""
    import torch
    tdt = {np.float64: torch.float64, np.int32: torch.int32}[np.dtype(dtype).type]
    t = torch.empty(shape, dtype=tdt, pin_memory=True)
    a = t.numpy()
    _PINNED[a.ctypes.data] = t
    return a


def pinned_release(a: np.ndarray) -> None:
    _PINNED.pop(a.ctypes.data, None)


class Solver:
    """One lpb context: a batch size, an LP shape and a kind, reused across solves."""

    def __init__(self, batch, m, n, kind=GENERAL, *, device=None, stream=None, **opts):
        import torch
        if device is None:
            device = torch.cuda.current_device() if torch.cuda.is_available() else 0
        if stream is None and torch.cuda.is_available():
            # torch's current stream; handle 0 is the legacy default stream, which the ABI
            # must receive as cudaStreamLegacy (0x1) -- NULL would mean "own stream"
            stream = torch.cuda.current_stream(device).cuda_stream or 0x1
        self.batch, self.m, self.n, self.kind = int(batch), int(m), int(n), kind
        self.device = device
        self.opts = default_options(device=int(device), stream=stream, **opts)
        self._ctx = P()
        rc = _lib.lpb_create(ctypes.byref(self._ctx), self.batch, self.m, self.n, kind,
                             ctypes.byref(self.opts))
        _check(rc)

    def close(self):
        if self._ctx:
            _lib.lpb_destroy(self._ctx)
            self._ctx = P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- solves --
    def solve_device(self, A, b, c, *, shared_box=False, shared_ab=False, want_x=True,
                     sync=False, timing=True):
        """Device tensors in; results stay in the context's device buffers (see
        ``device_results``).  Asynchronous on the context's stream unless ``sync``.
        ``shared_ab``: A (m x n) and b (m) are one constraint system for the whole batch."""
        flags = (DEVICE_PTRS | (SHARED_BOX if shared_box else 0) | (0 if want_x else NO_X) |
                 (SHARED_AB if shared_ab else 0))
        if not sync:
            flags |= ASYNC
        if not timing:
            flags |= NO_TIMING
        _check(_lib.lpb_solve_batch(self._ctx, _dptr(A), _dptr(b), _dptr(c), flags), self._ctx)

    def solve_host_into(self, A, b, c, status, obj, x=None, iters=None, *, shared_box=False,
                        shared_ab=False):
        """End-to-end path: host arrays in (pinned for overlap), results copied into host
        arrays, chunk by chunk on the library's streams; returns when done."""
        flags = ((SHARED_BOX if shared_box else 0) | (0 if x is not None else NO_X) |
                 (SHARED_AB if shared_ab else 0))
        _check(_lib.lpb_solve_batch_into(self._ctx, _hptr(A), _hptr(b), _hptr(c), flags,
                                         _hptr(status), _hptr(obj), _hptr(x), _hptr(iters)),
               self._ctx)

    def device_results(self, want_x=True):
        """torch CUDA tensors aliasing the context's result buffers (valid until next solve)."""
        import torch
        ps = [ctypes.c_void_p() for _ in range(4)]
        _check(_lib.lpb_result_device_ptrs(self._ctx, *[ctypes.byref(p) for p in ps]))
        B, n = self.batch, self.n
        out = {}
        for name, p, shape, dt in (("status", ps[0], (B,), torch.int32),
                                   ("obj", ps[1], (B,), torch.float64),
                                   ("x", ps[2], (B, n), torch.float64),
                                   ("iters", ps[3], (B, 2), torch.int32)):
            if name == "x" and not want_x:
                continue
            out[name] = _wrap_device(p.value, shape, dt, self.device)
        return out

    def sync(self):
        _check(_lib.lpb_sync(self._ctx), self._ctx)

    def timing(self):
        s, e = ctypes.c_double(), ctypes.c_double()
        _check(_lib.lpb_last_timing(self._ctx, ctypes.byref(s), ctypes.byref(e)), self._ctx)
        return s.value, e.value

    def kernel_ms(self):
        """Device time of the last device-pointer solve's dominant kernel."""
        k = ctypes.c_double()
        _check(_lib.lpb_last_kernel_timing(self._ctx, ctypes.byref(k)), self._ctx)
        return k.value

    def launch_info(self):
        n, k = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.lpb_last_launch_info(self._ctx, ctypes.byref(n), ctypes.byref(k)))
        return n.value, CLASS_NAMES.get(k.value, str(k.value))

    def launch_shape(self):
        """(CTAs per LP -- the L class's cluster size --, grid CTAs) of the last launch."""
        cl, g = ctypes.c_int32(), ctypes.c_int32()
        _check(_lib.lpb_last_launch_shape(self._ctx, ctypes.byref(cl), ctypes.byref(g)))
        return cl.value, g.value


def _wrap_device(ptr, shape, dtype, device):
    """Zero-copy torch view of library-owned device memory (via __cuda_array_interface__)."""
    import torch
    typestr = {torch.int32: "<i4", torch.float64: "<f8"}[dtype]

    class _Holder:
        __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                    "data": (ptr, False), "version": 3, "strides": None}
    with torch.cuda.device(device):
        return torch.as_tensor(_Holder(), device=f"cuda:{device}")


def solve(A, b, c, *, want_x=True, **opts):
    """One-shot solve of max c.x s.t. A x <= b, x >= 0 for a batch.
    A (B x m x n), b (B x m), c (B x n); or A (m x n) and b (m) shared by every LP (many
    objectives over one polytope, LPB_SHARED_AB).
    torch CUDA tensors -> torch results (device path, synchronous);
    numpy arrays -> numpy results (host pipeline)."""
    shared = len(A.shape) == 2
    if _is_torch(A):
        B, n = c.shape
        m = A.shape[-2]
        s = Solver(B, m, n, GENERAL, **opts)
        s.solve_device(A, b, c, want_x=want_x, sync=True, shared_ab=shared)
        res = {k: v.clone() for k, v in s.device_results(want_x).items()}
        s.close()
        return res
    A = np.ascontiguousarray(A, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    c = np.ascontiguousarray(c, np.float64)
    B, n = c.shape
    m = A.shape[-2]
    s = Solver(B, m, n, GENERAL, **opts)
    out = dict(status=np.empty(B, np.int32), obj=np.empty(B), iters=np.empty((B, 2), np.int32))
    out["x"] = np.empty((B, n)) if want_x else None
    s.solve_host_into(A, b, c, out["status"], out["obj"], out["x"], out["iters"],
                      shared_ab=shared)
    s.close()
    return out


def hyperbox(lo, hi, dirs, *, want_x=True, **opts):
    """Eq. (6) for a batch of directions over one shared box (the paper's setting).
    torch CUDA ``dirs`` -> torch results; numpy -> numpy."""
    if _is_torch(dirs):
        import torch
        B, n = dirs.shape
        box = torch.cat([torch.as_tensor(hi, dtype=torch.float64),
                         -torch.as_tensor(lo, dtype=torch.float64)]).to(dirs.device)
        s = Solver(B, 2 * n, n, HYPERBOX, **opts)
        s.solve_device(None, box, dirs, shared_box=True, want_x=want_x, sync=True)
        res = {k: v.clone() for k, v in s.device_results(want_x).items() if k != "iters"}
        s.close()
        return res
    dirs = np.ascontiguousarray(dirs, np.float64)
    B, n = dirs.shape
    box = np.ascontiguousarray(np.concatenate([np.asarray(hi, np.float64),
                                               -np.asarray(lo, np.float64)]))
    s = Solver(B, 2 * n, n, HYPERBOX, **opts)
    out = dict(status=np.empty(B, np.int32), obj=np.empty(B))
    out["x"] = np.empty((B, n)) if want_x else None
    s.solve_host_into(None, box, dirs, out["status"], out["obj"], out["x"], None,
                      shared_box=True)
    s.close()
    return out
