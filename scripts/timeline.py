"""Host-pipeline timeline (PAPER.md:185-206 stream pipeline; VERDICT r1 missing #3): per-chunk
device events of an end-to-end solve through the C ABI with pinned host buffers, for
n_chunks = 10 (default) and 1 (no overlap), from the development build's
lpb_set_timeline / lpb_last_timeline (include/dev/lpb_selftest.h).  nsys is not in the image;
CUDA events on each chunk's stream give the same per-chunk H2D / kernel / D2H intervals.

    python scripts/timeline.py cfg2 [cfg5 ...]  > profiles/<round>/timeline.txt
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "devbuild"))
sys.path.insert(1, ROOT)
import numpy as np  # noqa: E402

import lpgen  # noqa: E402
from paper_1609_08114_b200 import lpb  # noqa: E402

assert "devbuild" in lpb.LIB_PATH, lpb.LIB_PATH
L = lpb._lib
L.lpb_set_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int]
L.lpb_last_timeline.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_float), ctypes.c_int,
                                ctypes.POINTER(ctypes.c_int)]


def merged(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def union(iv):
    iv = sorted(iv)
    tot, cur = 0.0, None
    for a, b in iv:
        if cur is None or a > cur[1]:
            if cur:
                tot += cur[1] - cur[0]
            cur = [a, b]
        else:
            cur[1] = max(cur[1], b)
    return tot + (cur[1] - cur[0] if cur else 0.0)


def run(name, n_chunks):
    cfg = lpgen.CONFIGS[name]
    hyper = cfg["kind"] == "hyperbox"
    if hyper:
        lo, hi, dirs = lpgen.make_config(name)
        host = [None, np.concatenate([hi, -lo]), dirs]
        B, n = dirs.shape
        m = 2 * n
        kw = {}
    else:
        host = list(lpgen.make_config(name))
        B, m, n = host[0].shape
        kw = {"kmax_hint": lpgen.kmax_bound(name)}
    pin = [lpb.pinned_empty(v.shape) if v is not None else None for v in host]
    for d, s in zip(pin, host):
        if d is not None:
            d[...] = s
    st, ob = lpb.pinned_empty((B,), np.int32), lpb.pinned_empty((B,))
    x = lpb.pinned_empty((B, n))
    it = lpb.pinned_empty((B, 2), np.int32) if not hyper else None
    s = lpb.Solver(B, m, n, lpb.HYPERBOX if hyper else lpb.GENERAL, n_chunks=n_chunks, **kw)
    s.solve_host_into(*pin, st, ob, x, it, shared_box=hyper)  # warm-up
    L.lpb_set_timeline(s._ctx, 1)
    s.solve_host_into(*pin, st, ob, x, it, shared_box=hyper)
    e2e = s.timing()[1]
    buf = (ctypes.c_float * (4 * 64))()
    nq = ctypes.c_int()
    rc = L.lpb_last_timeline(s._ctx, buf, 64, ctypes.byref(nq))
    assert rc == 0, rc
    t = np.array(buf[: 4 * nq.value]).reshape(-1, 4)
    s.close()
    h2d = [(a, b) for a, b in t[:, 0:2]]
    ker = [(a, b) for a, b in t[:, 1:3]]
    d2h = [(a, b) for a, b in t[:, 2:4]]
    ksum = sum(b - a for a, b in ker)
    hsum = sum(b - a for a, b in h2d)
    # overlap: time during which some chunk's kernel interval and some chunk's H2D copy are
    # both in flight (intersection of the two interval unions)
    over = sum(max(0.0, min(kb, hb) - max(ka, ha))
               for ka, kb in merged(ker) for ha, hb in merged(h2d))
    return {"config": name, "n_chunks": int(nq.value), "e2e_ms": e2e, "B": int(B),
            "h2d_busy_ms": union(h2d), "kernel_busy_ms": union(ker), "d2h_busy_ms": union(d2h),
            "h2d_sum_ms": hsum, "kernel_sum_ms": ksum,
            "kernel_ms_under_h2d": over, "lps_per_s": B / (e2e / 1e3),
            "chunks": [[round(float(v), 3) for v in row] for row in t]}


def main():
    names = sys.argv[1:] or ["cfg2"]
    for name in names:
        for nch in (10, 1):
            r = run(name, nch)
            print(json.dumps(r))
            print(f"# {name} n_chunks={r['n_chunks']}: e2e {r['e2e_ms']:.2f} ms; H2D busy "
                  f"{r['h2d_busy_ms']:.2f} ms, kernels busy {r['kernel_busy_ms']:.2f} ms "
                  f"(sum {r['kernel_sum_ms']:.2f}), D2H busy {r['d2h_busy_ms']:.2f} ms; kernel time "
                  f"overlapped with H2D {r['kernel_ms_under_h2d']:.2f} ms", flush=True)


if __name__ == "__main__":
    main()
