"""End-to-end (host arrays) time vs pipeline depth: python scripts/chunk_probe.py cfg5 10 20 40"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
name = sys.argv[1]
cfg = lpgen.CONFIGS[name]
if cfg["kind"] == "hyperbox":
    lo, hi, dirs = lpgen.make_config(name)
    B, n = dirs.shape
    m = 2 * n
    host = (None, np.concatenate([hi, -lo]), dirs)
    kind = lpb.HYPERBOX
else:
    A, b, c = lpgen.make_config(name)
    B, m, n = A.shape
    host = (A, b, c)
    kind = lpb.GENERAL
pin = [lpb.pinned_empty(v.shape) if v is not None else None for v in host]
for d, s_ in zip(pin, host):
    if d is not None: d[...] = s_
out = (lpb.pinned_empty((B,), np.int32), lpb.pinned_empty((B,)), lpb.pinned_empty((B, n)),
       None if kind == lpb.HYPERBOX else lpb.pinned_empty((B, 2), np.int32))
for nch in map(int, sys.argv[2:]):
    s = lpb.Solver(B, m, n, kind, n_chunks=nch)
    ts = []
    for _ in range(4):
        s.solve_host_into(*pin, *out, shared_box=kind == lpb.HYPERBOX)
        ts.append(s.timing()[1])
    print(name, 'chunks', nch, 'e2e ms', ['%.2f' % t for t in ts[1:]], flush=True)
    s.close()
