"""Kernel-only time vs batch size (latency floor of small batches):
python scripts/lat_probe.py cfg1 R 1 10 100 1000"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
name, klass = sys.argv[1], sys.argv[2]
for B in map(int, sys.argv[3:]):
    A, b, c = lpgen.make_config(name, B)
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class=klass)
    for _ in range(5): s.solve_device(At, bt, ct, sync=True)
    ks, ts = [], []
    for _ in range(20):
        s.solve_device(At, bt, ct, sync=True); ks.append(s.kernel_ms()); ts.append(s.timing()[0])
    print(f"B={B}: kernel {1e3*np.median(ks):.1f} us, solve {1e3*np.median(ts):.1f} us", flush=True)
    s.close()
