"""Cluster-size A/B for the L class: python scripts/cl_probe.py cfg3:2000 2 4 8"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
name, B = sys.argv[1].split(':')
A, b, c = lpgen.make_config(name, int(B))
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
for cl in map(int, sys.argv[2:]):
    s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='L', cluster_ctas=cl)
    for _ in range(2): s.solve_device(At, bt, ct, sync=True)
    ts = []
    for _ in range(3):
        s.solve_device(At, bt, ct, sync=True); ts.append(s.kernel_ms())
    print(name, B, 'CL', cl, 'grid', s.launch_shape(), '%.2f ms' % min(ts), flush=True)
    s.close()
