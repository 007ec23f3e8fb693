"""Cluster-size A/B across builds: python scripts/cl_ab.py <pkgroot> cfg3:2000 2 4"""
import os, sys
sys.path.insert(0, os.path.abspath(sys.argv[1]))
sys.path.insert(1, os.path.abspath('.'))
import torch
import lpgen
from paper_1609_08114_b200 import lpb
name, B = sys.argv[2].split(':')
A, b, c = lpgen.make_config(name, int(B))
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
for cl in map(int, sys.argv[3:]):
    s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='L', cluster_ctas=cl)
    for _ in range(2): s.solve_device(At, bt, ct, sync=True)
    ts = []
    for _ in range(3):
        s.solve_device(At, bt, ct, sync=True); ts.append(s.kernel_ms())
    print(lpb.LIB_PATH.split('/')[-3], name, B, 'CL', cl, 'grid', s.launch_shape(), '%.2f ms' % min(ts), flush=True)
    s.close()
