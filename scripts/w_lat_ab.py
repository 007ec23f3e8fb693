import os, sys
sys.path.insert(0, os.path.abspath(sys.argv[1])); sys.path.insert(1, os.path.abspath('.'))
import numpy as np, torch, lpgen
from paper_1609_08114_b200 import lpb
for B in (1, 1000, 8192):
    A, b, c = lpgen.make_config('cfg1', B)
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='W')
    for _ in range(5): s.solve_device(At, bt, ct, sync=True)
    ks = []
    for _ in range(40):
        s.solve_device(At, bt, ct, sync=True); ks.append(s.kernel_ms())
    print(sys.argv[1], f"B={B}: kernel median {1e3*np.median(ks):.2f} us min {1e3*min(ks):.2f}", flush=True)
