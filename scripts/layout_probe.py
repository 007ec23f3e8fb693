import sys, numpy as np, torch, os
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
for (m, n) in ((60, 60), (64, 64), (56, 56)):
    A, b, c = lpgen.signed_bounded(50000, m, n, 3)
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    for kl, env in (("R", None), ("R", "3"), ("M", None)):
        if env: os.environ["LPB_REG_CFG"] = env
        else: os.environ.pop("LPB_REG_CFG", None)
        s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class=kl)
        for _ in range(2): s.solve_device(At, bt, ct, sync=True)
        ts = []
        for _ in range(3):
            s.solve_device(At, bt, ct, sync=True); ts.append(s.kernel_ms())
        print(m, n, kl, env, "%.3f ms" % min(ts), flush=True)
        s.close()
