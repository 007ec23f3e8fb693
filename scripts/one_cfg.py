"""One solve of a config for ncu captures: python scripts/one_cfg.py cfg1:1000000:S"""
import sys
sys.path.insert(0, '.')
import torch
import lpgen
from paper_1609_08114_b200 import lpb
name, B, kl = (sys.argv[1].split(':') + [None, None])[:3]
A, b, c = lpgen.make_config(name, int(B) if B else None)
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class=kl or None)
s.solve_device(At, bt, ct, sync=True)
s.solve_device(At, bt, ct, sync=True)
print('ok', s.kernel_ms(), s.launch_info())
