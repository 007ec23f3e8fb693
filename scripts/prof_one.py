"""Run one config a few times (for ncu captures): python scripts/prof_one.py cfg2:2000:R [reps]"""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
import lpgen
from paper_1609_08114_b200 import lpb
spec = sys.argv[1].split(':')
name = spec[0]; B = int(spec[1]) if len(spec) > 1 and spec[1] else None
kl = spec[2] if len(spec) > 2 and spec[2] else None
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = lpgen.CONFIGS[name]
if cfg['kind'] == 'hyperbox':
    lo, hi, dirs = lpgen.make_config(name, B)
    d = torch.from_numpy(dirs).cuda(); box = torch.from_numpy(np.concatenate([hi, -lo])).cuda()
    s = lpb.Solver(d.shape[0], 2 * d.shape[1], d.shape[1], lpb.HYPERBOX)
    f = lambda: s.solve_device(None, box, d, shared_box=True, sync=True)
else:
    A, b, c = lpgen.make_config(name, B)
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class=kl)
    f = lambda: s.solve_device(At, bt, ct, sync=True)
for _ in range(reps):
    f()
print('done', s.launch_info(), s.timing())
