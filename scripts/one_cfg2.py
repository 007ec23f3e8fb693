import sys; sys.path.insert(0,'.')
import torch, lpgen
from paper_1609_08114_b200 import lpb
A,b,c = lpgen.make_config('cfg2', 4000)
At,bt,ct = (torch.from_numpy(v).cuda() for v in (A,b,c))
s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='R')
s.solve_device(At,bt,ct,sync=True)
print('ok', s.kernel_ms())
