"""Per-phase cycle breakdown of the R-class kernel (warp 0 of each CTA):
python scripts/phase_prof.py cfg2:20000"""
import ctypes, os, sys
# the profiler is compiled in only with -DLPB_PROFILE: use (or build) that variant
if not os.path.exists('ab/prof/paper_1609_08114_b200/liblpb.so'):
    os.system(f'{sys.executable} paper_1609_08114_b200/build.py --variant ab/prof -DLPB_PROFILE')
sys.path.insert(0, 'ab/prof')
sys.path.insert(1, '.')
import numpy as np, torch
import lpgen
from paper_1609_08114_b200 import lpb
lpb._lib.lpb_set_profile_buffer.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
name, B = sys.argv[1].split(':')
A, b, c = lpgen.make_config(name, int(B))
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='R')
s.solve_device(At, bt, ct, sync=True)
buf = torch.zeros(4096 * 12, dtype=torch.int64, device='cuda')
lpb._lib.lpb_set_profile_buffer(s._ctx, ctypes.c_void_p(buf.data_ptr()))
s.solve_device(At, bt, ct, sync=True)
ms = s.timing()[0]
r = s.device_results()
piv = r['iters'].sum().item()
p = buf.view(-1, 12).sum(0).cpu().numpy().astype(float)
names = ['step1', 'publish', 'ratio_part', 'barrier1', 'reduce', 'prow', 'barrier2', 'loophead', 'update', '-', '-', '-']
ctas = (buf.view(-1, 12).sum(1) > 0).sum().item()
print(f'{name} B={B} ms={ms:.3f} pivots={piv} ctas={ctas}')
tot = p.sum()
for nm, v in zip(names, p):
    print(f'  {nm:14s} {v / piv:8.1f} cycles/pivot  {100 * v / tot:5.1f}%')
print(f'  total {tot / piv:.1f} cycles per LP-pivot (per CTA); wall per LP-pivot {ms * 1e-3 * 1.9e9 / (piv / ctas):.1f}')
