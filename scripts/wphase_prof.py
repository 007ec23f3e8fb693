"""Per-phase cycle breakdown of the W-class kernel for one warp (warp 0 of the grid):
python scripts/wphase_prof.py cfg1:1  (builds the -DLPB_PROFILE variant under ab/prof)"""
import ctypes, os, sys
if not os.path.exists('ab/prof/paper_1609_08114_b200/liblpb.so') or '--rebuild' in sys.argv:
    os.system(f'{sys.executable} paper_1609_08114_b200/build.py --variant ab/prof -DLPB_PROFILE')
sys.path.insert(0, 'ab/prof')
sys.path.insert(1, '.')
import torch
import lpgen
from paper_1609_08114_b200 import lpb
lpb._lib.lpb_set_profile_buffer.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
name, B = sys.argv[1].split(':')
A, b, c = lpgen.make_config(name, int(B))
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='W')
s.solve_device(At, bt, ct, sync=True)
buf = torch.zeros(16, dtype=torch.int64, device='cuda')
lpb._lib.lpb_set_profile_buffer(s._ctx, ctypes.c_void_p(buf.data_ptr()))
s.solve_device(At, bt, ct, sync=True)
p = buf.cpu().numpy().astype(float)
names = ['ticket', 'load+build', 'step1 shfl', 'colE shfl', 'ratio', 'pe/row shfl', 'divisions',
         'update', 'loop exit', 'extract', 'loop head', 'scan', 'argmax']
piv = max(p[15], 1)
print(f'{name} B={B} kernel {s.kernel_ms()*1e3:.1f} us; warp 0: {int(p[15])} pivots')
for nm, v in zip(names, p):
    print(f'  {nm:12s} {v:9.0f} cycles  ({v / piv:7.1f} per pivot)')
