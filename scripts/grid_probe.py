"""Per-pivot latency vs CTAs per SM (contention probe): python scripts/grid_probe.py cfg2:20000 148 296"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
name, B = sys.argv[1].split(':')
A, b, c = lpgen.make_config(name, int(B))
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
for g in sys.argv[2:]:
    s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class='R', grid_ctas=int(g))
    for _ in range(2): s.solve_device(At, bt, ct, sync=True)
    ts = []
    for _ in range(3):
        s.solve_device(At, bt, ct, sync=True); ts.append(s.timing()[0])
    piv = s.device_results()['iters'].sum().item()
    ms = min(ts)
    print(f"grid {g}: {ms:.3f} ms, {piv} pivots, cycles per LP-pivot per CTA "
          f"{ms * 1e-3 * 1.965e9 / (piv / int(g)):.0f}", flush=True)
    s.close()
