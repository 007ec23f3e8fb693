"""Step-time anatomy for small configs: torch events around back-to-back solves.
python scripts/step_probe.py cfg1"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
name = sys.argv[1]
A, b, c = lpgen.make_config(name)
At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
s = lpb.Solver(*A.shape, lpb.GENERAL)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for mode in ("noflush", "flush", "flush+sleep"):
    for _ in range(5): s.solve_device(At, bt, ct, timing=False)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    for i in range(20):
        if mode != "noflush":
            flush.fill_(float(i))
        if mode == "flush+sleep":
            torch.cuda._sleep(200000)
        ev[i][0].record(); s.solve_device(At, bt, ct, timing=False); ev[i][1].record()
    torch.cuda.synchronize()
    t = [a.elapsed_time(b_) * 1e3 for a, b_ in ev]
    print(mode, f"median step {np.median(t):.1f} us", flush=True)
