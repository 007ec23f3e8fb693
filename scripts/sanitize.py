"""Small batches through every kernel (size classes S, W, R (incl. the TMEM layouts), M, L on
2/4/8/16-CTA clusters (incl. the TMR variants), the phase-I warm start, hyperbox TMA-ring and
plain kernels), for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
    compute-sanitizer --tool racecheck python scripts/sanitize.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb


def run(A, b, c, **kw):
    At, bt, ct = (torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (A, b, c))
    B, n = ct.shape
    m = At.shape[-2]
    s = lpb.Solver(B, m, n, lpb.GENERAL, **kw)
    s.solve_device(At, bt, ct, sync=True, shared_ab=At.dim() == 2)
    r = s.device_results()
    out = (r["status"].cpu().numpy(), s.launch_info())
    s.close()
    return out


A, b, c = lpgen.status_mix(64, 6, 6, 1, infeasible_start=True)
# S: register kernel + deferred two-phase LPs in list mode; W: element layout + generic warps
for kl in ("S", "W", "R", "M", "L"):
    st, li = run(A, b, c, kernel_class=kl)
    print(kl, li, np.bincount(st, minlength=5))
A, b, c = lpgen.status_mix(20000, 5, 5, 7, infeasible_start=True)  # 128-thread S CTAs
st, li = run(A, b, c, kernel_class="S")
print("S 20000", li, np.bincount(st, minlength=5))
A, b, c = lpgen.signed_bounded(300, 7, 7, 8)  # W element layout only
st, li = run(A, b, c, kernel_class="W", pivot_rule="RPC", rpc_seed=1)
print("W elem RPC", li, np.bincount(st, minlength=5))
A, b, c = lpgen.twophase_signed(4, 40, 40, 2)
for cl in (2, 4, 8, 16):
    st, li = run(A, b, c, kernel_class="L", cluster_ctas=cl)
    print("L", cl, li, np.bincount(st, minlength=5))
A, b, c = lpgen.shared_polytope(16, 30, 30, 3, "G2")
st, li = run(A, b, c, kernel_class="M")  # phase-I record + warm start
print("warm", li, np.bincount(st, minlength=5))
A, b, c = lpgen.signed_bounded(8, 100, 100, 4)
st, li = run(A, b, c)
print("R 100x100", li, np.bincount(st, minlength=5))
A, b, c = lpgen.signed_bounded(8, 20, 20, 5)
st, li = run(A, b, c, pivot_rule="RPC", rpc_seed=3)
print("RPC", li, np.bincount(st, minlength=5))
# tensor-memory paths: R layouts 15 (cfg2 sizes) and 17 (cfg10), L-class TMR variants on
# 4-, 8- (two-phase: phase-switch copies) and 16-CTA clusters
for name, B in (("cfg2", 4), ("cfg10", 8), ("cfg6", 3), ("cfg8", 2), ("cfg7", 1)):
    A, b, c = lpgen.make_config(name, B)
    st, li = run(A, b, c)
    print("TMEM", name, li, np.bincount(st, minlength=5))
lo, hi, dirs = lpgen.hyperbox(256 * 8 * 3 + 17, 5, 6)
h = lpb.hyperbox(lo, hi, torch.from_numpy(dirs).cuda())
print("H tma", h["status"].sum().item())
g = np.random.default_rng(0)
lo2 = g.uniform(-1, 0, (300, 4))
s = lpb.Solver(300, 8, 4, lpb.HYPERBOX)
box = torch.from_numpy(np.concatenate([lo2 + 1, -lo2], axis=1)).cuda()
s.solve_device(None, box, torch.from_numpy(g.standard_normal((300, 4))).cuda(), sync=True)
print("H plain", s.device_results()["status"].sum().item())
print("sanitize run done")
