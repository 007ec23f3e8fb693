import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import lpgen
from paper_1609_08114_b200 import lpb
def tm(name, B=None, klass=None):
    cfg = lpgen.CONFIGS[name]
    if cfg['kind'] == 'hyperbox':
        lo, hi, dirs = lpgen.make_config(name, B)
        d = torch.from_numpy(dirs).cuda(); box = torch.from_numpy(np.concatenate([hi, -lo])).cuda()
        s = lpb.Solver(d.shape[0], 2*d.shape[1], d.shape[1], lpb.HYPERBOX)
        f = lambda: s.solve_device(None, box, d, shared_box=True)
    else:
        A, b, c = lpgen.make_config(name, B)
        At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
        s = lpb.Solver(*A.shape, lpb.GENERAL, kernel_class=klass)
        f = lambda: s.solve_device(At, bt, ct)
    for _ in range(3): f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        f(); ts.append(s.timing()[0])
    r = s.device_results()
    it = r['iters'].float().mean(0).tolist()
    print(name, B, 'class', s.launch_info(), 'ms', ['%.3f' % t for t in ts], 'LPs/s %.3e' % (s.batch / (min(ts) / 1e3)), 'iters', it, flush=True)
for a in sys.argv[1:]:
    parts = a.split(':')
    nm = parts[0]; B = int(parts[1]) if len(parts) > 1 and parts[1] else None
    kl = parts[2] if len(parts) > 2 else None
    tm(nm, B, kl)
