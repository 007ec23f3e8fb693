"""A/B of the hyperbox kernel across built variants (development tool; cf. scripts/ab.py):
    python scripts/hb_ab.py <root[@VAR=v,...]> ... -- cfg4 cfg5
Device time of the hyperbox kernel (min / median of 11 solves, L2 flushed between solves) and a
digest of (status, obj, x)."""
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, hashlib, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(1, {repo!r})
import lpgen
from paper_1609_08114_b200 import lpb
out = []
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for name in {specs!r}:
    lo, hi, dirs = lpgen.make_config(name)
    d = torch.from_numpy(dirs).cuda()
    box = torch.from_numpy(np.concatenate([hi, -lo])).cuda()
    s = lpb.Solver(d.shape[0], 2 * d.shape[1], d.shape[1], lpb.HYPERBOX)
    f = lambda: s.solve_device(None, box, d, shared_box=True, sync=True)
    for _ in range(3): f()
    ts = []
    for _ in range(11):
        flush.zero_(); torch.cuda.synchronize(); f(); ts.append(s.kernel_ms())
    r = {{k: v.cpu().numpy() for k, v in s.device_results().items() if k != "iters"}}
    h = hashlib.sha1(r["status"].tobytes() + r["obj"].tobytes() + r["x"].tobytes()).hexdigest()[:12]
    out.append(dict(spec=name, min_ms=min(ts), med_ms=sorted(ts)[5], digest=h))
    s.close()
print("AB-JSON " + json.dumps(out))
'''


def main():
    i = sys.argv.index("--")
    roots, specs = sys.argv[1:i], sys.argv[i + 1:]
    repo = os.path.abspath(".")
    for root in roots:
        path, _, envs = root.partition("@")
        env = dict(os.environ)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        p = subprocess.run([sys.executable, "-c", CHILD.format(root=os.path.abspath(path), repo=repo, specs=specs)],
                           capture_output=True, text=True, env=env)
        line = [l for l in p.stdout.splitlines() if l.startswith("AB-JSON ")]
        if not line:
            print(root, "FAILED", p.stderr[-1200:])
            continue
        for d in json.loads(line[0][8:]):
            print(f"{d['spec']:6s} {root:36s} min {d['min_ms']:8.4f} ms  med {d['med_ms']:8.4f}  digest {d['digest']}")


if __name__ == "__main__":
    main()
