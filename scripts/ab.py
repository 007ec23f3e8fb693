"""A/B kernel timing across built variants of the package (development tool).

    python scripts/ab.py <variant_root> [<variant_root> ...] -- cfg2:20000 cfg3:2000 ...

Each variant root holds a built paper_1609_08114_b200/ (build.py --variant <root> ...); a root
written <root>@VAR=value[,VAR=value] runs with those environment variables (the development
build's A/B switches, e.g. devbuild@LPB_NO_TMEM=1).  Every
variant runs in its own subprocess on the same inputs; prints the dominant kernel's device
time (min / median of 7 solves) and a digest of the results (status, iters, obj bits), so
variants that must be bit-identical can be checked at a glance."""
import hashlib
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
for spec in {specs!r}:
    parts = spec.split(':')
    name = parts[0]; B = int(parts[1]) if len(parts) > 1 and parts[1] else None
    klass = parts[2] if len(parts) > 2 and parts[2] else None
    clu = int(parts[3]) if len(parts) > 3 and parts[3] else 0
    A, b, c = lpgen.make_config(name, B)
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    kw = dict(kernel_class=klass) if klass else {{}}
    if clu: kw['cluster_ctas'] = clu
    kh = lpgen.kmax_bound(name)
    if 'kmax_hint' in [f[0] for f in lpb.Options._fields_]:
        kw['kmax_hint'] = kh
    s = lpb.Solver(c.shape[0], A.shape[-2], c.shape[1], lpb.GENERAL, **kw)
    f = lambda: s.solve_device(At, bt, ct, shared_ab=(A.ndim == 2), sync=True)
    try:
        f()
    except Exception as ex:
        print('skip', spec, ex, file=sys.stderr)
        continue
    for _ in range(2): f()
    ts = []
    for _ in range(7):
        f(); ts.append(s.kernel_ms())
    r = {{k: v.cpu().numpy() for k, v in s.device_results().items()}}
    h = hashlib.sha1(r['status'].tobytes() + r['iters'].tobytes() + r['obj'].tobytes()).hexdigest()[:12]
    piv = int(r['iters'].sum())
    out.append(dict(spec=spec, min_ms=min(ts), med_ms=sorted(ts)[3], klass=s.launch_info()[1] + str(s.launch_shape()),
                    digest=h, pivots=piv))
    s.close()
print('AB-JSON ' + json.dumps(out))
'''


def main():
    i = sys.argv.index('--')
    roots, specs = sys.argv[1:i], sys.argv[i + 1:]
    repo = os.path.abspath('.')
    res = {}
    for root in roots:
        path, _, envs = root.partition('@')
        env = dict(os.environ)
        for kv in filter(None, envs.split(',')):
            k, _, v = kv.partition('=')
            env[k] = v
        code = CHILD.format(root=os.path.abspath(path), repo=repo, specs=specs)
        p = subprocess.run([sys.executable, '-c', code], capture_output=True, text=True, env=env)
        line = [l for l in p.stdout.splitlines() if l.startswith('AB-JSON ')]
        if not line:
            print(root, 'FAILED', p.stdout[-800:], p.stderr[-1500:])
            continue
        res[root] = json.loads(line[0][8:])
    for spec in specs:
        print(spec)
        for root in roots:
            for d in res.get(root, []):
                if d['spec'] == spec:
                    ns = d['min_ms'] * 1e6 / max(d['pivots'], 1)
                    print(f"  {root:28s} {d['klass']} min {d['min_ms']:9.3f} ms  med {d['med_ms']:9.3f}"
                          f"  {ns:7.2f} ns/pivot  digest {d['digest']} pivots {d['pivots']}")


if __name__ == '__main__':
    main()
