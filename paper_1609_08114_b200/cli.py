"""Command-line surface (SPEC.md:403-471 commands gen / solve /
support-demo, as plumbing around the C ABI -- every LP is solved by the CUDA kernels).

    python -m paper_1609_08114_b200.cli gen --class feasible -n 100 -m 100 --count 1000 \\
        --seed 7 -o batch.npz
    python -m paper_1609_08114_b200.cli solve batch.npz [--pivot rpc --seed 1] [--repeat 10] \\
        [-o results.csv]
    python -m paper_1609_08114_b200.cli support-demo -n 5 --template random --count 4001000 \\
        --engine both

Exit codes: 0 success, 1 usage, 2 I/O / parse, 3 internal.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import numpy as np

STATUS_NAMES = ["optimal", "unbounded", "infeasible", "iter_limit", "numerical"]


def _lpgen():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    import lpgen
    return lpgen


def cmd_gen(a) -> int:
    """Seeded batch file (npz: A [N,m,n], b [N,m], c [N,n]; or lo, hi, dirs for --class box)."""
    g = _lpgen()
    if a.n <= 0 or a.count <= 0 or (a.klass != "box" and a.m <= 0):
        print("gen: -n, -m and --count must be positive", file=sys.stderr)
        return 1
    if a.klass == "feasible":
        A, b, c = g.signed_bounded(a.count, a.m, a.n, a.seed)
        np.savez(a.out, A=A, b=b, c=c)
    elif a.klass == "infeasible":
        A, b, c = g.twophase_signed(a.count, a.m, a.n, a.seed)
        np.savez(a.out, A=A, b=b, c=c)
    else:
        lo, hi, dirs = g.hyperbox(a.count, a.n, a.seed)
        np.savez(a.out, lo=lo, hi=hi, dirs=dirs)
    print(f"gen: {a.count} {a.klass} LPs, n={a.n}" + ("" if a.klass == "box" else f" m={a.m}")
          + f", seed {a.seed} -> {a.out}")
    return 0


def cmd_solve(a) -> int:
    import torch

    from . import lpb
    try:
        f = np.load(a.path)
    except (OSError, ValueError) as ex:
        print(f"solve: cannot read {a.path}: {ex}", file=sys.stderr)
        return 2
    box = "dirs" in f.files
    opts = {"pivot_rule": a.pivot.upper(), "rpc_seed": a.seed} if not box else {}
    if box:
        lo, hi, dirs = f["lo"], f["hi"], f["dirs"]
        B, n = dirs.shape
        s = lpb.Solver(B, 2 * n, n, lpb.HYPERBOX)
        args = (None, torch.from_numpy(np.concatenate([hi, -lo])).cuda(),
                torch.from_numpy(np.ascontiguousarray(dirs)).cuda())
        kw = dict(shared_box=True)
    else:
        A, b, c = f["A"], f["b"], f["c"]
        B, m, n = A.shape
        s = lpb.Solver(B, m, n, lpb.GENERAL, **opts)
        args = tuple(torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (A, b, c))
        kw = {}
    times = []
    for _ in range(max(1, a.repeat)):
        s.solve_device(*args, sync=True, **kw)
        times.append(s.timing()[0])
    r = {k: v.cpu().numpy() for k, v in s.device_results(want_x=False).items()}
    s.close()
    ms = statistics.median(times)
    st = r["status"]
    summary = {"lps": int(B), "median_ms": ms, "lps_per_s": B / (ms / 1e3),
               "status_counts": {STATUS_NAMES[i]: int(v)
                                 for i, v in enumerate(np.bincount(st, minlength=5)) if v},
               "engine": "hyperbox" if box else f"simplex/{a.pivot.lower()}"}
    if not box:
        summary["mean_iters"] = r["iters"].mean(axis=0).tolist()
    if a.out:
        with open(a.out, "w") as fo:
            fo.write("index,status,objective" + ("" if box else ",iters_phase1,iters_phase2")
                     + "\n")
            for k in range(B):
                row = f"{k},{STATUS_NAMES[st[k]]},{float(r['obj'][k])!r}"
                if not box:
                    row += f",{r['iters'][k, 0]},{r['iters'][k, 1]}"
                fo.write(row + "\n")
    print(json.dumps(summary))
    return 0


def cmd_support_demo(a) -> int:
    import torch

    from . import support
    g = _lpgen()
    n = a.n
    if n <= 0:
        print("support-demo: -n must be positive", file=sys.stderr)
        return 1
    if a.box == "paper" and n == 5:  # the five-dimensional benchmark's initial set
        lo, hi, _ = g.hyperbox(1, 5, 0)
    else:
        rg = g.rng(a.seed)
        lo = rg.uniform(-1.0, 0.0, size=n)
        hi = lo + rg.uniform(0.01, 1.0, size=n)
    if a.template == "box":
        dirs = g.box_directions(n)
    elif a.template == "oct":
        dirs = g.oct_directions(n)
    else:
        if a.count <= 0:
            print("support-demo: --count must be positive for the random template", file=sys.stderr)
            return 1
        dirs = g.hyperbox(a.count, n, a.seed)[2]
    engines = support.ENGINES if a.engine == "both" else (a.engine,)
    out = {"n": n, "template": a.template, "directions": int(dirs.shape[0])}
    vals = {}
    for e in engines:
        for _ in range(max(1, a.repeat)):  # first call pays module load / attribute setup
            r = support.support_box(lo, hi, dirs, engine=e)
        vals[e] = r["obj"].cpu().numpy()
        out[e] = {"device_ms": r["ms"], "directions_per_s": dirs.shape[0] / (r["ms"] / 1e3)}
        if "iters" in r:
            out[e]["mean_iters"] = r["iters"].float().mean(dim=0).tolist()
    if len(vals) == 2:
        v0, v1 = vals["closed-form"], vals["simplex"]
        out["max_abs_discrepancy"] = float(np.max(np.abs(v0 - v1)))
        out["max_rel_discrepancy"] = float(np.max(np.abs(v0 - v1) / np.maximum(1, np.abs(v0))))
    if a.out:
        np.savez(a.out, lo=lo, hi=hi, dirs=dirs, **{k.replace("-", "_"): v for k, v in vals.items()})
    print(json.dumps(out))
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_1609_08114_b200.cli")
    sub = ap.add_subparsers(dest="cmd", required=True)
    p = sub.add_parser("gen", help="write a seeded batch file (npz)")
    p.add_argument("--class", dest="klass", choices=["feasible", "infeasible", "box"],
                   default="feasible")
    p.add_argument("-n", type=int, required=True)
    p.add_argument("-m", type=int, default=0)
    p.add_argument("--count", type=int, required=True)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("-o", "--out", required=True)
    p = sub.add_parser("solve", help="solve a batch file on the GPU")
    p.add_argument("path")
    p.add_argument("--pivot", choices=["lpc", "rpc"], default="lpc")
    p.add_argument("--seed", type=int, default=0, help="RPC seed")
    p.add_argument("--repeat", type=int, default=10, help="median over repeats (P:230: 10 runs)")
    p.add_argument("-o", "--out", default=None, help="per-LP results CSV")
    p = sub.add_parser("support-demo", help="support-function sampling of a box (PAPER.md §7)")
    p.add_argument("-n", type=int, default=5)
    p.add_argument("--box", choices=["paper", "random"], default="paper")
    p.add_argument("--template", choices=["box", "oct", "random"], default="oct")
    p.add_argument("--count", type=int, default=0, help="random template size")
    p.add_argument("--engine", choices=["closed-form", "simplex", "both"], default="both")
    p.add_argument("--repeat", type=int, default=2, help="report the last of R runs")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("-o", "--out", default=None)
    try:
        a = ap.parse_args(argv)
    except SystemExit as ex:
        return 0 if ex.code == 0 else 1
    try:
        return {"gen": cmd_gen, "solve": cmd_solve, "support-demo": cmd_support_demo}[a.cmd](a)
    except Exception as ex:  # pragma: no cover - internal failure
        print(f"{a.cmd}: internal error: {ex}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
