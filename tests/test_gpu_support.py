"""GPU: support-function sampling -- the
closed-form engine (kernel H) bit-exact against the oracle's Eq. 6, the simplex engine
(shared-constraint general LPs) against the oracle's simplex on the same encoding, the two
engines within 1e-9 of each other, and the CLI commands end to end."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import lpgen
import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n,template,count", [(5, "oct", 0), (5, "random", 20000),
                                              (28, "oct", 0), (2, "box", 0)])
def test_support_engines(n, template, count):
    from paper_1609_08114_b200 import support
    from paper_1609_08114_b200.support import box_as_polytope
    lo, hi, rnd = lpgen.hyperbox(max(count, 1), n, 0 if n == 5 else 3)
    dirs = {"oct": lpgen.oct_directions(n), "box": lpgen.box_directions(n),
            "random": rnd}[template]
    cf = support.support_box(lo, hi, dirs, engine="closed-form")
    sx = support.support_box(lo, hi, dirs, engine="simplex")
    h = oracle.hyperbox(lo, hi, dirs)
    assert np.array_equal(cf["obj"].cpu().numpy(), h["obj"])
    A, b = box_as_polytope(lo, hi)
    B = dirs.shape[0]
    o = oracle.solve(np.broadcast_to(A, (B,) + A.shape), np.broadcast_to(b, (B, 2 * n)),
                     np.concatenate([dirs, -dirs], axis=1))
    assert np.array_equal(sx["status"].cpu().numpy(), o["status"])
    assert np.array_equal(sx["obj"].cpu().numpy(), o["obj"])
    assert np.array_equal(sx["iters"].cpu().numpy(), o["iters"])
    v0, v1 = cf["obj"].cpu().numpy(), sx["obj"].cpu().numpy()
    assert np.max(np.abs(v0 - v1) / np.maximum(1.0, np.abs(v0))) <= 1e-9


def test_support_polytope_general():
    """Many directions over one general polytope (the G1 generator's feasible region)."""
    from paper_1609_08114_b200 import support
    A, b, c = lpgen.shared_polytope(3000, 30, 30, 5, "G1")
    r = support.support_polytope(A, b, c, want_x=True)
    Ab = np.broadcast_to(A, (3000, 30, 30))
    bb = np.broadcast_to(b, (3000, 30))
    o = oracle.solve(Ab, bb, c)
    assert np.array_equal(r["status"].cpu().numpy(), o["status"])
    assert np.array_equal(r["obj"].cpu().numpy(), o["obj"])
    assert np.array_equal(r["x"].cpu().numpy(), o["x"])


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1609_08114_b200.cli", *args],
                          cwd=ROOT, capture_output=True, text=True)


def test_cli_end_to_end(tmp_path):
    f = tmp_path / "batch.npz"
    assert _cli("gen", "--class", "infeasible", "-n", "12", "-m", "12", "--count", "400",
                "--seed", "4", "-o", str(f)).returncode == 0
    csv = tmp_path / "res.csv"
    r = _cli("solve", str(f), "--repeat", "3", "-o", str(csv))
    assert r.returncode == 0, r.stderr
    s = json.loads(r.stdout.strip().splitlines()[-1])
    d = np.load(f)
    o = oracle.solve(d["A"], d["b"], d["c"])
    rows = open(csv).read().strip().splitlines()[1:]
    assert len(rows) == 400 and s["lps"] == 400
    objs = np.array([float(r_.split(",")[2]) for r_ in rows])
    assert np.array_equal(objs, o["obj"])
    r2 = _cli("solve", str(f), "--pivot", "rpc", "--seed", "1", "--repeat", "1", "-o", str(csv))
    objs2 = np.array([float(r_.split(",")[2]) for r_ in open(csv).read().strip().splitlines()[1:]])
    assert r2.returncode == 0
    assert np.max(np.abs(objs2 - objs) / np.maximum(1, np.abs(objs))) <= 1e-9  # rule-independent
    r3 = _cli("support-demo", "-n", "5", "--template", "random", "--count", "100000",
              "--engine", "both")
    assert r3.returncode == 0, r3.stderr
    out = json.loads(r3.stdout.strip().splitlines()[-1])
    assert out["directions"] == 100000 and out["max_rel_discrepancy"] <= 1e-9
    r4 = _cli("support-demo", "-n", "28", "--box", "random", "--template", "oct",
              "--engine", "closed-form")
    assert r4.returncode == 0 and json.loads(r4.stdout.strip().splitlines()[-1])["directions"] == 1568
