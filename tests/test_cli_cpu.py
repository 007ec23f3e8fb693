"""CLI host logic without a GPU: argument validation,
exit codes, seeded batch files, and the direction templates the support demo feeds kernel H."""
import os
import subprocess
import sys

import numpy as np

import lpgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1609_08114_b200.cli", *args],
                          cwd=ROOT, capture_output=True, text=True)


def test_gen_is_deterministic_and_validates(tmp_path):
    f1, f2 = tmp_path / "a.npz", tmp_path / "b.npz"
    for f in (f1, f2):
        r = _cli("gen", "--class", "infeasible", "-n", "6", "-m", "8", "--count", "5",
                 "--seed", "3", "-o", str(f))
        assert r.returncode == 0, r.stderr
    a, b = np.load(f1), np.load(f2)
    for k in ("A", "b", "c"):
        assert np.array_equal(a[k], b[k])
    assert a["A"].shape == (5, 8, 6) and np.all((a["b"] < 0).sum(axis=1) == 2)  # ceil(8/4)
    assert _cli("gen", "-n", "0", "-m", "3", "--count", "2", "-o", str(f1)).returncode == 1
    assert _cli("bogus").returncode == 1
    r = _cli("gen", "--class", "box", "-n", "28", "--count", "1", "-o", str(f1))
    assert r.returncode == 0 and np.load(f1)["lo"].shape == (28,)


def test_solve_reports_io_errors(tmp_path):
    assert _cli("solve", str(tmp_path / "missing.npz")).returncode == 2


def test_templates():
    assert lpgen.box_directions(2).tolist() == [[1, 0], [-1, 0], [0, 1], [0, -1]]
    for n, count in ((2, 8), (5, 50), (28, 1568)):
        d = lpgen.oct_directions(n)
        assert d.shape == (count, n)  # 2 n^2
        assert np.allclose(np.linalg.norm(d, axis=1), 1.0)
        assert len({tuple(r) for r in d}) == count  # deduplicated


def test_box_as_polytope_encoding():
    """The simplex engine's split-variable encoding has the box's support function as its LP
    optimum: checked against Eq. 6 with the oracle (both sides plain fp64)."""
    import oracle
    from paper_1609_08114_b200.support import box_as_polytope
    lo, hi, dirs = lpgen.hyperbox(300, 5, 0)
    A, b = box_as_polytope(lo, hi)
    B = dirs.shape[0]
    r = oracle.solve(np.broadcast_to(A, (B,) + A.shape), np.broadcast_to(b, (B, 10)),
                     np.concatenate([dirs, -dirs], axis=1))
    h = oracle.hyperbox(lo, hi, dirs)
    assert np.all(r["status"] == 0)
    assert np.max(np.abs(r["obj"] - h["obj"])) <= 1e-12
