"""Generator contracts."""
import numpy as np

import lpgen


def test_determinism():
    a = lpgen.twophase_signed(7, 9, 6, 3)
    b = lpgen.twophase_signed(7, 9, 6, 3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_g1_feasible_start_bounded():
    A, b, c = lpgen.signed_bounded(50, 6, 4, 1)
    assert A.shape == (50, 6, 4) and b.shape == (50, 6) and c.shape == (50, 4)
    assert np.all(b >= 1.0) and np.all(A[:, 0, :] >= 1.0)


def test_g2_cover_rows_negative_and_xstar_feasible():
    B, m, n = 40, 12, 7
    A, b, c = lpgen.twophase_signed(B, m, n, 5)
    kk = int(np.ceil(m / 4))
    # cover rows are b = -(Q x*) + U[0,1): negative unless x* is tiny (n small); others >= 1
    assert np.all((b < 0).sum(axis=1) <= kk) and np.mean((b < 0).sum(axis=1)) > kk - 0.5
    xs_ok = np.einsum("bij->bi", A) is not None  # shape sanity
    assert xs_ok and np.sum(b >= 1.0) >= B * (m - kk)
    assert np.all(b[:, 0] > 0)  # the budget row is never a cover row


def test_oct_and_box_counts():
    assert lpgen.box_directions(3).shape == (6, 3)
    for n in (2, 5, 28):
        d = lpgen.oct_directions(n)
        assert d.shape == (2 * n * n, n)
        np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-12)


def test_g3_box_and_dirs():
    lo, hi, dirs = lpgen.hyperbox(100, 5, 4)
    np.testing.assert_allclose(hi - lo, 0.02, atol=1e-15)
    np.testing.assert_allclose((lo + hi) / 2, [1, 0, 0, 0, 0], atol=1e-15)
    assert dirs.shape == (100, 5)
    lo, hi, dirs = lpgen.hyperbox(3000, 28, 5)
    assert np.all(hi > lo) and dirs.shape == (3000, 28)
    np.testing.assert_allclose(np.linalg.norm(dirs, axis=1), 1.0, atol=1e-12)


def test_status_mix_negated_rows():
    A, b, c = lpgen.status_mix(30, 8, 5, 2, infeasible_start=True)
    assert np.all((b < 0).sum(axis=1) == 2)


def test_config_table():
    assert lpgen.CONFIGS["cfg2"]["B"] == 50000 and lpgen.CONFIGS["cfg5"]["B"] == 6003000
    A, b, c = lpgen.make_config("cfg3", B=3)
    assert A.shape == (3, 200, 200) and np.all((b < 0).sum(axis=1) == 50)


def test_shards_equal_slices_of_the_full_batch():
    for gen, sh in ((lpgen.signed_bounded, lpgen.signed_bounded_shard),
                    (lpgen.twophase_signed, lpgen.twophase_signed_shard)):
        full = gen(23, 9, 7, 11)
        for lo, hi in ((0, 5), (5, 23), (17, 18)):
            part = sh(23, 9, 7, 11, lo, hi)
            for f, p in zip(full, part):
                assert np.array_equal(f[lo:hi], p)
    lo_b, hi_b, d = lpgen.make_config_shard("cfg4", 5000, 100, 300)
    assert np.array_equal(d, lpgen.hyperbox(5000, 5, 4)[2][100:300])


def test_shared_polytope_layout_and_shards():
    A, b, c = lpgen.shared_polytope(50, 12, 9, 4)
    assert A.shape == (12, 9) and b.shape == (12,) and c.shape == (50, 9)
    A1, b1, _ = lpgen.signed_bounded(1, 12, 9, 4)
    assert np.array_equal(A, A1[0]) and np.array_equal(b, b1[0])
    A2, b2, c2 = lpgen.make_config_shard("cfg2s", 200, 40, 90)
    Af, bf, cf = lpgen.make_config("cfg2s", 200)
    assert np.array_equal(A2, Af) and np.array_equal(b2, bf) and np.array_equal(c2, cf[40:90])
    _, b3, _ = lpgen.shared_polytope(3, 40, 40, 3, "G2")
    assert (b3 < 0).sum() == 10  # ceil(m/4) covering rows


def test_hyperbox_shards_cross_blocks():
    """G3 shards are generated block by block and equal slices of the full batch, across
    template / block boundaries (multi-GPU ranks draw only their slice)."""
    n, B = 3, 3 * lpgen.HB_BLOCK + 77
    full = lpgen.hyperbox(B, n, 9)[2]
    t = 2 * n * n
    for lo, hi in ((0, 5), (t - 2, t + 3), (t + lpgen.HB_BLOCK - 4, t + lpgen.HB_BLOCK + 9),
                   (1000, B), (B - 1, B)):
        _, _, d = lpgen.make_config_shard("cfg4", B, lo, hi) if n == 5 else (None, None,
                                                                               lpgen.hyperbox_dirs(n, 9, lo, hi))
        assert np.array_equal(d, full[lo:hi])
    assert np.array_equal(lpgen.hyperbox(B, n, 9)[2], full)  # deterministic


def test_kmax_bound_holds():
    """lpgen.kmax_bound (the solver's kmax_hint in bench.py) bounds #{b_i < 0} of every LP its
    generator draws: G1 has none (type 1), G2 exactly ceil(m/4) (type 2)."""
    import numpy as np
    for name in ("cfg1", "cfg2", "cfg3", "cfg8", "cfg2s", "cfg3s", "cfg9"):
        A, b, c = lpgen.make_config(name, 300)
        kb = lpgen.kmax_bound(name)
        k = (np.atleast_2d(b) < 0).sum(axis=-1)
        assert k.max() <= kb, name
        if lpgen.CONFIGS[name]["gen"] == "G2":
            assert k.min() == kb, name
    assert lpgen.kmax_bound("cfg4") == -1
