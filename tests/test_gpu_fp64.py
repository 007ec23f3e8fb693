"""The kernels' branch-free division (csrc/lpb_fp64.cuh) must be bit-identical to IEEE
round-to-nearest division: checked against __ddiv_rn on the GPU and against the CPU's IEEE
division (numpy) for operands spanning the whole exponent range, zeros, and the values the
simplex kernels meet (ratios, pivot-row entries)."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_div_fast_bit_exact():
    import torch

    from gpu_util import dev_lib
    dlib = dev_lib()  # the selftest kernel lives in the development build only
    g = np.random.Generator(np.random.PCG64(7))
    n = 2_000_000
    mant = g.uniform(1.0, 2.0, n) * np.where(g.uniform(0, 1, n) < 0.5, -1.0, 1.0)
    a = np.ldexp(mant, g.integers(-1070, 1020, n))
    b = np.ldexp(g.uniform(1.0, 2.0, n), g.integers(-1000, 1000, n))
    # simplex-like operands, exact zeros and signed zeros
    a[:200000] = g.uniform(-100, 100, 200000)
    b[:200000] = g.uniform(1e-9, 50, 200000)
    a[200000:200100] = 0.0
    a[200100:200200] = -0.0
    b[300000:310000] = -b[300000:310000]
    at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    q = torch.empty_like(at)
    out = (ctypes.c_int64 * 2)()
    rc = dlib.lpb_selftest_div(ctypes.c_void_p(at.data_ptr()), ctypes.c_void_p(bt.data_ptr()),
                                   ctypes.c_void_p(q.data_ptr()), ctypes.c_int64(n), out)
    assert rc == 0
    assert out[0] == 0, f"{out[0]} quotients differ from __ddiv_rn"
    with np.errstate(all="ignore"):
        ref = a / b
    qn = q.cpu().numpy()
    assert np.array_equal(qn.view(np.int64), ref.view(np.int64))
    # out[1] counts operands outside the fast range (extreme exponents): they take __ddiv_rn


def test_recip_approx_error_bound():
    """The S kernel's ratio test orders rows by approximate quotients (recip_approx) and
    treats rows within a relative 2^-30 of the minimum as ties that are divided exactly; the
    approximation's own relative error must be far below that window for every divisor the
    ratio test can meet (v > eps_piv = 1e-9, up to huge magnitudes)."""
    import torch

    from gpu_util import dev_lib
    dlib = dev_lib()
    dlib.lpb_selftest_rcp_approx.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
    g = np.random.Generator(np.random.PCG64(11))
    n = 2_000_000
    v = np.ldexp(g.uniform(1.0, 2.0, n), g.integers(-30, 1000, n))
    v[:100000] = g.uniform(1e-9, 100.0, 100000)
    v[100000:100010] = [1e-9, 1.0, 2.0, 3.0, 0.1, 1e300, 1.5, 1.9999999999999998, 1.0000000000000002, 7.0]
    vt = torch.from_numpy(v).cuda()
    rt = torch.empty_like(vt)
    assert dlib.lpb_selftest_rcp_approx(ctypes.c_void_p(vt.data_ptr()), ctypes.c_void_p(rt.data_ptr()),
                                        ctypes.c_int64(n)) == 0
    r = rt.cpu().numpy().astype(np.longdouble)
    rel = np.abs(r * v.astype(np.longdouble) - 1.0)
    assert np.all(np.isfinite(rel))
    assert rel.max() < 2.0 ** -36, float(rel.max())  # measured 9.8e-13 (2^-39.9)
