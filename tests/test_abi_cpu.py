"""C-ABI library checks that need no GPU: it loads, exports every symbol include/lpb.h
declares, and its argument validation / pure-host entry points behave as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "lpb.h")
LIB = os.path.join(ROOT, "paper_1609_08114_b200", "liblpb.so")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import subprocess
        import sys
        subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_1609_08114_b200", "build.py")])
    return ctypes.CDLL(LIB)


DEV_HDR = os.path.join(ROOT, "include", "dev", "lpb_selftest.h")
DEV_LIB = os.path.join(ROOT, "devbuild", "paper_1609_08114_b200", "liblpb.so")


def _declared(path=HDR):
    src = re.sub(r"/\*.*?\*/", "", open(path).read(), flags=re.S)
    return sorted(set(re.findall(r"\b(lpb_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    """Every call include/*.h declares is exported by the product library, which exports no
    development entry point (include/dev/)."""
    import glob
    names = sorted(set(sum((_declared(h) for h in glob.glob(os.path.join(ROOT, "include", "*.h"))), [])))
    assert len(names) >= 12
    for nm in names:
        assert hasattr(lib, nm), nm
    for nm in _declared(DEV_HDR):
        assert not hasattr(lib, nm), f"product library exports the diagnostic {nm}"


def test_dev_build_exports_diagnostics():
    """The development build (build.py --dev) exports include/dev/lpb_selftest.h as well."""
    if not os.path.exists(DEV_LIB):
        import subprocess
        import sys
        subprocess.check_call([sys.executable, os.path.join(ROOT, "paper_1609_08114_b200", "build.py"), "--dev"])
    dlib = ctypes.CDLL(DEV_LIB)
    for nm in _declared(HDR) + _declared(DEV_HDR):
        assert hasattr(dlib, nm), nm


def test_product_library_reads_no_environment():
    """Tuning / A-B switches are compiled into the development build only: the product
    library's own objects do not reference getenv (the statically linked CUDA runtime does,
    for CUDA_VISIBLE_DEVICES and friends)."""
    import glob
    import subprocess
    objs = glob.glob(os.path.join(ROOT, "paper_1609_08114_b200", "build_obj", "*.o"))
    assert objs
    for o in objs:
        out = subprocess.run(["nm", "--undefined-only", o], capture_output=True, text=True).stdout
        assert "getenv" not in out, o


def test_default_options_and_strerror(lib):
    from paper_1609_08114_b200 import lpb
    o = lpb.default_options()
    assert o.struct_size == ctypes.sizeof(lpb.Options)
    assert o.eps_enter == 1e-9 and o.eps_piv == 1e-9 and o.eps_phase1 == 1e-9
    assert o.max_iter == 0 and o.bland_after == 0 and o.device == -1 and o.n_chunks == 0
    lib.lpb_strerror.restype = ctypes.c_char_p
    assert lib.lpb_strerror(-5) == b"no compiled size class fits this LP size"
    assert lib.lpb_default_options(None) == -1


def test_create_shape_validation_without_gpu(lib):
    P = ctypes.c_void_p
    ctx = P()
    # invalid shapes / kinds are rejected before any CUDA call
    assert lib.lpb_create(ctypes.byref(ctx), 0, 5, 5, 0, None) == -1
    assert lib.lpb_create(ctypes.byref(ctx), 10, 0, 5, 0, None) == -1
    assert lib.lpb_create(ctypes.byref(ctx), 10, 5, 5, 7, None) == -1
    assert lib.lpb_create(ctypes.byref(ctx), 10, 5, 4, 1, None) == -1  # hyperbox needs m=2n
    assert lib.lpb_create(None, 10, 5, 5, 0, None) == -1
    assert lib.lpb_create(ctypes.byref(ctx), 10, 4000, 4000, 0, None) == -5  # too big
    assert lib.lpb_destroy(None) == 0


def test_binding_struct_matches_header():
    """ctypes Options mirrors lpb_options field by field (names and order)."""
    from paper_1609_08114_b200 import lpb
    src = re.sub(r"/\*.*?\*/", "", open(HDR).read(), flags=re.S)
    body = re.search(r"typedef struct \{(.*?)\} lpb_options;", src, re.S).group(1)
    fields = re.findall(r"(\w+)\s*;", body)
    assert fields == [f[0] for f in lpb.Options._fields_]


def test_binding_enums_match_header():
    """Every LPB_* enum constant of include/lpb.h has the same value in the Python binding."""
    from paper_1609_08114_b200 import lpb
    src = re.sub(r"/\*.*?\*/", "", open(HDR).read(), flags=re.S)
    consts = dict((k, int(v.rstrip("u"))) for k, v in re.findall(r"\b(LPB_[A-Z0-9_]+)\s*=\s*(-?\d+u?)", src))
    assert len(consts) >= 18
    for k, v in consts.items():
        name = k[4:]
        if hasattr(lpb, name):
            assert getattr(lpb, name) == v, k
    for k in ("DEVICE_PTRS", "SHARED_BOX", "NO_X", "ASYNC", "SHARED_AB", "NO_TIMING", "GENERAL",
              "HYPERBOX", "RULE_LPC", "RULE_RPC",
              "OPTIMAL", "UNBOUNDED", "INFEASIBLE", "ITER_LIMIT", "NUMERICAL"):
        assert getattr(lpb, k) == consts["LPB_" + k], k


def test_option_validation_without_gpu(lib):
    """Undefined entering rules and cluster sizes are LPB_EINVAL at create (include/lpb.h)."""
    from paper_1609_08114_b200 import lpb
    ctx = ctypes.c_void_p()
    for kw in (dict(pivot_rule=2), dict(pivot_rule=-1), dict(cluster_ctas=3),
               dict(cluster_ctas=32), dict(eps_enter=-1.0), dict(kernel_class=5),
               dict(kernel_class=6), dict(kernel_class=8), dict(kernel_class=-1),
               dict(kmax_hint=-2), dict(kmax_hint=6)):
        o = lpb.default_options(**kw)
        assert lib.lpb_create(ctypes.byref(ctx), 10, 5, 5, 0, ctypes.byref(o)) == -1, kw
    for kc in (1, 4, 7):  # a general class on a hyperbox context
        o = lpb.default_options(kernel_class=kc)
        assert lib.lpb_create(ctypes.byref(ctx), 10, 10, 5, 1, ctypes.byref(o)) == -1, kc
    o = lpb.default_options()
    o.struct_size = 8  # an older / foreign layout
    assert lib.lpb_create(ctypes.byref(ctx), 10, 5, 5, 0, ctypes.byref(o)) == -1


def test_create_argument_validation_without_gpu(lib):
    """Shape / kind errors are LPB_EINVAL and sizes no class holds are LPB_ETOOBIG, decided
    before any CUDA call (include/lpb.h, lpb_create)."""
    ctx = ctypes.c_void_p()
    lib.lpb_create.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                               ctypes.c_int32, ctypes.c_void_p]
    for B, m, n, kind in ((0, 5, 5, 0), (10, 0, 5, 0), (10, 5, -1, 0), (10, 5, 5, 7),
                          (10, 5, 5, 1), (2 ** 31, 5, 5, 0)):
        assert lib.lpb_create(ctypes.byref(ctx), B, m, n, kind, None) == -1, (B, m, n, kind)
    assert lib.lpb_create(ctypes.byref(ctx), 10, 600, 600, 0, None) == -5
    assert lib.lpb_create(None, 10, 5, 5, 0, None) == -1
