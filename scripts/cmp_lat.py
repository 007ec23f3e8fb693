import ctypes, sys
sys.path.insert(0, '.')
from paper_1609_08114_b200 import lpb
lpb._lib.lpb_selftest_cmp.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
o = (ctypes.c_longlong * 3)()
print('rc', lpb._lib.lpb_selftest_cmp(o), 'cycles/step: fp64 max', o[0], 'u64 max', o[1], 'dfma', o[2])
