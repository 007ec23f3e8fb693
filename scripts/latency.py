import ctypes, sys
sys.path.insert(0, '.')
from paper_1609_08114_b200 import lpb
lpb._lib.lpb_selftest_latency.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
names = ['redux_argmax', 'shfl_argmax', 'div_fast', 'dfma', 'syncthreads', 'shfl', 'redux', 'dsetp_sel', 'chk', 'recip_of', 'rcp64h']
for th in (32, 128, 256):
    out = (ctypes.c_longlong * 11)()
    rc = lpb._lib.lpb_selftest_latency(th, out)
    print(th, rc, {k: out[i] for i, k in enumerate(names)})
lpb._lib.lpb_selftest_prow.argtypes = [ctypes.POINTER(ctypes.c_longlong)]
out = (ctypes.c_longlong * 3)()
print('prow switch/select/divonly', lpb._lib.lpb_selftest_prow(out), list(out))
lpb._lib.lpb_selftest_fp64_peak.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
a, b = ctypes.c_double(), ctypes.c_double()
print('fp64 peak', lpb._lib.lpb_selftest_fp64_peak(ctypes.byref(a), ctypes.byref(b)), 'DFMA TFLOP/s', a.value, 'RCP64H Gops', b.value)
