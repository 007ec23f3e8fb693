#!/bin/bash
# Host-side AddressSanitizer + UndefinedBehaviorSanitizer run of the C ABI's host pipeline
# (lpb_api.cu: contexts, chunked H2D -> kernel -> D2H streams, launch memos) on the GPU box.
# Builds ab/asan (host code compiled with -fsanitize=address,undefined), preloads the
# sanitizer runtimes into python and drives host-pointer and device-pointer solves,
# including concurrent contexts on several host threads.  Output: gpurun_out/<dir>/asan.txt
set -u
OUT=${1:-gpurun_out/asan}
mkdir -p "$OUT"
python paper_1609_08114_b200/build.py --variant ab/asan \
  -Xcompiler=-fsanitize=address -Xcompiler=-fsanitize=undefined -Xcompiler=-fno-omit-frame-pointer > "$OUT/build.txt" 2>&1
ASAN_LIB=$(gcc -print-file-name=libasan.so)
UBSAN_LIB=$(gcc -print-file-name=libubsan.so)
LD_PRELOAD="$ASAN_LIB:$UBSAN_LIB" \
ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0:replace_intrin=0:abort_on_error=1 \
UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1 \
python - > "$OUT/asan.txt" 2>&1 <<'PY'
import sys, threading, numpy as np, torch
sys.path.insert(0, "ab/asan"); sys.path.insert(1, ".")
import lpgen
from paper_1609_08114_b200 import lpb
print("lib", lpb.LIB_PATH)
def host_solve(A, b, c, **kw):
    return lpb.solve(A, b, c, **kw)
runs = [("cfg2", 400, {}), ("cfg3", 20, {}), ("cfg2s", 500, {}), ("cfg3s", 50, {}),
        ("cfg1", 1000, {}), ("cfg1m", 20000, {}), ("cfg9", 2000, {})]
for name, B, kw in runs:
    A, b, c = lpgen.make_config(name, B)
    r = host_solve(A, b, c, **kw)
    print(name, B, "host path statuses", np.bincount(r["status"], minlength=6).tolist())
    At, bt, ct = (torch.from_numpy(v).cuda() for v in (A, b, c))
    rd = lpb.solve(At, bt, ct)
    assert np.array_equal(rd["status"].cpu().numpy(), r["status"])
    assert np.array_equal(rd["obj"].cpu().numpy(), r["obj"], equal_nan=True)
lo, hi, dirs = lpgen.make_config("cfg5", 300001)
h = lpb.hyperbox(lo, hi, dirs)
print("hyperbox host", h["obj"][:3])
# concurrent contexts from host threads (the C ABI drops the GIL inside ctypes calls)
errs = []
def worker(name, B, seed):
    try:
        A, b, c = lpgen.make_config(name, B)
        for _ in range(3):
            lpb.solve(A, b, c)
    except Exception as e:
        errs.append(repr(e))
ts = [threading.Thread(target=worker, args=(nm, B, i)) for i, (nm, B) in
      enumerate([("cfg2", 200), ("cfg2", 150), ("cfg3", 10), ("cfg9", 500), ("cfg1", 1000), ("cfg10", 300)])]
[t.start() for t in ts]; [t.join() for t in ts]
assert not errs, errs
print("ASAN-UBSAN-CLEAN")
PY
echo "rc=$?" >> "$OUT/asan.txt"
