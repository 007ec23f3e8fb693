"""Stall samples of an ncu SASS source export aggregated per CUDA source line.
    nvdisasm -g -c kernel.cubin > all.dis   (the cubin the profiled .so was linked from)
    python scripts/src_hot.py sass.csv all.dis <mangled kernel name> [top]
The SASS export's addresses are absolute; offsets from the first instruction index into
nvdisasm's line-annotated listing of the same kernel."""
import csv, re, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
body = rows[2:]
base = int(body[0][0], 16)
# offset -> (file, line) from the nvdisasm listing of the kernel
lines, cur, inside = {}, None, False
for ln in open(sys.argv[2]):
    if ln.startswith(sys.argv[3] + ":"):
        inside = True
        continue
    if inside and ln.startswith(".L_x_") is False and ln.startswith("//----"):
        if lines:
            break
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m:
        lines[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
tot = 0.0
for r in body:
    off = int(r[0], 16) - base
    key = lines.get(off, ("?", 0))
    smp = float(r[ix["# Samples"]] or 0)
    tot += smp
    a = agg[key]
    a[0] += smp
    a[1] += float(r[ix["Instructions Executed"]] or 0)
    for s in stalls:
        a[2][s[6:]] += float(r[ix[s]] or 0)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
print(f"total samples {tot:.0f}")
for key, (smp, ex, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    s2 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{key[0]:>18s}:{key[1]:<5d} {100 * smp / tot:5.1f}%  inst {ex:10.0f}  " +
          " ".join(f"{k}:{100 * v / max(smp, 1):.0f}%" for k, v in s2))
