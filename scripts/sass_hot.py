"""Per-instruction hot spots of an ncu source page (SASS) export:
    ncu -i rep --page source --csv --print-source sass > x.csv; python scripts/sass_hot.py x.csv
Prints executed instructions (warp-level counts) with their stall samples, top stall reason."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
minexec = float(sys.argv[2]) if len(sys.argv) > 2 else 1e5
tot = sum(float(r[ix["# Samples"]] or 0) for r in rows[2:])
print(f"total samples {tot:.0f}")
acc = 0
for r in rows[2:]:
    ex = float(r[ix["Instructions Executed"]] or 0)
    smp = float(r[ix["# Samples"]] or 0)
    if ex < minexec and smp < tot * 0.002:
        continue
    st = sorted(((float(r[ix[s]] or 0), s[6:]) for s in stalls), reverse=True)[:2]
    acc += smp
    print(f"{r[0][-5:]} {ex:10.0f} {smp:7.0f} {100*smp/tot:5.2f}% {acc/tot*100:5.1f}  "
          f"{st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}  | {r[1].strip()[:60]}")
