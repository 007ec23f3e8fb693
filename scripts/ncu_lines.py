"""Per-source-line instruction counts and stall samples from an ncu report's source page:
ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > X.csv
python scripts/ncu_lines.py X.csv [units] [min_instr_per_unit]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
fn = None; h = None
agg = collections.defaultdict(lambda: [0.0, 0.0, '', collections.Counter()])
def f(x):
    try: return float(x)
    except ValueError: return 0.0
for r in rows:
    if not r: continue
    if r[0] == 'File Path': fn = r[1].split('/')[-1]; continue
    if r[0] == 'Line No':
        h = r; iW = h.index('Warp Stall Sampling (All Samples)'); iE = h.index('Instructions Executed')
        st = [(i, k) for i, k in enumerate(h) if k.startswith('stall_') and 'Not Issued' not in k]
        continue
    if h is None: continue
    try: ln = int(r[0])
    except ValueError: continue
    k = (fn, ln); a = agg[k]
    a[0] += f(r[iE]); a[1] += f(r[iW]); a[2] = r[1][:70]
    for i, nm in st: a[3][nm[6:]] += f(r[i])
tot = sum(v[1] for v in agg.values()) or 1
print('total instr/unit %.1f' % (sum(v[0] for v in agg.values()) / units))
for k, v in sorted(agg.items()):
    if v[0] / units >= thr or v[1] / tot > 0.01:
        top = ', '.join('%s %.0f%%' % (n, 100 * c / (v[1] or 1)) for n, c in v[3].most_common(2))
        print('%-16s %4d i/u %7.1f samp %5.1f%% | %-60s | %s' % (k[0], k[1], v[0] / units, 100 * v[1] / tot, v[2].strip()[:60], top))
