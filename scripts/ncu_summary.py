"""Summarise an ncu report: instruction mix per pivot, stall reasons, hot windows.
python scripts/ncu_summary.py report.ncu-rep <pivots_total> <warps_per_lp>"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
piv = float(sys.argv[2]) * float(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv'], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = r[2:]
i_s = h.index('# Samples'); i_src = h.index('Source'); i_ex = h.index('Instructions Executed')
tot = sum(int(x[i_ex]) for x in rows)
print('instructions', tot, 'per warp-pivot', tot / piv if piv else '')
c = Counter(); s = Counter()
for x in rows:
    op = x[i_src].strip().split()
    op = [t for t in op if not t.startswith('@')][0].split('.')[0] if op else '?'
    c[op] += int(x[i_ex]); s[op] += int(x[i_s])
print(' '.join(f'{k}:{v/piv:.1f}' if piv else f'{k}:{v}' for k, v in c.most_common(20)))
raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines())); hh = rr[0]; vv = rr[2]
st = {}
for k, x in zip(hh, vv):
    if k.startswith('smsp__pcsamp_warps_issue_stalled') and not k.endswith('not_issued'):
        st[k.replace('smsp__pcsamp_warps_issue_stalled_', '')] = float(x.replace(',', ''))
    if k in ('gpu__time_duration.sum', 'sm__inst_executed.avg.per_cycle_active',
             'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
             'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
             'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__grid_size', 'launch__block_size'):
        print(k, x)
tt = sum(st.values())
print('stalls:', ' '.join(f'{k}:{v/tt*100:.0f}%' for k, v in sorted(st.items(), key=lambda t: -t[1]) if v / tt > 0.02))
