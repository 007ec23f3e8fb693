"""Summarise a round's GPU evidence (bench JSON lines, ncu launch lists, ncu full captures)
into profiles/<tag>.md.   python scripts/summarize_profiles.py gpurun_out/r01 profiles/r01.md"""
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

src, dst = sys.argv[1], sys.argv[2]
out = [f"# GPU evidence — {os.path.basename(src)}", ""]
gpu = os.path.join(src, "gpu.txt")
if os.path.exists(gpu):
    out += ["```", open(gpu).read().strip(), "```", ""]

out += ["## bench.py lines", ""]
for f in sorted(glob.glob(os.path.join(src, "bench_*.json"))) + sorted(glob.glob(os.path.join(src, "ref_*.json"))):
    txt = open(f).read().strip().splitlines()
    line = next((t for t in txt if t.startswith("{")), None)
    if not line:
        out += [f"- {os.path.basename(f)}: no JSON line", ""]
        continue
    j = json.loads(line)
    r = j.get("roofline") or {}
    e = j.get("e2e") or {}
    cb = j.get("cpu_baseline") or {}
    out.append(f"- **{j['config']['workload']}** ({j.get('impl', 'ours')}): "
               f"{j['value']:.4g} {j['unit']}, {j['ms_per_step']:.4g} ms/step; "
               f"roofline {r.get('bound')} {r.get('achieved', 0):.4g}/{r.get('peak', 0):.4g} "
               f"{r.get('unit', '')} = {100 * r.get('frac', 0):.2f}%; e2e {e.get('value', 0):.4g} "
               f"{e.get('unit', '')}; oracle {cb.get('value', 0):.4g} LPs/s on {cb.get('cores')} cores; "
               f"clocks {j.get('clocks')}")
    out.append("")
    out.append("  `" + line + "`")
    out.append("")

out += ["## ncu launch lists (gpu__time_duration.sum, cold-cache, serialised)", ""]
for f in sorted(glob.glob(os.path.join(src, "launches_*.csv"))):
    rows = list(csv.reader(l for l in open(f) if not l.startswith("==")))
    if not rows:
        continue
    h = rows[0]
    try:
        ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    except ValueError:
        continue
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if len(r) <= iv or r[im] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0][-60:]
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in agg.values()) or 1.0
    out += [f"### {os.path.basename(f)}", "", "| kernel | launches | total | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {c} | {t:.4g} | {100 * t / tot:.1f}% |")
    out.append("")

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed.avg.per_cycle_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__shared_mem_per_block_dynamic",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
out += ["## ncu full captures (--set full --clock-control none)", ""]
for f in sorted(glob.glob(os.path.join(src, "full_*.ncu-rep"))):
    raw = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    if len(rows) < 3:
        continue
    h, units, v = rows[0], rows[1], rows[2]
    kname = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    out += [f"### {os.path.basename(f)}: `{kname[:110]}`", "", "| metric | value |", "|---|---|"]
    for m in METRICS:
        if m in h:
            i = h.index(m)
            out.append(f"| {m} | {v[i]} {units[i]} |")
    st = {}
    for k, x in zip(h, v):
        if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued"):
            try:
                st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(x.replace(",", ""))
            except ValueError:
                pass
    tt = sum(st.values()) or 1.0
    top = sorted(st.items(), key=lambda t: -t[1])[:6]
    out.append("| top stall reasons (pc sampling) | " +
               ", ".join(f"{k} {100 * s / tt:.0f}%" for k, s in top) + " |")
    out.append("")

os.makedirs(os.path.dirname(dst), exist_ok=True)
open(dst, "w").write("\n".join(out) + "\n")
print(dst)
