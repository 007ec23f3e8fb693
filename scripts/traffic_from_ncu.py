"""Per-LP DRAM traffic of the dominant kernel, from one `ncu --set full` capture per config,
for bench.py's roofline.traffic (dram__bytes_read.sum + dram__bytes_write.sum per launch):
    python scripts/traffic_from_ncu.py profiles/traffic.json gpurun_out/r01b/full_cfg2.ncu-rep:cfg2:50000 ...
(spec = report:config:LPs in the captured launch)."""
import csv
import json
import subprocess
import sys

out = {}
for spec in sys.argv[2:]:
    rep, cfg, lps = spec.split(":")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(m)
        tot += float(v[i].replace(",", "")) * scale[units[i]]
    out[cfg] = {"dram_bytes_per_lp": tot / int(lps), "source": f"{rep} ({lps} LPs, "
                f"{v[h.index('Kernel Name')][:60]})"}
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(out, indent=1))
