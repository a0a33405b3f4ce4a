"""DRAM bytes per launch of each tier kernel over one full lpa() run (all passes), from an
ncu --set full report -> JSON for bench.py's roofline.traffic.
usage: python tools/ncu_traffic.py report.ncu-rep > profiles/<round>/ncu_traffic_r27.json"""
import collections
import csv
import json
import subprocess
import sys

TIER_OF = [("k_thread", "thread"), ("k_group<0, float, 0, 16", "half_warp"),
           ("k_group<0, float, 0, 32", "warp"), ("k_team<0, float, 0, 256, 32,", "team32"),
           ("k_team<0, float, 0, 256, 128,", "team128"), ("k_team<0, float, 0, 256, 256,", "team256"),
           ("k_team<0, float, 0, 512, 512,", "cta512"), ("k_wide", "wide"), ("k_cluster", "wide"),
           ("k_hub", "hub")]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units, data = rows[0], rows[1], rows[2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
acc = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in data:
    d = dict(zip(h, r))
    name = d["Kernel Name"].replace("(int)", "").replace("(bool)", "").replace("nulpa::dev::", "")
    tier = next((t for k, t in TIER_OF if k in name), None)
    if tier is None:
        continue
    b = sum(float(d[m]) * scale[units[h.index(m)]] for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    a = acc[tier]
    a[0] += 1
    a[1] += b
    a[2] += float(d["gpu__time_duration.sum"])
print(json.dumps({t: {"launches": c, "dram_bytes_per_launch": b / c, "ms_per_launch": ms / c}
                  for t, (c, b, ms) in acc.items()}, indent=1))
