#!/usr/bin/env python
"""profiles/ncu_traffic.json from an ncu --metrics CSV of a C5 bench run (bench.py's
roofline.traffic): per-launch DRAM bytes of the fused k_fs and the in-place k_ip launches.
usage: python scripts/traffic_json.py <metrics.csv> <particles> <K> <source-note>"""
import csv
import json
import sys
from collections import defaultdict

path, npart, K, note = sys.argv[1], float(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = defaultdict(dict)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
fam = defaultdict(list)
for (_, name), m in per.items():
    for f in ("k_fs", "k_ip"):
        if f"::{f}<" in name:
            fam[f].append(m)
out = {"workload": "C5", "particles": int(npart), "rebin_interval": K, "source": note}
for f, ms in fam.items():
    out[f] = sum(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"] for m in ms) / len(ms)
    out[f + "_launches"] = len(ms)
    if all("lts__t_sector_hit_rate.pct" in m for m in ms):
        out[f + "_l2_hit_pct"] = sum(m["lts__t_sector_hit_rate.pct"] for m in ms) / len(ms)
    if all("lts__t_sectors_op_red.sum" in m for m in ms):
        out[f + "_red_sectors"] = sum(m["lts__t_sectors_op_red.sum"] for m in ms) / len(ms)
    if all("gpu__time_duration.sum" in m for m in ms):
        out[f + "_ms"] = sum(m["gpu__time_duration.sum"] for m in ms) / len(ms) / 1e6
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
print(json.dumps(out))
