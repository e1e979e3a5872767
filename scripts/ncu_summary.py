#!/usr/bin/env python
"""Summarise an ncu report (--page raw) and a launch list CSV into markdown/JSON.

usage: python scripts/ncu_summary.py <report.ncu-rep> [launches.csv] [--out profiles/name]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sectors_op_red.sum", "L2 red sectors"),
    ("lts__t_sectors_op_atom.sum", "L2 atom sectors"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
]
STALLS = [
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
    "smsp__average_warp_latency_issue_stalled_short_scoreboard",
    "smsp__average_warp_latency_issue_stalled_lg_throttle",
    "smsp__average_warp_latency_issue_stalled_mio_throttle",
    "smsp__average_warp_latency_issue_stalled_wait",
    "smsp__average_warp_latency_issue_stalled_math_pipe_throttle",
    "smsp__average_warp_latency_issue_stalled_barrier",
    "smsp__average_warp_latency_issue_stalled_membar",
    "smsp__average_warp_latency_issue_stalled_no_instruction",
    "smsp__average_warp_latency_issue_stalled_not_selected",
    "smsp__average_warp_latency_issue_stalled_selected",
    "smsp__average_warp_latency_issue_stalled_dispatch_stall",
    "smsp__average_warp_latency_issue_stalled_drain",
]


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m, name in METRICS:
            if m in hdr:
                d[name] = (r[hdr.index(m)], units[hdr.index(m)])
        st = {}
        for m in hdr:
            if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("_not_issued"):
                try:
                    st[m.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[hdr.index(m)].replace(",", ""))
                except ValueError:
                    pass
        tot = sum(st.values()) or 1.0
        d["stall_samples_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]}
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    t, c = defaultdict(float), defaultdict(int)
    for r in rows[h + 1:]:
        if len(r) > vi:
            try:
                name = r[ki].split("(")[0][-60:]
                t[name] += float(r[vi].replace(",", ""))
                c[name] += 1
            except ValueError:
                pass
    tot = sum(t.values())
    return [(k, v / 1e6, c[k], 100 * v / tot) for k, v in sorted(t.items(), key=lambda x: -x[1])]


def main():
    args = sys.argv[1:]
    out = None
    if "--out" in args:
        i = args.index("--out")
        out = args[i + 1]
        args = args[:i] + args[i + 2:]
    rep = args[0]
    lines = [f"# ncu summary: {rep}", ""]
    data = {"report": rep, "kernels": raw(rep)}
    for k in data["kernels"]:
        lines.append(f"## {k['kernel'][:120]}")
        for m, name in METRICS:
            if name in k:
                lines.append(f"- {name}: {k[name][0]} {k[name][1]}")
        lines.append(f"- top stall reasons (pc samples %): {k['stall_samples_pct']}")
        lines.append("")
    if len(args) > 1:
        ls = launches(args[1])
        data["launch_list"] = ls
        lines.append("## launch list (cold-cache, serialised; compare shares)")
        lines.append("| kernel | total ms | launches | share % |")
        lines.append("|---|---|---|---|")
        for k, ms, n, sh in ls[:20]:
            lines.append(f"| {k} | {ms:.3f} | {n} | {sh:.1f} |")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out + ".md", "w").write(text + "\n")
        json.dump(data, open(out + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
