#!/usr/bin/env python3
"""Summarise an ncu report: key throughput metrics, stall reasons and the
hottest SASS lines (used to write profiles/*.md)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h, units, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fp64.avg.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct",
        "smsp__inst_executed.sum", "launch__occupancy_limit", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
for i, name in enumerate(h):
    if any(name == w or name.startswith(w + ".") or (w.endswith("pct") and name.startswith(w)) or
           (w == "launch__occupancy_limit" and name.startswith(w)) for w in want):
        print(f"{name:70s} {v[i]} {units[i]}".rstrip())
print("-- stalls per issue --")
for i, name in enumerate(h):
    if "average_warps_issue_stalled" in name and name.endswith("per_issue_active.ratio"):
        try:
            if float(v[i]) > 0.05:
                print(f"  {name.replace('smsp__average_warps_issue_stalled_', ''):50s} {v[i]}")
        except ValueError:
            pass
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(src.splitlines()))
    hh = rows[1]
    idx = {n: i for i, n in enumerate(hh)}
    data = rows[2:]
    key = "Warp Stall Sampling (All Samples)"
    tot = sum(int(x[idx[key]] or 0) for x in data)
    print(f"-- SASS: {len(data)} instructions, {tot} stall samples; top lines --")
    for x in sorted(data, key=lambda x: -int(x[idx[key]] or 0))[:int(sys.argv[2])]:
        print(f"  {x[idx['Source']][:70]:72s} {x[idx[key]]:>6s}")
