#!/usr/bin/env python
"""Key metrics and warp-stall reasons (cycles per issued instruction) of every kernel in an ncu
report.   python tools/ncu_stalls.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
txt = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[0]
for row in rows[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:70])
    for k in KEYS:
        if k in d:
            print(f"  {k} = {d[k]}")
    st = []
    for k, v in d.items():
        if "smsp__average_warps_issue_stalled" in k and "per_issue_active" in k:
            try:
                st.append((float(v), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    st.sort(reverse=True)
    print("  stalls:", ", ".join(f"{n} {v:.2f}" for v, n in st[:9]))
