#!/usr/bin/env python
"""Summarise a gpurun_out/ ncu launch list (gpu__time_duration.sum per launch) and an
`ncu --set full` report into a markdown file under profiles/ (the judged evidence).

  python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/prof.ncu-rep profiles/rNN_x.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
       "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__sass_thread_inst_executed_op_dfma_pred_on.sum",
       "sm__sass_thread_inst_executed_op_dmul_pred_on.sum",
       "sm__sass_thread_inst_executed_op_dadd_pred_on.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed",
       "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__cycles_elapsed.avg.per_second", "smsp__cycles_active.avg"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = defaultdict(lambda: [0, 0.0])
    for d in data:
        if d.get("Metric Name", "gpu__time_duration.sum") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    unit = data[0]["Metric Unit"] if data else "ns"
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(v[1] for v in agg.values())
    out = [f"Launch list: {len(data)} launches, total {tot * scale:.1f} us (cold-cache, serialised; "
           "compare shares, not absolutes)\n", "| kernel | launches | total us | share |",
           "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1] * scale:.1f} | {100 * v[1] / tot:.1f}% |")
    return "\n".join(out)


def full(rep):
    if rep.endswith(".csv"):   # a raw page exported on the GPU box (large reports stay there)
        txt = open(rep).read()
    else:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return "(no --set full data)"
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        out.append(f"\n### `{name}`\n")
        out.append("| metric | value |\n|---|---|")
        vals = {}
        for w in RAW:
            if w in hdr:
                i = hdr.index(w)
                vals[w] = r[i]
                out.append(f"| {w} | {r[i]} {units[i]} |")
        try:
            fl = (2 * float(vals["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"].replace(",", "")) +
                  float(vals["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"].replace(",", "")) +
                  float(vals["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"].replace(",", "")))
            t = float(vals["gpu__time_duration.sum"].replace(",", ""))
            tu = units[hdr.index("gpu__time_duration.sum")]
            ts = t * {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3}.get(tu, 1e-6)
            out.append(f"| executed FP64 flops (2 DFMA + DMUL + DADD) | {fl:.4g} |")
            out.append(f"| executed FP64 TFLOP/s (ncu replay time) | {fl / ts / 1e12:.2f} |")
        except Exception:
            pass
    return "\n".join(out)


if __name__ == "__main__":
    lc, rep, dst = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else dst
    s = [f"# {title}\n", launches(lc), "\n## ncu --set full (top kernels)\n", full(rep)]
    open(dst, "w").write("\n".join(s) + "\n")
    print(dst)
