#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum, dram__bytes_read/write.sum per launch)
of a bench / solve command: the LAST solve (launches from the last tensor_seed_kernel on), per
kernel: launches, ms, share of the solve, DRAM bytes.  Optionally records the per-step DRAM bytes
of each kernel into profiles/ncu_traffic.json under --config.

  python tools/launch_summary.py gpurun_out/x_launch_c5.csv [--config C5 --traffic-json F] [--md out.md]
"""
import argparse
import collections
import csv
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--config")
    ap.add_argument("--traffic-json")
    ap.add_argument("--md")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.csv)))
    hdr, byid = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            e = byid.setdefault(d["ID"], {"name": d["Kernel Name"].split("(")[0]})
            e[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    ids = list(byid.values())
    starts = [i for i, e in enumerate(ids) if "tensor_seed_kernel" in e["name"]]
    last = ids[starts[-1]:] if starts else ids
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for e in last:
        k = e["name"].replace("void ", "").replace("cyl::", "").split("<")[0]
        agg[k][0] += 1
        agg[k][1] += e.get("gpu__time_duration.sum", 0.0)
        agg[k][2] += e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    lines = [f"launch list: {a.csv} (last solve: {len(last)} launches, {tot / 1e6:.3f} ms "
             f"serialised, cold-cache ncu times)", "",
             "| kernel | launches | ms | share | DRAM GB |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {v[0]} | {v[1] / 1e6:.3f} | {v[1] / tot:.3f} | {v[2] / 1e9:.3f} |")
    print("\n".join(lines))
    if a.md:
        open(a.md, "w").write("\n".join(lines) + "\n")
    if a.traffic_json and a.config:
        try:
            j = json.load(open(a.traffic_json))
        except Exception:
            j = {}
        j.setdefault("per_step_dram_bytes", {})[a.config] = {k: int(v[2]) for k, v in agg.items()}
        j["source"] = ("ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                       "--clock-control none of `python bench.py --steps 1 --warmup 3 "
                       "--no-cpu-baseline --no-e2e [--config C]`, last solve (tools/launch_summary.py)")
        json.dump(j, open(a.traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main()
