#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples of an ncu report (--page source, cuda,sass).
   python tools/ncu_lines.py report.ncu-rep [N] [launch index]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
sel = ["--launch-skip", sys.argv[3], "--launch-count", "1"] if len(sys.argv) > 3 else []
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + sel,
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, ""])
fname = ""
hdr = None
for r in csv.reader(io.StringIO(txt)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0] not in ("", "-"):
        try:
            s = int(r[4])
            ins = int(r[7])
        except ValueError:
            continue
        k = (fname, int(r[0]))
        agg[k][0] += s
        agg[k][1] += ins
        agg[k][2] = r[1][:100]
tot = sum(v[0] for v in agg.values()) or 1
for (f, l), (s, ins, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{s / tot:6.3f} {f}:{l:<5d} inst={ins:<12d} {src}")
