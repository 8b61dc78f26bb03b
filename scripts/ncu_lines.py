#!/usr/bin/env python
"""Per-CUDA-source-line instruction and stall-sample totals from an ncu report
(`ncu -i rep --page source --csv --print-source cuda,sass`).

  python scripts/ncu_lines.py gpurun_out/prof.ncu-rep [launch_index] [top]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
launch = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", str(launch), "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    ii = hdr.index("Instructions Executed")
    si = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        inst = float(r[ii] or 0)
        st = float(r[si] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    agg[key][0] += inst
    agg[key][1] += st
    agg[key][2] = r[1][:90]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp-instructions {ti:.4e}, stall samples {ts:.0f}")
for (f, l), (i, s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{i / ti * 100:5.1f}% inst {s / ts * 100:5.1f}% stall  {f}:{l:<5d} {src}")
