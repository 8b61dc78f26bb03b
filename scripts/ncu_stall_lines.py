#!/usr/bin/env python
"""Top source lines of an ncu report by warp-stall samples, with the dominant stall reason per line.
  python scripts/ncu_stall_lines.py rep.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
fname, hdr = "", None
agg = defaultdict(lambda: defaultdict(float))
src = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    src[key] = r[1][:70]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") or h.startswith("Warp Stall Sampling (All"):
            try:
                agg[key][h] += float(r[i])
            except ValueError:
                pass
tot = sum(v.get("Warp Stall Sampling (All Samples)", 0) for v in agg.values()) or 1
reasons = [h for h in (hdr or []) if h.startswith("stall_")]
print(f"stall samples {tot:.0f}; per-line reason columns: {len(reasons)}")
for key, v in sorted(agg.items(), key=lambda x: -x[1].get("Warp Stall Sampling (All Samples)", 0))[:top]:
    s = v.get("Warp Stall Sampling (All Samples)", 0)
    rs = sorted(((v[h], h) for h in reasons), reverse=True)[:2]
    rtxt = ", ".join(f"{h[6:]} {x / s * 100:.0f}%" for x, h in rs if s > 0 and x > 0)
    print(f"{s / tot * 100:5.1f}%  {key[0]}:{key[1]:<5d} {rtxt:40s} {src[key]}")
