#!/usr/bin/env python
"""Per-CUDA-line stall samples (with reason split) from an ncu report.
  python scripts/ncu_stalls.py gpurun_out/prof.ncu-rep [launch] [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
launch = sys.argv[2] if len(sys.argv) > 2 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
fname = ""
agg = collections.defaultdict(collections.Counter)
src = {}
cols = ["stall_barrier", "stall_short_sb", "stall_long_sb", "stall_wait", "stall_mio", "stall_selected",
        "stall_branch_resolving", "Warp Stall Sampling (All Samples)", "Instructions Executed"]
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
    key = (fname, int(r[0]))
    src[key] = r[1][:70]
    for c in cols:
        try:
            agg[key][c] += float(r[hdr.index(c)] or 0)
        except (ValueError, IndexError):
            pass
tot = sum(v["Warp Stall Sampling (All Samples)"] for v in agg.values()) or 1
ti = sum(v["Instructions Executed"] for v in agg.values()) or 1
print(f"samples {tot:.0f}, warp-instructions {ti:.3e}")
for k, v in sorted(agg.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"])[:top]:
    s = v["Warp Stall Sampling (All Samples)"]
    print(f"{s / tot * 100:5.1f}% i{v['Instructions Executed'] / ti * 100:4.1f} bar{v['stall_barrier'] / tot * 100:4.1f} "
          f"ssb{v['stall_short_sb'] / tot * 100:4.1f} lsb{v['stall_long_sb'] / tot * 100:4.1f} "
          f"w{v['stall_wait'] / tot * 100:4.1f} {k[0]}:{k[1]} {src[k]}")
