#!/usr/bin/env python
"""Opcode histogram (executed warp-instructions) of one launch in an ncu report.
  python scripts/ncu_sass_ops.py rep.ncu-rep [launch] [units]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]; launch = sys.argv[2] if len(sys.argv) > 2 else "0"
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch, "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[1]
ops = collections.Counter(); stall = collections.Counter(); tot = 0; tots = 0
for r in rows[2:]:
    if len(r) < len(hdr) - 2: continue
    try:
        n = float(r[hdr.index("Instructions Executed")] or 0); s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError: continue
    t = r[1].strip().split()
    if not t: continue
    op = t[1] if t[0].startswith("@") else t[0]
    op = op.split(".")[0]
    ops[op] += n; stall[op] += s; tot += n; tots += s
for k, v in ops.most_common(45):
    print(f"{k:10s} {v / tot * 100:5.1f}% inst {stall[k] / tots * 100:5.1f}% stall  {v / units:9.0f} per unit")
print("total", tot / units, "per unit")
