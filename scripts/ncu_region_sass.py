#!/usr/bin/env python
"""SASS of a dg_stage.cu line range with executed counts (per unit) and stall samples.
  python scripts/ncu_region_sass.py rep.ncu-rep launch units lo hi"""
import csv, io, subprocess, sys
rep, launch, units, lo, hi = sys.argv[1], sys.argv[2], float(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None; fname = ""; ln = 0; seen = set(); out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0].isdigit(): ln = int(r[0]); continue
    if fname != "dg_stage.cu" or not (lo <= ln <= hi): continue
    if r[2] in ("", "...", "-") or r[2] in seen: continue
    seen.add(r[2])
    n = float(r[hdr.index("Instructions Executed")] or 0); s = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    out.append((int(r[2], 16), ln, n / units, s, r[3].strip()))
for a, ln, n, s, t in sorted(out):
    if n > 0: print(f"{ln:5d} {n:7.2f} {s:6.0f}  {t[:70]}")
