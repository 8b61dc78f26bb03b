#!/usr/bin/env python
"""Per-source-line instructions / stall samples of dg_stage.cu lines in [lo, hi] from an ncu report.
  python scripts/ncu_lines2.py rep.ncu-rep lo hi [launch]"""
import csv, io, subprocess, sys
rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
launch = sys.argv[4] if len(sys.argv) > 4 else "0"
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
src = open("paper_2404_16648_b200/csrc/dg_stage.cu").read().splitlines()
hdr = None; fname = ""; tot_i = tot_s = 0; out = []
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit(): continue
    def num(cn):
        try: return float(r[hdr.index(cn)] or 0)
        except ValueError: return 0.0
    i, s = num("Instructions Executed"), num("Warp Stall Sampling (All Samples)")
    tot_i += i; tot_s += s
    ln = int(r[0])
    if fname == "dg_stage.cu" and lo <= ln <= hi and (i or s):
        out.append((ln, i, s))
for ln, i, s in out:
    print(f"{ln:5d} {i/tot_i*100:5.1f}%i {s/tot_s*100:5.1f}%s  {src[ln-1].strip()[:90]}")
