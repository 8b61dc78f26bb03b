#!/usr/bin/env python
"""Attribute ncu per-line instructions/stall samples to the stage kernel's phases
(by source line ranges of the named device functions in dg_stage.cu).
  python scripts/ncu_phases.py gpurun_out/prof.ncu-rep [launch]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
launch = sys.argv[2] if len(sys.argv) > 2 else "0"
src = open("paper_2404_16648_b200/csrc/dg_stage.cu").read().splitlines()
# function start lines
starts = []
for i, l in enumerate(src, 1):
    m = re.match(r"^(?:__device__|__global__).*?\b(\w+)\(", l)
    if m:
        starts.append((i, m.group(1)))
def func_of(line):
    name = "?"
    for s, n in starts:
        if s <= line:
            name = n
    return name
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None
fname = ""
agg = collections.defaultdict(lambda: [0.0, 0.0])
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
    key = func_of(int(r[0])) if fname == "dg_stage.cu" else fname
    def num(c):
        try:
            return float(r[hdr.index(c)] or 0)
        except ValueError:
            return 0.0
    agg[key][0] += num("Instructions Executed")
    agg[key][1] += num("Warp Stall Sampling (All Samples)")
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, (i, s) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{s / ts * 100:5.1f}% stall  {i / ti * 100:5.1f}% inst  {k}")
