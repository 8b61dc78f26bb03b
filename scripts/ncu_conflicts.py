#!/usr/bin/env python
"""Shared-memory bank-conflict wavefronts (excessive) per source line of an ncu report.
  python scripts/ncu_conflicts.py gpurun_out/prof.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, hdr, fname, out = list(csv.reader(io.StringIO(txt))), None, "", []
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
    def num(c):
        try:
            return float(r[hdr.index(c)] or 0)
        except ValueError:
            return 0.0
    out.append((num("L1 Wavefronts Shared Excessive"), num("L1 Wavefronts Shared"), fname, r[0], r[1][:90]))
tot = sum(o[0] for o in out) or 1
print(f"total excessive shared wavefronts {tot:.3e}, total shared wavefronts {sum(o[1] for o in out):.3e}")
for e, w, f, l, s in sorted(out, key=lambda x: -x[0])[:n]:
    print(f"{e / tot * 100:5.1f}% exc {e:.2e} of {w:.2e}  {f}:{l} {s}")
