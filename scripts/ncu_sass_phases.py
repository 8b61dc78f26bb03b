#!/usr/bin/env python
"""Stall samples per SASS address range (program-order phases) of one kernel in an ncu report.
  python scripts/ncu_sass_phases.py rep.ncu-rep file.cu name:line [name:line ...]
A phase starts at the lowest SASS address attributed to its marker line of file.cu and runs to
the next phase's start (addresses in program order; inlined helpers count with their caller)."""
import collections, csv, io, subprocess, sys
rep, fn = sys.argv[1], sys.argv[2]
marks = [(a.split(":")[0], int(a.split(":")[1])) for a in sys.argv[3:]]
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None; fname = ""; cur = None; seen = {}
def num(r, c):
    try: return float(r[hdr.index(c)] or 0)
    except (ValueError, IndexError): return 0.0
cols = ["stall_short_sb", "stall_wait", "stall_long_sb", "stall_selected", "stall_no_inst", "stall_branch_resolving", "stall_math", "stall_mio", "stall_lg"]
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if len(r) < 5: continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0].isdigit(): cur = (fname, int(r[0])); continue
    if r[2] in ("", "-", "...") or r[2] in seen: continue
    seen[r[2]] = (int(r[2], 16), cur, num(r, "Warp Stall Sampling (All Samples)"), num(r, "Instructions Executed"),
                  {c: num(r, c) for c in cols})
ins = sorted(seen.values())
starts = []
for name, ln in marks:
    a = [x[0] for x in ins if x[1] == (fn, ln)]
    if a: starts.append((min(a), name))
    else: print("no SASS for", name, ln)
starts.sort()
T = sum(x[2] for x in ins); I = sum(x[3] for x in ins)
agg = collections.defaultdict(collections.Counter)
for addr, cur, s, n, st in ins:
    ph = "pre"
    for a0, name in starts:
        if addr >= a0: ph = name
    agg[ph]["samp"] += s; agg[ph]["inst"] += n
    for c in cols: agg[ph][c] += st[c]
print("phase".ljust(12) + "samp%".rjust(7) + "inst%".rjust(7) + "".join(c.replace("stall_", "")[:7].rjust(8) for c in cols))
for _, name in [(0, "pre")] + starts:
    d = agg[name]
    print(name.ljust(12) + f"{d['samp'] / T * 100:7.1f}{d['inst'] / I * 100:7.1f}" + "".join(f"{d[c] / T * 100:8.1f}" for c in cols))
