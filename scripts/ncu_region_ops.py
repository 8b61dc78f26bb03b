#!/usr/bin/env python
"""Per source-region opcode classes (FP64 / DMMA / LDS-STS / global / int+control) of a kernel
in an ncu report, regions given as dg_stage.cu line ranges.
  python scripts/ncu_region_ops.py rep.ncu-rep units name:lo-hi [name:lo-hi ...]"""
import collections, csv, io, subprocess, sys
rep, units = sys.argv[1], float(sys.argv[2])
regs = []
for a in sys.argv[3:]:
    n, r = a.split(":"); lo, hi = r.split("-"); regs.append((n, int(lo), int(hi)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", "0", "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = None; fname = ""; cur = None; seen = set()
agg = collections.defaultdict(collections.Counter)
def cls(op):
    if op in ("DFMA", "DADD", "DMUL", "DSETP", "DMNMX"): return "fp64"
    if op == "DMMA": return "dmma"
    if op in ("LDS", "STS", "LDSM"): return "smem"
    if op in ("LDG", "STG", "LDGSTS", "LDL", "STL"): return "gmem"
    if op in ("MUFU",): return "mufu"
    return "int/ctl"
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0].isdigit():
        ln = int(r[0]); cur = "other"
        if fname == "dg_stage.cu":
            for n, lo, hi in regs:
                if lo <= ln <= hi: cur = n; break
        else: cur = fname
        continue
    if r[2] in ("", "...", "-") or r[2] in seen: continue
    seen.add(r[2])
    t = r[3].strip().split()
    if not t: continue
    op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    try: n = float(r[hdr.index("Instructions Executed")] or 0)
    except ValueError: continue
    agg[cur][cls(op)] += n
C = ["fp64", "dmma", "smem", "gmem", "mufu", "int/ctl"]
print("region".ljust(18) + "".join(c.rjust(9) for c in C) + "    total")
tt = collections.Counter()
for k, d in sorted(agg.items(), key=lambda x: -sum(x[1].values())):
    print(k.ljust(18) + "".join(f"{d[c] / units:9.0f}" for c in C) + f"{sum(d.values()) / units:9.0f}")
    tt.update(d)
print("TOTAL".ljust(18) + "".join(f"{tt[c] / units:9.0f}" for c in C) + f"{sum(tt.values()) / units:9.0f}")
