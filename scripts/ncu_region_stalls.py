#!/usr/bin/env python
"""Per source-region instructions and stall reasons (sample shares) of one launch.
  python scripts/ncu_region_stalls.py rep.ncu-rep launch units name:lo-hi [...]"""
import collections, csv, io, subprocess, sys
rep, launch, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
regs = []
for a in sys.argv[4:]:
    n, r = a.split(":"); lo, hi = r.split("-"); regs.append((n, int(lo), int(hi)))
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--launch-skip", launch, "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cols = ["stall_short_sb", "stall_wait", "stall_barrier", "stall_long_sb", "stall_math", "stall_mio", "stall_selected",
        "stall_not_selected", "stall_branch_resolving", "stall_lg", "stall_no_inst", "stall_dispatch"]
hdr = None; fname = ""; cur = None; seen = set()
agg = collections.defaultdict(collections.Counter)
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
    def num(c):
        try: return float(r[hdr.index(c)] or 0)
        except ValueError: return 0.0
    agg[cur]["inst"] += num("Instructions Executed")
    for c in cols: agg[cur][c] += num(c)
T = sum(sum(d[c] for c in cols) for d in agg.values())
print("region".ljust(14) + "inst/u".rjust(8) + "stall%".rjust(8) + "".join(c.replace("stall_", "")[:8].rjust(9) for c in cols))
for k, d in sorted(agg.items(), key=lambda x: -x[1]["inst"]):
    st = sum(d[c] for c in cols)
    print(k.ljust(14) + f"{d['inst'] / units:8.0f}" + f"{st / T * 100:8.1f}" + "".join(f"{d[c] / T * 100:9.1f}" for c in cols))
