#!/usr/bin/env python
"""Per source line (all files) instructions and stall-sample shares of one kernel in an ncu report.
  python scripts/ncu_line_stalls.py rep.ncu-rep [top] [file-filter]"""
import collections, csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cols = ["stall_short_sb", "stall_wait", "stall_barrier", "stall_long_sb", "stall_math", "stall_mio", "stall_selected",
        "stall_not_selected", "stall_branch_resolving", "stall_lg", "stall_no_inst", "stall_dispatch", "stall_membar",
        "stall_sleep", "stall_tex", "stall_drain", "stall_misc"]
hdr = None; fname = ""; cur = None; seen = set()
agg = collections.defaultdict(collections.Counter)
src = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0].isdigit():
        cur = (fname, int(r[0])); src[cur] = r[1][:70]
        continue
    if r[2] in ("", "...", "-") or r[2] in seen: continue
    seen.add(r[2])
    def num(c):
        try: return float(r[hdr.index(c)] or 0) if c in hdr else 0.0
        except ValueError: return 0.0
    agg[cur]["inst"] += num("Instructions Executed")
    agg[cur]["samples"] += num("Warp Stall Sampling (All Samples)")
    for c in cols: agg[cur][c] += num(c)
T = sum(d["samples"] for d in agg.values())
I = sum(d["inst"] for d in agg.values())
print(f"total samples {T:.0f} inst {I:.0f}")
used = [c for c in cols if sum(d[c] for d in agg.values()) > 0.005 * T]
print("file:line".ljust(24) + "inst%".rjust(7) + "samp%".rjust(7) + "".join(c.replace("stall_", "")[:7].rjust(8) for c in used) + "  source")
for k, d in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:top]:
    print(f"{k[0][:16]}:{k[1]}".ljust(24) + f"{d['inst'] / I * 100:7.1f}{d['samples'] / T * 100:7.1f}" +
          "".join(f"{d[c] / T * 100:8.1f}" for c in used) + "  " + src.get(k, ""))
