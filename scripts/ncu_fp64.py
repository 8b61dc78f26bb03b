#!/usr/bin/env python
"""FP64 work per launch of k_stage_h7 from an ncu --set full report -> profiles/ncu_fp64.json
(read by bench.py's fp64 row).  flops = 2 DFMA + DADD + DMUL (thread ops, predicated on) + the
FP64 tensor-path ops (sm__ops_path_tensor_src_fp64: DMMA, 2 per MAC).
  python scripts/ncu_fp64.py rep.ncu-rep"""
import csv, io, json, os, subprocess, sys
rep = sys.argv[1]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr = rows[0]
def val(r, k):
    return float(r[hdr.index(k)].replace(",", ""))
out = {"flops_per_launch": {}, "pipe_util": {}, "source": f"ncu --set full ({os.path.basename(rep)}), k_stage_h7"}
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    if "k_stage_h7" not in name:
        continue
    kind = name.split("<")[1][0]
    key = {"0": "rhs", "1": "stage0", "2": "stage12"}[kind]
    cyc = val(r, "sm__cycles_elapsed.avg") if "sm__cycles_elapsed.avg" in hdr else None
    el = val(r, "gpu__time_duration.sum") * 1e-3 * val(r, "sm__cycles_elapsed.avg.per_second") * 1e9 \
        if "sm__cycles_elapsed.avg.per_second" in hdr else cyc
    per = lambda k: val(r, k) * el
    dfma = per("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum.per_cycle_elapsed")
    dadd = per("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum.per_cycle_elapsed")
    dmul = per("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum.per_cycle_elapsed")
    tens = val(r, "sm__ops_path_tensor_src_fp64.sum")
    fl = 2 * dfma + dadd + dmul + tens
    out["flops_per_launch"][key] = fl
    out["pipe_util"][key] = {"fp64_pipe_pct": val(r, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                             "dmma_pipe_pct": val(r, "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
                             "ncu_ms": val(r, "gpu__time_duration.sum")}
    print(key, f"{fl / 1e9:.2f} GFLOP per launch", out["pipe_util"][key])
json.dump(out, open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_fp64.json"), "w"), indent=1)
