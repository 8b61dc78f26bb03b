#!/usr/bin/env python
"""Summarise an ncu --set full report (.ncu-rep) or a launch-list CSV into profiles/.

  python scripts/ncu_summary.py full  gpurun_out/prof.ncu-rep  profiles/r01_x_ncu.txt [--traffic-key k_stage_3_7]
  python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_x_launches.txt

`full` writes the key metrics of every captured launch and the mean DRAM bytes
per launch; with --traffic-key it also records that mean in
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).
`launches` aggregates the per-launch gpu__time_duration list by kernel name
(count, total, share) -- ncu's launch list is cold-cache and serialised, so the
share of the step is what compares with bench.py, not the absolute time.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "gcc__cache_requests_type_instruction.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
    "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_global_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
]


def full(rep, out, traffic_key=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {os.path.basename(rep)}"]
    dram = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"\n## launch {r[hdr.index('ID')] if 'ID' in hdr else '?'}: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"{k} = {r[i]} {units[i]}")
        st = [(hdr[i], r[i]) for i in range(len(hdr))
              if "pcsamp_warps_issue_stalled" in hdr[i] and not hdr[i].endswith("not_issued")]
        st = sorted(((k, float(v)) for k, v in st if v.replace(".", "", 1).isdigit()), key=lambda x: -x[1])[:8]
        tot = sum(v for _, v in st) or 1.0
        lines.append("top stall reasons (pc samples): " +
                     ", ".join(f"{k.split('stalled_')[1]} {v / tot * 100:.0f}%" for k, v in st))
        ib, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        dram.append(float(r[ib]) * scale.get(units[ib], 1) + float(r[iw]) * scale.get(units[iw], 1))
    mean = sum(dram) / len(dram) if dram else None
    lines.append(f"\nmean dram bytes (read+write) per launch: {mean:.4e}" if mean else "")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_key and mean:
        p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "profiles", "ncu_traffic.json")
        d = json.load(open(p)) if os.path.exists(p) else {}
        d[traffic_key] = mean
        d[traffic_key + "_source"] = os.path.basename(out)
        json.dump(d, open(p, "w"), indent=1)
    print("\n".join(lines))


def launches(src, out):
    agg = OrderedDict()
    with open(src) as f:
        body = [l for l in f if not l.startswith("==")]
    rows = list(csv.DictReader(io.StringIO("".join(body))))
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}.get(unit, 1.0)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values()) or 1.0
    lines = [f"# launch list summary of {os.path.basename(src)} (ncu gpu__time_duration, cold-cache, serialised)",
             f"{'launches':>8} {'total_us':>12} {'mean_us':>10} {'share':>6}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{n:8d} {t:12.1f} {t / n:10.1f} {t / tot * 100:5.1f}%  {k[:120]}")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    mode, src, out = sys.argv[1:4]
    tk = sys.argv[sys.argv.index("--traffic-key") + 1] if "--traffic-key" in sys.argv else None
    full(src, out, tk) if mode == "full" else launches(src, out)
