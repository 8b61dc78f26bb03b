#!/usr/bin/env python
"""NEXT-1 + NEXT-2: the paper's tree-based AMR vortex run:
32 x 32 root elements, N = 3, one refinement level, buffer B = 2 cells, forward
Euler dt = 2.5e-4 s to t = 3 s, regridding every T steps on the density
perturbation |rho - rho_bar| (R36, R39) through the C ABI (indicator kernel ->
host plan -> mesh upload -> transfer kernels).  Error against the closed form
on the final mesh.  Prints one JSON line.
  python scripts/vortex_amr.py [--every 400] [--refine 0.01] [--coarsen 0.005] [--out f.json]"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402


def run(nx=32, order=3, every=400, refine=0.01, coarsen=0.005, buffer=2, t_end=3.0, dt=2.5e-4):
    p = W.vortex_params(nx, order)
    p.max_level = 1
    lv, an = W.uniform_morton(p)
    ctx = D.DG(p)
    ctx.mesh_upload(lv, an)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(W.vortex_background(p)).cuda())
    q = D.to_device(W.vortex_state(p, lv, an), stride)
    n = int(round(t_end / dt))
    counts, regrid_ms = [], []
    ev = lambda: torch.cuda.Event(enable_timing=True)
    step_ms = 0.0
    a = None
    for s0 in range(0, n, every):
        e0, e1 = ev(), ev()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q, plan = ctx.regrid(q, 1, refine, coarsen, buffer)
        torch.cuda.synchronize()
        regrid_ms.append((time.perf_counter() - t0) * 1e3)
        counts.append(int(q.shape[0]))
        a = torch.empty_like(q)
        e0.record()
        for _ in range(min(every, n - s0)):
            ctx.rk_stage(0, dt, q, q, a)
            q, a = a, q
        e1.record()
        torch.cuda.synchronize()
        step_ms += e0.elapsed_time(e1)
    lv2, an2 = plan["level"], plan["anchor"]
    qh = D.from_device(q, F, Np)
    err = W.vortex_l2(p, qh, W.vortex_state(p, lv2, an2, n * dt), lv2)
    return {"workload": f"AMR vortex {nx}x{nx} N={order}, max_level 1, B={buffer}, regrid every {every} steps "
                        f"on |rho'| (refine > {refine}, coarsen < {coarsen})",
            "steps": n, "dt": dt, "t": n * dt, "l2_rms": err["rms"], "l2_quad": err["l2"], "l2_max": err["max"], "paper_l2": 8.75e-4,
            "elements_min": min(counts), "elements_max": max(counts), "elements_final": counts[-1],
            "uniform_fine_elements": 4 * nx * nx, "regrids": len(counts),
            "regrid_ms_mean": float(np.mean(regrid_ms[1:] or regrid_ms)), "us_per_step": step_ms * 1e3 / n,
            "finite": bool(np.isfinite(qh).all())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--every", type=int, default=400)
    ap.add_argument("--refine", type=float, default=0.01)
    ap.add_argument("--coarsen", type=float, default=0.005)
    ap.add_argument("--buffer", type=int, default=2)
    ap.add_argument("--t", type=float, default=3.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = run(every=a.every, refine=a.refine, coarsen=a.coarsen, buffer=a.buffer, t_end=a.t)
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
