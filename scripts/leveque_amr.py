#!/usr/bin/env python
"""The paper's LeVeque swirl (§4.2; readings R43, R44): a cosine-bell
tracer in the time-reversing deformation wind on [0,1]^2, N = 4, T = 5, through the
kinematic tracer kernels (dg_tracer_rk_stage, SSP-RK3) -- uniform 16^2 and 64^2 meshes,
and tree-based AMR on a 16^2 root with two levels, B = 2, 80 regrids over the period
(indicator max |C| per element; refine > 0.05, coarsen < 0.01), with mortars and with
the pointwise-interpolation baseline.  Reports the error at t = T against the initial
bell (the exact solution), the tracer-mass drift and the wall time.  One JSON line.
  python scripts/leveque_amr.py [--out f.json]"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402

T = W.LEVEQUE_T


def run(nx, max_level, amr, ncmode=0, dt=1.0 / 1600.0, regrids=80, refine=0.05, coarsen=0.01, buffer=2):
    p = W.leveque_params(nx, 4, max_level)
    lv, an = W.uniform_morton(p)
    ctx = D.DG(p)
    ctx.mesh_upload(lv, an)
    ctx.set_background(torch.ones((int(W.row_offsets(p)[-1]), 3), dtype=torch.float64, device="cuda"))
    ctx.set_nonconforming(ncmode)
    E, F, Np, stride = ctx.state_layout()
    s = D.to_device(W.leveque_state(p, lv, an, 0.0), stride)

    def coords(lv, an):
        X = torch.from_numpy(W.node_coords(p, lv, an)).cuda()
        return torch.sin(math.pi * X[:, 0]) ** 2 * torch.sin(2 * math.pi * X[:, 1]), \
            -torch.sin(math.pi * X[:, 1]) ** 2 * torch.sin(2 * math.pi * X[:, 0])

    def regrid(s, lv, an):
        C = s[:, :Np].cpu().numpy()
        eta = np.abs(C).max(axis=1)
        s2, plan = ctx.regrid_eta(s, eta, refine, coarsen, buffer)
        return s2, plan["level"], plan["anchor"]

    if amr:
        for _ in range(max_level):  # refine around the initial bell
            s, lv, an = regrid(s, lv, an)
    u0, v0 = coords(lv, an)
    mass0 = ctx.integrals(s)[0]
    n = int(round(T / dt))
    every = n // regrids if amr else n + 1
    counts, drift = [], 0.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a, b = torch.empty_like(s), torch.empty_like(s)
    for k in range(n):
        if amr and k > 0 and k % every == 0:
            s, lv, an = regrid(s, lv, an)
            u0, v0 = coords(lv, an)
            a, b = torch.empty_like(s), torch.empty_like(s)
            counts.append(len(lv))
            drift = max(drift, abs(ctx.integrals(s)[0] - mass0) / mass0)
        t = k * dt
        for st, (src, dst, ts) in enumerate(((s, a, t), (a, b, t + dt), (b, a, t + 0.5 * dt))):
            g = math.cos(math.pi * ts / T)
            src[:, Np:2 * Np] = u0 * g
            src[:, 2 * Np:3 * Np] = v0 * g
            ctx.tracer_rk_stage(st, dt, s, src, dst)
        s, a = a, s
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    mass = ctx.integrals(s)[0]
    drift = max(drift, abs(mass - mass0) / mass0)
    C = D.from_device(s, F, Np)
    Cex = W.leveque_state(p, lv, an, 0.0)
    err = W.vortex_l2(p, C[:, :1], Cex[:, :1], lv)  # quadrature L2 and max of field 0
    return {"mesh": (f"AMR {nx}^2 root, {max_level} levels, B={buffer}, {regrids} regrids, "
                     f"{'mortar' if ncmode == 0 else 'pointwise'}") if amr else f"uniform {nx}^2",
            "steps": n, "dt": dt, "l2": err["l2"], "max_err": err["max"], "mass_drift_rel": drift,
            "elements_final": len(lv), "elements_max": max(counts) if counts else len(lv),
            "elements_min": min(counts) if counts else len(lv), "wall_s": wall}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    runs = [run(16, 0, False), run(64, 0, False), run(16, 2, True, 0), run(16, 2, True, 1)]
    res = {"workload": "LeVeque swirl (P:422-556): [0,1]^2, N=4, T=5, SSP-RK3 dt=1/1600",
           "paper_wall_s": {"tree_amr": 11, "uniform_16": 18, "uniform_32": 51}, "runs": runs}
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
