#!/usr/bin/env python
"""Long run of the bench workload (c5: 3D N = 7, 335.5 M DOF, periodic x/y, walls z) through the
fused RK3 stages: n steps, then the relative drift of the mass and Theta integrals (dg_integrals,
compensated) and the extreme values.  Prints one JSON line.
  python scripts/c5_long_run.py [steps]"""
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

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500
w = W.c5()
ctx = D.DG(w.params)
ctx.mesh_upload(w.level, w.anchor)
E, F, Np, stride = ctx.state_layout()
ctx.set_background(torch.from_numpy(w.bg).cuda())
q = D.to_device(w.q0, stride)
del w
a, b = torch.empty_like(q), torch.empty_like(q)
I0 = ctx.integrals(q)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(n):
    ctx.rk_stage(0, 0.005, q, q, a)
    ctx.rk_stage(1, 0.005, q, a, b)
    ctx.rk_stage(2, 0.005, q, b, a)
    q, a = a, q
torch.cuda.synchronize()
wall = time.perf_counter() - t0
I1 = ctx.integrals(q)
qf = q[:, :F * Np].view(E, F, Np)
print(json.dumps({"workload": "c5 (3D N=7, 64x64x32), SSP-RK3 dt=0.005 s", "steps": n, "t": n * 0.005,
                  "wall_s": wall, "ms_per_step": wall * 1e3 / n,
                  "mass_drift_rel": float((I1[0] - I0[0]) / I0[0]), "theta_drift_rel": float((I1[4] - I0[4]) / I0[4]),
                  "finite": bool(torch.isfinite(qf).all().item()),
                  "max_abs_w": float(qf[:, 3].abs().max().item())}))
