#!/usr/bin/env python
"""A/B timing of one SSP-RK3 step of a workload (default c5) through whichever libdg DG_LIB names:
per-stage CUDA-event times, median of n steps after warm-up.  python scripts/ab_c5.py [c5] [n]"""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = W.get(name)
ctx = D.DG(w.params); ctx.mesh_upload(w.level, w.anchor)
E, F, Np, stride = ctx.state_layout()
ctx.set_background(torch.from_numpy(w.bg).cuda())
qn = D.to_device(w.q0, stride); a = torch.empty_like(qn); b = torch.empty_like(qn)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
res = []
for it in range(n + 3):
    ev[0].record(); ctx.rk_stage(0, w.dt, qn, qn, a)
    ev[1].record(); ctx.rk_stage(1, w.dt, qn, a, b)
    ev[2].record(); ctx.rk_stage(2, w.dt, qn, b, a)
    ev[3].record(); torch.cuda.synchronize()
    if it >= 3:
        res.append([ev[i].elapsed_time(ev[i + 1]) for i in range(3)])
r = np.median(np.array(res), axis=0)
print(f"{os.environ.get('DG_LIB', 'libdg.so').split('/')[-1]:22s} {name}: stage ms {r[0]:.4f} {r[1]:.4f} {r[2]:.4f} step {r.sum():.4f}")
