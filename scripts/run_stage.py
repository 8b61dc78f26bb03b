#!/usr/bin/env python
"""Run n RK stages (stage 1) of a config through the C ABI (for ncu captures).
  python scripts/run_stage.py c4 6"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = W.get(name)
ctx = D.DG(w.params)
ctx.mesh_upload(w.level, w.anchor)
E, F, Np, stride = ctx.state_layout()
ctx.set_background(torch.from_numpy(w.bg).cuda())
q = D.to_device(w.q0, stride)
a, b = torch.empty_like(q), torch.empty_like(q)
ctx.rk_stage(0, w.dt, q, q, a)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for i in range(n):
    ctx.rk_stage(1, w.dt, q, a, b)
ev1.record()
torch.cuda.synchronize()
print(f"{name}: E={E} {ev0.elapsed_time(ev1) / n:.4f} ms per stage-1 launch")
