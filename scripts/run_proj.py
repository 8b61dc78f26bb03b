#!/usr/bin/env python
"""c4 refine -> coarsen projection pass (R25) through the C ABI, for ncu captures."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402

w = W.c4()
ctx = D.DG(w.params)
ctx.mesh_upload(w.level, w.anchor)
E, F, Np, stride = ctx.state_layout()
q = D.to_device(w.q0, stride)
flags = W.c4_projection_flags(w)
isf = np.zeros(E, bool)
isf[flags] = True
size = np.where(isf, 8, 1)
start = np.concatenate([[0], np.cumsum(size)[:-1]]).astype(np.int32)
E2 = int(size.sum())
T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()
par, ch0 = T(flags), T(start[flags])
fine = torch.empty((E2, stride), dtype=torch.float64, device="cuda")
back = torch.empty_like(q)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    ctx.amr_project_refine(len(flags), par, ch0, q, fine)
    ctx.amr_project_coarsen(len(flags), ch0, par, fine, back)
torch.cuda.synchronize()
print("ok", len(flags))
