#!/usr/bin/env python
"""SHA-256 of the RHS and of the three RK stage outputs of a workload through whichever libdg DG_LIB
names (bitwise regression check between kernel variants):  python scripts/hash_stage.py c4 [c3 ...]"""
import hashlib, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402
import numpy as np  # noqa: E402
for name in sys.argv[1:] or ["c3"]:
    w = W.get(name)
    ctx = D.DG(w.params); ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(w.bg).cuda())
    rng = np.random.default_rng(7)
    q0 = w.q0.copy(); d = w.params.dim
    q0[:, 1:1 + d] += q0[:, :1] * rng.uniform(-0.5, 0.5, size=q0[:, 1:1 + d].shape)
    q0[:, d + 1] *= 1.0 + 1e-4 * rng.uniform(-1.0, 1.0, size=q0[:, d + 1].shape)
    qn = D.to_device(q0, stride); a = torch.empty_like(qn); b = torch.empty_like(qn); r = torch.empty_like(qn)
    ctx.rhs(qn, r); ctx.rk_stage(0, w.dt, qn, qn, a); ctx.rk_stage(1, w.dt, qn, a, b); ctx.rk_stage(2, w.dt, qn, b, a)
    torch.cuda.synchronize()
    hs = [hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:12] for t in (r, b, a)]
    print(f"{os.environ.get('DG_LIB', 'libdg.so').split('/')[-1]:22s} {name}: rhs {hs[0]} stage1 {hs[1]} stage2 {hs[2]}")
