#!/usr/bin/env python
"""Small end-to-end run of every stage/transfer/monitor kernel through the C ABI, sized for
compute-sanitizer (memcheck / racecheck / synccheck): c1, c2 (2D, mortars), a 3D N = 4 AMR forest
(k_stage<3,4> with 3D mortars), the c5 element type on a 4 x 4 x 2 box (k_stage_h7, RHS and all
three RK kinds), a 3D N = 7 AMR forest (k_stage_h7's mortar path), refine -> coarsen, copy,
integrals and check_state.  Prints one line per case; exits non-zero on any library error."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402


def run(name, p, level, anchor, bg, q0, dt):
    ctx = D.DG(p)
    ctx.mesh_upload(level, anchor)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(np.ascontiguousarray(bg)).cuda())
    q = D.to_device(q0, stride)
    a, b, r = torch.zeros_like(q), torch.zeros_like(q), torch.zeros_like(q)
    ctx.rhs(q, r)
    ctx.rk_stage(0, dt, q, q, a)
    ctx.rk_stage(1, dt, q, a, b)
    ctx.rk_stage(2, dt, q, b, a)
    nch = 1 << p.dim
    k = min(E, 4)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.int32)).cuda()
    par, ch0 = T(np.arange(k)), T(nch * np.arange(k))
    fine = torch.zeros((nch * k, stride), dtype=torch.float64, device="cuda")
    ctx.amr_project_refine(k, par, ch0, q, fine)
    ctx.amr_project_coarsen(k, ch0, par, fine, b)
    ctx.copy_elements(k, par, par, q, b)
    I = ctx.integrals(a)
    chk = ctx.check_state(a)
    torch.cuda.synchronize()
    print(f"{name}: E={E} finite={bool(torch.isfinite(a).all())} integrals={I[0]:.6e} check={chk}", flush=True)
    ctx.close()


def moving(p, lv, an, seed):
    from test_oracle_rhs import _bubble_state
    return _bubble_state(p, lv, an, seed)


sys.path.insert(0, os.path.join(ROOT, "tests"))
for name in ("c1", "c2"):
    w = W.get(name)
    run(name, w.params, w.level, w.anchor, w.bg, w.q0, w.dt)
p, lv, an = W.random_forest(7, 3, order=4, max_level=2)
p.hi = tuple(250.0 * r for r in p.root)
bg, q = moving(p, lv, an, 7)
run("amr3d N4", p, lv, an, bg, q, 5e-4)
w = W.c5(root=(4, 4, 2))
run("c5 box N7", w.params, w.level, w.anchor, w.bg, w.q0, w.dt)
p, lv, an = W.random_forest(6, 3, order=7, max_level=1)
p.hi = tuple(250.0 * r for r in p.root)
bg, q = moving(p, lv, an, 6)
run("amr3d N7", p, lv, an, bg, q, 5e-4)
print("sanitize_run: done")
