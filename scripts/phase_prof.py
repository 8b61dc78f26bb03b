#!/usr/bin/env python
"""Debug: per-phase clock shares of the fused stage kernel (DG_PHASE_PROF=1, on a libdg built with
-DDG_PHASE_PROF: the hooks are compiled out of the default build).

  DG_PHASE_PROF=1 python scripts/phase_prof.py [c5|c4|c3] [n_stages]
Slots: 0 issue (bulk/trace/desc), 1 wait q + barrier, 2 mortars + nodes,
3 wait traces + barrier, 4 fine projection + faces, 5 pass x, 6 passes y, z, 7 epilogue.
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("DG_PHASE_PROF", "1")
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
w = W.get(name)
ctx = D.DG(w.params)
ctx.mesh_upload(w.level, w.anchor)
E, F, Np, stride = ctx.state_layout()
ctx.set_background(torch.from_numpy(w.bg).cuda())
q = D.to_device(w.q0, stride)
a, b = torch.empty_like(q), torch.empty_like(q)
fn = D.lib.dg_debug_phase_clocks
fn.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(16, np.uint64)
ctx.rk_stage(0, w.dt, q, q, a)
torch.cuda.synchronize()
fn(buf.ctypes.data, 1)
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
for i in range(n):
    ctx.rk_stage(1, w.dt, q, a, b)
ev1.record()
torch.cuda.synchronize()
fn(buf.ctypes.data, 1)
if w.params.order == 7 and w.params.dim == 3:
    names = ["end+issue next", "wait q", "EOS+x+y+Fz", "barrier 1", "z pass", "faces", "barrier 2", "epilogue"]
    print(f"{name}: {ev0.elapsed_time(ev1) / n:.3f} ms per stage-1 launch (warp 0 | warp 7, share of its loop time)")
    t0, t7 = buf[:8].sum(), buf[8:].sum()
    for k, v0, v7 in zip(names, buf[:8], buf[8:]):
        print(f"  {k:14s} {v0 / t0 * 100:5.1f}%  {v7 / t7 * 100:5.1f}%")
else:
    names = ["issue:desc", "wait q", "mortar+nodes", "wait traces", "faces", "pass x", "pass y", "pass z+RK",
             "issue:fence", "issue:bulk", "issue:prefetch", "issue:traces", "", "", "", ""]
    tot = buf.sum()
    print(f"{name}: {ev0.elapsed_time(ev1) / n:.3f} ms per stage-1 launch")
    for k, v in zip(names, buf):
        if k:
            print(f"  {k:14s} {v / tot * 100:5.1f}%")
