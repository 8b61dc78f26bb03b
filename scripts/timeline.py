#!/usr/bin/env python
"""Debug (DG_LIB built with -DDG_TIMELINE): per-warp phase timeline of the two CTAs on SM 0
for 6 consecutive elements of one c5 stage-1 launch.  Marks: 0 top (q_n prefetch), 1 q landed,
2 warp-local volume done, 3 barrier 1 passed (+ next issue), 4 z pass done, 5 faces done,
6 barrier 2 passed, 7 epilogue done."""
import ctypes as C, os, sys
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402
w = W.get(sys.argv[1] if len(sys.argv) > 1 else "c5")
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = D.DG(w.params); ctx.mesh_upload(w.level, w.anchor)
E, F, Np, stride = ctx.state_layout()
ctx.set_background(torch.from_numpy(w.bg).cuda())
q = D.to_device(w.q0, stride); a = torch.empty_like(q); b = torch.empty_like(q)
fn = D.lib.dg_debug_timeline; fn.argtypes = [C.c_void_p, C.c_int]; fn.restype = C.c_int
buf = np.zeros(2 * 6 * 8 * 8, np.int64)
ctx.rk_stage(0, w.dt, q, q, a); ctx.rk_stage(1, w.dt, q, a, b); torch.cuda.synchronize()
fn(buf.ctypes.data, buf.size)
if stage == 0:
    ctx.rk_stage(0, w.dt, q, q, b)
else:
    ctx.rk_stage(1, w.dt, q, a, b)
torch.cuda.synchronize()
n = fn(buf.ctypes.data, buf.size)
t = buf.reshape(2, 6, 8, 8)
t0 = t[t > 0].min()
print(f"stage {stage}; mean per-phase cycles over warps/elements:",
      " ".join(f"{x:.0f}" for x in np.diff(t[:, :, :, :], axis=3).mean(axis=(0, 1, 2))))
for sl in range(2):
    print(f"CTA slot {sl} (cycles from the first mark; per element: warp rows, marks 0..7)")
    for it in range(6):
        base = t[sl, it, :, 0].min()
        print(f" element +{it}: start {base - t0:8d}, length {t[sl, it, :, 7].max() - base:6d}")
        for wp in range(8):
            print("   w%d " % wp + " ".join(f"{v - base:6d}" for v in t[sl, it, wp]))
