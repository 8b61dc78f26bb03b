#!/usr/bin/env python
"""NEXT-2: the paper's isentropic-vortex run on the GPU path:
32 x 32 elements, N = 3, forward Euler (= SSP-RK3 stage 0, q + dt L(q)) with
dt = 2.5e-4 s to t = 3 s, error against the translated closed form (R36).
Also the same run with SSP-RK3.  Prints one JSON line.
  python scripts/vortex_run.py [--nx 32] [--order 3] [--t 3.0] [--out profiles/r01_vortex.json]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_16648_b200 import dg as D  # noqa: E402
import workloads as W  # noqa: E402

PAPER_L2 = 8.75e-4  # P:384, tree-based AMR (one refinement level), t = 3 s


def run(nx, order, t_end, dt, scheme):
    w = W.vortex(nx, order)
    ctx = D.DG(w.params)
    ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(w.bg).cuda())
    n = int(round(t_end / dt))
    q = D.to_device(w.q0, stride)
    a, b = torch.empty_like(q), torch.empty_like(q)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(n):
        if scheme == "euler":
            ctx.rk_stage(0, dt, q, q, a)
            q, a = a, q
        else:
            ctx.rk_stage(0, dt, q, q, a)
            ctx.rk_stage(1, dt, q, a, b)
            ctx.rk_stage(2, dt, q, b, a)
            q, a = a, q
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    qh = D.from_device(q, F, Np)
    err = W.vortex_l2(w.params, qh, W.vortex_state(w.params, w.level, w.anchor, n * dt), w.level)
    launches = n * (1 if scheme == "euler" else 3)
    return {"scheme": scheme, "steps": n, "dt": dt, "t": n * dt, "ms_total": ms, "us_per_launch": ms * 1e3 / launches,
            "l2_rms": err["rms"], "l2_quad": err["l2"], "l2_paper_formula": err["paper"], "max_abs": err["max"],
            "finite": bool(np.isfinite(qh).all())}


def run_graph(nx, order, t_end, dt, k=200):
    """Forward Euler with the launches captured in a CUDA graph (k steps per replay)."""
    w = W.vortex(nx, order)
    ctx = D.DG(w.params)
    ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(w.bg).cuda())
    n = int(round(t_end / dt))
    assert n % k == 0 and k % 2 == 0
    q = D.to_device(w.q0, stride)
    a = torch.empty_like(q)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(k):  # even k: ends with the state back in q
            src, dst = (q, a) if i % 2 == 0 else (a, q)
            ctx.rk_stage(0, dt, src, src, dst, s)
    q.copy_(D.to_device(w.q0, stride))  # capture does not execute; reset anyway
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):  # replay() launches on the current stream
        ev0.record()
        for _ in range(n // k):
            g.replay()
        ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    qh = D.from_device(q, F, Np)
    err = W.vortex_l2(w.params, qh, W.vortex_state(w.params, w.level, w.anchor, n * dt), w.level)
    return {"scheme": "euler, CUDA graph of %d launches" % k, "steps": n, "dt": dt, "t": n * dt, "ms_total": ms,
            "us_per_launch": ms * 1e3 / n, "l2_rms": err["rms"], "l2_quad": err["l2"], "l2_paper_formula": err["paper"],
            "max_abs": err["max"], "finite": bool(np.isfinite(qh).all())}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nx", type=int, default=32)
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--t", type=float, default=3.0)
    ap.add_argument("--dt", type=float, default=2.5e-4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"workload": f"vortex {a.nx}x{a.nx} N={a.order}", "paper_l2": PAPER_L2,
           "runs": [run(a.nx, a.order, a.t, a.dt, s) for s in ("euler", "rk3")] + [run_graph(a.nx, a.order, a.t, a.dt)]}
    line = json.dumps(res)
    print(line)
    if a.out:
        with open(a.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
