"""Checkpoint / resume ("the state is plain arrays; the mesh is the leaf list").

A checkpoint is one .npz holding the context parameters, the leaf list
(level[E] int8, anchor[E][dim] int32, upload order = state row order), the
state in the compact layout [E][F][Np] fp64 (padding of the device rows is not
stored), the background table (rows (rho_bar, Theta_bar, P_bar), R3) and the
context settings that change the operator -- the 2:1 face treatment (ncmode,
NEXT-3) and the artificial viscosity mu (R42) -- plus the simulated time and step
count.  Host logic only: the device copies are `dg.to_device` / `dg.from_device`.
`restore` rebuilds a context from the file alone (mesh upload on the stored leaf
list, so the state rows line up with the element order; background, ncmode, mu).
"""
from __future__ import annotations

import numpy as np

PARAM_KEYS = ("dim", "order", "root", "lo", "hi", "periodic", "max_level", "gamma", "R", "cp", "p0", "g")
VERSION = 2


def save(path, params, level, anchor, q, t=0.0, step=0, bg=None, ncmode=0, mu=0.0):
    """Write params, leaf list, compact state q[E][F][Np], the background table bg (rows
    (rho_bar, Theta_bar, P_bar)), ncmode, mu and (t, step) to `path` (.npz)."""
    level = np.ascontiguousarray(level, np.int8)
    anchor = np.ascontiguousarray(anchor, np.int32)
    q = np.ascontiguousarray(q, np.float64)
    E = level.shape[0]
    if anchor.shape != (E, params.dim) or q.ndim != 3 or q.shape[0] != E:
        raise ValueError(f"checkpoint: inconsistent shapes level {level.shape} anchor {anchor.shape} q {q.shape}")
    n1 = params.order + 1
    if q.shape[1] != params.dim + 2 or q.shape[2] != n1 ** params.dim:
        raise ValueError(f"checkpoint: q {q.shape} does not match dim {params.dim}, order {params.order}")
    if bg is None:
        raise ValueError("checkpoint: the background table is part of the state (pass bg)")
    bg = np.ascontiguousarray(bg, np.float64)
    if bg.ndim != 2 or bg.shape[1] != 3:
        raise ValueError(f"checkpoint: background table {bg.shape} is not [rows][3]")
    if int(ncmode) not in (0, 1) or not (float(mu) >= 0.0):
        raise ValueError("checkpoint: ncmode must be 0 or 1 and mu >= 0")
    arrays = {f"param_{k}": np.asarray(getattr(params, k)) for k in PARAM_KEYS}
    np.savez(path, version=np.int64(VERSION), level=level, anchor=anchor, q=q, t=np.float64(t),
             step=np.int64(step), bg=bg, ncmode=np.int64(ncmode), mu=np.float64(mu), **arrays)


def load(path):
    """Read a checkpoint: dict with params (SimpleNamespace), level, anchor, q, t, step."""
    from types import SimpleNamespace
    with np.load(path) as z:
        if int(z["version"]) != VERSION:
            raise ValueError(f"checkpoint: version {int(z['version'])} != {VERSION}")
        p = {}
        for k in PARAM_KEYS:
            v = z[f"param_{k}"]
            p[k] = tuple(v.tolist()) if v.ndim else v.item()
        params = SimpleNamespace(**p)
        params.n1 = params.order + 1
        params.n_fields = params.dim + 2
        params.n_nodes = params.n1 ** params.dim
        return {"params": params, "level": z["level"].copy(), "anchor": z["anchor"].copy(), "q": z["q"].copy(),
                "t": float(z["t"]), "step": int(z["step"]), "bg": z["bg"].copy(), "ncmode": int(z["ncmode"]),
                "mu": float(z["mu"])}


def restore(path, stream=None):
    """Cold restart from the file alone: (ctx, q_device, checkpoint dict).  Creates the context,
    uploads the stored leaf list, sets the stored background table, 2:1 treatment and
    viscosity, and copies the state to the device (padded rows)."""
    import torch
    from . import dg as D
    ck = load(path)
    ctx = D.DG(ck["params"])
    ctx.mesh_upload(ck["level"], ck["anchor"], stream)
    ctx.set_background(torch.from_numpy(ck["bg"]).cuda(), stream)
    ctx.set_nonconforming(ck["ncmode"])
    ctx.set_viscosity(ck["mu"])
    _, _, _, stride = ctx.state_layout()
    return ctx, D.to_device(ck["q"], stride), ck
