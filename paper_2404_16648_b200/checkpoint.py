"""Checkpoint / resume ("the state is plain arrays; the mesh is the leaf list").

A checkpoint is one .npz holding the context parameters, the leaf list
(level[E] int8, anchor[E][dim] int32, upload order = state row order) and the
state in the compact layout [E][F][Np] fp64 (padding of the device rows is not
stored), plus the simulated time and step count.  Host logic only: the device
copies are `dg.to_device` / `dg.from_device`.  Resuming re-runs dg_mesh_upload
on the stored leaf list, so the state rows line up with the element order.
"""
from __future__ import annotations

import numpy as np

PARAM_KEYS = ("dim", "order", "root", "lo", "hi", "periodic", "max_level", "gamma", "R", "cp", "p0", "g")
VERSION = 1


def save(path, params, level, anchor, q, t=0.0, step=0):
    """Write params, leaf list, compact state q[E][F][Np] and (t, step) to `path` (.npz)."""
    level = np.ascontiguousarray(level, np.int8)
    anchor = np.ascontiguousarray(anchor, np.int32)
    q = np.ascontiguousarray(q, np.float64)
    E = level.shape[0]
    if anchor.shape != (E, params.dim) or q.ndim != 3 or q.shape[0] != E:
        raise ValueError(f"checkpoint: inconsistent shapes level {level.shape} anchor {anchor.shape} q {q.shape}")
    n1 = params.order + 1
    if q.shape[1] != params.dim + 2 or q.shape[2] != n1 ** params.dim:
        raise ValueError(f"checkpoint: q {q.shape} does not match dim {params.dim}, order {params.order}")
    arrays = {f"param_{k}": np.asarray(getattr(params, k)) for k in PARAM_KEYS}
    np.savez(path, version=np.int64(VERSION), level=level, anchor=anchor, q=q, t=np.float64(t),
             step=np.int64(step), **arrays)


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
                "t": float(z["t"]), "step": int(z["step"])}
