"""Checkpoint / resume: host round trip of params, leaf list and
state; on the GPU, a run resumed from a checkpoint is bitwise identical to the
uninterrupted run."""
import numpy as np
import pytest

import workloads as W
from paper_2404_16648_b200 import checkpoint as CK


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_round_trip(tmp_path, name):
    w = W.get(name)
    path = tmp_path / "ck.npz"
    CK.save(path, w.params, w.level, w.anchor, w.q0, t=1.25, step=7)
    r = CK.load(path)
    for k in CK.PARAM_KEYS:
        a, b = getattr(w.params, k), getattr(r["params"], k)
        assert (tuple(a) == tuple(b)) if isinstance(a, (tuple, list)) else a == b, k
    assert np.array_equal(r["level"], w.level) and np.array_equal(r["anchor"], w.anchor)
    assert np.array_equal(r["q"], w.q0) and r["q"].dtype == np.float64
    assert r["t"] == 1.25 and r["step"] == 7


def test_shape_checks(tmp_path):
    w = W.get("c1")
    with pytest.raises(ValueError):
        CK.save(tmp_path / "a.npz", w.params, w.level, w.anchor, w.q0[:-1])
    with pytest.raises(ValueError):
        CK.save(tmp_path / "b.npz", w.params, w.level, w.anchor, w.q0[:, :3])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_resume_bitwise(tmp_path, name):
    import torch
    from paper_2404_16648_b200 import dg as D
    w = W.get(name)

    def run(params, level, anchor, q0, n_steps):
        ctx = D.DG(params)
        ctx.mesh_upload(level, anchor)
        E, F, Np, stride = ctx.state_layout()
        ctx.set_background(torch.from_numpy(np.ascontiguousarray(w.bg)).cuda())
        q = D.to_device(q0, stride)
        a, b = torch.empty_like(q), torch.empty_like(q)
        for _ in range(n_steps):
            ctx.rk_stage(0, w.dt, q, q, a)
            ctx.rk_stage(1, w.dt, q, a, b)
            ctx.rk_stage(2, w.dt, q, b, a)
            q = a.clone()
        torch.cuda.synchronize()
        return D.from_device(q, F, Np)

    straight = run(w.params, w.level, w.anchor, w.q0, 2)
    half = run(w.params, w.level, w.anchor, w.q0, 1)
    CK.save(tmp_path / "ck.npz", w.params, w.level, w.anchor, half, t=w.dt, step=1)
    r = CK.load(tmp_path / "ck.npz")
    resumed = run(r["params"], r["level"], r["anchor"], r["q"], 1)
    assert np.array_equal(resumed, straight)
