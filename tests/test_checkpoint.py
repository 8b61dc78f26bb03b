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
    CK.save(path, w.params, w.level, w.anchor, w.q0, t=1.25, step=7, bg=w.bg, ncmode=1, mu=1.5)
    r = CK.load(path)
    assert np.array_equal(r["bg"], w.bg) and r["ncmode"] == 1 and r["mu"] == 1.5
    for k in CK.PARAM_KEYS:
        a, b = getattr(w.params, k), getattr(r["params"], k)
        assert (tuple(a) == tuple(b)) if isinstance(a, (tuple, list)) else a == b, k
    assert np.array_equal(r["level"], w.level) and np.array_equal(r["anchor"], w.anchor)
    assert np.array_equal(r["q"], w.q0) and r["q"].dtype == np.float64
    assert r["t"] == 1.25 and r["step"] == 7


def test_shape_checks(tmp_path):
    w = W.get("c1")
    with pytest.raises(ValueError):
        CK.save(tmp_path / "a.npz", w.params, w.level, w.anchor, w.q0[:-1], bg=w.bg)
    with pytest.raises(ValueError):
        CK.save(tmp_path / "b.npz", w.params, w.level, w.anchor, w.q0[:, :3], bg=w.bg)
    with pytest.raises(ValueError):  # the background is part of the state
        CK.save(tmp_path / "c.npz", w.params, w.level, w.anchor, w.q0)
    with pytest.raises(ValueError):
        CK.save(tmp_path / "d.npz", w.params, w.level, w.anchor, w.q0, bg=w.bg, ncmode=2)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c3"])
def test_resume_bitwise(tmp_path, name):
    """A run resumed from a checkpoint (cold restart: everything from the file) is bitwise
    identical to the uninterrupted run."""
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
    CK.save(tmp_path / "ck.npz", w.params, w.level, w.anchor, half, t=w.dt, step=1, bg=w.bg)
    # cold restart from the file alone: context, mesh, background and settings from the checkpoint
    ctx, q, ck = CK.restore(tmp_path / "ck.npz")
    E, F, Np, stride = ctx.state_layout()
    a, b = torch.empty_like(q), torch.empty_like(q)
    ctx.rk_stage(0, w.dt, q, q, a)
    ctx.rk_stage(1, w.dt, q, a, b)
    ctx.rk_stage(2, w.dt, q, b, a)
    torch.cuda.synchronize()
    assert np.array_equal(D.from_device(a, F, Np), straight)
    ctx.close()


@pytest.mark.gpu
def test_restore_applies_settings(tmp_path):
    """ncmode and mu stored in the checkpoint change the restored context's operator exactly as
    setting them by hand does (NEXT-3 pointwise 2:1 treatment, R41; viscosity, R42)."""
    import torch
    from paper_2404_16648_b200 import dg as D
    w = W.c2()
    CK.save(tmp_path / "ck.npz", w.params, w.level, w.anchor, w.q0, bg=w.bg, ncmode=1, mu=1.5)
    ctx, q, ck = CK.restore(tmp_path / "ck.npz")
    ref = D.DG(w.params)
    ref.mesh_upload(w.level, w.anchor)
    ref.set_background(torch.from_numpy(np.ascontiguousarray(w.bg)).cuda())
    ref.set_nonconforming(1)
    ref.set_viscosity(1.5)
    r1, r2 = torch.zeros_like(q), torch.zeros_like(q)
    ctx.rhs(q, r1)
    ref.rhs(q, r2)
    torch.cuda.synchronize()
    assert torch.equal(r1, r2)
    ctx.close()
    ref.close()
