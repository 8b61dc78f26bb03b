"""NEXT-3 passive tracer of the Euler flow on the GPU (dg_passive_rhs / dg_passive_rk_stage;
C = rho c; reading R45) against the oracle at R19 (field 0, 1e-12 of its max): c1, c2
(2D mortars), c3, c4 (3D mortars) and a random 3D forest, moving Euler states and discontinuous
mixing ratios; an RK stage on identical inputs; conservation of the GPU's dC/dt."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import Gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-12


def _moving(p, lv, an, q0, amp=4.0):
    X = W.node_coords(p, lv, an)
    q = q0.copy()
    L = max(p.hi[d] - p.lo[d] for d in range(p.dim))
    for d in range(p.dim):
        q[:, 1 + d] += amp * q[:, 0] * np.sin(4 * np.pi * X[:, (d + 1) % p.dim] / L + d) * np.cos(2 * np.pi * X[:, d] / L)
    return q


def _cases():
    for name in ("c1", "c2", "c3", "c4"):
        w = W.get(name)
        yield name, w.params, w.level, w.anchor, w.bg, w.q0
    from test_oracle_rhs import _bubble_state
    p, lv, an = W.random_forest(7, 3, order=4, max_level=2)
    p.hi = tuple(250.0 * r for r in p.root)
    bg, q = _bubble_state(p, lv, an, 7)
    yield "forest7", p, lv, an, bg, q


def _rel(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: c[0])
def test_passive_matches_oracle(case):
    name, p, lv, an, bg, q0 = case
    q = _moving(p, lv, an, q0)
    rng = np.random.default_rng(5)
    C = q[:, 0] * rng.uniform(0.0, 1.0, size=q[:, 0].shape)
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    cfull = np.zeros_like(q)
    cfull[:, 0] = C
    qd, cd = g.dev(q), g.dev(cfull)
    out = g.empty()
    g.ctx.passive_rhs(qd, cd, out)
    gpu = g.host(out)[:, 0]
    ora = oracle.passive_rhs(m, bg, q, C)
    assert _rel(gpu, ora) <= TOL, (name, _rel(gpu, ora))
    # conservation of the GPU result (mortars, mirror walls)
    a = np.zeros_like(q)
    a[:, 0] = gpu
    b = np.zeros_like(q)
    b[:, 0] = np.abs(gpu)
    assert abs(oracle.integrals(m, a)[0] / oracle.integrals(m, b)[0]) < 1e-14
    # RK stages 0 and 1 on identical inputs (stage 1 fed the GPU's stage-0 output)
    dt = 1e-3
    s0 = g.empty()
    g.ctx.passive_rk_stage(0, dt, qd, cd, cd, s0)
    s0h = g.host(s0)[:, 0]
    assert _rel(s0h, oracle.passive_rk_stage(m, bg, 0, dt, q, C, C)) <= TOL
    s1 = g.empty()
    g.ctx.passive_rk_stage(1, dt, qd, cd, s0, s1)
    assert _rel(g.host(s1)[:, 0], oracle.passive_rk_stage(m, bg, 1, dt, q, C, s0h)) <= TOL


def test_passive_rejects_pointwise_mode():
    from paper_2404_16648_b200 import dg as D
    w = W.c2()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    g.ctx.set_nonconforming(1)
    q = g.dev(w.q0)
    with pytest.raises(D.DGError):
        g.ctx.passive_rhs(q, q.clone(), g.empty())


def test_passive_mass_conserved_over_a_run():
    """c2 (2D quadtree, 2:1 faces), the cold bubble falling: 100 SSP-RK3 steps of the Euler state
    with the passive tracer alongside (each tracer stage with the Euler stage's input); the tracer
    mass changes by rounding only (the paper's tracer loss ~1e-14; mortars)."""
    w = W.c2()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    X = W.node_coords(w.params, w.level, w.anchor)
    c0 = np.zeros_like(w.q0)
    c0[:, 0] = w.q0[:, 0] * (X[:, 1] < 2000.0)  # discontinuous: tracer in the lowest 2 km
    q, c = g.dev(w.q0), g.dev(c0)
    qa, qb, ca, cb = g.empty(), g.empty(), g.empty(), g.empty()
    for _ in range(100):
        g.ctx.rk_stage(0, w.dt, q, q, qa)
        g.ctx.passive_rk_stage(0, w.dt, q, c, c, ca)
        g.ctx.rk_stage(1, w.dt, q, qa, qb)
        g.ctx.passive_rk_stage(1, w.dt, qa, c, ca, cb)
        g.ctx.rk_stage(2, w.dt, q, qb, qa)
        g.ctx.passive_rk_stage(2, w.dt, qb, c, cb, ca)
        q, qa = qa, q
        c, ca = ca, c
    ch = g.host(c)
    assert np.isfinite(ch[:, 0]).all()
    I0 = oracle.integrals(m, c0)[0]
    I1 = oracle.integrals(m, ch)[0]
    assert abs(I1 - I0) / abs(I0) < 1e-13, (I0, I1)
    assert np.abs(ch[:, 0] - c0[:, 0]).max() > 1e-9  # it moved
