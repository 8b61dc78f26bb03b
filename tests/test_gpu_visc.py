"""NEXT-3 artificial viscosity on the GPU (dg_set_viscosity, reading R42):
the viscous term V (= RHS with mu minus RHS without) against the oracle's, exact
for the Neumann polynomial of tests/test_oracle_visc.py across 2:1 faces,
conservative, and a full RK stage with viscosity against the oracle."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import Gpu, _check
from test_oracle_visc import _meshes, _poly_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

MU = 1.5


def _visc_gpu(g, q):
    g.ctx.set_viscosity(0.0)
    r0 = g.rhs(q)
    g.ctx.set_viscosity(MU)
    r1 = g.rhs(q)
    g.ctx.set_viscosity(0.0)
    return r1 - r0, r1


def _random_state(p, lv, an, bg, seed):
    rng = np.random.default_rng(seed)
    rest = W.pressure_balanced_state(p, W.node_background(p, bg, lv, an), np.zeros((len(lv), p.n_nodes)))
    X = W.node_coords(p, lv, an)
    L = max(p.hi[d] - p.lo[d] for d in range(p.dim))
    q = rest.copy()
    for k in range(p.n_fields):
        ph = rng.uniform(0, 2 * np.pi, size=p.dim)
        wave = np.prod([np.sin(2 * np.pi * X[:, d] / L * (1 + d) + ph[d]) for d in range(p.dim)], axis=0)
        q[:, k] += (0.02 if k in (0, p.dim + 1) else 3.0) * wave * (np.abs(rest[:, k]).max() if k in (0, p.dim + 1) else 1.0)
    return q


@pytest.mark.parametrize("i", range(3))
def test_visc_exact_polynomial_on_gpu(i):
    p, lv, an = list(_meshes())[i]
    p.periodic = (0,) * p.dim
    bg = W.background_table(p)
    q, lap = _poly_state(p, lv, an, bg)
    g = Gpu(p, lv, an, bg)
    V, _ = _visc_gpu(g, q)
    assert np.abs(V - MU * lap).max() <= 1e-8 * np.abs(MU * lap).max()


@pytest.mark.parametrize("case", ["c2", "forest3d"])
def test_visc_matches_oracle_and_conserves(case):
    if case == "c2":
        w = W.c2()
        p, lv, an, bg = w.params, w.level, w.anchor, w.bg
    else:
        p, lv, an = W.random_forest(5, 3, order=3, max_level=2, frac=0.35)
        bg = W.background_table(p)
    q = _random_state(p, lv, an, bg, 3)
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    V, r1 = _visc_gpu(g, q)
    Vo = oracle.visc(m, bg, q, MU)
    scale = np.abs(Vo).max(axis=(0, 2))
    err = np.abs(V - Vo).max(axis=(0, 2)) / scale
    assert np.all(err <= 1e-9), err
    _check(r1, oracle.rhs(m, bg, q) + Vo, what=f"{case} rhs with viscosity")
    I, A = oracle.integrals(m, Vo), oracle.integrals(m, np.abs(Vo))
    Ig = oracle.integrals(m, V)
    assert np.all(np.abs(Ig) <= 1e-11 * A), Ig / A
    # one RK stage (stage 1) with viscosity
    dt = 0.01
    q1 = oracle.rk_stage_visc(m, bg, 0, dt, q, q, MU)
    g.ctx.set_viscosity(MU)
    qn, qi, out = g.dev(q), g.dev(q1), g.empty()
    g.ctx.rk_stage(1, dt, qn, qi, out)
    _check(g.host(out), oracle.rk_stage_visc(m, bg, 1, dt, q, q1, MU), what=f"{case} stage 1 with viscosity")


def test_visc_rejected_on_partitioned_context():
    from paper_2404_16648_b200 import dg as D
    w = W.c2()
    ctx = D.DG(w.params)
    ctx.mesh_upload_part(w.level, w.anchor, 2, 0)
    with pytest.raises(D.DGError):
        ctx.set_viscosity(1.5)
    with pytest.raises(D.DGError):
        D.DG(w.params).set_viscosity(-1.0)
