"""NEXT-3 baseline on the GPU: the pointwise-interpolation treatment of 2:1 faces
(dg_set_nonconforming(ctx, 1); R41) against the oracle at R19, and
the conservation contrast with the mortar method."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import Gpu, _check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _moving(p, lv, an, q0):
    X = W.node_coords(p, lv, an)
    q = q0.copy()
    L = max(p.hi[d] - p.lo[d] for d in range(p.dim))
    for d in range(p.dim):  # a few m/s with O(1) momentum RHS in every component (R19 is per field)
        q[:, 1 + d] += 4.0 * q[:, 0] * np.sin(4 * np.pi * X[:, (d + 1) % p.dim] / L + d) * np.cos(2 * np.pi * X[:, d] / L)
    return q


def _cases():
    w = W.c2()
    yield "c2", w.params, w.level, w.anchor, w.bg, w.q0
    for seed, dim, order in [(3, 3, 4), (5, 3, 3), (2, 2, 5)]:
        p, lv, an = W.random_forest(seed, dim, order=order, max_level=2, frac=0.35)
        bg = W.background_table(p)
        X = W.node_coords(p, lv, an)
        c = np.array([0.5 * (p.hi[d] + p.lo[d]) for d in range(dim)])
        r = np.sqrt(((X - c[None, :, None]) ** 2).sum(axis=1)) / (0.3 * (p.hi[0] - p.lo[0]))
        q = W.pressure_balanced_state(p, W.node_background(p, bg, lv, an), 0.5 * W.cosine_bubble(r))
        yield f"forest{seed}", p, lv, an, bg, q


@pytest.mark.parametrize("case", list(_cases()), ids=lambda c: c[0])
def test_pointwise_matches_oracle_and_mortar_conserves(case):
    name, p, lv, an, bg, q0 = case
    q = _moving(p, lv, an, q0)
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    assert m.faces()[1].shape[0] > 0
    r_mortar = g.rhs(q)
    g.ctx.set_nonconforming(1)
    r_point = g.rhs(q)
    _check(r_point, oracle.rhs(m, bg, q, ncmode=1), what=f"{name} pointwise")
    g.ctx.set_nonconforming(0)
    _check(g.rhs(q), oracle.rhs(m, bg, q), what=f"{name} mortar")
    for f in (0, p.dim + 1):
        im = oracle.integrals(m, r_mortar)[f] / oracle.integrals(m, np.abs(r_mortar))[f]
        ip = oracle.integrals(m, r_point)[f] / oracle.integrals(m, np.abs(r_point))[f]
        assert abs(im) < 1e-14 and abs(ip) > 1e-13, (name, f, im, ip)


def test_pointwise_mode_n7():
    """3D N = 7 with the pointwise baseline runs on the generic tile kernel (k_stage_h7 keeps
    the mortar method only): RHS and an RK stage against the oracle on a 2:1 forest."""
    p, lv, an = W.random_forest(10, 3, order=7, max_level=1, frac=0.4)
    bg = W.background_table(p)
    X = W.node_coords(p, lv, an)
    c = np.array([0.5 * (p.hi[d] + p.lo[d]) for d in range(3)])
    r = np.sqrt(((X - c[None, :, None]) ** 2).sum(axis=1)) / (0.3 * (p.hi[0] - p.lo[0]))
    q = _moving(p, lv, an, W.pressure_balanced_state(p, W.node_background(p, bg, lv, an), 0.5 * W.cosine_bubble(r)))
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    assert m.faces()[1].shape[0] > 0
    g.ctx.set_nonconforming(1)
    _check(g.rhs(q), oracle.rhs(m, bg, q, ncmode=1), what="N=7 pointwise rhs")
    out = g.empty()
    g.ctx.rk_stage(0, 1e-3, g.dev(q), g.dev(q), out)
    # stage 0 of R17 on the oracle's pointwise RHS: q + dt L (the same rounded operations)
    _check(g.host(out), q + 1e-3 * oracle.rhs(m, bg, q, ncmode=1), what="N=7 pointwise stage 0")
