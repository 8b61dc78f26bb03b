"""NEXT-3: the passive tracer of the Euler flow in the oracle (C = rho c, P:73-89 eq.
eulervector; reading R45).  Pins, none of which re-types the oracle's formula:

* polynomial exactness: uniform rho, Theta (P' = 0, g = 0), velocity v and mixing ratio c global
  polynomials of degree <= N/2 on 2:1 forests -> C v in Q_N is continuous, every jump vanishes, and
  dC/dt = -div(C v) exactly at the nodes of elements not touching a wall (mortars exact
  for polynomials);
* consistency with the continuity equation (whose RHS is pinned in test_oracle_rhs.py): a constant
  mixing ratio, C = c0 rho, gives dC/dt = c0 drho/dt to rounding on a conforming mesh with gravity and
  on a 2:1 forest with a constant background (the mortar projection preserves constants);
* conservation: the quadrature of dC/dt vanishes to rounding for a discontinuous random C on a
  moving state with walls and 2:1 faces (the mortar method);
* rest: U = 0 with a continuous C gives exactly 0."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_oracle_rhs import Poly, amr_forest, const_bg, interior_elements, rand_poly


def _moving(p, lv, an, q0, amp=4.0):
    X = W.node_coords(p, lv, an)
    q = q0.copy()
    L = max(p.hi[d] - p.lo[d] for d in range(p.dim))
    for d in range(p.dim):
        q[:, 1 + d] += amp * q[:, 0] * np.sin(4 * np.pi * X[:, (d + 1) % p.dim] / L + d) * np.cos(2 * np.pi * X[:, d] / L)
    return q


@pytest.mark.parametrize("dim", [2, 3])
def test_passive_polynomial_exactness(dim):
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=4, root=(4, 4) if dim == 2 else (3, 3, 3))
    p.g = 0.0
    rb, Tb = 1.1, 320.0
    bg = const_bg(p, rb, Tb)
    mesh = oracle.Mesh(p, level, anchor)
    assert len(mesh.faces()[1]) > 0
    X = W.node_coords(p, level, anchor)
    L = [p.hi[d] for d in range(dim)]
    rng = np.random.default_rng(8 + dim)
    N = p.order
    v = [rand_poly(rng, dim, N // 2).scale(5.0) for _ in range(dim)]
    cp = rand_poly(rng, dim, N // 2).scale(0.3)
    q = np.zeros((len(level), p.n_fields, p.n_nodes))
    q[:, 0] = rb
    q[:, dim + 1] = Tb
    for j in range(dim):
        q[:, 1 + j] = rb * v[j](X, L)
    C = rb * cp(X, L)
    flux = [cp * v[d] for d in range(dim)]  # C u / rho_bar
    acc = flux[0].deriv(0, L)
    for d in range(1, dim):
        acc = acc + flux[d].deriv(d, L)
    exact = -rb * acc(X, L)
    r = oracle.passive_rhs(mesh, bg, q, C)
    sel = interior_elements(p, level, anchor)
    assert len(np.intersect1d(sel, mesh.faces()[1][:, 0])) > 0  # coarse sides of 2:1 faces among them
    err = np.abs(r[sel] - exact[sel]).max() / np.abs(exact[sel]).max()
    assert err < 1e-11, err
    # a wrong sign in the face term would show at every face node; so would a transposed P_b
    assert np.abs(exact[sel]).max() > 1e-3


def test_constant_mixing_ratio_follows_continuity_conforming():
    w = W.c3()
    mesh = oracle.Mesh(w.params, w.level, w.anchor)
    q = _moving(w.params, w.level, w.anchor, w.q0, amp=2.0)
    c0 = 0.37
    r = oracle.passive_rhs(mesh, w.bg, q, c0 * q[:, 0])
    drho = oracle.rhs(mesh, w.bg, q)[:, 0]
    err = np.abs(r - c0 * drho).max() / np.abs(c0 * drho).max()
    assert err < 1e-10, err


@pytest.mark.parametrize("dim", [2, 3])
def test_constant_mixing_ratio_follows_continuity_amr(dim):
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=6, root=(4, 4) if dim == 2 else (3, 3, 3))
    p.g = 0.0
    bg = const_bg(p)
    mesh = oracle.Mesh(p, level, anchor)
    assert len(mesh.faces()[1]) > 0
    rng = np.random.default_rng(9)
    q0 = W.pressure_balanced_state(p, W.node_background(p, bg, level, anchor),
                                   rng.uniform(-0.5, 0.5, size=(len(level), p.n_nodes)))
    q = _moving(p, level, anchor, q0)
    c0 = 2.5
    r = oracle.passive_rhs(mesh, bg, q, c0 * q[:, 0])
    drho = oracle.rhs(mesh, bg, q)[:, 0]
    err = np.abs(r - c0 * drho).max() / np.abs(c0 * drho).max()
    assert err < 1e-10, err


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_passive_conservation(name):
    w = W.get(name)
    mesh = oracle.Mesh(w.params, w.level, w.anchor)
    q = _moving(w.params, w.level, w.anchor, w.q0)
    rng = np.random.default_rng(11)
    C = q[:, 0] * rng.uniform(0.0, 1.0, size=q[:, 0].shape)  # discontinuous mixing ratio
    r = oracle.passive_rhs(mesh, w.bg, q, C)
    a = np.zeros_like(q)
    a[:, 0] = r
    b = np.zeros_like(q)
    b[:, 0] = np.abs(r)
    rel = oracle.integrals(mesh, a)[0] / oracle.integrals(mesh, b)[0]
    assert abs(rel) < 1e-14, rel


def test_passive_rest_is_exactly_zero():
    """U = 0 and a continuous C (both sides of every face see the same values): no flux, no jump."""
    w = W.c1()
    mesh = oracle.Mesh(w.params, w.level, w.anchor)
    X = W.node_coords(w.params, w.level, w.anchor)
    C = 1.0 + 0.1 * np.sin(X[:, 0] / 300.0) * np.cos(X[:, 1] / 200.0)
    rest = W.pressure_balanced_state(w.params, W.node_background(w.params, w.bg, w.level, w.anchor),
                                     np.zeros((w.n_elem, w.params.n_nodes)))
    assert np.all(oracle.passive_rhs(mesh, w.bg, rest, C) == 0.0)
