"""NEXT-3 artificial viscosity in the oracle (reading R42): pins.

* exactness: for a perturbation that is a global polynomial of degree <= N with
  zero normal derivative on the walls (f(s) = s^2 (3 - 2 s) per axis, s = x / L),
  the BR1 operator returns mu times its Laplacian exactly -- also across 2:1
  faces, where the mortar projections of a degree-N polynomial are exact;
* conservation: every field's integral of V vanishes (walls carry no diffusive
  flux, interior and mortar fluxes are single-valued);
* rest: V = 0 for the background state."""
import numpy as np

import oracle
import workloads as W


def _f(s):
    return s * s * (3.0 - 2.0 * s)


def _d2f(s):
    return 6.0 - 12.0 * s


def _poly_state(p, lv, an, bg):
    X = W.node_coords(p, lv, an)
    bgn = W.node_background(p, bg, lv, an)
    L = [p.hi[d] - p.lo[d] for d in range(p.dim)]
    g = sum(_f((X[:, d] - p.lo[d]) / L[d]) for d in range(p.dim))
    lap = sum(_d2f((X[:, d] - p.lo[d]) / L[d]) / L[d] ** 2 for d in range(p.dim))
    amp = np.array([0.01, 1.0, 2.0, 3.0, 0.1])[: p.n_fields]
    amp[-1] = 0.1
    q = np.empty((len(lv), p.n_fields, p.n_nodes))
    q[:, 0] = bgn[:, :, 0] + amp[0] * g
    for j in range(p.dim):
        q[:, 1 + j] = amp[1 + j] * g
    q[:, -1] = bgn[:, :, 1] + amp[-1] * g
    return q, amp[None, :, None] * lap[:, None, :]


def _meshes():
    p = W.Params(2, 4, (4, 3), (0.0, 0.0), (400.0, 300.0), (0, 0), 1)
    yield p, *W.uniform_morton(p)
    yield W.random_forest(2, 2, order=4, max_level=2, frac=0.4)
    yield W.random_forest(3, 3, order=3, max_level=1, frac=0.4)


def test_visc_exact_for_neumann_polynomial():
    mu = 1.5
    for p, lv, an in _meshes():
        p.periodic = (0,) * p.dim
        bg = W.background_table(p)
        q, lap = _poly_state(p, lv, an, bg)
        m = oracle.Mesh(p, lv, an)
        V = oracle.visc(m, bg, q, mu)
        scale = np.abs(mu * lap).max()
        assert np.abs(V - mu * lap).max() <= 1e-9 * scale, np.abs(V - mu * lap).max() / scale


def test_visc_conservative_and_zero_at_rest():
    rng = np.random.default_rng(11)
    for p, lv, an in _meshes():
        bg = W.background_table(p)
        m = oracle.Mesh(p, lv, an)
        rest = W.pressure_balanced_state(p, W.node_background(p, bg, lv, an), np.zeros((len(lv), p.n_nodes)))
        assert np.all(oracle.visc(m, bg, rest, 1.5) == 0.0)
        q = rest + 0.01 * rng.standard_normal(rest.shape) * np.abs(rest).max(axis=(0, 2))[None, :, None]
        V = oracle.visc(m, bg, q, 1.5)
        I, A = oracle.integrals(m, V), oracle.integrals(m, np.abs(V))
        assert np.all(np.abs(I) <= 1e-13 * A), I / A
