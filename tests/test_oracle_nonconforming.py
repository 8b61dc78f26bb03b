"""NEXT-3 baseline in the oracle: pointwise interpolation on the coarse side of
2:1 faces (R41).  Pins: identical to the mortar method where there
is nothing to interpolate (no 2:1 faces; rest state), and -- the paper's point
 -- not conservative where the mortar method is."""
import numpy as np

import oracle
import workloads as W


def _moving(w):
    X = W.node_coords(w.params, w.level, w.anchor)
    q = w.q0.copy()
    q[:, 1] += 0.5 * q[:, 0] * np.sin(X[:, 1] / 2000.0)
    q[:, 2] += 0.3 * q[:, 0] * np.cos(X[:, 0] / 3000.0)
    return q


def test_same_as_mortar_without_two_to_one_faces_or_at_rest():
    w = W.c1()  # conforming
    m = oracle.Mesh(w.params, w.level, w.anchor)
    assert np.array_equal(oracle.rhs(m, w.bg, w.q0, ncmode=1), oracle.rhs(m, w.bg, w.q0))
    w = W.c2()  # 2:1 faces, hydrostatic rest far from the bubble: both exactly at rest there
    m = oracle.Mesh(w.params, w.level, w.anchor)
    rest = W.pressure_balanced_state(w.params, W.node_background(w.params, w.bg, w.level, w.anchor),
                                     np.zeros((w.n_elem, w.params.n_nodes)))
    assert np.all(oracle.rhs(m, w.bg, rest, ncmode=1) == 0.0)


def test_not_conservative_where_mortar_is():
    w = W.c2()
    m = oracle.Mesh(w.params, w.level, w.anchor)
    q = _moving(w)
    I = {}
    for mode in (0, 1):
        r = oracle.rhs(m, w.bg, q, ncmode=mode)
        I[mode] = oracle.integrals(m, r) / oracle.integrals(m, np.abs(r))
    for f in (0, 3):  # mass and Theta: no sources, walls are no-flux
        assert abs(I[0][f]) < 1e-14
        assert abs(I[1][f]) > 1e-12
