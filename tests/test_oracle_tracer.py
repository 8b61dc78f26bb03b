"""Kinematic tracer in the oracle (the paper's LeVeque test; R43): pins.

* with a constant wind on a periodic mesh the RHS converges to -u . grad C at the
  spatial order of the strong-form derivative;
* with the LeVeque wind (no normal component on the walls) the tracer mass is
  conserved to round-off by the mortar method and not by the pointwise baseline
  (P:551-555);
* a constant tracer in a constant wind is a steady state (RHS 0 to round-off)."""
import numpy as np

import oracle
import workloads as W


def _periodic(nx, order=3):
    p = W.Params(2, order, (nx, nx), (0.0, 0.0), (1.0, 1.0), (1, 1), 0)
    lv, an = W.uniform_morton(p)
    return p, lv, an


def test_constant_wind_converges_to_advection():
    errs = []
    for nx in (4, 8, 16):
        p, lv, an = _periodic(nx)
        X = W.node_coords(p, lv, an)
        s = np.zeros((len(lv), 4, p.n_nodes))
        s[:, 0] = np.sin(2 * np.pi * X[:, 0]) * np.sin(2 * np.pi * X[:, 1])
        s[:, 1], s[:, 2] = 1.0, 0.5
        exact = -(2 * np.pi * np.cos(2 * np.pi * X[:, 0]) * np.sin(2 * np.pi * X[:, 1])
                  + 0.5 * 2 * np.pi * np.sin(2 * np.pi * X[:, 0]) * np.cos(2 * np.pi * X[:, 1]))
        r = oracle.tracer_rhs(oracle.Mesh(p, lv, an), s)
        errs.append(np.abs(r - exact).max() / np.abs(exact).max())
    assert errs[0] / errs[1] > 4 and errs[1] / errs[2] > 5, errs
    # constant tracer in a constant wind: steady (to the round-off of the D row sums)
    s[:, 0] = 0.7
    assert np.abs(oracle.tracer_rhs(oracle.Mesh(p, lv, an), s)).max() <= 1e-12 * 0.7 * 2 * 16 * 16


def test_mortar_conserves_tracer_pointwise_does_not():
    p, lv, an = W.random_forest(2, 2, order=4, max_level=2, frac=0.4)
    p = W.Params(2, 4, p.root, (0.0, 0.0), (1.0, 1.0), (0, 0), 2)
    s = W.leveque_state(p, lv, an, t=0.7)
    X = W.node_coords(p, lv, an)
    s[:, 0] = np.exp(-((X[:, 0] - 0.4) ** 2 + (X[:, 1] - 0.45) ** 2) / 0.05)
    m = oracle.Mesh(p, lv, an)
    assert m.faces()[1].shape[0] > 0
    for mode, lo, hi in ((0, None, 1e-14), (1, 1e-12, None)):
        r = oracle.tracer_rhs(m, s, ncmode=mode)
        tmp = np.zeros_like(s)
        tmp[:, 0] = r
        I = oracle.integrals(m, tmp)[0]
        tmp[:, 0] = np.abs(r)
        rel = abs(I) / oracle.integrals(m, tmp)[0]
        if hi is not None:
            assert rel < hi, (mode, rel)
        if lo is not None:
            assert rel > lo, (mode, rel)
