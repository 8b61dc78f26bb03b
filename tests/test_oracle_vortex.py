"""NEXT-2: the oracle against the closed-form isentropic vortex
(§4.1; reading R36).  The exact solution is a translation of
the t = 0 vortex at (1, 1) m/s, so

* the oracle RHS at t = 0 must converge to dq/dt = -(c . grad) q0 (taken here as
  a central difference in time of the closed form) at the spatial order of the
  strong-form DGSEM derivative, O(h^N): ratio ~ 2^N per halving of h;
* RK3 trajectories must converge to the translated vortex at O(h^(N+1)).

A dropped flux term, a wrong sign or a transposed operand gives an O(1) error
that does not converge, so these pin the whole RHS, not just its pieces."""
import numpy as np

import oracle
import workloads as W


def _case(nx, order=3):
    p = W.vortex_params(nx, order)
    lv, an = W.uniform_morton(p)
    bg = W.vortex_background(p)
    return p, lv, an, bg, oracle.Mesh(p, lv, an)


def test_vortex_state_is_isentropic_translation():
    p = W.vortex_params(8, 3)
    lv, an = W.uniform_morton(p)
    q0 = W.vortex_state(p, lv, an, 0.0)
    # theta = Theta / rho = 1 (isentropic), far field = free stream
    assert np.array_equal(q0[:, 3], q0[:, 0])
    X = W.node_coords(p, lv, an)
    far = np.hypot(X[:, 0], X[:, 1]) > 5.9
    assert np.allclose(q0[:, 0][far], 1.0, atol=1e-12)
    assert np.allclose(q0[:, 1][far] / q0[:, 0][far], 1.0, atol=1e-12)
    # one full period of the periodic square (12 m at 1 m/s) returns the same state
    assert np.allclose(W.vortex_state(p, lv, an, 12.0), q0, atol=1e-12)


def test_vortex_rhs_converges_to_exact_time_derivative():
    errs = []
    for nx in (8, 16, 32):
        p, lv, an, bg, m = _case(nx)
        q0 = W.vortex_state(p, lv, an, 0.0)
        r = oracle.rhs(m, bg, q0)
        eps = 1e-4
        dq = (W.vortex_state(p, lv, an, eps) - W.vortex_state(p, lv, an, -eps)) / (2 * eps)
        errs.append(np.abs(r - dq).max() / np.abs(dq).max())
    assert errs[2] < 1e-2, errs
    assert errs[0] / errs[1] > 4.0 and errs[1] / errs[2] > 5.0, errs


def test_vortex_rk3_converges_to_translated_vortex():
    T = 0.25
    rms = []
    for nx in (16, 32):
        p, lv, an, bg, m = _case(nx)
        q = W.vortex_state(p, lv, an, 0.0)
        n = int(round(T / (0.15 / nx)))
        dt = T / n
        for _ in range(n):
            q = oracle.rk3_step(m, bg, dt, q)
        rms.append(W.vortex_l2(p, q, W.vortex_state(p, lv, an, T))["rms"])
    assert rms[1] < 1e-4, rms
    assert rms[0] / rms[1] > 8.0, rms
