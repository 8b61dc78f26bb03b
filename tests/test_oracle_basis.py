"""Pins of the oracle's 1D operators against closed
forms, exact integrals and an independent Vandermonde / numpy-Gauss
construction of the paper's L2 projections (Sec. 3.3)."""
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _closed_forms():
    out = {}
    with open(os.path.join(GOLD, "lgl_closed_forms.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            n, xs, ws = [s.strip() for s in line.split("|")]
            ev = lambda s: [float(eval(t, {"sqrt": math.sqrt})) for t in s.split(",")]
            out[int(n)] = (np.array(ev(xs)), np.array(ev(ws)))
    return out


@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_lgl_closed_forms(N):
    x, w = oracle.lgl(N)
    xr, wr = _closed_forms()[N]
    np.testing.assert_allclose(x, xr, rtol=0, atol=1e-15)
    np.testing.assert_allclose(w, wr, rtol=0, atol=1e-15)


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 6, 7, 8])
def test_lgl_quadrature_exactness(N):
    x, w = oracle.lgl(N)
    assert abs(w.sum() - 2.0) < 1e-15 * 4
    assert np.all(np.diff(x) > 0) and x[0] == -1.0 and x[-1] == 1.0
    np.testing.assert_array_equal(x, -x[::-1])
    for k in range(2 * N):
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs(np.dot(w, x ** k) - exact) < 1e-14
    # degree 2N is NOT integrated exactly by LGL (guards against Gauss nodes)
    exact = 2.0 / (2 * N + 1)
    assert abs(np.dot(w, x ** (2 * N)) - exact) > 1e-6


def _interp_matrix(xfrom, tto):
    """Lagrange interpolation matrix via a Vandermonde solve (independent of the oracle)."""
    n = len(xfrom)
    V = np.vander(xfrom, n, increasing=True)
    T = np.vander(tto, n, increasing=True)
    return np.linalg.solve(V.T, T.T).T


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 7, 8])
def test_dmat(N):
    x, w = oracle.lgl(N)
    D = oracle.dmat(N)
    assert np.abs(D @ np.ones(N + 1)).max() < 1e-13
    for k in range(1, N + 1):
        np.testing.assert_allclose(D @ x ** k, k * x ** (k - 1), atol=1e-13 * max(1, N ** 2))
    assert abs(D[0, 0] + N * (N + 1) / 4.0) < 1e-13
    # summation by parts: W D + D^T W = diag(-1, 0, ..., 0, 1)
    Wm = np.diag(w)
    B = np.zeros((N + 1, N + 1))
    B[0, 0], B[N, N] = -1.0, 1.0
    assert np.abs(Wm @ D + D.T @ Wm - B).max() < 1e-13


@pytest.mark.parametrize("N", [1, 2, 3, 4, 5, 7])
def test_mortar_projection_definition(N):
    """P_b = (M^Xi)^-1 S and R_b = s M^-1 S^T with s = 1/2,
    rebuilt from the L2 definitions with a 24-point numpy Gauss rule."""
    x, w = oracle.lgl(N)
    M, S, P, R = oracle.mortar_ops(N)
    y, W = np.polynomial.legendre.leggauss(24)
    Ly = _interp_matrix(x, y)             # l_j(y_q)
    Mref = (Ly * W[:, None]).T @ Ly
    np.testing.assert_allclose(M, Mref, atol=1e-15 * 10)
    for b, xi in enumerate([(y - 1) / 2, (y + 1) / 2]):
        Lxi = _interp_matrix(x, xi)
        Sref = (Ly * W[:, None]).T @ Lxi
        np.testing.assert_allclose(S[b], Sref, atol=1e-14)
        Pref = np.linalg.solve(Mref, Sref)
        Rref = 0.5 * np.linalg.solve(Mref, Sref.T)
        np.testing.assert_allclose(P[b], Pref, atol=1e-13)
        np.testing.assert_allclose(R[b], Rref, atol=1e-13)
        # L2 projection of a degree-N polynomial is the interpolant on the half interval
        interp = _interp_matrix(x, (x - 1) / 2 if b == 0 else (x + 1) / 2)
        assert np.abs(P[b] - interp).max() < 1e-14 * max(1, N)
        # S_b 1 = w (integral of each mortar cardinal)
        np.testing.assert_allclose(S[b] @ np.ones(N + 1), w, atol=1e-15 * 8)
        # conservation: w^T R_b = 1/2 w^T  (integral of the back projection)
        np.testing.assert_allclose(w @ R[b], 0.5 * w, atol=1e-15 * 8)
        # constants map to constants both ways
        np.testing.assert_allclose(P[b] @ np.ones(N + 1), np.ones(N + 1), atol=1e-14)
    np.testing.assert_allclose(R[0] @ np.ones(N + 1) + R[1] @ np.ones(N + 1), np.ones(N + 1), atol=1e-14)
    # round trip face -> mortars -> face is the identity on degree-N polynomials
    np.testing.assert_allclose(R[0] @ P[0] + R[1] @ P[1], np.eye(N + 1), atol=1e-14 * max(1, N))


def test_mortar_n1_lower_example():
    """field xi at N=1 projected to the lower mortar -> nodal values {-1, 0}."""
    _, _, P, _ = oracle.mortar_ops(1)
    np.testing.assert_allclose(P[0] @ np.array([-1.0, 1.0]), [-1.0, 0.0], atol=1e-15)
    np.testing.assert_allclose(P[1] @ np.array([-1.0, 1.0]), [0.0, 1.0], atol=1e-15)


def test_mortar_scale_factor_golden():
    """s = 0.5 for 2:1: R_b 1 summed over a constant mortar flux of 1 gives 1."""
    vals = {}
    with open(os.path.join(GOLD, "paper_values.txt")) as fh:
        for line in fh:
            if line.startswith("#") or not line.strip():
                continue
            k, v, tol, _ = [s.strip() for s in line.split("|")]
            vals[k] = (float(v), float(tol))
    s, _ = vals["mortar_scale_2to1"]
    N = 4
    x, w = oracle.lgl(N)
    M, S, P, R = oracle.mortar_ops(N)
    np.testing.assert_allclose(R[0], s * np.linalg.solve(M, S[0].T), atol=1e-14)
