"""Pins of the oracle's point physics: EOS, perturbation form
(PAPER.md:96-103), sound speed, hydrostatic background
 and the Rusanov flux -- SURVEY C.3 P4-P6."""
import os

import numpy as np
import pytest

import oracle
import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _p(dim=3, **kw):
    p = W.Params(dim, 4, (1,) * dim, (0.0,) * dim, (1.0,) * dim, (0,) * dim, 0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def _pt(p, rho, U, Th, bg):
    """(rho', U, Theta', rho_bar, Theta_bar, P_bar) from full variables."""
    rb, Tb, Pb = bg
    return np.array([rho - rb] + list(U[: p.dim]) + [Th - Tb, rb, Tb, Pb])


def _consistent_bg(p, Tb, rb=1.0):
    return (rb, Tb, p.p0 * (p.R * Tb / p.p0) ** p.gamma)


def test_eos_fixed_point_and_scaling():
    p = _p()
    Tb = p.p0 / p.R                     # R Theta = p0  =>  P = p0
    bg = _consistent_bg(p, Tb)
    assert bg[2] == pytest.approx(p.p0, rel=1e-15)
    _, der = oracle.point_flux(p, 0, _pt(p, 1.0, [0, 0, 0], Tb, bg))
    assert der[3] == pytest.approx(p.p0, rel=1e-15) and der[2] == 0.0
    # Theta doubled => P = p0 2^gamma
    _, der = oracle.point_flux(p, 0, _pt(p, 1.0, [0, 0, 0], 2 * Tb, bg))
    assert der[3] == pytest.approx(p.p0 * 2 ** p.gamma, rel=1e-14)


@pytest.mark.parametrize("seed", range(5))
def test_eos_perturbation_form_matches_paper_eos(seed):
    """P' + P_bar reproduces P = p0 (R Theta/p0)^gamma for any
    Theta, given the consistent background P_bar = p0 (R Theta_bar/p0)^gamma."""
    rng = np.random.default_rng(seed)
    p = _p()
    for _ in range(50):
        Tb = rng.uniform(190, 350)
        Th = Tb * (1 + rng.uniform(-0.2, 0.2))
        bg = _consistent_bg(p, Tb)
        _, der = oracle.point_flux(p, 0, _pt(p, 1.0, [0, 0, 0], Th, bg))
        P_paper = p.p0 * (p.R * Th / p.p0) ** p.gamma
        assert der[3] == pytest.approx(P_paper, rel=1e-13)
        # P' itself accurate (cancellation-free, reading R2)
        assert der[2] == pytest.approx(P_paper - bg[2], rel=1e-9, abs=1e-9)


def test_pprime_small_perturbation_accuracy():
    """R2: P' relative error at Theta'/Theta_bar = 1e-6 must be ~1e-15, which
    the naive pow form cannot deliver; compare to the 2-term Taylor expansion."""
    p = _p()
    Tb = 320.0
    bg = _consistent_bg(p, Tb)
    for eps in (1e-6, 1e-9, -3e-7):
        pt = np.array([0.0, 0.0, 0.0, 0.0, Tb * eps, bg[0], bg[1], bg[2]])  # Theta' given directly
        _, der = oracle.point_flux(p, 0, pt)
        eps = (Tb * eps) / Tb
        # exact: P_bar((1+eps)^g - 1) = P_bar(g eps + g(g-1)/2 eps^2 + g(g-1)(g-2)/6 eps^3 + ...)
        g = p.gamma
        exact = bg[2] * (g * eps + g * (g - 1) / 2 * eps ** 2 + g * (g - 1) * (g - 2) / 6 * eps ** 3)
        assert der[2] == pytest.approx(exact, rel=1e-14)


def test_sound_speed_paper_value():
    """a = sqrt(gamma P/rho) at the theta0 = 300 K surface state vs the
    paper's 347.3 m/s within 0.5 m/s."""
    vals = {}
    with open(os.path.join(GOLD, "paper_values.txt")) as fh:
        for line in fh:
            if not line.startswith("#") and line.strip():
                k, v, tol, _ = [s.strip() for s in line.split("|")]
                vals[k] = (float(v), float(tol))
    ref, tol = vals["sound_speed_surface_mps"]
    p = W.Params(2, 4, (1, 1), (0.0, 0.0), (1000.0, 1000.0), (0, 0), 0)
    bg = W.background_table(p)[0]          # z = 0 row
    assert bg[2] == p.p0
    _, der = oracle.point_flux(p, 0, _pt(p, bg[0], [0, 0], bg[1], bg))
    assert abs(der[4] - ref) < tol
    assert der[4] == pytest.approx(np.sqrt(p.gamma * p.R * 300.0), rel=1e-14)


def test_sound_speed_homogeneity():
    p = _p()
    Tb = 300.0
    bg = _consistent_bg(p, Tb, rb=1.1)
    _, d1 = oracle.point_flux(p, 0, _pt(p, 1.1, [0, 0, 0], Tb, bg))
    assert d1[4] == pytest.approx(np.sqrt(p.gamma * bg[2] / 1.1), rel=1e-15)


def test_flux_rows():
    """F = (U, U u_d + P' e_d, Theta u_d) (reading R5)."""
    p = _p()
    bg = _consistent_bg(p, 300.0, rb=1.0)
    U = np.array([1.0, 2.0, -0.5])
    pt = _pt(p, 2.0, U, 310.0, bg)
    for d in range(3):
        F, der = oracle.point_flux(p, d, pt)
        u = U / 2.0
        np.testing.assert_allclose(F[0], U[d], rtol=1e-15)
        for j in range(3):
            np.testing.assert_allclose(F[1 + j], U[j] * u[d] + (der[2] if j == d else 0), rtol=1e-15)
        np.testing.assert_allclose(F[4], 310.0 * u[d], rtol=1e-15)


def test_hydrostatic_background_closed_form():
    """P_bar(0) = p0, Theta_bar(0) = p0/R, rho_bar(0) = Theta_bar/theta0, and the
    table rows follow P = p0 (1 - g z/(cp theta0))^(cp/R)."""
    p = W.Params(2, 4, (10, 10), (0.0, 0.0), (1000.0, 1000.0), (0, 0), 1)
    bg = W.background_table(p)
    z = W.table_heights(p)
    assert bg[0, 2] == p.p0
    assert bg[0, 1] == pytest.approx(p.p0 / p.R, rel=1e-15)
    assert bg[0, 0] == pytest.approx(p.p0 / p.R / 300.0, rel=1e-15)
    assert bg[0, 0] == pytest.approx(1.161440, abs=1e-6)
    np.testing.assert_allclose(bg[:, 2], p.p0 * (1 - p.g * z / (p.cp * 300.0)) ** 3.5, rtol=1e-14)
    # EOS consistency of the background (needed for the well-balanced rest state)
    np.testing.assert_allclose(bg[:, 2], p.p0 * (p.R * bg[:, 1] / p.p0) ** p.gamma, rtol=1e-14)


def test_discrete_hydrostatic_residual_decays():
    """||(2/h) D P_bar + rho_bar g|| / (rho_bar g) decays spectrally in N."""
    res = []
    for N in (2, 3, 4):
        p = W.Params(2, N, (1, 10), (0.0, 0.0), (100.0, 1000.0), (0, 0), 0)
        bg = W.background_table(p)
        D = oracle.dmat(N)
        r = 0.0
        for iz in range(10):
            rows = bg[iz * (N + 1):(iz + 1) * (N + 1)]
            resid = (2.0 / 100.0) * D @ rows[:, 2] + rows[:, 0] * p.g
            r = max(r, np.abs(resid).max() / (rows[:, 0] * p.g).max())
        res.append(r)
    assert res[0] > res[1] > res[2]
    assert res[2] < 1e-11 and res[0] < 1e-4


# ------------------------------ Rusanov (P6) ------------------------------
def _rand_pt(rng, p):
    Tb = rng.uniform(250, 340)
    bg = _consistent_bg(p, Tb, rb=Tb / 300.0)
    rho = bg[0] * (1 + rng.uniform(-0.05, 0.05))
    U = rng.uniform(-20, 20, 3)
    Th = Tb * (1 + rng.uniform(-0.05, 0.05))
    return _pt(p, rho, U, Th, bg)


@pytest.mark.parametrize("dim", [2, 3])
def test_rusanov_consistency_and_antisymmetry(dim):
    p = _p(dim)
    rng = np.random.default_rng(7)
    for _ in range(40):
        L, R = _rand_pt(rng, p), _rand_pt(rng, p)
        for d in range(dim):
            for s in (1.0, -1.0):
                # consistency: F*(q, q, n) = F(q).n exactly
                F, _ = oracle.point_flux(p, d, L)
                np.testing.assert_array_equal(oracle.rusanov(p, d, s, L, L), s * F)
                # conservation: F*(q-, q+, n) = -F*(q+, q-, -n) bitwise
                a = oracle.rusanov(p, d, s, L, R)
                b = oracle.rusanov(p, d, -s, R, L)
                np.testing.assert_array_equal(a, -b)


def test_rusanov_mirror_wall_zero_mass_and_theta_flux():
    """Reading R9: mirror ghost gives exactly zero mass and Theta flux through a wall."""
    p = _p(3)
    rng = np.random.default_rng(9)
    for _ in range(20):
        L = _rand_pt(rng, p)
        for d in range(3):
            R = L.copy()
            R[1 + d] = -L[1 + d]
            for s in (1.0, -1.0):
                Fs = oracle.rusanov(p, d, s, L, R)
                assert Fs[0] == 0.0 and Fs[4] == 0.0


def test_rusanov_dissipation_is_upwinding():
    """The jump term dissipates: for a pure density jump at rest the mass flux
    is lambda/2 (rho'- - rho'+) with lambda = max(a-, a+) (PAPER.md:129-131,
    readings R6-R7), i.e. mass moves from the denser to the lighter side."""
    p = _p(3)
    Tb = 300.0
    bg = _consistent_bg(p, Tb, rb=1.0)
    L = _pt(p, 1.2, [0, 0, 0], Tb, bg)
    R = _pt(p, 1.0, [0, 0, 0], Tb, bg)
    Fs = oracle.rusanov(p, 0, 1.0, L, R)
    aL, aR = np.sqrt(p.gamma * bg[2] / 1.2), np.sqrt(p.gamma * bg[2] / 1.0)
    assert Fs[0] > 0
    assert Fs[0] == pytest.approx(0.5 * max(aL, aR) * 0.2, rel=1e-14)
    # and the wave speed includes |u.n|: supersonic-free check with u = 10
    L2 = _pt(p, 1.2, [12.0, 0, 0], Tb, bg)
    R2 = _pt(p, 1.0, [10.0, 0, 0], Tb, bg)
    F2 = oracle.rusanov(p, 0, 1.0, L2, R2)
    lam = max(10.0 + aL, 10.0 + aR)
    assert F2[0] == pytest.approx(0.5 * (12 + 10) + 0.5 * lam * 0.2, rel=1e-14)
