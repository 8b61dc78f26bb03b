"""Pins of the oracle's dGSEM right-hand side and RK stage:
free-stream preservation, the well-balanced rest state, exactness on
polynomial fluxes (against analytic derivatives), discrete conservation, an
independent dense weak-form assembly on tiny AMR meshes (PAPER.md:116-133,
290-310), and the SSP-RK3 stability polynomial (reading R17)."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W
from test_oracle_mesh import brute_force_faces


# ----------------------------------------------------------------- helpers
def const_bg(p, rb=1.1, Tb=320.0):
    rows = W.row_offsets(p)[-1]
    Pb = p.p0 * (p.R * Tb / p.p0) ** p.gamma
    return np.tile(np.array([[rb, Tb, Pb]]), (rows, 1))


def amr_forest(dim, periodic, seed=0, root=None, max_level=2):
    rng = np.random.default_rng(seed)
    root = root or ((4, 3) if dim == 2 else (3, 2, 2))
    p = W.Params(dim, 4, root, (0.0,) * dim, tuple(250.0 * r for r in root), periodic, max_level)
    f = W.Forest(p)
    for lev in range(max_level):
        cand = sorted(x for x in f.leaves if x[0] == lev)
        for leaf in cand:
            if rng.random() < 0.35:
                f.split(leaf)
    f.balance()
    level, anchor = f.ordered()
    return p, level, anchor


def field_rel(a, b):
    """Per-field max|a-b| / max|b| (reading R19)."""
    out = []
    for f in range(a.shape[1]):
        den = np.abs(b[:, f]).max()
        num = np.abs(a[:, f] - b[:, f]).max()
        out.append(num / den if den > 0 else num)
    return np.array(out)


def quad_weights(p, level):
    """J * prod_d w_{i_d} per (element, node) with the generator's nodes."""
    N, n1 = p.order, p.n1
    x = W.lgl_nodes(N)
    y, wq = np.polynomial.legendre.leggauss(2 * N + 2)
    V = np.vander(x, n1, increasing=True)
    L = np.vander(y, n1, increasing=True) @ np.linalg.inv(V)
    w = wq @ L
    node = np.arange(p.n_nodes)
    wn = np.ones(p.n_nodes)
    J = np.ones(len(level))
    for d in range(p.dim):
        wn = wn * w[(node // n1 ** d) % n1]
        J = J * 0.5 * ((p.hi[d] - p.lo[d]) / p.root[d]) / 2.0 ** level.astype(np.float64)
    return J[:, None] * wn[None, :]


# ------------------------------------------------------- P7a free stream
@pytest.mark.parametrize("dim", [2, 3])
def test_free_stream_periodic_amr(dim):
    p, level, anchor = amr_forest(dim, (1,) * dim, seed=1)
    p.g = 0.0
    mesh = oracle.Mesh(p, level, anchor)
    assert len(mesh.faces()[1]) > 0
    bg = const_bg(p)
    E = len(level)
    q = np.zeros((E, p.n_fields, p.n_nodes))
    rho = 1.1 * 1.07
    vel = np.array([3.0, -2.0, 1.5])[:dim]
    q[:, 0] = rho
    q[:, 1:1 + dim] = (rho * vel)[None, :, None]
    q[:, dim + 1] = 320.0 * 1.05
    r = oracle.rhs(mesh, bg, q)
    Pp = bg[0, 2] * (1.05 ** p.gamma - 1)
    Fmax = max(rho * vel.max() ** 2 + Pp, 320 * 1.05 * vel.max())
    hmin = min((p.hi[d] - p.lo[d]) / p.root[d] for d in range(dim)) / 2 ** level.max()
    assert np.abs(r).max() <= 1e-12 * Fmax * 2 / hmin


# ------------------------------------------------------- P7b rest state
@pytest.mark.parametrize("case", ["c1", "c2", "amr3d"])
def test_rest_state_is_exactly_zero(case):
    if case == "amr3d":
        p, level, anchor = amr_forest(3, (1, 0, 0), seed=2)
    elif case == "c2":
        p, f = W.c2_forest()
        level, anchor = f.ordered()
    else:
        w = W.c1()
        p, level, anchor = w.params, w.level, w.anchor
    bg = W.background_table(p)
    mesh = oracle.Mesh(p, level, anchor)
    q = W.pressure_balanced_state(p, W.node_background(p, bg, level, anchor), 0.0)
    r = oracle.rhs(mesh, bg, q)
    assert np.all(r == 0.0)
    # and the state is bitwise unchanged by RK3 steps (zero RHS)
    q1 = oracle.rk3_step(mesh, bg, 0.01, q)
    assert np.array_equal(q1, q)


# ----------------------------------------------- P7c polynomial exactness
class Poly:
    """Multivariate polynomial {exponent tuple: coeff} in scaled coordinates."""

    def __init__(self, terms, dim):
        self.t = {k: v for k, v in terms.items() if v != 0.0}
        self.dim = dim

    def __mul__(self, o):
        out = {}
        for a, ca in self.t.items():
            for b, cb in o.t.items():
                k = tuple(i + j for i, j in zip(a, b))
                out[k] = out.get(k, 0.0) + ca * cb
        return Poly(out, self.dim)

    def __add__(self, o):
        out = dict(self.t)
        for k, v in o.t.items():
            out[k] = out.get(k, 0.0) + v
        return Poly(out, self.dim)

    def scale(self, s):
        return Poly({k: v * s for k, v in self.t.items()}, self.dim)

    def deriv(self, d, L):
        out = {}
        for k, v in self.t.items():
            if k[d] > 0:
                kk = list(k)
                kk[d] -= 1
                out[tuple(kk)] = out.get(tuple(kk), 0.0) + v * k[d] / L[d]
        return Poly(out, self.dim)

    def __call__(self, X, L):
        out = np.zeros(X.shape[0:1] + X.shape[2:])
        for k, v in self.t.items():
            term = np.full(out.shape, v)
            for d in range(self.dim):
                term = term * (X[:, d] / L[d]) ** k[d]
            out += term
        return out


def rand_poly(rng, dim, deg):
    terms = {}
    for k in itertools.product(range(deg + 1), repeat=dim):
        terms[k] = rng.uniform(-1, 1)
    return Poly(terms, dim)


def interior_elements(p, level, anchor):
    conf, nonc, bnd = oracle.Mesh(p, level, anchor).faces()
    touch = np.zeros(len(level), bool)
    touch[bnd[:, 0]] = True
    return np.nonzero(~touch)[0]


@pytest.mark.parametrize("dim", [2, 3])
def test_polynomial_exactness(dim):
    """g = 0, rho and Theta constant = background (P' = 0), U = rho0 v with v a
    global polynomial of degree <= N/2 per coordinate: every flux is in Q_N and
    continuous, so the RHS equals -div F exactly at the nodes (mortars too)."""
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=3, root=(4, 4) if dim == 2 else (3, 3, 3))
    p.g = 0.0
    rb, Tb = 1.1, 320.0
    bg = const_bg(p, rb, Tb)
    mesh = oracle.Mesh(p, level, anchor)
    assert len(mesh.faces()[1]) > 0
    X = W.node_coords(p, level, anchor)
    Lsc = [p.hi[d] for d in range(dim)]
    rng = np.random.default_rng(11)
    v = [rand_poly(rng, dim, p.order // 2).scale(5.0) for _ in range(dim)]
    q = np.zeros((len(level), p.n_fields, p.n_nodes))
    q[:, 0] = rb
    q[:, dim + 1] = Tb
    for j in range(dim):
        q[:, 1 + j] = rb * v[j](X, Lsc)
    r = oracle.rhs(mesh, bg, q)
    exact = np.zeros_like(r)
    divv = v[0].deriv(0, Lsc)
    for d in range(1, dim):
        divv = divv + v[d].deriv(d, Lsc)
    exact[:, 0] = -rb * divv(X, Lsc)
    exact[:, dim + 1] = -Tb * divv(X, Lsc)
    for j in range(dim):
        acc = (v[j] * v[0]).deriv(0, Lsc)
        for d in range(1, dim):
            acc = acc + (v[j] * v[d]).deriv(d, Lsc)
        exact[:, 1 + j] = -rb * acc(X, Lsc)
    sel = interior_elements(p, level, anchor)
    conf, nonc, bnd = mesh.faces()
    mort = np.zeros(len(level), bool)
    mort[nonc[:, 0]] = True
    mort[nonc[:, 2::2].ravel()] = True
    plain = sel[~mort[sel]]
    assert len(plain) > 0 and mort[sel].any()
    err = field_rel(r[plain], exact[plain])
    assert err.max() < 5e-13, err      # rounding of sum_m D F with row sums |D| ~ 16
    # on mortar faces the projected trace equals the fine trace only to rounding,
    # and the Rusanov jump term amplifies that by lambda/2 (2/h)/w0: bound it so
    x, w = oracle.lgl(p.order)
    lam = np.sqrt(p.gamma * bg[0, 2] / rb) + np.abs(q[:, 1:1 + dim] / rb).max()
    hmin = min(p.hi[d] / p.root[d] for d in range(dim)) / 2 ** level.max()
    for f in range(p.n_fields):
        bound = 1e-13 * np.abs(exact[sel, f]).max() + 4e-15 * lam * np.abs(q[:, f]).max() * 2 / hmin / w[0]
        assert np.abs(r[sel, f] - exact[sel, f]).max() <= bound, f


@pytest.mark.parametrize("dim", [2, 3])
def test_mass_row_exact_for_degree_N(dim):
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=4, root=(4, 4) if dim == 2 else (3, 3, 3))
    p.g = 0.0
    bg = const_bg(p)
    mesh = oracle.Mesh(p, level, anchor)
    X = W.node_coords(p, level, anchor)
    Lsc = [p.hi[d] for d in range(dim)]
    rng = np.random.default_rng(12)
    U = [rand_poly(rng, dim, p.order).scale(0.01) for _ in range(dim)]
    q = np.zeros((len(level), p.n_fields, p.n_nodes))
    q[:, 0] = 1.1
    q[:, dim + 1] = 320.0
    for j in range(dim):
        q[:, 1 + j] = U[j](X, Lsc)
    r = oracle.rhs(mesh, bg, q)
    div = U[0].deriv(0, Lsc)
    for d in range(1, dim):
        div = div + U[d].deriv(d, Lsc)
    sel = interior_elements(p, level, anchor)
    ex = -div(X, Lsc)[sel]
    assert np.abs(r[sel, 0] - ex).max() < 5e-13 * np.abs(ex).max()


# ------------------------------------------------------- P7d conservation
def _bubble_state(p, level, anchor, seed):
    bg = W.background_table(p)
    X = W.node_coords(p, level, anchor)
    c = [0.5 * (p.hi[d] + p.lo[d]) for d in range(p.dim)]
    r = np.sqrt(sum((X[:, d] - c[d]) ** 2 for d in range(p.dim))) / (0.3 * p.hi[0])
    q = W.pressure_balanced_state(p, W.node_background(p, bg, level, anchor), 2.0 * W.cosine_bubble(r))
    rng = np.random.default_rng(seed)
    q[:, 1:1 + p.dim] = q[:, :1] * rng.uniform(-1.0, 1.0, size=(len(level), p.dim, p.n_nodes))
    q[:, p.dim + 1] *= 1 + 1e-3 * rng.uniform(-1, 1, size=(len(level), p.n_nodes))
    return bg, q


@pytest.mark.parametrize("case", [("2d", (1, 0)), ("2d", (0, 0)), ("3d", (1, 1, 0)), ("3d", (0, 0, 0))])
def test_conservation_rhs_and_step(case):
    dim = 2 if case[0] == "2d" else 3
    p, level, anchor = amr_forest(dim, case[1], seed=5)
    mesh = oracle.Mesh(p, level, anchor)
    bg, q = _bubble_state(p, level, anchor, 6)
    r = oracle.rhs(mesh, bg, q)
    Jw = quad_weights(p, level)
    for f in (0, dim + 1):   # mass and Theta
        tot = (Jw * r[:, f]).sum()
        scale = (Jw * np.abs(r[:, f])).sum()
        assert abs(tot) <= 1e-13 * scale, (f, tot, scale)
    q1 = oracle.rk3_step(mesh, bg, 0.01, q)
    I0, I1 = oracle.integrals(mesh, q), oracle.integrals(mesh, q1)
    for f in (0, dim + 1):
        assert abs(I1[f] - I0[f]) <= 1e-13 * abs(I0[f])
        # and relative to the amount actually moved
        moved = 0.01 * (Jw * np.abs(r[:, f])).sum()
        assert abs(I1[f] - I0[f]) <= 1e-11 * moved


def test_integrals_match_generator_quadrature():
    w = W.c1()
    mesh = oracle.Mesh(w.params, w.level, w.anchor)
    I = oracle.integrals(mesh, w.q0)
    ref = (quad_weights(w.params, w.level)[:, None, :] * w.q0).sum(axis=(0, 2))
    np.testing.assert_allclose(I, ref, rtol=1e-13)
    # constant field integrates to the domain volume
    ones = np.ones_like(w.q0)
    np.testing.assert_allclose(oracle.integrals(mesh, ones), 1e6, rtol=1e-14)


# ------------------------------------------ P7e dense weak-form assembly
class Basis:
    def __init__(self, N):
        self.N = N
        x = W.lgl_nodes(N)
        self.x = x
        n1 = N + 1
        Vinv = np.linalg.inv(np.vander(x, n1, increasing=True))
        self.L = lambda t: np.vander(t, n1, increasing=True) @ Vinv
        k = np.arange(n1)
        self.dL = lambda t: (np.vander(t, n1, increasing=True)[:, :-1] * k[1:][None, :]) @ Vinv[1:, :]
        y, wq = np.polynomial.legendre.leggauss(2 * N + 2)
        Ly, dLy = self.L(y), self.dL(y)
        self.w = wq @ Ly
        self.K = (dLy * wq[:, None]).T @ Ly          # K[i][j] = int l_i' l_j
        M = (Ly * wq[:, None]).T @ Ly
        self.P, self.R = [], []
        for b in range(2):
            Sb = (Ly * wq[:, None]).T @ self.L((y - 1) / 2 if b == 0 else (y + 1) / 2)
            self.P.append(np.linalg.solve(M, Sb))
            self.R.append(0.5 * np.linalg.solve(M, Sb.T))


def np_point(p, q, bgr):
    """Vectorised point physics (readings R2, R5, R6)."""
    dim = p.dim
    rho, Th = q[0], q[dim + 1]
    rp, Tp = rho - bgr[0], Th - bgr[1]
    Pp = bgr[2] * np.expm1(p.gamma * np.log1p(Tp / bgr[1]))
    P = bgr[2] + Pp
    u = q[1:1 + dim] / rho
    a = np.sqrt(p.gamma * P / rho)
    return rp, Tp, Pp, u, a


def np_flux(p, q, bgr, d):
    dim = p.dim
    rp, Tp, Pp, u, a = np_point(p, q, bgr)
    F = np.empty_like(q)
    F[0] = q[1 + d]
    for j in range(dim):
        F[1 + j] = q[1 + j] * u[d] + (Pp if j == d else 0.0)
    F[dim + 1] = q[dim + 1] * u[d]
    return F


def np_rusanov(p, d, sgn, qL, bL, qR, bR):
    FL, FR = np_flux(p, qL, bL, d), np_flux(p, qR, bR, d)
    _, _, _, uL, aL = np_point(p, qL, bL)
    _, _, _, uR, aR = np_point(p, qR, bR)
    lam = np.maximum(np.abs(uL[d]) + aL, np.abs(uR[d]) + aR)
    jL, jR = qL.copy(), qR.copy()
    jL[0] -= bL[0]
    jR[0] -= bR[0]
    jL[p.dim + 1] -= bL[1]
    jR[p.dim + 1] -= bR[1]
    return 0.5 * sgn * (FL + FR) + 0.5 * lam * (jL - jR)


def dense_weak_rhs(p, level, anchor, bg, q):
    """Weak-form dGSEM assembled element by element with dense 1D stiffness
    (Gauss quadrature), lumped LGL mass, LGL face quadrature, and mortar fluxes
    projected with M^-1 S matrices built here; neighbours found geometrically."""
    B = Basis(p.order)
    dim, n1, Np, F = p.dim, p.n1, p.n_nodes, p.n_fields
    X = W.node_coords(p, level, anchor)
    bgn = W.node_background(p, bg, level, anchor)        # [E, Np, 3]
    E = len(level)
    node = np.arange(Np)
    idx = np.stack([(node // n1 ** d) % n1 for d in range(dim)])  # [dim, Np]
    conf, nonc, bnd = brute_force_faces(p, level, anchor)
    h = np.stack([((p.hi[d] - p.lo[d]) / p.root[d]) / 2.0 ** level.astype(float) for d in range(dim)], 1)
    J = np.prod(h / 2, axis=1)
    wn = np.prod(B.w[idx], axis=0)
    res = np.zeros((E, F, Np))
    # volume: + sum_d int dphi/dx_d F^d (tangential LGL quadrature)
    for e in range(E):
        for d in range(dim):
            Fd = np_flux(p, q[e], bgn[e].T, d)
            for i in range(Np):
                line = [n for n in range(Np) if all(idx[t, n] == idx[t, i] for t in range(dim) if t != d)]
                line.sort(key=lambda n: idx[d, n])
                wt = np.prod([B.w[idx[t, i]] for t in range(dim) if t != d])
                res[e, :, i] += J[e] * (2.0 / h[e, d]) * wt * (B.K[idx[d, i]] @ Fd[:, line].T)
        # source (mass-lumped)
        res[e, 1 + p.vert] += J[e] * wn * (-(q[e, 0] - bgn[e, :, 0]) * p.g)

    def face_nodes(e, f):
        d, s = f // 2, f % 2
        ns = [n for n in range(Np) if idx[d, n] == (p.order if s else 0)]
        tang = [t for t in range(dim) if t != d]
        ns.sort(key=lambda n: tuple(X[e, t, n] for t in reversed(tang)))
        return ns, tang

    def surf(e, f, ns, tang, Fn):
        d = f // 2
        Jf = np.prod([h[e, t] / 2 for t in tang])
        for k, n in enumerate(ns):
            wt = np.prod([B.w[idx[t, n]] for t in tang])
            res[e, :, n] -= Jf * wt * Fn[:, k]

    for e, f in bnd:
        ns, tang = face_nodes(e, f)
        d, sgn = f // 2, (1.0 if f % 2 else -1.0)
        qL = q[e][:, ns]
        qR = qL.copy()
        qR[1 + d] *= -1
        b = bgn[e][ns].T
        surf(e, f, ns, tang, np_rusanov(p, d, sgn, qL, b, qR, b))
    for eL, fL, eR, fR in conf:
        nL, tang = face_nodes(eL, fL)
        nR, _ = face_nodes(eR, fR)
        for t in tang:   # geometric match of the face nodes
            assert np.array_equal(X[eL, t, nL], X[eR, t, nR])
        d = fL // 2
        Fs = np_rusanov(p, d, 1.0, q[eL][:, nL], bgn[eL][nL].T, q[eR][:, nR], bgn[eR][nR].T)
        surf(eL, fL, nL, tang, Fs)
        surf(eR, fR, nR, tang, -Fs)
    nsub = 1 << (dim - 1)
    for row in nonc:
        eC, fC = row[0], row[1]
        nC, tang = face_nodes(eC, fC)
        d, sC = fC // 2, (1.0 if fC % 2 else -1.0)
        qc = q[eC][:, nC].copy()
        qc[0] -= bgn[eC][nC, 0]
        qc[dim + 1] -= bgn[eC][nC, 1]
        Fc = np.zeros((F, len(nC)))
        for b in range(nsub):
            eF, fF = row[2 + 2 * b], row[3 + 2 * b]
            nF, _ = face_nodes(eF, fF)
            # mortar position from geometry (fine face lies in the lower/upper half)
            bits = []
            for t in tang:
                mid = 0.5 * (X[eC, t, nC].min() + X[eC, t, nC].max())
                bits.append(0 if X[eF, t, nF].mean() < mid else 1)
            Pm = B.P[bits[0]] if dim == 2 else np.kron(B.P[bits[1]], B.P[bits[0]])
            Rm = B.R[bits[0]] if dim == 2 else np.kron(B.R[bits[1]], B.R[bits[0]])
            qm = qc @ Pm.T
            bF = bgn[eF][nF].T
            qm[0] += bF[0]
            qm[dim + 1] += bF[1]
            Fb = np_rusanov(p, d, sC, qm, bF, q[eF][:, nF], bF)
            surf(eF, fF, nF, tang, -Fb)
            Fc += Fb @ Rm.T
        surf(eC, fC, nC, tang, Fc)
    return res / (J[:, None, None] * wn[None, None, :])


@pytest.mark.parametrize("case", ["2d_walls", "3d_periodic_x"])
def test_dense_weak_form_assembly(case):
    if case == "2d_walls":
        p = W.Params(2, 3, (2, 2), (0.0, 0.0), (800.0, 800.0), (0, 0), 1)
        f = W.Forest(p)
        f.split((0, 0, 0, 0))
    else:
        p = W.Params(3, 2, (2, 2, 2), (0.0,) * 3, (600.0, 600.0, 600.0), (1, 0, 0), 1)
        f = W.Forest(p)
        f.split((0, 1, 0, 0))
    level, anchor = f.ordered()
    bg, q = _bubble_state(p, level, anchor, 21)
    q[:, 0] *= 1 + 0.01 * np.random.default_rng(3).uniform(-1, 1, q[:, 0].shape)
    mesh = oracle.Mesh(p, level, anchor)
    assert len(mesh.faces()[1]) > 0
    r = oracle.rhs(mesh, bg, q)
    d = dense_weak_rhs(p, level, anchor, bg, q)
    err = field_rel(r, d)
    assert err.max() < 1e-12, err


# ------------------------------------------------------------- P8 RK3
def test_rk3_zero_rhs_and_arguments():
    w = W.c1()
    mesh = oracle.Mesh(w.params, w.level, w.anchor)
    with pytest.raises(oracle.OracleError):
        oracle.rk_stage(mesh, w.bg, 3, 0.01, w.q0, w.q0)
    with pytest.raises(oracle.OracleError):
        oracle.rk_stage(mesh, w.bg, 0, 0.0, w.q0, w.q0)


def test_rk3_stability_polynomial():
    """Linearised about the exact rest state (RHS = 0), one SSP-RK3 step must
    apply 1 + z + z^2/2 + z^3/6 (z = dt J) to a small perturbation."""
    w = W.c1()
    p = w.params
    mesh = oracle.Mesh(p, w.level, w.anchor)
    bg = w.bg
    rest = W.pressure_balanced_state(p, W.node_background(p, bg, w.level, w.anchor), 0.0)
    rng = np.random.default_rng(8)
    eps = 1e-7
    y0 = eps * rest * rng.uniform(-1, 1, rest.shape)

    def Jv(v):
        s = eps * np.abs(rest).max() / max(np.abs(v).max(), 1e-300)
        return oracle.rhs(mesh, bg, rest + s * v) / s

    dt = 0.1
    y1 = Jv(y0)
    y2 = Jv(y1)
    y3 = Jv(y2)
    poly = y0 + dt * y1 + dt ** 2 / 2 * y2 + dt ** 3 / 6 * y3
    step = oracle.rk3_step(mesh, bg, dt, rest + y0) - rest
    err = np.abs(step - poly).max() / np.abs(poly - y0).max()
    assert err < 2e-3, err
    # a wrong coefficient (e.g. forward Euler) is far outside that tolerance
    wrong = y0 + dt * y1
    assert np.abs(step - wrong).max() / np.abs(poly - y0).max() > 100 * err
