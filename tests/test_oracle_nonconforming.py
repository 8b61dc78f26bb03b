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


# ----------------------------------------------------------------- value pins (2:1 faces)
# A continuous global polynomial state of degree <= N has exact traces on every face:
# the fine trace evaluated at a coarse node (pointwise, R41) IS the coarse value, so every
# jump vanishes and F* = F(q-).n.  Where the fluxes are polynomials of degree <= N the RHS
# is then -div F exactly at the nodes, in the pointwise mode as in the mortar
# mode.  A wrong sub-face coordinate evaluates the fine polynomial elsewhere and fails.
import pytest  # noqa: E402

from test_oracle_rhs import Poly, amr_forest, const_bg, field_rel, interior_elements, rand_poly  # noqa: E402


def _poly_case(dim, variant):
    """(mesh, bg, q, exact, rows): rows = fields whose flux is a polynomial of degree <= N."""
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=5, root=(4, 4) if dim == 2 else (3, 3, 3))
    p.g = 0.0
    rb, Tb = 1.1, 320.0
    bg = const_bg(p, rb, Tb)
    mesh = oracle.Mesh(p, level, anchor)
    X = W.node_coords(p, level, anchor)
    L = [p.hi[d] for d in range(dim)]
    rng = np.random.default_rng(21 + variant)
    N = p.order
    one = Poly({(0,) * dim: 1.0}, dim)
    if variant == 0:    # rho, Theta = background (P' = 0), v of degree N/2: all rows
        rho, Th, v = one.scale(rb), one.scale(Tb), [rand_poly(rng, dim, N // 2).scale(5.0) for _ in range(dim)]
        rows = list(range(dim + 2))
    elif variant == 1:  # rho' of degree N/2, Theta = background, v of degree N/4: all rows
        rho = one.scale(rb) + rand_poly(rng, dim, N // 2).scale(0.05)
        Th, v = one.scale(Tb), [rand_poly(rng, dim, N // 4).scale(5.0) for _ in range(dim)]
        rows = list(range(dim + 2))
    else:               # Theta' of degree N/2 (P' != 0: momentum not polynomial), rho const: mass and Theta rows
        rho, Th = one.scale(rb), one.scale(Tb) + rand_poly(rng, dim, N // 2).scale(2.0)
        v = [rand_poly(rng, dim, N // 2).scale(5.0) for _ in range(dim)]
        rows = [0, dim + 1]
    q = np.zeros((len(level), p.n_fields, p.n_nodes))
    q[:, 0] = rho(X, L)
    q[:, dim + 1] = Th(X, L)
    U = [rho * v[j] for j in range(dim)]
    for j in range(dim):
        q[:, 1 + j] = U[j](X, L)

    def div(vec):
        acc = vec[0].deriv(0, L)
        for d in range(1, dim):
            acc = acc + vec[d].deriv(d, L)
        return -acc(X, L)
    exact = np.zeros_like(q)
    exact[:, 0] = div(U)
    exact[:, dim + 1] = div([Th * v[d] for d in range(dim)])
    for j in range(dim):
        exact[:, 1 + j] = div([U[j] * v[d] for d in range(dim)])
    return p, level, anchor, mesh, bg, q, exact, rows


def _bound(p, level, bg, q, exact, sel, f):
    # rounding of sum_m D F (row sums |D| ~ 16) plus the Rusanov jump term, which multiplies
    # rounding-level trace differences by lambda/2 (2/h)/w0 (as in test_polynomial_exactness)
    x, w = oracle.lgl(p.order)
    dim = p.dim
    lam = np.sqrt(p.gamma * bg[0, 2] / q[:, 0].min()) + np.abs(q[:, 1:1 + dim] / q[:, :1]).max()
    hmin = min(p.hi[d] / p.root[d] for d in range(dim)) / 2 ** level.max()
    return 1e-13 * np.abs(exact[sel, f]).max() + 4e-15 * lam * np.abs(q[:, f]).max() * 2 / hmin / w[0]


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("variant", [0, 1, 2])
def test_pointwise_polynomial_exactness(dim, variant):
    p, level, anchor, mesh, bg, q, exact, rows = _poly_case(dim, variant)
    conf, nonc, bnd = mesh.faces()
    assert len(nonc) > 0
    sel = interior_elements(p, level, anchor)
    coarse = np.intersect1d(sel, nonc[:, 0])
    assert len(coarse) > 0
    worst = {}
    for mode in (0, 1, 2, 3):
        r = oracle.rhs(mesh, bg, q, ncmode=mode)
        worst[mode] = max(np.abs(r[sel, f] - exact[sel, f]).max() / _bound(p, level, bg, q, exact, sel, f)
                          for f in rows)
    assert worst[0] <= 1.0 and worst[1] <= 1.0, worst
    # the mirrored xi-map (mutant 2) is caught by the same bound, by orders of magnitude; mutant 3
    # (the midpoint node read from the upper sub-face at xi = -1, the same physical point) cannot
    # differ on continuous data -- the sub-face dependency test below catches it
    assert worst[2] > 1e3, worst


def _tracer_case(dim, deg_c, deg_u, seed):
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=seed, root=(4, 4) if dim == 2 else (3, 3, 3))
    mesh = oracle.Mesh(p, level, anchor)
    X = W.node_coords(p, level, anchor)
    L = [p.hi[d] for d in range(dim)]
    rng = np.random.default_rng(seed)
    Cp = rand_poly(rng, dim, deg_c)
    u = [rand_poly(rng, dim, deg_u).scale(3.0) for _ in range(dim)]
    s = np.zeros((len(level), p.n_fields, p.n_nodes))
    s[:, 0] = Cp(X, L)
    for d in range(dim):
        s[:, 1 + d] = u[d](X, L)
    acc = (Cp * u[0]).deriv(0, L)
    for d in range(1, dim):
        acc = acc + (Cp * u[d]).deriv(d, L)
    return p, level, anchor, mesh, s, -acc(X, L)


@pytest.mark.parametrize("dim", [2, 3])
def test_tracer_polynomial_exactness_both_modes(dim):
    """C and u continuous polynomials with deg C + deg u <= N: every trace is exact, so
    both 2:1 treatments give -div(C u) exactly at the nodes (R43); the two mutants fail."""
    p, level, anchor, mesh, s, exact = _tracer_case(dim, 2, 2, seed=6)
    assert len(mesh.faces()[1]) > 0
    sel = interior_elements(p, level, anchor)
    x, w = oracle.lgl(p.order)
    hmin = min(p.hi[d] / p.root[d] for d in range(dim)) / 2 ** level.max()
    umax = np.abs(s[:, 1:1 + dim]).max()
    bound = 1e-13 * np.abs(exact[sel]).max() + 4e-15 * umax * np.abs(s[:, 0]).max() * 2 / hmin / w[0]
    worst = {m: np.abs(oracle.tracer_rhs(mesh, s, ncmode=m)[sel] - exact[sel]).max() / bound for m in (0, 1, 2, 3)}
    assert worst[0] <= 1.0 and worst[1] <= 1.0, worst
    assert worst[2] > 1e3, worst


def _coarse_nodes_by_subface(p, mesh):
    """For a 2:1 face: (eC, fC, eF list, per coarse face node t the sub-face b(t) of R41)."""
    conf, nonc, bnd = mesh.faces()
    x, _ = oracle.lgl(p.order)
    row = nonc[0]
    eC, fC = int(row[0]), int(row[1])
    nsub = 2 ** (p.dim - 1)
    eF = [int(row[2 + 2 * b]) for b in range(nsub)]
    n1 = p.order + 1
    Nf = n1 ** (p.dim - 1)
    bt = []
    for t in range(Nf):
        t1, t2 = t % n1, t // n1
        bt.append(int(x[t1] > 0) + (2 * int(x[t2] > 0) if p.dim == 3 else 0))
    return eC, fC, eF, np.array(bt)


def _face_nodes(p, f):
    """Volume node index of the face nodes of local face f (R28: tangential axes ascending)."""
    n1 = p.order + 1
    d, e = f // 2, (p.order if f % 2 else 0)
    idx = []
    for t in range(n1 ** (p.dim - 1)):
        t1, t2 = t % n1, t // n1
        ijk = [0, 0, 0]
        tang = [a for a in range(p.dim) if a != d]
        ijk[d] = e
        ijk[tang[0]] = t1
        if p.dim == 3:
            ijk[tang[1]] = t2
        idx.append(ijk[0] + n1 * ijk[1] + n1 * n1 * ijk[2])
    return np.array(idx)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("which", ["euler", "tracer"])
def test_pointwise_reads_only_the_subface_containing_the_node(dim, which):
    """R41: in the pointwise mode the coarse-side value at face node t comes
    from the fine element whose sub-face contains it (x = 0 -> the lower one) and from no
    other: perturbing fine element b changes the coarse RHS exactly at the nodes with
    b(t) = b.  The mortar mode mixes all sub-faces into every node."""
    p, level, anchor = amr_forest(dim, (0,) * dim, seed=7, root=(4, 4) if dim == 2 else (3, 3, 3))
    mesh = oracle.Mesh(p, level, anchor)
    eC, fC, eF, bt = _coarse_nodes_by_subface(p, mesh)
    nodes = _face_nodes(p, fC)
    rng = np.random.default_rng(8)
    if which == "euler":
        bg = W.background_table(p)
        q = W.pressure_balanced_state(p, W.node_background(p, bg, level, anchor), 0.0)
        q[:, 1:1 + dim] = 0.01 * rng.uniform(-1, 1, size=(len(level), dim, p.n_nodes))
        run = lambda s, mode: oracle.rhs(mesh, bg, s, ncmode=mode)[eC][:, nodes]
        pert = lambda s, e: s[e, 1:1 + dim].__iadd__(0.003 * rng.uniform(-1, 1, size=(dim, p.n_nodes)))
    else:
        s0 = np.zeros((len(level), p.n_fields, p.n_nodes))
        s0[:, 0] = rng.uniform(0, 1, size=(len(level), p.n_nodes))
        s0[:, 1:1 + dim] = 0.3
        s0[:, 1 + fC // 2] = -0.5 if fC % 2 else 0.5  # inflow into the coarse element: upwind = the fine side
        q = s0
        run = lambda s, mode: oracle.tracer_rhs(mesh, s, ncmode=mode)[eC][nodes][None]
        pert = lambda s, e: s[e, 0].__iadd__(0.1 * rng.uniform(0, 1, size=p.n_nodes))
    for b, ef in enumerate(eF):
        q2 = q.copy()
        pert(q2, ef)
        for mode, expect in ((1, bt == b), (3, None)):
            # changed beyond rounding (an upwind flux still rounds differently when the
            # downwind value changes)
            changed = np.any(np.abs(run(q2, mode) - run(q, mode)) > 1e-9 * np.abs(run(q, mode)).max(), axis=0)
            if mode == 1:
                assert np.array_equal(changed, expect), (b, changed, expect)
            elif b == 0:
                # mutant 3 moves the midpoint node (x = 0) to the upper sub-face: caught here
                assert not np.array_equal(changed, bt == b)
        dm = np.abs(run(q2, 0) - run(q, 0))
        assert np.all(np.any(dm > 1e-9 * np.abs(run(q, 0)).max(), axis=0))  # mortar: every node sees sub-face b
