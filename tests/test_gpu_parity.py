"""GPU parity: libdg (sm_100a, through the C ABI) against the CPU oracle on the
same seeded inputs.  Bar (reading R19): per field
max|gpu - oracle| / max|oracle| <= 1e-12; a field whose oracle values are all
zero must be exactly zero on the GPU.  Connectivity is bit-exact."""
import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-12


def _lib():
    from paper_2404_16648_b200 import dg as D
    return D


def rel_err(a, b):
    out = []
    for f in range(a.shape[1]):
        den = np.abs(b[:, f]).max()
        num = np.abs(a[:, f] - b[:, f]).max()
        out.append(num / den if den > 0 else (0.0 if num == 0 else np.inf))
    return np.array(out)


class Gpu:
    """Device-side run of one workload through the C ABI."""

    def __init__(self, p, level, anchor, bg):
        D = _lib()
        self.D = D
        self.p = p
        self.ctx = D.DG(p)
        self.ctx.mesh_upload(level, anchor)
        self.E, self.F, self.Np, self.stride = self.ctx.state_layout()
        self.bg = torch.from_numpy(np.ascontiguousarray(bg)).cuda()
        self.ctx.set_background(self.bg)

    def dev(self, q):
        return self.D.to_device(q, self.stride)

    def host(self, t):
        torch.cuda.synchronize()
        return self.D.from_device(t, self.F, self.Np)

    def empty(self):
        return torch.zeros((self.E, self.stride), dtype=torch.float64, device="cuda")

    def rhs(self, q):
        out = self.empty()
        self.ctx.rhs(self.dev(q), out)
        return self.host(out)

    def stages(self, q0, dt, n_stages, every_step=None):
        """n_stages consecutive rk_stage calls cycling 0,1,2 (reading R31)."""
        qn = self.dev(q0)
        qin = qn
        bufs = [self.empty(), self.empty()]
        k = 0
        outs = []
        for i in range(n_stages):
            s = i % 3
            out = bufs[k]
            k ^= 1
            self.ctx.rk_stage(s, dt, qn, qin, out)
            qin = out
            if s == 2:
                qn = out.clone()
                qin = qn
                if every_step is not None:
                    outs.append(self.host(qn))
        return self.host(qin), outs


def _check(gpu, ora, tol=TOL, what=""):
    err = rel_err(gpu, ora)
    assert np.all(err <= tol), f"{what} per-field rel err {err}"
    return err


def _check_traj(gpu, ora, p, bg, dt, n_stages, hmin, what=""):
    """Multi-step trajectory parity (reading R19b): rho and Theta at
    R19 <= 1e-12; momentum at 1e-12 of its own max plus the propagation bound of
    one-ulp differences in the stored Theta (full-variable storage, R1): each
    such ulp is a pressure perturbation gamma P/Theta ulp(Theta), lifted with at
    most (2/h)/w0 per unit time, over n_stages stages of size dt."""
    err = rel_err(gpu, ora)
    dim = p.dim
    for f in (0, dim + 1):
        assert err[f] <= TOL, f"{what} field {f} rel err {err}"
    x, w = oracle.lgl(p.order)
    kappa = p.gamma * np.max(bg[:, 2] / bg[:, 1]) * np.spacing(np.max(bg[:, 1]) * 1.1)
    bound = 4.0 * n_stages * dt * (2.0 / hmin) / w[0] * kappa
    for f in range(1, dim + 1):
        d = np.abs(gpu[:, f] - ora[:, f]).max()
        assert d <= TOL * np.abs(ora[:, f]).max() + bound, f"{what} momentum {f}: |d| {d:.3e} bound {bound:.3e} rel {err}"
    return err


def _hmin(p, level):
    return min((p.hi[d] - p.lo[d]) / p.root[d] for d in range(p.dim)) / 2.0 ** int(np.max(level))


# ------------------------------------------------------------------- c1
def test_c1_rhs_and_10_steps():
    w = W.c1()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    _check(g.rhs(w.q0), oracle.rhs(m, w.bg, w.q0), what="c1 rhs")
    _, steps = g.stages(w.q0, w.dt, 30, every_step=True)
    q = w.q0
    for k in range(10):
        q = oracle.rk3_step(m, w.bg, w.dt, q)
        if k == 0:
            for f in (0, w.params.dim + 1):
                _check((steps[k] - w.q0)[:, f:f + 1], (q - w.q0)[:, f:f + 1], tol=1e-9, what="c1 increment 0")
        _check_traj(steps[k], q, w.params, w.bg, w.dt, 3 * (k + 1), _hmin(w.params, w.level), what=f"c1 step {k}")


def test_rest_state_bitwise_zero_on_gpu():
    for case in ("c1", "c2", "amr3d"):
        if case == "amr3d":
            from test_oracle_rhs import amr_forest
            p, lv, an = amr_forest(3, (1, 0, 0), seed=2)
        elif case == "c2":
            p, f = W.c2_forest()
            lv, an = f.ordered()
        else:
            w = W.c1()
            p, lv, an = w.params, w.level, w.anchor
        bg = W.background_table(p)
        g = Gpu(p, lv, an, bg)
        q = W.pressure_balanced_state(p, W.node_background(p, bg, lv, an), 0.0)
        r = g.rhs(q)
        assert np.all(r == 0.0), case
        qT, _ = g.stages(q, 0.01, 300)
        assert np.array_equal(qT, q), case   # 100 RK3 steps leave the rest state bitwise unchanged


# ------------------------------------------------------------------- c2
def test_c2_rhs_and_100_stages():
    w = W.c2()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    assert len(m.faces()[1]) > 0
    _check(g.rhs(w.q0), oracle.rhs(m, w.bg, w.q0), what="c2 rhs")
    final, steps = g.stages(w.q0, w.dt, 100, every_step=True)
    qn = w.q0
    qin = qn
    for i in range(100):
        s = i % 3
        out = oracle.rk_stage(m, w.bg, s, w.dt, qn, qin)
        qin = out
        if s == 2:
            qn = out
            _check_traj(steps[i // 3], qn, w.params, w.bg, w.dt, i + 1, _hmin(w.params, w.level),
                        what=f"c2 step {i // 3}")
    _check_traj(final, qin, w.params, w.bg, w.dt, 100, _hmin(w.params, w.level), what="c2 after 100 stages")


# ------------------------------------------------------------------- c3
def test_c3_rhs_and_10_steps():
    w = W.c3()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    _check(g.rhs(w.q0), oracle.rhs(m, w.bg, w.q0), what="c3 rhs")
    _, steps = g.stages(w.q0, w.dt, 30, every_step=True)
    q = w.q0
    for k in range(10):
        q = oracle.rk3_step(m, w.bg, w.dt, q)
        if k == 0:
            for f in (0, w.params.dim + 1):
                _check((steps[k] - w.q0)[:, f:f + 1], (q - w.q0)[:, f:f + 1], tol=1e-9, what="c3 increment 0")
        _check_traj(steps[k], q, w.params, w.bg, w.dt, 3 * (k + 1), _hmin(w.params, w.level), what=f"c3 step {k}")


# ------------------------------------------------------------------- c4
@pytest.fixture(scope="module")
def c4w():
    return W.c4()


def test_c4_rhs_and_step(c4w):
    w = c4w
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    _check(g.rhs(w.q0), oracle.rhs(m, w.bg, w.q0), what="c4 rhs")
    q1, _ = g.stages(w.q0, w.dt, 3)
    ref = oracle.rk3_step(m, w.bg, w.dt, w.q0)
    _check_traj(q1, ref, w.params, w.bg, w.dt, 3, _hmin(w.params, w.level), what="c4 step")
    for f in (0, 4):
        _check((q1 - w.q0)[:, f:f + 1], (ref - w.q0)[:, f:f + 1], tol=1e-9, what=f"c4 increment field {f}")
    # conservation of mass and Theta through the step (1e-13 relative)
    I0, I1 = g.ctx.integrals(g.dev(w.q0)), g.ctx.integrals(g.dev(q1))
    for f in (0, 4):
        assert abs(I1[f] - I0[f]) <= 1e-13 * abs(I0[f])
    np.testing.assert_allclose(I0, oracle.integrals(m, w.q0), rtol=1e-13)


def projection_maps(w, flags):
    """Harness-side maps for the refine->coarsen pass (R25): each flagged
    element is replaced in place by its 2^d children (Morton order)."""
    nch = 1 << w.params.dim
    E = w.n_elem
    is_f = np.zeros(E, bool)
    is_f[flags] = True
    size = np.where(is_f, nch, 1)
    start = np.concatenate([[0], np.cumsum(size)[:-1]]).astype(np.int32)
    E2 = int(size.sum())
    keep = np.nonzero(~is_f)[0].astype(np.int32)
    return E2, flags.astype(np.int32), start[flags].astype(np.int32), keep, start[keep].astype(np.int32)


def test_c4_projection_pass(c4w):
    w = c4w
    p = w.params
    g = Gpu(p, w.level, w.anchor, w.bg)
    flags = W.c4_projection_flags(w)
    assert len(flags) > 1000
    E2, par, ch0, keep, keep_dst = projection_maps(w, flags)
    T = lambda a: torch.from_numpy(a).cuda()
    q = g.dev(w.q0)
    fine = torch.zeros((E2, g.stride), dtype=torch.float64, device="cuda")
    g.ctx.amr_project_refine(len(par), T(par), T(ch0), q, fine)
    g.ctx.copy_elements(len(keep), T(keep), T(keep_dst), q, fine)
    back = torch.zeros_like(q)
    g.ctx.amr_project_coarsen(len(par), T(ch0), T(par), fine, back)
    g.ctx.copy_elements(len(keep), T(keep_dst), T(keep), fine, back)
    fine_h = g.D.from_device(fine, g.F, g.Np)
    back_h = g.host(back)
    ref_f = oracle.refine(3, p.order, par, ch0, w.q0, E2)
    ref_f[keep_dst] = w.q0[keep]
    _check(fine_h, ref_f, what="c4 refine")
    ref_b = oracle.coarsen(3, p.order, ch0, par, ref_f, w.n_elem)
    ref_b[keep] = ref_f[keep_dst]
    _check(back_h, ref_b, what="c4 coarsen")
    _check(back_h, w.q0, what="c4 round trip")
    # conservation through the pass (integrals on the new, unbalanced element set)
    isf = np.isin(np.arange(w.n_elem), flags)
    lv2 = np.repeat(w.level + isf, np.where(isf, 8, 1)).astype(np.int8)
    Jw_f = _quad_weights(p, lv2)
    Jw_0 = _quad_weights(p, w.level)
    for f in (0, 4):
        I0 = (Jw_0 * w.q0[:, f]).sum()
        I1 = (Jw_f * fine_h[:, f]).sum()
        assert abs(I1 - I0) <= 1e-13 * abs(I0)


def _quad_weights(p, level):
    from test_oracle_rhs import quad_weights
    return quad_weights(p, level)


# ------------------------------------------------------------------- c5 (sampled, full size)
def _neigh(m, E):
    conf, nonc, bnd = m.faces()
    nb = [[] for _ in range(E)]
    for eL, _, eR, _ in conf:
        nb[eL].append(eR)
        nb[eR].append(eL)
    return nb


def test_c5_sampled_rhs_and_step():
    """BASELINE configs[4] at full size in the bench's launch configuration;
    the oracle computes only sampled elements (and their dependency cone)."""
    w = W.c5()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    rng = np.random.default_rng(55)
    S2 = np.unique(np.concatenate([rng.choice(w.n_elem, 48, replace=False), [0, w.n_elem - 1]]))
    nb = _neigh(m, w.n_elem)
    grow = lambda S: np.unique(np.concatenate([S] + [np.array(nb[e]) for e in S]))
    S1 = grow(S2)
    S0 = grow(S1)
    r_gpu = g.rhs(w.q0)
    r_ora = oracle.rhs(m, w.bg, w.q0, elems=S2)
    _check(r_gpu[S2], r_ora[S2], what="c5 rhs (sampled)")
    # smooth, U = 0 at t = 0 (reading R26): d rho/dt and d Theta/dt vanish exactly everywhere
    assert np.all(r_gpu[:, 0] == 0.0) and np.all(r_gpu[:, 4] == 0.0)
    q1, _ = g.stages(w.q0, w.dt, 3)
    a = oracle.rk_stage(m, w.bg, 0, w.dt, w.q0, w.q0, elems=S0)
    b = oracle.rk_stage(m, w.bg, 1, w.dt, w.q0, a, elems=S1)
    c = oracle.rk_stage(m, w.bg, 2, w.dt, w.q0, b, elems=S2)
    _check_traj(q1[S2], c[S2], w.params, w.bg, w.dt, 3, _hmin(w.params, w.level), what="c5 step (sampled)")


# ------------------------------------------------------------------- random AMR, other orders
@pytest.mark.parametrize("dim,order,seed", [(2, 2, 0), (2, 3, 1), (3, 2, 2), (3, 3, 3), (2, 7, 4), (3, 5, 5), (3, 7, 6), (3, 4, 7), (3, 8, 8)])
def test_random_amr_orders(dim, order, seed):
    from test_oracle_rhs import _bubble_state
    p, lv, an = W.random_forest(seed, dim, order=order, max_level=2)
    p.hi = tuple(250.0 * r for r in p.root)
    bg, q = _bubble_state(p, lv, an, seed)
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    _check(g.rhs(q), oracle.rhs(m, bg, q), what=f"rhs dim{dim} N{order}")
    q1, _ = g.stages(q, 0.01, 3)
    _check_traj(q1, oracle.rk3_step(m, bg, 0.01, q), p, bg, 0.01, 3, _hmin(p, lv), what="step")


def test_free_stream_and_conservation_gpu():
    from test_oracle_rhs import amr_forest, const_bg, _bubble_state
    p, lv, an = amr_forest(3, (1, 1, 1), seed=1)
    p.g = 0.0
    bg = const_bg(p)
    q = np.zeros((len(lv), p.n_fields, p.n_nodes))
    q[:, 0] = 1.177
    q[:, 1:4] = (1.177 * np.array([3.0, -2.0, 1.5]))[None, :, None]
    q[:, 4] = 336.0
    g = Gpu(p, lv, an, bg)
    r = g.rhs(q)
    assert np.abs(r).max() < 1e-12 * 7000 * 2 / 62.5
    p2, lv2, an2 = amr_forest(3, (1, 1, 0), seed=5)
    bg2, q2 = _bubble_state(p2, lv2, an2, 6)
    g2 = Gpu(p2, lv2, an2, bg2)
    out = g2.empty()
    g2.ctx.rhs(g2.dev(q2), out)
    I = g2.ctx.integrals(out)
    absI = g2.ctx.integrals(out.abs())
    for f in (0, 4):
        assert abs(I[f]) <= 1e-13 * absI[f]


# ------------------------------------------------------------------- ABI behaviour
def test_host_variants_match_device_path():
    w = W.c3()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    r_dev = g.rhs(w.q0)
    qh = torch.from_numpy(np.ascontiguousarray(w.q0)).pin_memory()
    rh = torch.zeros_like(qh).pin_memory()
    g.ctx.rhs_host(qh, rh)
    assert np.array_equal(rh.numpy(), r_dev)
    q2, _ = g.stages(w.q0, w.dt, 6)
    g.ctx.rk3_step_host(w.dt, 2, qh)
    assert np.array_equal(qh.numpy(), q2)


def test_argument_errors():
    D = _lib()
    w = W.c1()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    a, b = g.dev(w.q0), g.empty()
    for bad in [lambda: g.ctx.rk_stage(3, 0.01, a, a, b), lambda: g.ctx.rk_stage(0, 0.0, a, a, b),
                lambda: g.ctx.rk_stage(0, float("nan"), a, a, b), lambda: g.ctx.rk_stage(1, 0.01, a, a, b),
                lambda: g.ctx.rk_stage(0, 0.01, a, a, a), lambda: g.ctx.rhs(a, a)]:
        with pytest.raises(D.DGError) as ex:
            bad()
        assert ex.value.code == -1
    with pytest.raises(D.DGError) as ex:
        g.ctx.set_background(g.bg[:-1])
    assert ex.value.code == -5
    n0 = g.ctx.launch_count()
    g.ctx.rhs(a, b)
    assert g.ctx.launch_count() == n0 + 1


# ------------------------------------------------------------------- projection at other dims / orders
@pytest.mark.parametrize("dim,order,seed", [(2, 1, 0), (2, 4, 1), (2, 7, 2), (3, 2, 3), (3, 5, 4), (3, 7, 5), (3, 8, 6)])
def test_projection_orders(dim, order, seed):
    """refine -> coarsen through the C ABI vs the oracle's Kronecker loops, all
    leaves of a small uniform mesh flagged (R16); the round trip is the identity
    and mass / Theta integrals are conserved on the refined element set."""
    root = (3, 2) if dim == 2 else (2, 2, 1)
    p = W.Params(dim, order, root, (0.0,) * dim, tuple(250.0 * r for r in root), (0,) * dim, 1)
    lv, an = W.uniform_morton(p)
    from test_oracle_rhs import _bubble_state
    bg, q0 = _bubble_state(p, lv, an, seed)
    g = Gpu(p, lv, an, bg)
    E = len(lv)
    nch = 1 << dim
    par = np.arange(E, dtype=np.int32)
    ch0 = (nch * par).astype(np.int32)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.int32)).cuda()
    q = g.dev(q0)
    fine = torch.zeros((E * nch, g.stride), dtype=torch.float64, device="cuda")
    back = torch.zeros_like(q)
    g.ctx.amr_project_refine(E, T(par), T(ch0), q, fine)
    g.ctx.amr_project_coarsen(E, T(ch0), T(par), fine, back)
    fine_h = g.D.from_device(fine, g.F, g.Np)
    back_h = g.host(back)
    ref_f = oracle.refine(dim, order, par, ch0, q0, E * nch)
    _check(fine_h, ref_f, what=f"refine d{dim} N{order}")
    _check(back_h, oracle.coarsen(dim, order, ch0, par, ref_f, E), what=f"coarsen d{dim} N{order}")
    _check(back_h, q0, what=f"round trip d{dim} N{order}")
    Jw0 = _quad_weights(p, lv)
    Jw1 = _quad_weights(p, np.repeat(lv + 1, nch).astype(np.int8))
    for f in (0, dim + 1):
        I0, I1 = (Jw0 * q0[:, f]).sum(), (Jw1 * fine_h[:, f]).sum()
        assert abs(I1 - I0) <= 1e-13 * abs(I0)


def test_copy_elements_permutation():
    w = W.c1()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    rng = np.random.default_rng(9)
    perm = rng.permutation(w.n_elem).astype(np.int32)
    T = lambda x: torch.from_numpy(np.ascontiguousarray(x, np.int32)).cuda()
    out = g.empty()
    g.ctx.copy_elements(w.n_elem, T(np.arange(w.n_elem, dtype=np.int32)), T(perm), g.dev(w.q0), out)
    got = g.host(out)
    assert np.array_equal(got[perm], w.q0)


# ------------------------------------------------------------------- degenerate meshes
@pytest.mark.parametrize("dim,order,per", [(3, 7, (1, 1, 1)), (3, 4, (1, 1, 1)), (3, 7, (1, 1, 0)),
                                           (2, 4, (1, 0)), (2, 7, (1, 1))])
def test_single_element_periodic(dim, order, per):
    """One element whose periodic faces are conforming faces with itself (the neighbour
    trace is its own opposite face), through the same fused kernels as the configs
    (3D N = 7 -> k_stage_h7): RHS and one RK3 step against the oracle."""
    from test_oracle_rhs import _bubble_state
    root = (1,) * dim
    p = W.Params(dim, order, root, (0.0,) * dim, (250.0,) * dim, per, 0)
    lv, an = W.uniform_morton(p)
    bg, q = _bubble_state(p, lv, an, 11)
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    _check(g.rhs(q), oracle.rhs(m, bg, q), what=f"rhs single element d{dim} N{order}")
    q1, _ = g.stages(q, 0.01, 3)
    _check_traj(q1, oracle.rk3_step(m, bg, 0.01, q), p, bg, 0.01, 3, _hmin(p, lv), what="single element step")


def test_zero_size_transfers_are_noops():
    w = W.c1()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    q = g.dev(w.q0)
    out = g.empty()
    e = torch.zeros(0, dtype=torch.int32, device="cuda")
    n0 = g.ctx.launch_count()
    g.ctx.amr_project_refine(0, e, e, q, out)
    g.ctx.amr_project_coarsen(0, e, e, q, out)
    g.ctx.copy_elements(0, e, e, q, out)
    torch.cuda.synchronize()
    assert g.ctx.launch_count() == n0 and torch.count_nonzero(out).item() == 0
