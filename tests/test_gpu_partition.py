"""NEXT-4 on one GPU: a partitioned run equals the whole-mesh run bit for bit.
Each part of an SFC partition (dg_mesh_upload_part) is computed by its own
context with its halo rows filled from the other parts' outputs -- the
exchange of the multi-GPU path, emulated sequentially (one GPU here, so no
concurrently-waiting ranks) -- for the RHS and a full SSP-RK3 step, on the
2D AMR c2, the 3D AMR c4 and an N = 7 sample (k_stage_h7)."""
import numpy as np
import pytest

import workloads as W
from test_gpu_parity import Gpu

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _case(name):
    if name == "c5s":
        w = W.c5(root=(8, 8, 4))
    else:
        w = W.get(name)
    return w


class Parts:
    def __init__(self, w, n_parts):
        from paper_2404_16648_b200 import dg as D
        self.D, self.n = D, n_parts
        self.ctx, self.b, self.nl, self.halo = [], [], [], []
        lists = []
        for k in range(n_parts):
            c = D.DG(w.params)
            c.mesh_upload_part(w.level, w.anchor, n_parts, k)
            c.set_background(torch.from_numpy(np.ascontiguousarray(w.bg)).cuda())
            info = c.part_info()
            self.ctx.append(c)
            self.b.append(info["global_begin"])
            self.nl.append(info["n_local"])
            lists.append(c.part_exchange_lists())
        # halo rows of part k, in order: from each peer j (ascending) the rows j sends to k
        for k in range(n_parts):
            h = []
            for j in range(n_parts):
                sc, _, idx = lists[j]
                off = int(sc[:k].sum())
                h.extend((self.b[j] + idx[off:off + sc[k]]).tolist())
            assert len(h) == lists[k][1].sum()
            self.halo.append(np.array(h, np.int64))
        self.stride = self.ctx[0].state_layout()[3]

    def scatter(self, G):
        """Global [E, stride] device tensor -> per-part [n_local + n_halo, stride] (the exchange)."""
        out = []
        for k in range(self.n):
            rows = np.concatenate([np.arange(self.b[k], self.b[k] + self.nl[k]), self.halo[k]])
            out.append(G[torch.from_numpy(rows).cuda()].contiguous())
        return out

    def gather(self, parts, E):
        G = torch.empty((E, self.stride), dtype=torch.float64, device="cuda")
        for k in range(self.n):
            G[self.b[k]:self.b[k] + self.nl[k]] = parts[k][:self.nl[k]]
        return G


@pytest.mark.parametrize("name,n_parts", [("c2", 3), ("c4", 3), ("c5s", 4), ("c4", 7)])
def test_partitioned_rhs_and_step_bitwise(name, n_parts):
    w = _case(name)
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    q = g.dev(w.q0)
    r_glob = g.empty()
    g.ctx.rhs(q, r_glob)
    a, b = g.empty(), g.empty()
    dt = w.dt
    g.ctx.rk_stage(0, dt, q, q, a)
    g.ctx.rk_stage(1, dt, q, a, b)
    g.ctx.rk_stage(2, dt, q, b, a)
    step_glob = a
    P = Parts(w, n_parts)
    E = w.n_elem
    row = w.params.n_fields * w.params.n_nodes  # padding columns are never written (dg.h)
    qs = P.scatter(q)
    outs = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rhs(qs[k], outs[k])
    assert torch.equal(P.gather(outs, E)[:, :row], r_glob[:, :row])
    # RK3 step with the halo exchange emulated between stages
    s0 = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rk_stage(0, dt, qs[k], qs[k], s0[k])
    s0 = P.scatter(P.gather(s0, E))
    s1 = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rk_stage(1, dt, qs[k], s0[k], s1[k])
    s1 = P.scatter(P.gather(s1, E))
    s2 = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rk_stage(2, dt, qs[k], s1[k], s2[k])
    assert torch.equal(P.gather(s2, E)[:, :row], step_glob[:, :row])
    # per-part integrals add up to the whole-mesh integrals
    I = sum(P.ctx[k].integrals(s2[k]) for k in range(n_parts))
    Ig = g.ctx.integrals(step_glob)
    scale = g.ctx.integrals(step_glob.abs())
    assert np.all(np.abs(I - Ig) <= 1e-14 * scale), (I, Ig)


@pytest.mark.parametrize("name,n_parts", [("c2", 3), ("c4", 4), ("c5s", 3)])
def test_face_exchange_halo_is_enough(name, n_parts):
    """Halo rows filled with NaN except the face-node values moved by the face-trace
    exchange (dg_pack_faces on the owner, dg_unpack_faces on the receiver): the RHS and
    an RK3 step still equal the whole-mesh run bit for bit, so the kernels read nothing
    else of a remote element."""
    w = _case(name)
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    q = g.dev(w.q0)
    r_glob = g.empty()
    g.ctx.rhs(q, r_glob)
    a, b = g.empty(), g.empty()
    dt = w.dt
    g.ctx.rk_stage(0, dt, q, q, a)
    g.ctx.rk_stage(1, dt, q, a, b)
    g.ctx.rk_stage(2, dt, q, b, a)
    P = Parts(w, n_parts)
    E = w.n_elem
    row = w.params.n_fields * w.params.n_nodes
    lists = [c.part_face_lists() for c in P.ctx]
    F, Nf = w.params.n_fields, w.params.n_nodes // (w.params.order + 1)

    def exchange(arrs):
        for k in range(n_parts):  # receiver
            nl = P.nl[k]
            arrs[k][nl:] = float("nan")
            _, rc, _, rp = lists[k]
            for j in range(n_parts):
                if j == k or rc[j] == 0:
                    continue
                sc_j, _, sp_j, _ = lists[j]
                s0 = int(sc_j[:k].sum())
                pairs_s = torch.from_numpy(np.ascontiguousarray(sp_j[s0:s0 + sc_j[k]])).cuda()
                r0 = int(rc[:j].sum())
                pairs_r = torch.from_numpy(np.ascontiguousarray(rp[r0:r0 + rc[j]])).cuda()
                buf = torch.empty((int(sc_j[k]), F, Nf), dtype=torch.float64, device="cuda")
                P.ctx[j].pack_faces(len(pairs_s), pairs_s, arrs[j], buf)
                P.ctx[k].unpack_faces(len(pairs_r), pairs_r, buf, arrs[k])
        return arrs

    qs = exchange(P.scatter(q))
    outs = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rhs(qs[k], outs[k])
    assert torch.equal(P.gather(outs, E)[:, :row], r_glob[:, :row])
    s0 = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rk_stage(0, dt, qs[k], qs[k], s0[k])
    s0 = exchange(s0)
    s1 = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rk_stage(1, dt, qs[k], s0[k], s1[k])
    s1 = exchange(s1)
    s2 = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rk_stage(2, dt, qs[k], s1[k], s2[k])
    assert torch.equal(P.gather(s2, E)[:, :row], a[:, :row])


def test_viscosity_rejected_on_partitioned_mesh_in_either_order():
    """Viscosity needs the halo's gradients, which the exchange does not move: a stage on a
    partitioned context with mu > 0 must fail (DG_ERR_UNSUPPORTED), also when set_viscosity
    came BEFORE mesh_upload_part (the check used to sit in set_viscosity only)."""
    from paper_2404_16648_b200 import dg as D
    w = W.c2()
    c = D.DG(w.params)
    c.set_viscosity(1.5)
    c.mesh_upload_part(w.level, w.anchor, 2, 0)
    c.set_background(torch.from_numpy(np.ascontiguousarray(w.bg)).cuda())
    rows, F, Np, stride = c.state_layout()
    q = torch.zeros((rows, stride), dtype=torch.float64, device="cuda")
    out = torch.zeros_like(q)
    with pytest.raises(D.DGError) as ex:
        c.rk_stage(0, w.dt, q, q, out)
    assert ex.value.code == -2
    with pytest.raises(D.DGError) as ex:
        c.rhs(q, out)
    assert ex.value.code == -2
    c.close()


@pytest.mark.parametrize("name,n_parts", [("c2", 3), ("amr3d", 4), ("c5s", 3)])
def test_partitioned_vs_oracle(name, n_parts):
    """NEXT-4 against the ORACLE (not the whole-mesh GPU run): a moving state (velocity and
    Theta noise) through the partitioned contexts, halo exchanged between stages, matches the
    oracle's RHS and every SSP-RK3 stage on identical inputs at R19 (1e-12 per field)."""
    import oracle
    import sys
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from __graft_entry__ import _moving
    from test_gpu_parity import _check
    if name == "amr3d":
        from test_oracle_rhs import _bubble_state
        p, lv, an = W.random_forest(7, 3, order=4, max_level=2)
        p.hi = tuple(250.0 * r for r in p.root)
        bg, q0 = _bubble_state(p, lv, an, 7)
        w = W.Workload("amr3d", p, lv, an, bg, q0, 5e-4, "3D N=4 random forest, moving bubble state")
    else:
        w = _case(name)
        q0 = _moving(w, 11)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    P = Parts(w, n_parts)
    E = w.n_elem
    D = P.D
    row = w.params.n_fields * w.params.n_nodes
    stride = P.stride
    G = torch.zeros((E, stride), dtype=torch.float64, device="cuda")
    G[:, :row] = torch.from_numpy(np.ascontiguousarray(q0).reshape(E, row)).cuda()
    host = lambda T: T[:, :row].cpu().numpy().reshape(q0.shape)
    qs = P.scatter(G)
    outs = [torch.empty_like(x) for x in qs]
    for k in range(n_parts):
        P.ctx[k].rhs(qs[k], outs[k])
    _check(host(P.gather(outs, E)), oracle.rhs(m, w.bg, q0), what=f"{name} partitioned rhs")
    qin_h, qin = q0, qs
    for s in range(3):
        out = [torch.empty_like(x) for x in qs]
        for k in range(n_parts):
            P.ctx[k].rk_stage(s, w.dt, qs[k], qin[k], out[k])
        Gs = P.gather(out, E)
        got = host(Gs)
        _check(got, oracle.rk_stage(m, w.bg, s, w.dt, q0, qin_h), what=f"{name} partitioned stage {s}")
        qin_h, qin = got, P.scatter(Gs)


@pytest.mark.parametrize("name,n_parts", [("c2", 3), ("c4", 4), ("c5s", 3), ("c3", 3)])
def test_overlap_interior_then_boundary(name, n_parts):
    """The overlapped stage of NEXT-4 (HaloExchange.rk3_step_overlap): each part computes its
    interior elements (dg_rk_stage_elems) with the halo rows still NaN -- they read none -- then,
    after the face-trace exchange, its boundary elements; the RK3 step equals the whole-mesh
    run bit for bit (c2, c4: generic kernel; c5s: k_stage_h7; c3: k_stage_h4)."""
    from paper_2404_16648_b200.halo import HaloExchange
    w = _case(name)
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    q = g.dev(w.q0)
    a, b = g.empty(), g.empty()
    dt = w.dt
    g.ctx.rk_stage(0, dt, q, q, a)
    g.ctx.rk_stage(1, dt, q, a, b)
    g.ctx.rk_stage(2, dt, q, b, a)
    P = Parts(w, n_parts)
    E = w.n_elem
    row = w.params.n_fields * w.params.n_nodes
    lists = [c.part_face_lists() for c in P.ctx]
    F, Nf = w.params.n_fields, w.params.n_nodes // (w.params.order + 1)
    splits = []
    for k in range(n_parts):
        inner, bnd = HaloExchange(P.ctx[k], None, "cpu").split()
        splits.append((torch.from_numpy(inner).cuda(), torch.from_numpy(bnd).cuda()))
        assert len(inner) > 0 and len(bnd) > 0

    def exchange(arrs):
        for k in range(n_parts):
            _, rc, _, rp = lists[k]
            for j in range(n_parts):
                if j == k or rc[j] == 0:
                    continue
                sc_j, _, sp_j, _ = lists[j]
                s0 = int(sc_j[:k].sum())
                pairs_s = torch.from_numpy(np.ascontiguousarray(sp_j[s0:s0 + sc_j[k]])).cuda()
                r0 = int(rc[:j].sum())
                pairs_r = torch.from_numpy(np.ascontiguousarray(rp[r0:r0 + rc[j]])).cuda()
                buf = torch.empty((int(sc_j[k]), F, Nf), dtype=torch.float64, device="cuda")
                P.ctx[j].pack_faces(len(pairs_s), pairs_s, arrs[j], buf)
                P.ctx[k].unpack_faces(len(pairs_r), pairs_r, buf, arrs[k])

    qs = P.scatter(q)
    for k in range(n_parts):
        qs[k][P.nl[k]:] = float("nan")
    exchange(qs)
    cur = qs
    for s in range(3):
        outs = [torch.full_like(x, float("nan")) for x in qs]
        for k in range(n_parts):  # interior first: the halo rows of cur are NaN here ...
            halo = cur[k][P.nl[k]:].clone()
            cur[k][P.nl[k]:] = float("nan")
            P.ctx[k].rk_stage_elems(s, dt, qs[k], cur[k], outs[k], splits[k][0])
            cur[k][P.nl[k]:] = halo  # ... then the exchanged values, and the boundary elements
            P.ctx[k].rk_stage_elems(s, dt, qs[k], cur[k], outs[k], splits[k][1])
        for k in range(n_parts):
            outs[k][P.nl[k]:] = float("nan")
        exchange(outs)
        cur = outs
    assert torch.equal(P.gather(cur, E)[:, :row], a[:, :row])


@pytest.mark.parametrize("name", ["c2", "c3", "c4", "c5s"])
def test_element_list_launch(name):
    """dg_rhs_elems / dg_rk_stage_elems: two disjoint random lists give the full call's result bit
    for bit, and rows not listed are not written (all stage kernels: generic, h4, h7)."""
    w = _case(name)
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    rng = np.random.default_rng(3)
    X = w.q0.copy()
    X[:, 1:1 + w.params.dim] += X[:, :1] * rng.uniform(-0.5, 0.5, size=X[:, 1:1 + w.params.dim].shape)
    q = g.dev(X)
    perm = rng.permutation(g.E).astype(np.int32)
    L1 = torch.from_numpy(np.sort(perm[: g.E // 3])).cuda()
    L2 = torch.from_numpy(perm[g.E // 3:]).cuda()  # unsorted on purpose
    full, part = g.empty(), torch.full_like(g.empty(), 7.0)
    g.ctx.rhs(q, full)
    g.ctx.rhs_elems(q, part, L1)
    untouched = torch.ones(g.E, dtype=torch.bool, device="cuda")
    untouched[L1.long()] = False
    assert torch.all(part[untouched] == 7.0)
    g.ctx.rhs_elems(q, part, L2)
    row = w.params.n_fields * w.params.n_nodes
    assert torch.equal(part[:, :row], full[:, :row])
    s0, s1, p0, p1 = g.empty(), g.empty(), g.empty(), g.empty()
    g.ctx.rk_stage(0, w.dt, q, q, s0)
    g.ctx.rk_stage_elems(0, w.dt, q, q, p0, L1)
    g.ctx.rk_stage_elems(0, w.dt, q, q, p0, L2)
    assert torch.equal(p0[:, :row], s0[:, :row])
    g.ctx.rk_stage(1, w.dt, q, s0, s1)
    g.ctx.rk_stage_elems(1, w.dt, q, s0, p1, L2)
    g.ctx.rk_stage_elems(1, w.dt, q, s0, p1, L1)
    assert torch.equal(p1[:, :row], s1[:, :row])


def test_overlap_step_plumbing_single_part():
    """HaloExchange.rk3_step_overlap on a one-part partition (no peers: the exchange is empty, every
    element interior): the side stream, events and element-list launches give the plain RK3 step
    bit for bit."""
    from paper_2404_16648_b200 import dg as D
    from paper_2404_16648_b200.halo import HaloExchange
    w = _case("c5s")
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    q = g.dev(w.q0)
    a, b = g.empty(), g.empty()
    g.ctx.rk_stage(0, w.dt, q, q, a)
    g.ctx.rk_stage(1, w.dt, q, a, b)
    g.ctx.rk_stage(2, w.dt, q, b, a)
    c = D.DG(w.params)
    c.mesh_upload_part(w.level, w.anchor, 1, 0)
    c.set_background(torch.from_numpy(np.ascontiguousarray(w.bg)).cuda())
    hx = HaloExchange(c, None, torch.device("cuda"))
    inner, bnd = hx.split()
    assert len(bnd) == 0 and len(inner) == w.n_elem
    q2 = g.dev(w.q0)
    a2, b2 = g.empty(), g.empty()
    out = hx.rk3_step_overlap(w.dt, q2, a2, b2, torch.cuda.current_stream())
    torch.cuda.synchronize()
    row = w.params.n_fields * w.params.n_nodes
    assert torch.equal(out[:, :row], a[:, :row])
