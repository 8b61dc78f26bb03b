"""NEXT-4 host logic: the SFC partition and halo lists of libdg
(dg_mesh_build_part, no GPU) against an independent derivation from the
oracle's face lists, and the halo exchange protocol (paper_2404_16648_b200.halo)
on gloo ranks with CPU tensors (world size 2 and 3)."""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads as W
from paper_2404_16648_b200 import dg as D

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _adjacency(p, lv, an):
    """Face adjacency from the oracle's canonical face lists (conforming pairs and
    coarse <-> fine across 2:1 faces)."""
    conf, nonconf, _ = oracle.Mesh(p, lv, an).faces()
    adj = [set() for _ in range(len(lv))]
    for r in conf:
        adj[r[0]].add(int(r[2]))
        adj[r[2]].add(int(r[0]))
    for r in nonconf:
        for eF in r[2::2]:
            adj[r[0]].add(int(eF))
            adj[eF].add(int(r[0]))
    return adj


def _cuts(lv, an, n_parts):
    """Family-aligned SFC cuts (R40 + SURVEY 8(e)): n k / n_parts moved forward while the leaf
    before the cut and the leaf after it are siblings (same level >= 1, same parent)."""
    n = len(lv)
    par = [tuple(int(x) >> 1 for x in a) for a in np.asarray(an).reshape(n, -1)]
    bnd = [0]
    for k in range(1, n_parts):
        g = max(n * k // n_parts, bnd[-1])
        while 0 < g < n and lv[g] == lv[g - 1] and lv[g] > 0 and par[g] == par[g - 1]:
            g += 1
        bnd.append(g)
    return bnd + [n]


def _expected(adj, n, n_parts, part, lv=None, an=None):
    bnd = _cuts(lv, an, n_parts) if lv is not None else [n * k // n_parts for k in range(n_parts + 1)]
    owner = lambda g: max(k for k in range(n_parts) if bnd[k] <= g)  # noqa: E731
    b, e = bnd[part], bnd[part + 1]
    halo = [sorted({h for g in range(b, e) for h in adj[g] if owner(h) == k}) for k in range(n_parts)]
    send = [sorted({g for g in range(b, e) if any(owner(h) == k for h in adj[g])}) if k != part else []
            for k in range(n_parts)]
    halo[part] = []
    return b, e, halo, send


CASES = [("c2", None), ("forest2", 2), ("forest3", 3), ("forest3b", 5)]


def _mesh(name):
    if name == "c2":
        w = W.c2()
        return w.params, w.level, w.anchor
    seed = {"forest2": 2, "forest3": 1, "forest3b": 5}[name]
    dim = 2 if name == "forest2" else 3
    return W.random_forest(seed, dim, order=2, max_level=2, frac=0.35)


@pytest.mark.parametrize("name", [c[0] for c in CASES])
@pytest.mark.parametrize("n_parts", [2, 3, 4])
def test_partition_lists_match_face_adjacency(name, n_parts):
    p, lv, an = _mesh(name)
    adj = _adjacency(p, lv, an)
    for part in range(n_parts):
        ctx = D.DG(p)
        ctx.mesh_build_part(lv, an, n_parts, part)
        info = ctx.part_info()
        b, e, halo, send = _expected(adj, len(lv), n_parts, part, lv, an)
        assert info["global_begin"] == b and info["n_local"] == e - b
        assert info["n_halo"] == sum(len(h) for h in halo)
        sc, rc, idx = ctx.part_exchange_lists()
        assert rc.tolist() == [len(h) for h in halo]
        assert sc.tolist() == [len(s) for s in send]
        assert idx.tolist() == [g - b for k in range(n_parts) for g in send[k]]
        assert ctx.state_layout()[0] == info["n_local"] + info["n_halo"]


def test_partition_errors():
    p, lv, an = _mesh("forest2")
    ctx = D.DG(p)
    with pytest.raises(D.DGError):
        ctx.mesh_build_part(lv, an, 2, 2)
    with pytest.raises(D.DGError):
        ctx.mesh_build_part(lv, an, len(lv) + 1, 0)  # empty part
    ctx.mesh_build_part(lv, an, 2, 0)
    with pytest.raises(D.DGError):
        ctx.regrid_plan(np.zeros(len(lv)), 1.0, 0.0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, name, out, mode="rows"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_16648_b200.halo import HaloExchange
    p, lv, an = _mesh(name)
    ctx = D.DG(p)
    ctx.mesh_build_part(lv, an, world, rank)
    info = ctx.part_info()
    rows, _, _, stride = ctx.state_layout()
    # global state: a unique value per (element, column)
    qg = np.arange(len(lv), dtype=np.float64)[:, None] * 1000.0 + np.arange(stride)[None, :]
    b, nl = info["global_begin"], info["n_local"]
    q = torch.full((rows, stride), -1.0, dtype=torch.float64)
    q[:nl] = torch.from_numpy(qg[b:b + nl])
    hx = HaloExchange(ctx, dist, "cpu", mode=mode)
    hx.exchange(q)
    out[rank] = q.numpy().copy()
    # whole-mesh sum of per-rank vectors: identical on every rank (rank-order Neumaier)
    out[("sum", rank)] = hx.allsum(np.array([1e16 * (rank + 1), 1.0 + rank, -0.5 * rank]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,name", [(2, "forest3"), (3, "c2")])
def test_halo_exchange_gloo(world, name):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, out, "rows"), nprocs=world, join=True)
    p, lv, an = _mesh(name)
    adj = _adjacency(p, lv, an)
    for rank in range(world):
        b, e, halo, _ = _expected(adj, len(lv), world, rank, lv, an)
        q = out[rank]
        glob = list(range(b, e)) + [h for k in range(world) for h in halo[k]]
        assert q.shape[0] == len(glob)
        assert np.array_equal(q[:, 0], np.array(glob, dtype=np.float64) * 1000.0)
        assert np.array_equal(q[:, 1] - q[:, 0], np.ones(len(glob)))
    sums = [out[("sum", r)] for r in range(world)]
    exact = np.array([1e16 * world * (world + 1) / 2, sum(1.0 + r for r in range(world)),
                      sum(-0.5 * r for r in range(world))])
    for x in sums:
        assert np.array_equal(x, sums[0]) and np.array_equal(x, exact)


@pytest.mark.parametrize("world,name", [(2, "forest3"), (3, "c2")])
def test_face_exchange_gloo(world, name):
    """Face-trace mode: every face node of a halo element that touches this part arrives;
    the rest of the halo row is left untouched (-1)."""
    from paper_2404_16648_b200.halo import face_nodes
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), name, out, "faces"), nprocs=world, join=True)
    p, lv, an = _mesh(name)
    adj = _adjacency(p, lv, an)
    n1 = p.order + 1
    for rank in range(world):
        b, e, halo, _ = _expected(adj, len(lv), world, rank, lv, an)
        q = out[rank]
        ctx = D.DG(p)
        ctx.mesh_build_part(lv, an, world, rank)
        _, _, _, rp = ctx.part_face_lists()
        glob = list(range(b, e)) + [h for k in range(world) for h in halo[k]]
        got = set()
        for row, face in rp:
            g = glob[row]
            for f in range(p.n_fields):
                nodes = f * p.n_nodes + face_nodes(p.dim, n1, face)
                assert np.array_equal(q[row, nodes], g * 1000.0 + nodes)
            got.add((row, face))
        # every halo element has at least one delivered face, and local rows are intact
        assert {r for r, _ in got} == set(range(e - b, len(glob)))
        assert np.array_equal(q[: e - b, 0], np.arange(b, e) * 1000.0)


def test_cuts_never_split_a_sibling_family():
    """a part boundary never falls between two sibling leaves (same level >= 1, same
    parent), and the libdg cuts equal the independent rule; on these forests some cuts had to move
    off the plain SFC position n k / n_parts."""
    moved = 0
    for name in [c[0] for c in CASES]:
        p, lv, an = _mesh(name)
        n = len(lv)
        par = [tuple(int(x) >> 1 for x in a) for a in np.asarray(an).reshape(n, -1)]
        for n_parts in (2, 3, 4, 5):
            cuts = []
            for part in range(n_parts):
                ctx = D.DG(p)
                ctx.mesh_build_part(lv, an, n_parts, part)
                cuts.append(ctx.part_info()["global_begin"])
            assert cuts == _cuts(lv, an, n_parts)[:-1]
            for g in cuts[1:]:
                assert not (lv[g] == lv[g - 1] and lv[g] > 0 and par[g] == par[g - 1]), (name, n_parts, g)
            moved += sum(g != n * k // n_parts for k, g in enumerate(cuts))
    assert moved > 0


@pytest.mark.parametrize("name", [c[0] for c in CASES])
@pytest.mark.parametrize("n_parts", [2, 3])
@pytest.mark.parametrize("mode", ["faces", "rows"])
def test_interior_boundary_split(name, n_parts, mode):
    """HaloExchange.split (the overlap of NEXT-4): boundary = own elements with a face neighbour
    owned by another part (independently from the oracle's face adjacency), interior = the rest."""
    from paper_2404_16648_b200.halo import HaloExchange
    p, lv, an = _mesh(name)
    adj = _adjacency(p, lv, an)
    bnd_all = _cuts(lv, an, n_parts)
    owner = lambda g: max(k for k in range(n_parts) if bnd_all[k] <= g)  # noqa: E731
    for part in range(n_parts):
        ctx = D.DG(p)
        ctx.mesh_build_part(lv, an, n_parts, part)
        b, e = bnd_all[part], bnd_all[part + 1]
        inner, bnd = HaloExchange(ctx, None, "cpu", mode).split()
        want = [g - b for g in range(b, e) if any(owner(h) != part for h in adj[g])]
        assert bnd.tolist() == want
        assert sorted(inner.tolist() + bnd.tolist()) == list(range(e - b))
