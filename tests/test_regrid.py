"""NEXT-1: the regrid plan -- oracle pins from the paper / SPEC
examples and invariants, then libdg's host planner (C ABI, no GPU needed)
bit-exact against the oracle on seeded random forests (R37-R39)."""
import numpy as np
import pytest

import oracle
import oracle.regrid as OR
import workloads as W
from paper_2404_16648_b200 import dg as D


def _uniform(dim, root, max_level, periodic=None, order=2):
    per = periodic or (0,) * dim
    p = W.Params(dim, order, tuple(root), (0.0,) * dim, tuple(100.0 * r for r in root), per, max_level)
    lv, an = W.uniform_morton(p)
    return p, lv, an


def _idx(an, cell):
    return [i for i in range(len(an)) if tuple(an[i]) == tuple(cell)][0]


def _leafset(pl):
    return {(int(l),) + tuple(int(x) for x in a) for l, a in zip(pl["level"], pl["anchor"])}


def _check_invariants(p, lv, an, pl):
    dim = p.dim
    # tiling: volumes at max_level sum to the domain
    vol = sum(1 << (dim * (p.max_level - int(l))) for l in pl["level"])
    dom = 1
    for d in range(dim):
        dom *= p.root[d] << p.max_level
    assert vol == dom
    # the oracle's own mesh build checks overlap, gaps and 2:1 balance (raises otherwise)
    oracle.Mesh(p, pl["level"], pl["anchor"])
    # every new leaf is covered exactly once by the maps; at most one level of change
    En, nch = len(pl["level"]), 1 << dim
    cover = np.zeros(En, int)
    cover[pl["copy_dst"]] += 1
    for c0 in pl["refine_child0"]:
        cover[c0:c0 + nch] += 1
    cover[pl["coarsen_parent"]] += 1
    assert np.all(cover == 1)
    for s, d in zip(pl["copy_src"], pl["copy_dst"]):
        assert lv[s] == pl["level"][d] and tuple(an[s]) == tuple(pl["anchor"][d])
    for s, c0 in zip(pl["refine_parent"], pl["refine_child0"]):
        assert pl["level"][c0] == lv[s] + 1 and tuple(pl["anchor"][c0]) == tuple(2 * an[s])
    for c0, d in zip(pl["coarsen_child0"], pl["coarsen_parent"]):
        assert pl["level"][d] == lv[c0] - 1 and tuple(2 * pl["anchor"][d]) == tuple(an[c0])


# ----------------------------------------------------------------- oracle pins
@pytest.mark.parametrize("dim", [2, 3])
def test_one_cell_buffer_two_is_the_centred_block(dim):
    """one interior cell tagged, B = 2 -> the 5x5(x5) block around it is refined."""
    p, lv, an = _uniform(dim, (8,) * dim, 1)
    eta = np.zeros(len(lv))
    centre = (4,) * dim
    eta[_idx(an, centre)] = 1.0
    pl = OR.plan(p, lv, an, eta, 0.5, -1.0, 2)
    got = {tuple(an[i]) for i in pl["refine_parent"]}
    want = {c for c in np.ndindex(*(8,) * dim) if all(abs(c[d] - 4) <= 2 for d in range(dim))}
    assert got == want
    _check_invariants(p, lv, an, pl)


def test_buffer_clipped_at_walls_and_wrapped_on_periodic_axes():
    p, lv, an = _uniform(2, (8, 8), 1)
    eta = np.zeros(len(lv))
    eta[_idx(an, (0, 0))] = 1.0
    got = {tuple(an[i]) for i in OR.plan(p, lv, an, eta, 0.5, -1.0, 2)["refine_parent"]}
    assert got == {(i, j) for i in range(3) for j in range(3)}
    p, lv, an = _uniform(2, (8, 8), 1, periodic=(1, 0))
    got = {tuple(an[i]) for i in OR.plan(p, lv, an, eta, 0.5, -1.0, 1)["refine_parent"]}
    assert got == {(i % 8, j) for i in (-1, 0, 1) for j in (0, 1)}


def test_refine_one_cell_of_two_by_two():
    """refining one cell of a 2x2 patch gives 7 leaves and 2 nonconforming faces."""
    p, lv, an = _uniform(2, (2, 2), 1)
    eta = np.zeros(4)
    eta[_idx(an, (0, 0))] = 1.0
    pl = OR.plan(p, lv, an, eta, 0.5, -1.0, 0)
    assert len(pl["level"]) == 7
    assert oracle.Mesh(p, pl["level"], pl["anchor"]).faces()[1].shape[0] == 2
    _check_invariants(p, lv, an, pl)


def test_balance_ripple_refines_the_coarse_neighbour_once():
    """refining a cell next to a neighbour one level coarser refines that neighbour once."""
    p = W.Params(2, 2, (2, 1), (0.0, 0.0), (200.0, 100.0), (0, 0), 2)
    f = W.Forest(p)
    f.split((0, 0, 0, 0))
    lv, an = f.ordered()
    eta = np.zeros(len(lv))
    eta[[i for i in range(len(lv)) if lv[i] == 1 and tuple(an[i]) == (1, 0)][0]] = 1.0
    pl = OR.plan(p, lv, an, eta, 0.5, -1.0, 0)
    leaves = _leafset(pl)
    assert (0, 1, 0) not in leaves and all((1, 2 + i, j) in leaves for i in (0, 1) for j in (0, 1))
    assert {(2, 2 + i, j) for i in (0, 1) for j in (0, 1)} <= leaves
    _check_invariants(p, lv, an, pl)


def test_refine_then_coarsen_round_trip_and_identity():
    """refine a family and coarsen it back -> identical leaves;
    no tags -> unchanged mesh (identity copy)."""
    p, lv, an = _uniform(2, (4, 4), 1)
    eta = np.zeros(len(lv))
    pl0 = OR.plan(p, lv, an, eta, 0.5, -1.0, 2)
    assert np.array_equal(pl0["level"], lv) and np.array_equal(pl0["anchor"], an)
    assert np.array_equal(pl0["copy_src"], np.arange(len(lv))) and len(pl0["refine_parent"]) == 0
    eta[_idx(an, (1, 1))] = 1.0
    pl1 = OR.plan(p, lv, an, eta, 0.5, -1.0, 0)
    eta1 = np.zeros(len(pl1["level"]))
    pl2 = OR.plan(p, pl1["level"], pl1["anchor"], eta1, 0.5, 0.1, 0)
    assert np.array_equal(pl2["level"], lv) and np.array_equal(pl2["anchor"], an)
    assert len(pl2["coarsen_parent"]) == 1


def test_saturation_and_coarsen_blocked_by_balance():
    """every cell above threshold -> every leaf below max_level refined.
    S:141: a family next to a leaf two levels finer (after the merge) is kept."""
    p, lv, an = _uniform(2, (2, 2), 2)
    pl = OR.plan(p, lv, an, np.ones(4), 0.5, -1.0, 0)
    assert len(pl["level"]) == 16 and set(pl["level"]) == {1}
    # level-1 everywhere, then refine one level-1 leaf to level 2; the level-1 family
    # containing it cannot coarsen, a neighbouring family whose parent would touch a
    # level-2 leaf must not coarsen either
    p2 = W.Params(2, 2, (2, 1), (0.0, 0.0), (200.0, 100.0), (0, 0), 2)
    f = W.Forest(p2)
    f.split((0, 0, 0, 0))
    f.split((0, 1, 0, 0))
    f.split((1, 2, 0, 0))  # level-2 leaves at the left edge of the right root cell
    f.balance()
    lv2, an2 = f.ordered()
    eta = np.where(lv2 == 2, 0.2, 0.0)  # level-2 leaves stay (above coarsen_below, below refine_above)
    pl2 = OR.plan(p2, lv2, an2, eta, 0.5, 0.1, 0)
    leaves = _leafset(pl2)
    assert (0, 0, 0) not in leaves  # left family would touch level-2 leaves -> kept at level 1
    assert {(1, 0, 0), (1, 1, 0), (1, 0, 1), (1, 1, 1)} <= leaves
    _check_invariants(p2, lv2, an2, pl2)


@pytest.mark.parametrize("seed", range(8))
def test_random_forest_invariants(seed):
    dim = 2 + seed % 2
    p, lv, an = W.random_forest(seed, dim, order=2, max_level=3 if dim == 2 else 2, frac=0.3)
    rng = np.random.default_rng(500 + seed)
    eta = rng.random(len(lv))
    pl = OR.plan(p, lv, an, eta, 0.9, 0.5, seed % 3)
    _check_invariants(p, lv, an, pl)


def _bump_eta(p, lv, an, rng):
    """Smooth indicator: a Gaussian bump of the element centres (whole regions fall
    below the coarsening threshold, so families merge) plus a little noise."""
    cen = np.empty((len(lv), p.dim))
    for d in range(p.dim):
        h = (p.hi[d] - p.lo[d]) / p.root[d] / (2.0 ** lv.astype(np.float64))
        cen[:, d] = p.lo[d] + (an[:, d] + 0.5) * h
    c = np.array([rng.uniform(p.lo[d], p.hi[d]) for d in range(p.dim)])
    L = max(p.hi[d] - p.lo[d] for d in range(p.dim))
    r2 = ((cen - c) ** 2).sum(axis=1) / (0.25 * L) ** 2
    return np.exp(-r2) + 0.02 * rng.random(len(lv))


# ------------------------------------------------------ libdg planner vs oracle
@pytest.mark.parametrize("seed", range(16))
def test_libdg_plan_matches_oracle(seed):
    dim = 2 + seed % 2
    p, lv, an = W.random_forest(seed, dim, order=2, max_level=3 if dim == 2 else 2, frac=0.35)
    rng = np.random.default_rng(700 + seed)
    if seed % 4 < 2:
        eta = _bump_eta(p, lv, an, rng)
        thr_r, thr_c, B = 0.6, 0.3, int(rng.integers(0, 3))
    else:
        eta = rng.random(len(lv))
        thr_r, thr_c, B = 0.8 + 0.15 * rng.random(), 0.6 * rng.random(), int(rng.integers(0, 3))
    ctx = D.DG(p)
    ctx.mesh_build(lv, an)
    got = ctx.regrid_plan(eta, thr_r, thr_c, B)
    want = OR.plan(p, lv, an, eta, thr_r, thr_c, B)
    for k in want:
        assert np.array_equal(got[k], want[k]), k


def test_libdg_plan_repeated_regrids_match_oracle():
    """A sequence of plans (each plan's output is the next input) stays bit-exact."""
    p, lv, an = _uniform(2, (8, 8), 2, periodic=(1, 1))
    rng = np.random.default_rng(9)
    n_coarsen = 0
    for it in range(6):
        eta = _bump_eta(p, lv, an, rng) * 2.0
        ctx = D.DG(p)
        ctx.mesh_build(lv, an)
        got = ctx.regrid_plan(eta, 1.5, 0.7, 1)
        want = OR.plan(p, lv, an, eta, 1.5, 0.7, 1)
        for k in want:
            assert np.array_equal(got[k], want[k]), (it, k)
        n_coarsen += len(want["coarsen_parent"])
        lv, an = want["level"], want["anchor"]
    assert n_coarsen > 0


def test_libdg_plan_argument_errors():
    p, lv, an = _uniform(2, (4, 4), 1)
    ctx = D.DG(p)
    with pytest.raises(D.DGError):
        ctx.regrid_plan(np.zeros(len(lv)), 0.5, 0.1, 0)  # no mesh yet
    ctx.mesh_build(lv, an)
    with pytest.raises(D.DGError):
        ctx.regrid_plan(np.zeros(len(lv)), 0.5, 0.1, -1)
    with pytest.raises(D.DGError):
        ctx.regrid_plan(np.zeros(len(lv)), float("nan"), 0.1, 0)
    # siblings not consecutive (non-Morton upload order) -> rejected when a family would merge
    p2, lv2, an2 = _uniform(2, (2, 2), 1)
    pl = OR.plan(p2, lv2, an2, np.array([1.0, 0, 0, 0]), 0.5, -1.0, 0)
    perm = np.arange(len(pl["level"]))[::-1].copy()
    ctx2 = D.DG(p2)
    ctx2.mesh_build(pl["level"][perm], pl["anchor"][perm])
    with pytest.raises(D.DGError):
        ctx2.regrid_plan(np.zeros(len(perm)), 0.5, 0.1, 0)
