"""CPU-side tests of the C ABI (no compute calls without a GPU): the library
loads and exports every symbol include/dg.h declares, validates arguments, and
its host connectivity build is bit-exact against the oracle's face lists
(R29) on the configs and on seeded random balanced forests."""
import os
import re

import numpy as np
import pytest

import oracle
import workloads as W
from paper_2404_16648_b200 import dg as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "dg.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(dg_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_header_symbol():
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(D.lib, s), s
    assert sorted(D.SYMBOLS) == syms


def test_create_validation():
    p = W.c1().params
    for bad in [dict(dim=4), dict(order=0), dict(order=9), dict(max_level=9), dict(gamma=1.0)]:
        q = W.Params(**{**p.__dict__, **bad})
        with pytest.raises(D.DGError) as ex:
            D.DG(q)
        assert ex.value.code in (-1, -2)
    q = W.Params(**{**p.__dict__, "hi": (0.0, 1000.0)})
    with pytest.raises(D.DGError):
        D.DG(q)


def test_calls_without_mesh_fail_cleanly():
    ctx = D.DG(W.c1().params)
    with pytest.raises(D.DGError) as ex:
        ctx.mesh_face_counts()
    assert ex.value.code == -3
    with pytest.raises(D.DGError) as ex:
        ctx.rhs(1, 2)
    assert ex.value.code == -3
    e, f, n, s = ctx.state_layout()
    assert (e, f, n) == (0, 4, 25) and s % 16 == 0 and s >= f * n


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4"])
def test_config_connectivity_bit_exact(name):
    if name == "c4":
        p, f = W.c4_forest(np.random.default_rng(4))
        lv, an = f.ordered()
    elif name == "c2":
        p, f = W.c2_forest()
        lv, an = f.ordered()
    else:
        w = W.get(name)
        p, lv, an = w.params, w.level, w.anchor
    ctx = D.DG(p)
    ctx.mesh_build(lv, an)
    mine = ctx.mesh_faces()
    ref = oracle.Mesh(p, lv, an).faces()
    for a, b in zip(mine, ref):
        assert a.dtype == b.dtype and np.array_equal(a, b)
    assert ctx.state_layout()[0] == len(lv)


def test_c5_connectivity_counts():
    p = W.Params(3, 7, (64, 64, 32), (0.0,) * 3, (1e4, 1e4, 5e3), (1, 1, 0), 0)
    lv, an = W.uniform_morton(p)
    ctx = D.DG(p)
    ctx.mesh_build(lv, an)
    nc, nn, nb = ctx.mesh_face_counts()
    assert (nc, nn, nb) == (64 * 64 * 32 * 3 - 64 * 64, 0, 2 * 64 * 64)


@pytest.mark.parametrize("seed", range(25))
@pytest.mark.parametrize("dim", [2, 3])
def test_random_forest_bit_exact(seed, dim):
    p, lv, an = W.random_forest(seed, dim, max_level=3 if dim == 2 else 2)
    ctx = D.DG(p)
    ctx.mesh_build(lv, an)
    for a, b in zip(ctx.mesh_faces(), oracle.Mesh(p, lv, an).faces()):
        assert np.array_equal(a, b)


def test_mesh_errors_match_oracle():
    p = W.Params(2, 2, (3, 1), (0.0, 0.0), (3.0, 1.0), (0, 0), 2)
    f = W.Forest(p)
    f.split((0, 1, 0, 0))
    f.split((1, 2, 0, 0))
    lv, an = f.ordered()
    ctx = D.DG(p)
    with pytest.raises(D.DGError) as ex:
        ctx.mesh_build(lv, an)
    assert ex.value.code == -4
    with pytest.raises(D.DGError) as ex:     # overlap
        ctx.mesh_build(np.array([0, 0, 0, 1], np.int8), np.array([[0, 0], [1, 0], [2, 0], [0, 0]], np.int32))
    assert ex.value.code == -3
    with pytest.raises(D.DGError) as ex:     # gap
        ctx.mesh_build(np.array([0, 0], np.int8), np.array([[0, 0], [1, 0]], np.int32))
    assert ex.value.code == -3
    with pytest.raises(D.DGError) as ex:     # out of range
        ctx.mesh_build(np.array([0, 0, 0], np.int8), np.array([[0, 0], [1, 0], [3, 0]], np.int32))
    assert ex.value.code == -3
    with pytest.raises(D.DGError) as ex:     # level beyond max_level
        ctx.mesh_build(np.array([3], np.int8), np.array([[0, 0]], np.int32))
    assert ex.value.code == -3


def test_empty_leaf_list_rejected():
    """An empty leaf list cannot cover the root grid: rejected like a gap (oracle: ARG)."""
    p = W.Params(2, 3, (1, 1), (0.0, 0.0), (250.0, 250.0), (1, 0), 0)
    ctx = D.DG(p)
    with pytest.raises(D.DGError) as ex:
        ctx.mesh_build(np.zeros(0, np.int8), np.zeros((0, 2), np.int32))
    assert ex.value.code in (-1, -3)


@pytest.mark.parametrize("dim,per", [(3, (1, 1, 1)), (2, (1, 0))])
def test_single_element_self_neighbour_lists(dim, per):
    """Degenerate periodic mesh of one element: its periodic faces are conforming faces
    with itself (one per periodic axis); face lists bit-exact against the oracle."""
    root = (1,) * dim
    p = W.Params(dim, 3, root, (0.0,) * dim, (250.0,) * dim, per, 0)
    lv, an = W.uniform_morton(p)
    ctx = D.DG(p)
    ctx.mesh_build(lv, an)
    got = ctx.mesh_faces()
    ref = oracle.Mesh(p, lv, an).faces()
    for g, r in zip(got, ref):
        assert np.array_equal(g, r)
    assert len(got[0]) == sum(per)
