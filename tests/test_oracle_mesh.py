"""Pins of the oracle's connectivity: SPEC tiny meshes,
closed-form counts of uniform meshes, the face-slot identity, and an O(E^2)
brute-force geometric adjacency search on seeded random balanced forests
(PAPER.md:181-182 forest of active leaves; PAPER.md:281 2:1 faces; R15, R29)."""
import numpy as np
import pytest

import oracle
import workloads as W


def brute_force_faces(p, level, anchor):
    """Canonical face lists from pairwise box contacts at the finest resolution."""
    E = len(level)
    dim = p.dim
    L = int(level.max())
    lev = level.astype(np.int64)
    lo = anchor.astype(np.int64) << (L - lev)[:, None]
    hi = lo + (1 << (L - lev))[:, None]
    ext = np.array([p.root[d] << L for d in range(dim)])
    conf, nonc, bnd = [], {}, []
    touched = np.zeros((E, 2 * dim), bool)
    for d in range(dim):
        tang = [a for a in range(dim) if a != d]
        # i's +d face against j's -d face
        hit = hi[:, d][:, None] == lo[:, d][None, :]
        if p.periodic[d]:
            hit |= (hi[:, d][:, None] == ext[d]) & (lo[:, d][None, :] == 0)
        for t in tang:
            hit &= (np.minimum(hi[:, t][:, None], hi[:, t][None, :]) >
                    np.maximum(lo[:, t][:, None], lo[:, t][None, :]))
        for i, j in zip(*np.nonzero(hit)):
            touched[i, 2 * d + 1] = touched[j, 2 * d] = True
            if lev[i] == lev[j]:
                conf.append((i, 2 * d + 1, j, 2 * d))
            else:
                assert abs(lev[i] - lev[j]) == 1
                c, fc, f, ff = (i, 2 * d + 1, j, 2 * d) if lev[i] < lev[j] else (j, 2 * d, i, 2 * d + 1)
                b = sum(((int(anchor[f, t]) & 1) << k) for k, t in enumerate(tang))
                nonc.setdefault((c, fc), {})[b] = (f, ff)
    for e in range(E):
        for f in range(2 * dim):
            if not touched[e, f]:
                bnd.append((e, f))
    conf = np.array(sorted(conf), np.int32).reshape(-1, 4)
    nsub = 1 << (dim - 1)
    rows = []
    for (c, fc) in sorted(nonc):
        kids = nonc[(c, fc)]
        assert sorted(kids) == list(range(nsub))
        rows.append([c, fc] + [v for b in range(nsub) for v in kids[b]])
    nonc = np.array(rows, np.int32).reshape(-1, 2 + 2 * nsub)
    bnd = np.array(sorted(bnd), np.int32).reshape(-1, 2)
    return conf, nonc, bnd


def _mesh(p, level, anchor):
    return oracle.Mesh(p, level, anchor).faces()


def test_spec_single_root_refined():
    """single root refined -> 4 leaves, 4 internal conforming faces."""
    p = W.Params(2, 2, (1, 1), (0.0, 0.0), (1.0, 1.0), (0, 0), 1)
    f = W.Forest(p)
    f.split((0, 0, 0, 0))
    lv, an = f.ordered()
    conf, nonc, bnd = _mesh(p, lv, an)
    assert len(lv) == 4 and len(conf) == 4 and len(nonc) == 0 and len(bnd) == 8


def test_spec_2x2_one_refined():
    """refine one cell of a 2x2 patch -> 7 leaves, 2 nonconforming faces."""
    p = W.Params(2, 2, (2, 2), (0.0, 0.0), (2.0, 2.0), (0, 0), 1)
    f = W.Forest(p)
    f.split((0, 0, 0, 0))
    lv, an = f.ordered()
    conf, nonc, bnd = _mesh(p, lv, an)
    assert len(lv) == 7 and len(nonc) == 2
    assert len(conf) == 4 + 2   # 4 among the children + 2 among the three coarse cells
    # the coarse owners see their fine neighbours in b order
    for row in nonc:
        assert lv[row[0]] == 0 and lv[row[2]] == 1 and lv[row[4]] == 1


def test_balance_ripple_and_rejection():
    """SPEC S:132 ripple: refining twice next to a coarse cell forces the coarse
    neighbour to refine once; the oracle rejects the unbalanced forest."""
    p = W.Params(2, 2, (3, 1), (0.0, 0.0), (3.0, 1.0), (0, 0), 2)
    f = W.Forest(p)
    f.split((0, 1, 0, 0))
    f.split((1, 2, 0, 0))          # level-2 cells touch root cell 0
    lv, an = f.ordered()
    with pytest.raises(oracle.OracleError) as ex:
        oracle.Mesh(p, lv, an)
    assert ex.value.code == -4
    f.balance()
    lv, an = f.ordered()
    assert (0, 0, 0, 0) not in f.leaves        # neighbour auto-refined once
    assert max(l for l, *_ in f.leaves if l >= 0) == 2
    conf, nonc, bnd = _mesh(p, lv, an)
    assert len(nonc) > 0


def test_overlap_and_gap_rejected():
    p = W.Params(2, 2, (2, 1), (0.0, 0.0), (2.0, 1.0), (0, 0), 1)
    lv = np.array([0, 0, 1], np.int8)
    an = np.array([[0, 0], [1, 0], [0, 0]], np.int32)       # overlap
    with pytest.raises(oracle.OracleError) as ex:
        oracle.Mesh(p, lv, an)
    assert ex.value.code == -3
    lv = np.array([0], np.int8)
    an = np.array([[0, 0]], np.int32)                         # gap
    with pytest.raises(oracle.OracleError) as ex:
        oracle.Mesh(p, lv, an)
    assert ex.value.code == -3
    lv = np.array([0, 0], np.int8)
    an = np.array([[0, 0], [0, 0]], np.int32)                 # duplicate
    with pytest.raises(oracle.OracleError):
        oracle.Mesh(p, lv, an)


@pytest.mark.parametrize("nx,nz", [(1, 1), (3, 2), (10, 10), (5, 7)])
def test_uniform_2d_wall_counts(nx, nz):
    p = W.Params(2, 3, (nx, nz), (0.0, 0.0), (1.0, 1.0), (0, 0), 0)
    lv, an = W.uniform_morton(p)
    conf, nonc, bnd = _mesh(p, lv, an)
    assert len(conf) == (nx - 1) * nz + nx * (nz - 1)
    assert len(bnd) == 2 * (nx + nz) and len(nonc) == 0


def test_uniform_3d_periodic_counts():
    p = W.Params(3, 2, (4, 3, 2), (0.0,) * 3, (1.0,) * 3, (1, 1, 0), 0)
    lv, an = W.uniform_morton(p)
    conf, nonc, bnd = _mesh(p, lv, an)
    assert len(conf) == 4 * 3 * 2 * 2 + 4 * 3 * 1
    assert len(bnd) == 2 * 4 * 3


def _slot_identity(p, n, conf, nonc, bnd):
    return 2 * len(conf) + len(bnd) + (1 + (1 << (p.dim - 1))) * len(nonc) == 2 * p.dim * n


@pytest.mark.parametrize("name,counts", [("c1", (100, 180, 0, 40)), ("c3", (4096, 12032, 0, 512))])
def test_config_meshes(name, counts):
    w = W.get(name)
    conf, nonc, bnd = _mesh(w.params, w.level, w.anchor)
    assert (w.n_elem, len(conf), len(nonc), len(bnd)) == counts
    assert _slot_identity(w.params, w.n_elem, conf, nonc, bnd)


def test_c2_mesh():
    p, f = W.c2_forest()
    lv, an = f.ordered()
    conf, nonc, bnd = _mesh(p, lv, an)
    assert len(nonc) > 0 and _slot_identity(p, len(lv), conf, nonc, bnd)
    bf = brute_force_faces(p, lv, an)
    np.testing.assert_array_equal(conf, bf[0])
    np.testing.assert_array_equal(nonc, bf[1])
    np.testing.assert_array_equal(bnd, bf[2])


@pytest.mark.parametrize("seed", range(30))
@pytest.mark.parametrize("dim", [2, 3])
def test_random_forest_brute_force(seed, dim):
    p, lv, an = W.random_forest(seed, dim, max_level=3 if dim == 2 else 2)
    conf, nonc, bnd = _mesh(p, lv, an)
    bf = brute_force_faces(p, lv, an)
    np.testing.assert_array_equal(conf, bf[0])
    np.testing.assert_array_equal(nonc, bf[1])
    np.testing.assert_array_equal(bnd, bf[2])
    assert _slot_identity(p, len(lv), conf, nonc, bnd)
