"""Pins of the oracle's conservative parent<->child projection (PAPER.md:279,
313; readings R16): constants, polynomial reproduction at the
children's own nodes, refine->coarsen identity, and conservation of every
field integral."""
import itertools

import numpy as np
import pytest

import oracle
import workloads as W


def _family(dim, N):
    """One root cell (parent) and its 2^d children as two separate 'meshes'."""
    p = W.Params(dim, N, (1,) * dim, (0.0,) * dim, tuple(100.0 * (d + 1) for d in range(dim)), (0,) * dim, 1)
    par_l = np.zeros(1, np.int8)
    par_a = np.zeros((1, dim), np.int32)
    f = W.Forest(p)
    f.split((0, 0, 0, 0))
    ch_l, ch_a = f.ordered()
    return p, (par_l, par_a), (ch_l, ch_a)


def _poly_field(p, X, rng, deg):
    F = p.n_fields
    out = np.zeros((X.shape[0], F, X.shape[2]))
    for f in range(F):
        for k in itertools.product(range(deg + 1), repeat=p.dim):
            c = rng.uniform(-1, 1)
            term = np.full(X.shape[0:1] + X.shape[2:], c)
            for d in range(p.dim):
                term = term * (X[:, d] / p.hi[d]) ** k[d]
            out[:, f] += term
    return out


@pytest.mark.parametrize("dim,N", [(2, 4), (3, 4), (3, 2), (2, 7), (3, 7)])
def test_refine_reproduces_polynomials_and_coarsen_inverts(dim, N):
    p, (pl, pa), (cl, ca) = _family(dim, N)
    rng = np.random.default_rng(dim * 10 + N)
    Xp = W.node_coords(p, pl, pa)
    Xc = W.node_coords(p, cl, ca)
    qp = _poly_field(p, Xp, rng, N)
    qc = oracle.refine(dim, N, [0], [0], qp, 1 << dim)
    # children are the same polynomial sampled at their own nodes (Morton child order, R27)
    ref = _poly_field(p, Xc, np.random.default_rng(dim * 10 + N), N)
    assert np.abs(qc - ref).max() <= 1e-12 * np.abs(ref).max()
    back = oracle.coarsen(dim, N, [0], [0], qc, 1)
    assert np.abs(back - qp).max() <= 1e-12 * np.abs(qp).max()
    # constants exactly (to rounding) both ways
    one = np.ones_like(qp) * 3.5
    assert np.abs(oracle.refine(dim, N, [0], [0], one, 1 << dim) - 3.5).max() < 1e-13
    onec = np.ones_like(qc) * 3.5
    assert np.abs(oracle.coarsen(dim, N, [0], [0], onec, 1) - 3.5).max() < 1e-13


@pytest.mark.parametrize("dim,N", [(2, 4), (3, 4), (3, 7)])
def test_projection_conserves_integrals(dim, N):
    """Arbitrary (non-polynomial) data: refine and coarsen conserve every field's
    integral (PAPER.md:273-279 'conservative coarsening')."""
    p, (pl, pa), (cl, ca) = _family(dim, N)
    rng = np.random.default_rng(5)
    mp = oracle.Mesh(p, pl, pa)
    mc = oracle.Mesh(p, cl, ca)
    qp = rng.uniform(0.5, 2.0, size=(1, p.n_fields, p.n_nodes))
    qc = oracle.refine(dim, N, [0], [0], qp, 1 << dim)
    np.testing.assert_allclose(oracle.integrals(mc, qc), oracle.integrals(mp, qp), rtol=1e-13)
    qc2 = rng.uniform(0.5, 2.0, size=(1 << dim, p.n_fields, p.n_nodes))
    qp2 = oracle.coarsen(dim, N, [0], [0], qc2, 1)
    np.testing.assert_allclose(oracle.integrals(mp, qp2), oracle.integrals(mc, qc2), rtol=1e-13)


def test_refine_kron_against_vandermonde():
    """child_b = (kron P_b) parent with P_b = interpolation to the half interval,
    built here from a Vandermonde solve."""
    dim, N = 3, 3
    x = W.lgl_nodes(N)
    n1 = N + 1
    V = np.vander(x, n1, increasing=True)
    rng = np.random.default_rng(0)
    qp = rng.standard_normal((1, 5, n1 ** 3))
    qc = oracle.refine(dim, N, [0], [0], qp, 8)
    for b in range(8):
        mats = []
        for a in range(3):
            t = (x - 1) / 2 if not (b >> a) & 1 else (x + 1) / 2
            mats.append(np.linalg.solve(V.T, np.vander(t, n1, increasing=True).T).T)
        K = np.kron(mats[2], np.kron(mats[1], mats[0]))
        np.testing.assert_allclose(qc[b], qp[0] @ K.T, atol=1e-13)


def test_multi_family_indexing():
    """Several families with scattered parent/child indices go to the right slots."""
    dim, N = 2, 3
    rng = np.random.default_rng(1)
    n1 = N + 1
    qsrc = rng.standard_normal((5, 4, n1 ** 2))
    parents = np.array([4, 0, 2], np.int32)
    child0 = np.array([8, 0, 4], np.int32)
    out = oracle.refine(dim, N, parents, child0, qsrc, 12)
    for pi, c0 in zip(parents, child0):
        one = oracle.refine(dim, N, [0], [0], qsrc[pi:pi + 1], 4)
        np.testing.assert_array_equal(out[c0:c0 + 4], one)
    back = oracle.coarsen(dim, N, child0, parents, out, 5)
    for pi in parents:
        np.testing.assert_allclose(back[pi], qsrc[pi], atol=1e-12)
