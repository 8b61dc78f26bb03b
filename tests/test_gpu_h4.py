"""k_stage_h4 (3D, N = 4, warp per element) on meshes WITH 2:1 faces.

By default the library runs 3D N = 4 meshes that have 2:1 faces on the generic tile kernel
and conforming ones on k_stage_h4; DG_H4_AMR=1 (inline mortar steps) or 2 (mortar pre-pass) at
context creation puts AMR meshes on k_stage_h4 too, so its mortar steps (coarse side A-E and the
fine-side projection, R35; §3.3) stay covered: strict identical-input stage parity
(R19, every field) and the RHS against the oracle on c4 and on random balanced forests."""
import numpy as np
import pytest

import oracle
import workloads as W
from test_gpu_parity import Gpu, _check
from test_gpu_stage_strict import _strict_chain

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(params=["1", "2"], ids=["inline", "prepass"])
def h4_amr(monkeypatch, request):
    """DG_H4_AMR=1: k_stage_h4 with its inline mortar steps; 2: the mortar pre-pass (k_mortar_h4,
    one warp per coarse face) writes the coarse-side lifts, k_stage_h4 copies them in."""
    monkeypatch.setenv("DG_H4_AMR", request.param)


def test_h4_forced_c4(h4_amr):
    w = W.c4()
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    assert len(m.faces()[1]) > 0
    _check(g.rhs(w.q0), oracle.rhs(m, w.bg, w.q0), what="c4 rhs (k_stage_h4)")
    _strict_chain(g, m, w.bg, w.dt, w.q0, 1, what="c4 (k_stage_h4)")


@pytest.mark.parametrize("seed", [7, 9, 11])
def test_h4_forced_random_amr(h4_amr, seed):
    from test_oracle_rhs import _bubble_state
    p, lv, an = W.random_forest(seed, 3, order=4, max_level=2)
    p.hi = tuple(250.0 * r for r in p.root)
    bg, q = _bubble_state(p, lv, an, seed)
    g = Gpu(p, lv, an, bg)
    m = oracle.Mesh(p, lv, an)
    assert len(m.faces()[1]) > 0
    _check(g.rhs(q), oracle.rhs(m, bg, q), what=f"amr seed {seed} rhs (k_stage_h4)")
    _strict_chain(g, m, bg, 5e-4, q, 2, what=f"amr seed {seed} (k_stage_h4)")


def test_h4_c5n4_sampled_rhs_and_step():
    """The c5 mesh at N = 4 (131,072 elements: the multi-warp-CTA launch of k_stage_h4, the bench's
    c5n4 leg) at full size on a moving state (seeded velocity and Theta noise: every face has
    jumps); the oracle computes sampled elements and their dependency cone."""
    from test_gpu_parity import _check_traj, _hmin, _neigh
    w = W.get("c5n4")
    rng = np.random.default_rng(56)
    q0 = w.q0.copy()
    q0[:, 1:4] += q0[:, :1] * rng.uniform(-0.5, 0.5, size=q0[:, 1:4].shape)
    q0[:, 4] *= 1.0 + 1e-4 * rng.uniform(-1.0, 1.0, size=q0[:, 4].shape)
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    S2 = np.unique(np.concatenate([rng.choice(w.n_elem, 48, replace=False), [0, 11, 12, w.n_elem - 1]]))
    nb = _neigh(m, w.n_elem)
    grow = lambda S: np.unique(np.concatenate([S] + [np.array(nb[e]) for e in S]))
    S1 = grow(S2)
    S0 = grow(S1)
    _check(g.rhs(q0)[S2], oracle.rhs(m, w.bg, q0, elems=S2)[S2], what="c5n4 rhs (sampled)")
    q1, _ = g.stages(q0, w.dt, 3)
    a = oracle.rk_stage(m, w.bg, 0, w.dt, q0, q0, elems=S0)
    b = oracle.rk_stage(m, w.bg, 1, w.dt, q0, a, elems=S1)
    c = oracle.rk_stage(m, w.bg, 2, w.dt, q0, b, elems=S2)
    _check_traj(q1[S2], c[S2], w.params, w.bg, w.dt, 3, _hmin(w.params, w.level), what="c5n4 step (sampled)")
