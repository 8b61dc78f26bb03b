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
