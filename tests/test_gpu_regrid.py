"""NEXT-1 on the GPU: the refinement indicator kernel bit-exact against the
oracle, and a whole regrid (indicator -> host plan -> mesh upload -> transfer
kernels) against the oracle's plan and transfer (R16, R19, R37-R39)."""
import numpy as np
import pytest

import oracle
import oracle.regrid as OR
import workloads as W
from test_gpu_parity import Gpu, _check

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg,kind", [("c2", 0), ("c2", 1), ("c4", 0), ("c3", 1)])
def test_indicator_bit_exact(cfg, kind):
    w = W.get(cfg)
    g = Gpu(w.params, w.level, w.anchor, w.bg)
    eta = torch.empty(w.n_elem, dtype=torch.float64, device="cuda")
    g.ctx.amr_indicator(kind, g.dev(w.q0), eta)
    want = OR.indicator(w.params, w.level, w.anchor, w.bg, w.q0, kind)
    assert np.array_equal(eta.cpu().numpy(), want)


def _case(cfg):
    """(params, level, anchor, bg, q0, kind, thresholds, buffer)."""
    if cfg == "vortex":  # 2D refinement: the vortex on 16 x 16 with one level allowed
        p = W.vortex_params(16, 3)
        p.max_level = 1
        lv, an = W.uniform_morton(p)
        return p, lv, an, W.vortex_background(p), W.vortex_state(p, lv, an), 1, (0.05, 0.005), 1
    if cfg == "c2":  # 2D coarsening away from the bubble
        w = W.c2()
        return w.params, w.level, w.anchor, w.bg, w.q0, 0, (1.0, 0.05), 1
    # 3D: seeded random forest, warm bubble, both refinement and coarsening
    p, lv, an = W.random_forest(3, 3, order=3, max_level=2, frac=0.4)
    bg = W.background_table(p)
    X = W.node_coords(p, lv, an)
    c = np.array([0.5 * (p.hi[d] + p.lo[d]) for d in range(3)])
    r = np.sqrt(((X - c[None, :, None]) ** 2).sum(axis=1)) / (0.3 * (p.hi[0] - p.lo[0]))
    q = W.pressure_balanced_state(p, W.node_background(p, bg, lv, an), 0.5 * W.cosine_bubble(r))
    return p, lv, an, bg, q, 0, (0.2, 0.01), 1


@pytest.mark.parametrize("cfg", ["vortex", "c2", "forest3d"])
def test_regrid_matches_oracle(cfg):
    p, lv, an, bg, q0, kind, thr, B = _case(cfg)
    g = Gpu(p, lv, an, bg)
    q = g.dev(q0)
    I0 = g.ctx.integrals(q)
    absI = g.ctx.integrals(q.abs())
    q_new, plan = g.ctx.regrid(q, kind, thr[0], thr[1], B)
    eta = OR.indicator(p, lv, an, bg, q0, kind)
    want = OR.plan(p, lv, an, eta, thr[0], thr[1], B)
    for k in want:
        assert np.array_equal(plan[k], want[k]), k
    assert len(want["refine_parent"]) + len(want["coarsen_parent"]) > 0
    got = g.D.from_device(q_new, g.F, g.Np)
    _check(got, OR.transfer(p, q0, want), what=f"{cfg} regrid state")
    # conservative transfer (R16): integrals unchanged
    I1 = g.ctx.integrals(q_new)
    for f in range(p.n_fields):
        assert abs(I1[f] - I0[f]) <= 1e-13 * absI[f], (f, I0[f], I1[f])
    # the context now holds the new mesh: the RHS on it matches the oracle
    m2 = oracle.Mesh(p, plan["level"], plan["anchor"])
    out = torch.empty_like(q_new)
    g.ctx.rhs(q_new, out)
    _check(g.D.from_device(out, g.F, g.Np), oracle.rhs(m2, bg, got), what=f"{cfg} rhs after regrid")


def test_rrtb_amr_run_conserves_mass_to_roundoff():
    """with mortars (R11-R14) and conservative transfers (R16), an AMR run of
    the rising thermal bubble with regrids keeps the mass and Theta integrals to
    round-off (here 100 s, 4 regrids, two levels, B = 2)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from rrtb_amr import run as run_rrtb
    r = run_rrtb(t_end=100.0, every_s=25.0)
    assert r["finite"]
    assert r["elements_max"] > 100 and r["regrids"] >= 4
    assert r["max_abs_mass_rel"] < 1e-14 and r["max_abs_theta_rel"] < 1e-14, r
