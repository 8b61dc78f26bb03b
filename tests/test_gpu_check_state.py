"""dg_check_state (SPEC.md:193-194 positivity monitor, SPEC.md:740 NaN failure)
through the C ABI against oracle.check_state: integer results, bit-exact.
Bad values are planted at seeded positions; NaN in the row padding must not be
counted (the scan reads only the F*Np state doubles of each row)."""
import numpy as np
import pytest

import oracle
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _ctx(w):
    from paper_2404_16648_b200 import dg as D
    ctx = D.DG(w.params)
    ctx.mesh_upload(w.level, w.anchor)
    return D, ctx


def _plant(q, rng, k):
    E, F, Np = q.shape
    q = q.copy()
    cells = rng.permutation(E * Np)[:5 * k]
    vals = [np.nan, -0.5, 0.0, -np.inf, np.inf]
    fields = [1, 0, F - 1, 0, F - 2]
    for j, (v, f) in enumerate(zip(vals, fields)):
        for c in cells[j * k:(j + 1) * k]:
            q[c // Np, f, c % Np] = v
    return q


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5s"])
def test_check_state_parity(name):
    w = W.c5(root=(4, 4, 2)) if name == "c5s" else W.get(name)
    D, ctx = _ctx(w)
    E, F, Np, stride = ctx.state_layout()
    assert ctx.check_state(D.to_device(w.q0, stride)) == oracle.check_state(w.q0) == (0, 0, 0, -1)
    rng = np.random.default_rng(11)
    for k in (1, 3, 17):
        q = _plant(w.q0, rng, min(k, E * Np // 5))
        t = D.to_device(q, stride)
        if stride > F * Np:
            t[:, F * Np:] = float("nan")  # padding is never read
        got = ctx.check_state(t)
        torch.cuda.synchronize()
        assert got == oracle.check_state(q), (name, k)
    # tail: only the last element bad
    q = w.q0.copy()
    q[-1, 0, Np - 1] = -1.0
    assert ctx.check_state(D.to_device(q, stride)) == (0, 1, 0, E - 1)


def test_check_state_full_c5_planted():
    """BASELINE configs[4] at full size (131,072 elements, 2.68 GB): healthy rows
    built on the device, bad values planted at seeded positions; the counts must
    equal the numbers planted (a property that holds at any size)."""
    from types import SimpleNamespace
    p = W.Params(3, 7, (64, 64, 32), (0.0, 0.0, 0.0), (10000.0, 10000.0, 5000.0), (1, 1, 0), 0)
    level, anchor = W.uniform_morton(p)
    D, ctx = _ctx(SimpleNamespace(params=p, level=level, anchor=anchor))
    assert ctx.state_layout()[0] == 131072
    E, F, Np, stride = ctx.state_layout()
    q = torch.zeros((E, stride), dtype=torch.float64, device="cuda")
    q[:, :Np] = 1.2
    q[:, (F - 1) * Np:F * Np] = 350.0
    assert ctx.check_state(q) == (0, 0, 0, -1)
    g = torch.Generator().manual_seed(5)
    e = torch.randint(0, E, (40,), generator=g)
    n = torch.randint(0, Np, (40,), generator=g)
    pairs = sorted(set(zip(e.tolist(), n.tolist())))[:30]
    for j, (ee, nn) in enumerate(pairs):
        if j % 3 == 0:
            q[ee, 2 * Np + nn] = float("nan")
        elif j % 3 == 1:
            q[ee, nn] = -1.0
        else:
            q[ee, (F - 1) * Np + nn] = -2.0
    exp = (len(pairs[0::3]), len(pairs[1::3]), len(pairs[2::3]), min(p[0] for p in pairs))
    assert ctx.check_state(q) == exp
