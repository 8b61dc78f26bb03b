"""Pins of oracle.check_state (SPEC.md:193-194 positivity monitor, SPEC.md:740
NaN failure): bad values are planted at seeded positions on a healthy state,
so the expected counts are the numbers planted, not a re-run of the scan."""
import numpy as np
import pytest

import oracle


def _healthy(E, F, Np, rng):
    q = rng.uniform(-1.0, 1.0, (E, F, Np))
    q[:, 0] = rng.uniform(0.5, 1.5, (E, Np))   # rho > 0
    q[:, -1] = rng.uniform(100.0, 400.0, (E, Np))  # rho*theta > 0
    return q


@pytest.mark.parametrize("F,Np", [(4, 25), (5, 125), (5, 512)])
def test_clean_state(F, Np):
    q = _healthy(7, F, Np, np.random.default_rng(1))
    assert oracle.check_state(q) == (0, 0, 0, -1)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_planted_counts(seed):
    rng = np.random.default_rng(seed)
    E, F, Np = 40, 5, 125
    q = _healthy(E, F, Np, rng)
    cells = rng.permutation(E * Np)[:60]
    nan_mom = cells[:10]     # NaN in a momentum field: non-finite only
    neg_rho = cells[10:25]   # rho < 0 (finite)
    zero_th = cells[25:33]   # rho*theta == 0 (finite, counts: <= 0)
    inf_rho = cells[33:38]   # -inf in rho: non-finite AND rho <= 0
    nan_rho = cells[38:42]   # NaN in rho: non-finite, not <= 0
    for c in nan_mom:
        q[c // Np, 2, c % Np] = np.nan
    for c in neg_rho:
        q[c // Np, 0, c % Np] = -0.25
    for c in zero_th:
        q[c // Np, F - 1, c % Np] = 0.0
    for c in inf_rho:
        q[c // Np, 0, c % Np] = -np.inf
    for c in nan_rho:
        q[c // Np, 0, c % Np] = np.nan
    first = int(min(cells[:42]) // Np)
    assert oracle.check_state(q) == (10 + 5 + 4, 15 + 5, 8, first)


def test_positive_inf_is_nonfinite_not_nonpositive():
    q = _healthy(3, 4, 25, np.random.default_rng(5))
    q[2, 0, 7] = np.inf
    q[1, 3, 0] = -0.0  # -0 <= 0
    assert oracle.check_state(q) == (1, 0, 1, 1)
