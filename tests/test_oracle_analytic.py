"""Pins for oracle/analytic.py (Eqs. 1-6, Theorem 1; §3.3)."""
import json
import os

import numpy as np
import pytest

from oracle import analytic as A

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "analytic_worked_values.json")))
GRID_A = [round(0.05 * k, 2) for k in range(1, 20)]
GRID_G = list(range(1, 17))


def test_golden_worked_values():
    for e in GOLD["rho_steady_state"]:
        assert A.rho_steady_state(e["alpha"], e["gamma"]) == pytest.approx(e["value"], abs=1e-12), e
    for e in GOLD["expected_tokens"]:
        assert A.expected_tokens(e["alpha"], e["gamma"], e["rho"]) == pytest.approx(e["value"], abs=1e-12)
    for e in GOLD["pipespec_rate"]:
        assert A.pipespec_rate(e["alpha"], e["gamma"]) == pytest.approx(e["value"], abs=e.get("tol", 1e-12)), e
    for e in GOLD["sd_speedup"]:
        assert A.sd_speedup(e["alpha"], e["gamma"], e["c"]) == pytest.approx(e["value"], abs=1e-12), e
    for e in GOLD["pipespec_ideal"]:
        assert A.pipespec_ideal(e["alpha"], e["gamma"]) == pytest.approx(e["value"], abs=1e-12), e


def test_eq2_fixed_point_is_eq3():
    """SPEC criterion 1: iterate Eq.2 to its fixed point; equals Eq.3 within 1e-9."""
    for a in GRID_A:
        for g in GRID_G:
            last = A.rho_recursion(a, g, 10_000)[-1]
            r = A.rho_steady_state(a, g)
            assert abs(last - r) < 1e-9
            # exact fixed point of Eq.2's right-hand side
            assert abs(r * a ** (g + 1) + (1 - r) * a - r) < 1e-12


def test_eq3_cesaro_average_converges():
    """Eq.3 is written as a Cesaro average; the O(1/n) transient vanishes (reading R5)."""
    a, g = 0.8, 4
    r = A.rho_steady_state(a, g)
    e1 = abs(A.rho_cesaro(a, g, 1_000) - r)
    e2 = abs(A.rho_cesaro(a, g, 10_000) - r)
    assert e2 < e1 / 5 and e2 < 1e-4


def test_recursion_boundary_values():
    assert A.rho_recursion(0.0, 4, 3) == [0.0, 0.0, 0.0]
    assert A.rho_recursion(1.0, 4, 3) == [1.0, 1.0, 1.0]


def test_theorem1_rate_above_one():
    """Theorem 1: PipeSpec(P) > 1 for 0 < alpha < 1, gamma > 0."""
    for a in GRID_A + [1e-3, 0.999]:
        for g in GRID_G:
            assert A.pipespec_rate(a, g) > 1.0


def test_ratio_form_equals_summation_form():
    for a in GRID_A:
        for g in GRID_G:
            assert A.geom_sum(a, g) == pytest.approx((1 - a ** (g + 1)) / (1 - a), rel=1e-12)


def test_eq5_limits():
    for g in (1, 4, 8):
        for c in (2.0, 4.0, 10.0):
            assert A.sd_speedup(1.0, g, c) == pytest.approx((g + 1) / (g / c + 1))
            assert A.sd_speedup(0.0, g, c) < 1.0   # "performs worse than autoregressive"
    # Eq.6 dominates Eq.5 for every c > 0 -- but exact Eq.4 need not (reading R14)
    assert A.pipespec_ideal(0.8, 4) > A.sd_speedup(0.8, 4, 10.0)
    assert A.pipespec_rate(0.8, 4) < A.sd_speedup(0.8, 4, 10.0)
    assert A.pipespec_rate(0.8, 8) > A.sd_speedup(0.8, 8, 10.0)


def test_monotone_in_alpha_and_gamma():
    for g in GRID_G:
        v = [A.pipespec_rate(a, g) for a in GRID_A]
        assert all(x <= y + 1e-12 for x, y in zip(v, v[1:]))
    for a in GRID_A:
        v = [A.pipespec_rate(a, g) for g in GRID_G]
        assert all(x <= y + 1e-12 for x, y in zip(v, v[1:]))


def test_verify_branch_tokens_by_monte_carlo():
    """Leviathan et al.'s count that Eq.1 cites: with gamma drafts each
    accepted independently w.p. alpha, a verify step appends the accepted prefix
    plus one token; its mean is sum_{j<=gamma} alpha^j.  Simulated, not restated."""
    rng = np.random.default_rng(5)
    for a, g in [(0.5, 2), (0.8, 4), (0.95, 8)]:
        acc = rng.random((200_000, g)) < a
        prefix = np.where(acc.all(1), g, np.argmin(acc, axis=1))
        est = (prefix + 1).mean()
        assert est == pytest.approx(A.geom_sum(a, g), rel=0.01)


def test_two_state_chain_matches_eq3_eq1():
    """[V4] An independent simulation of the verification state: after a verify
    step the next step verifies iff all gamma drafts AND the draft at the bonus
    position agree (alpha^(gamma+1)); after a 1-token step iff one draft agrees
    (alpha).  Long-run verify frequency and tokens/step match Eq.3 and Eq.1."""
    rng = np.random.default_rng(11)
    for a, g in [(0.8, 4), (0.5, 8), (0.95, 2)]:
        n = 200_000
        u = rng.random((n, g + 1)) < a
        V = True  # rho(t_0) = alpha: the first step verifies iff the first draft agrees
        V = bool(u[0, 0])
        nv, tok = 0, 0
        for s in range(1, n):
            if V:
                nv += 1
                acc = u[s, :g]
                k = g if acc.all() else int(np.argmin(acc))
                tok += k + 1
                V = bool(acc.all() and u[s, g])
            else:
                tok += 1
                V = bool(u[s, 0])
        rho = nv / (n - 1)
        assert rho == pytest.approx(A.rho_steady_state(a, g), abs=0.01)
        assert tok / (n - 1) == pytest.approx(A.pipespec_rate(a, g), rel=0.02)
