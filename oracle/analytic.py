"""The paper's analytic throughput model, Eqs. 1-6 and Theorem 1.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §3.3.  Geometric sums are written in summation form
sum_{j=0}^{gamma} alpha^j, which equals the paper's ratio form
(1 - alpha^(gamma+1)) / (1 - alpha) for alpha < 1 and stays finite at
alpha = 1.  Notation: alpha = alpha_{i-1,i}, gamma = gamma_i,
c = c_{d,t} = t_t / t_d (reading R13), rho = rho_i.
"""
from __future__ import annotations


def geom_sum(alpha: float, gamma: int) -> float:
    """sum_{j=0}^{gamma} alpha^j  (Eq.1's (1-alpha^(gamma+1))/(1-alpha))."""
    return sum(alpha ** j for j in range(gamma + 1))


def rho_recursion(alpha: float, gamma: int, steps: int) -> list[float]:
    """Eq.2: rho(t_0) = alpha;
    rho(t_j) = rho(t_{j-1}) * alpha^(gamma+1) + (1 - rho(t_{j-1})) * alpha."""
    out = [alpha]
    for _ in range(steps - 1):
        r = out[-1]
        out.append(r * alpha ** (gamma + 1) + (1.0 - r) * alpha)
    return out


def rho_steady_state(alpha: float, gamma: int) -> float:
    """Eq.3: rho = alpha / (1 - alpha^(gamma+1) + alpha)."""
    return alpha / (1.0 - alpha ** (gamma + 1) + alpha)


def rho_cesaro(alpha: float, gamma: int, n: int) -> float:
    """Eq.3's left-hand side: (1/(n+1)) sum_{j=0}^{n} rho(t_j)."""
    seq = rho_recursion(alpha, gamma, n + 1)
    return sum(seq) / (n + 1)


def expected_tokens(alpha: float, gamma: int, rho: float) -> float:
    """Eq.1: E(N(M_i)) = (1-rho)*1 + rho * sum_{j=0}^{gamma} alpha^j."""
    return (1.0 - rho) + rho * geom_sum(alpha, gamma)


def pipespec_rate(alpha: float, gamma: int) -> float:
    """Eq.4 / Theorem 1: Eq.1 evaluated at the Eq.3 steady state."""
    return expected_tokens(alpha, gamma, rho_steady_state(alpha, gamma))


def sd_speedup(alpha: float, gamma: int, c: float) -> float:
    """Eq.5: sum_{j=0}^{gamma} alpha^j / (gamma/c + 1)."""
    return geom_sum(alpha, gamma) / (gamma / c + 1.0)


def pipespec_ideal(alpha: float, gamma: int) -> float:
    """Eq.6: sum_{j=0}^{gamma} alpha^j."""
    return geom_sum(alpha, gamma)
