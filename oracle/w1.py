"""Closed forms used as pins — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* w1_exact: the unregularised 1D Wasserstein-1 distance of Eq. (kantorovich)
   on a uniform grid, by the classical CDF identity
  W1 = h * sum_{k<N} |sum_{i<=k} (u_i - v_i)|.  It is the
  eps -> 0 limit of the entropic problem.
* n2_plan: the exact entropic optimal plan for N = 2.  The Gibbs form
  gamma = diag(phi) K diag(psi) fixes the cross ratio
  gamma11 gamma22 / (gamma12 gamma21) = 1/lambda^2; with the marginals this
  leaves the quadratic (1-l^2) x^2 - (l^2 (1-a1-b1) + a1 + b1) x + a1 b1 = 0
  for x = gamma11.  Cost = h (gamma12 + gamma21) = h (a1+b1-2x).
"""
from __future__ import annotations

import math

import numpy as np


def w1_exact(a, b, h: float) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(h * np.sum(np.abs(np.cumsum(a - b)[:-1])))


def n2_plan(a1: float, b1: float, lam: float):
    """Return (gamma11, cost/h) of the N=2 entropic plan with total mass 1."""
    A = 1.0 - lam * lam
    Bc = lam * lam * (1.0 - a1 - b1) + a1 + b1
    C = a1 * b1
    lo, hi = max(0.0, a1 + b1 - 1.0), min(a1, b1)
    if A == 0.0:
        x = C / Bc
    else:
        # Bc^2 - 4AC expanded into non-negative terms (no cancellation):
        # (a1-b1)^2 + l^2 (2 s d + 4 a1 b1) + l^4 d^2,  s = a1+b1, d = 1-s
        s, d, l2 = a1 + b1, 1.0 - a1 - b1, lam * lam
        disc = math.sqrt((a1 - b1) ** 2 + l2 * (2 * s * d + 4 * a1 * b1) + l2 * l2 * d * d)
        # small root without cancellation: (Bc - disc)/(2A) == 2C/(Bc + disc)
        roots = [2 * C / (Bc + disc), (Bc + disc) / (2 * A)]
        x = [r for r in roots if lo - 1e-15 <= r <= hi + 1e-15][0]
    # off-diagonal mass gamma12 + gamma21 = (a1 - x) + (b1 - x)
    return x, (a1 - x) + (b1 - x)


def entropy(p) -> float:
    p = np.asarray(p, dtype=np.float64).ravel()
    p = p[p > 0]
    return float(-np.sum(p * np.log(p)))
