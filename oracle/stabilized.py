"""The paper's log-domain-stabilised FS-1 in fp64 — TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py).

Algorithm 1 with the absorption of Remark 2.1
and the replacement recursions of Remark 3.2:

  state      alpha, beta (absorbed potentials), phi, psi (scalings)
  kernel     K~ = diag(e^{alpha/eps}) K diag(e^{beta/eps})                  Remark 2.1
  line 1     lambda = e^{-h/eps}; phi = psi = 1/N; alpha = beta = 0; l = 0
  line 2     while l < itr_max and sum_j |psi_j (K~^T phi)_j - v_j| > tol
  l. 3-6     K~^T phi by lines 5-6 of Remark 3.2 (oracle.recur.stab_sweep, own = beta)
  line 7     psi = v / (K~^T phi)
  l. 8-11    K~ psi by lines 10-11 of Remark 3.2 (own = alpha)
  line 12    phi = u / (K~ psi)
  line 13    l = l + 1
  absorb     if max(|phi|_inf, |psi|_inf) > tau: alpha += eps ln phi, beta += eps ln psi,
             phi = psi = 1                                                   Remark 2.1
  line 14    return sum_ij gamma_ij |i-j| h,  gamma = diag(e^{alpha/eps} phi) K diag(e^{beta/eps} psi)

Readings: R8 — the absorption is alpha <- alpha + eps ln phi (the printed
"alpha <- alpha + ln phi" is dimensionally inconsistent with the e^{alpha/eps} rescaling);
the potentials are kept divided by eps (A = alpha/eps, B = beta/eps, so the absorption is
A <- A + ln phi); R29 — line 3's r_1 = phi_1 becomes r_1 = e^{(alpha_1+beta_1)/eps} phi_1
(and p_1 likewise), the value the replaced recursion gives for an empty prefix; R30 —
tau is unstated: 1e10 (SPEC.md's reading), tested after every full iteration (after the
non-finite check; "exceed" = strictly greater).  The other readings are the plain
oracle's (R2-R7 in oracle/sinkhorn.py).  Outputs are log-scalings F = A + ln phi,
G = B + ln psi, so they compare directly with oracle.sinkhorn's.
"""
from __future__ import annotations

import math

import numpy as np

from . import dense, recur
from .sinkhorn import CONVERGED, ITR_MAX, NONFINITE


def stab_apply_dense(x, own, other, lam):
    """The definition: diag(e^own) K diag(e^other) x with K_ij = lambda^|i-j| materialised
    (Remark 2.1's rescaled kernel; powers by stepwise multiplication, Remark 3.3)."""
    K = dense.kernel(len(x), lam)
    Kt = np.exp(np.asarray(own, np.float64))[:, None] * K * np.exp(np.asarray(other, np.float64))[None, :]
    return Kt @ np.asarray(x, np.float64)


def absorb(A, B, phi, psi):
    """Remark 2.1: alpha <- alpha + eps ln phi, beta <- beta + eps ln psi (divided by eps),
    phi, psi <- 1.  Returns the new (A, B, phi, psi)."""
    return A + np.log(phi), B + np.log(psi), np.ones_like(phi), np.ones_like(psi)


def solve_stab(a, b, *, n, h, eps, itr_max, tol=0.0, tau=1e10, check_interval=1, absorb_at=()):
    """Stabilised Algorithm 1 on one pair (fp64).  ``absorb_at``: iterations l (after line 13)
    at which to absorb regardless of tau (absorption-transparency tests).

    Returns dict F, G (log-scalings), iters, err, flags, cost, absorptions (list of l)."""
    u = np.asarray(a, np.float64).ravel()
    v = np.asarray(b, np.float64).ravel()
    assert u.size == n and v.size == n
    lam = dense.lam(h, eps)
    phi = np.full(n, 1.0 / n)
    psi = np.full(n, 1.0 / n)
    A = np.zeros(n)
    B = np.zeros(n)
    absorb_at = set(absorb_at)
    l = 0
    err = math.nan
    flag = 0
    absorptions = []
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        while True:
            check = l >= itr_max or (tol > 0 and l % check_interval == 0)
            t = recur.stab_sweep(phi, B, A, lam)                    # K~^T phi, lines 3-6
            if check:
                err = float(np.sum(np.abs(psi * t - v)))             # line 2
                if l >= itr_max or err <= tol:
                    flag = CONVERGED if (tol > 0 and err <= tol) else ITR_MAX
                    break
            psi = v / t                                              # line 7
            phi = u / recur.stab_sweep(psi, A, B, lam)               # lines 8-12
            l += 1                                                   # line 13
            if not (np.isfinite(phi).all() and np.isfinite(psi).all()):
                flag = NONFINITE
                err = math.nan
                break
            if max(np.max(np.abs(phi)), np.max(np.abs(psi))) > tau or l in absorb_at:
                A, B, phi, psi = absorb(A, B, phi, psi)               # Remark 2.1
                absorptions.append(l)
        F = A + np.log(phi)
        G = B + np.log(psi)
    if flag == NONFINITE:
        cost = math.nan
    else:                                                            # line 14 on gamma(F, G)
        c = h / eps
        cost = recur.sum_exp2(F, recur.wsweep_log(G, c, h))
    return {"F": F[None], "G": G[None], "iters": np.array([l]), "err": np.array([err]),
            "flags": np.array([flag]), "cost": np.array([cost]), "absorptions": absorptions}
