"""Algorithm 1 / Algorithm 2 loops in fp64 — TEST INFRASTRUCTURE ONLY.

Follows PAPER.md line by line (numbering without EndFor lines):

  line 1   lambda = e^{-h/eps}; phi^0 = psi^0 = 1/N (2D: 1/(NM))
  line 2   while l < itr_max and sum_i |psi_i (K^T phi)_i - v_i| > tol PAPER.md:148
  l. 3-7   psi = v / (K^T phi)  (K symmetric: K^T phi = K phi)
  l. 8-12  phi = u / (K psi)
  line 13  l = l + 1
  line 14  return sum_ij phi_i psi_j lambda^{|i-j|} |i-j| h           PAPER.md:163 (2D: :339)

Readings: psi is updated first (R2); the marginal error of
line 2 is evaluated with phi^(l), psi^(l) before the psi update (R3); stop
when err <= tol (R4); tol = 0 means "fixed iterations": the check is skipped
inside the loop and err is evaluated once at exit (R5); a non-finite phi or
psi after an iteration stops that problem with the NONFINITE flag (the
paper's "terminates abnormally") (R6); the returned value is
<C, gamma> without the entropy term (R7).

Log domain: F = log phi, G = log psi, the same updates written with
log-sum-exp (BASELINE.json north_star; Remark 2.1 PAPER.md:100-108 is the
paper's motivation).  In exact arithmetic its iterates equal the scaling
domain's; tests/test_oracle_solve.py pins that.

Kernel applies:  apply="dense" uses oracle.dense (O(N^2) definition);
apply="recur" uses oracle.recur (the paper's O(N) recursion in plain C),
itself pinned equal to dense.
"""
from __future__ import annotations

import math

import numpy as np

from . import dense, recur

CONVERGED, NONFINITE, ITR_MAX = 1, 2, 4


class _Ops1D:
    def __init__(self, n, h, eps, apply):
        self.n, self.h, self.c = n, h, h / eps
        self.lam = dense.lam(h, eps)
        self.mode = apply
        if apply == "dense":
            self.K = dense.kernel(n, self.lam)
            self.W = dense.weighted_kernel(n, self.lam, h)

    # x: [N, B] linear
    def K_(self, x):
        if self.mode == "dense":
            return self.K @ x
        return np.stack([recur.sweep(x[:, j], self.lam) for j in range(x.shape[1])], axis=1)

    def Klog(self, X):
        if self.mode == "dense":
            return np.stack([dense.apply_log(X[:, j], self.c) for j in range(X.shape[1])], axis=1)
        return np.stack([recur.sweep_log(X[:, j], self.c) for j in range(X.shape[1])], axis=1)

    def cost(self, phi, psi):
        if self.mode == "dense":
            return np.einsum("ib,ib->b", phi, self.W @ psi)
        with np.errstate(divide="ignore"):
            return self.cost_log(np.log(phi), np.log(psi))

    def cost_log(self, F, G):
        out = []
        for j in range(F.shape[1]):
            if self.mode == "dense":
                LW = dense.weighted_apply_log(G[:, j], self.c, self.h)
            else:
                LW = recur.wsweep_log(G[:, j], self.c, self.h)
            out.append(recur.sum_exp2(F[:, j], LW))
        return np.array(out)


class _Ops2D:
    """Column-major (N, M) arrays flattened as j*N + i."""

    def __init__(self, n, m, h1, h2, eps, apply):
        self.n, self.m = n, m
        self.h1, self.h2 = h1, h2
        self.c1, self.c2 = h1 / eps, h2 / eps
        self.l1, self.l2 = dense.lam(h1, eps), dense.lam(h2, eps)
        self.mode = apply
        if apply == "dense":
            self.K1, self.K2 = dense.kernel(n, self.l1), dense.kernel(m, self.l2)
            self.W1 = dense.weighted_kernel(n, self.l1, h1)
            self.W2 = dense.weighted_kernel(m, self.l2, h2)

    def _mat(self, x):
        return x.reshape(self.m, self.n).T

    def _flat(self, X):
        return X.T.ravel()

    def K_(self, x):
        out = np.empty_like(x)
        for j in range(x.shape[1]):
            X = self._mat(x[:, j])
            if self.mode == "dense":
                Y = self.K1 @ X @ self.K2          # K0 on columns, then lambda2 mixing
            else:
                Y = recur.sweep(recur.sweep(X, self.l1, axis=1), self.l2, axis=2)
            out[:, j] = self._flat(Y)
        return out

    def Klog(self, X):
        out = np.empty_like(X)
        for j in range(X.shape[1]):
            M = self._mat(X[:, j])
            if self.mode == "dense":
                Y = dense.apply_2d_log(M, self.c1, self.c2)
            else:
                Y = recur.sweep_log(recur.sweep_log(M, self.c1, axis=1), self.c2, axis=2)
            out[:, j] = self._flat(Y)
        return out

    def cost(self, phi, psi):
        if self.mode != "dense":
            with np.errstate(divide="ignore"):
                return self.cost_log(np.log(phi), np.log(psi))
        out = []
        for j in range(phi.shape[1]):
            P, S = self._mat(phi[:, j]), self._mat(psi[:, j])
            T = self.W1 @ S @ self.K2 + self.K1 @ S @ self.W2
            out.append(float(np.sum(P * T)))
        return np.array(out)

    def cost_log(self, F, G):
        out = []
        for j in range(F.shape[1]):
            Fm, Gm = self._mat(F[:, j]), self._mat(G[:, j])
            if self.mode == "dense":
                # log of the two separable terms, each = LSE over (i', j') with weights
                n, m = self.n, self.m
                d1, d2 = dense.dist(n), dense.dist(m)
                with np.errstate(divide="ignore"):
                    w1 = np.log(d1 * self.h1) - self.c1 * d1
                    w2 = np.log(d2 * self.h2) - self.c2 * d2
                full1 = Gm[None, :, None, :] + w1[:, :, None, None] - self.c2 * d2[None, None]
                full2 = Gm[None, :, None, :] - self.c1 * d1[:, :, None, None] + w2[None, None]
                L1 = dense.lse(dense.lse(full1, axis=3), axis=1)
                L2 = dense.lse(dense.lse(full2, axis=3), axis=1)
            else:
                L1 = recur.sweep_log(recur.wsweep_log(Gm, self.c1, self.h1, axis=1), self.c2, axis=2)
                L2 = recur.wsweep_log(recur.sweep_log(Gm, self.c1, axis=1), self.c2, self.h2, axis=2)
            out.append(recur.sum_exp2(Fm, L1) + recur.sum_exp2(Fm, L2))
        return np.array(out)


class _Ops3D:
    """The separable extension to three axes ("easily extended to
    high-dimensional cases"): K = T_L(lambda3) (x) T_M(lambda2) (x) T_N(lambda1) on
    column-major (N, M, L) arrays flattened as (z M + j) N + i, applied per axis (dense
    per-axis kernels); cost with the weighted kernel on one axis at a time.  Scaling
    domain, dense applies only."""

    def __init__(self, n, m, l, h1, h2, h3, eps, apply):
        assert apply == "dense"
        self.n, self.m, self.l = n, m, l
        self.K = [dense.kernel(n, dense.lam(h1, eps)), dense.kernel(m, dense.lam(h2, eps)),
                  dense.kernel(l, dense.lam(h3, eps))]
        self.W = [dense.weighted_kernel(n, dense.lam(h1, eps), h1), dense.weighted_kernel(m, dense.lam(h2, eps), h2),
                  dense.weighted_kernel(l, dense.lam(h3, eps), h3)]

    def _t(self, x):        # flat -> [i, j, z]
        return x.reshape(self.l, self.m, self.n).transpose(2, 1, 0)

    def _f(self, X):
        return X.transpose(2, 1, 0).ravel()

    def _app(self, mats, x):
        # (K1 (x) K2 (x) K3) X, one axis at a time: Y_ijz = sum_abc K1_ia K2_jb K3_zc X_abc
        X = self._t(x)
        X = np.einsum("ia,ajz->ijz", mats[0], X)
        X = np.einsum("jb,ibz->ijz", mats[1], X)
        X = np.einsum("zc,ijc->ijz", mats[2], X)
        return self._f(X)

    def K_(self, x):
        return np.stack([self._app(self.K, x[:, j]) for j in range(x.shape[1])], axis=1)

    def cost(self, phi, psi):
        out = []
        for j in range(phi.shape[1]):
            t = 0.0
            for w in range(3):
                mats = [self.W[a] if a == w else self.K[a] for a in range(3)]
                t += float(phi[:, j] @ self._app(mats, psi[:, j]))
            out.append(t)
        return np.array(out)


def solve(a, b, *, n, m=1, h1, h2=0.0, eps, itr_max, tol=0.0, domain="scaling",
          input_is_log=False, apply="dense", check_interval=1, u0=None, v0=None,
          trace=None, l=1, h3=0.0):
    """Run Algorithm 1 (m == 1) or Algorithm 2 (m > 1; l > 1: its 3D extension) on one
    or many pairs.

    a, b: [size] or [B, size]; promoted to fp64 (R16).
    Returns dict with F, G (log scalings, [B, size]), iters, err, flags, cost ([B]).
    ``trace`` (optional list) receives (l, half, F, G) after every half-step.
    """
    a = np.atleast_2d(np.asarray(a, dtype=np.float64))
    b = np.atleast_2d(np.asarray(b, dtype=np.float64))
    B, size = a.shape
    assert size == n * m * l
    if l > 1:
        assert domain == "scaling", "3D: scaling domain only"
        ops = _Ops3D(n, m, l, h1, h2, h3, eps, apply)
    else:
        ops = _Ops1D(n, h1, eps, apply) if m == 1 else _Ops2D(n, m, h1, h2, eps, apply)
    # work on [size, B] (pairs as columns; BLAS-friendly)
    a, b = a.T.copy(), b.T.copy()
    log_dom = domain == "log"
    if log_dom:
        with np.errstate(divide="ignore"):
            la = a if input_is_log else np.log(a)
            lb = b if input_is_log else np.log(b)
        blin = np.exp(lb)
        F = np.full((size, B), -math.log(size)) if u0 is None else np.atleast_2d(u0).T.astype(np.float64).copy()
        G = np.full((size, B), -math.log(size)) if v0 is None else np.atleast_2d(v0).T.astype(np.float64).copy()
    else:
        if input_is_log:
            a, b = np.exp(a), np.exp(b)
        phi = np.full((size, B), 1.0 / size) if u0 is None else np.atleast_2d(u0).T.astype(np.float64).copy()
        psi = np.full((size, B), 1.0 / size) if v0 is None else np.atleast_2d(v0).T.astype(np.float64).copy()

    iters = np.zeros(B, dtype=np.int64)
    err = np.full(B, np.nan)
    flags = np.zeros(B, dtype=np.int64)
    active = np.ones(B, dtype=bool)
    l = 0
    while active.any():
        idx = np.nonzero(active)[0]
        check = (l >= itr_max) or (tol > 0 and l % check_interval == 0)
        if log_dom:
            T = ops.Klog(F[:, idx])                                  # log K^T phi
            if check:
                with np.errstate(over="ignore"):
                    e = np.sum(np.abs(np.exp(G[:, idx] + T) - blin[:, idx]), axis=0)
        else:
            t = ops.K_(phi[:, idx])                                  # K^T phi (lines 3-6)
            if check:
                e = np.sum(np.abs(psi[:, idx] * t - b[:, idx]), axis=0)
        if check:
            err[idx] = e
            stop = (l >= itr_max) | (e <= tol)
            if stop.any():
                s = idx[stop]
                active[s] = False
                iters[s] = l
                flags[s] = np.where((tol > 0) & (e[stop] <= tol), CONVERGED, ITR_MAX)
            keep = ~stop
            idx = idx[keep]
            if log_dom:
                T = T[:, keep]
            else:
                t = t[:, keep]
            if idx.size == 0:
                break
        with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
            if log_dom:
                G[:, idx] = lb[:, idx] - T                           # line 7
                if trace is not None:
                    trace.append((l, 0, F.copy(), G.copy()))
                F[:, idx] = la[:, idx] - ops.Klog(G[:, idx])         # lines 8-12
                if trace is not None:
                    trace.append((l, 1, F.copy(), G.copy()))
                bad = np.isnan(F[:, idx]).any(0) | np.isnan(G[:, idx]).any(0) | \
                    np.isposinf(F[:, idx]).any(0) | np.isposinf(G[:, idx]).any(0)
            else:
                psi[:, idx] = b[:, idx] / t                          # line 7
                if trace is not None:
                    trace.append((l, 0, np.log(phi), np.log(psi)))
                phi[:, idx] = a[:, idx] / ops.K_(psi[:, idx])        # lines 8-12
                if trace is not None:
                    trace.append((l, 1, np.log(phi), np.log(psi)))
                bad = ~(np.isfinite(phi[:, idx]).all(0) & np.isfinite(psi[:, idx]).all(0))
        l += 1                                                       # line 13
        if bad.any():
            s = idx[bad]
            active[s] = False
            iters[s] = l
            flags[s] = NONFINITE
            err[s] = np.nan

    with np.errstate(divide="ignore", over="ignore", invalid="ignore"):
        if log_dom:
            cost = ops.cost_log(F, G)                                # line 14 (log form)
            Fo, Go = F, G
        else:
            cost = ops.cost(phi, psi)                                # line 14
            Fo, Go = np.log(phi), np.log(psi)
    return {"F": Fo.T.copy(), "G": Go.T.copy(), "iters": iters, "err": err,
            "flags": flags, "cost": cost}


# ---------------------------------------------------------------------------------------
# Steps either side of the loop

def log_gibbs(n, m, h1, h2, eps):
    """-C_kl / eps for the flat (column-major, k = j n + i) grid points: the exponent of
    the Gibbs kernel K_kl = lambda1^{|di|} lambda2^{|dj|}."""
    i = np.tile(np.arange(n), m)
    j = np.repeat(np.arange(m), n)
    C = np.abs(i[:, None] - i[None, :]) * h1 + np.abs(j[:, None] - j[None, :]) * h2
    return -C / eps


def dual_objective(a, b, F, G, *, n, m=1, h1, h2=0.0, eps):
    """The dual of the entropic problem Eq. (2.3) at log-scalings F, G,
    written out densely (small problems):

        D = eps (<F, a> + <G, b> - sum_kl gamma_kl) + eps (sum a + sum b) / 2,
        gamma_kl = exp(F_k + G_l - C_kl / eps)

    From the Lagrangian of PAPER.md:77-83 with gamma = exp((alpha_k + beta_l - C_kl)/eps - 1)
    and F = alpha/eps - 1/2, G = beta/eps - 1/2 (the paper's phi = e^{-1/2 - alpha/eps}
    with the multiplier sign flipped).  By weak duality D <= sum gamma C + eps sum gamma
    ln gamma for every feasible gamma, with equality at the optimum; every Sinkhorn
    half-step maximises D over one block.  Terms with a_k = 0 (F_k = -inf) count 0."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    F = np.asarray(F, np.float64)
    G = np.asarray(G, np.float64)
    L = log_gibbs(n, m, h1, h2, eps)
    with np.errstate(invalid="ignore"):
        fa = np.where(a > 0, F * a, 0.0).sum()
        gb = np.where(b > 0, G * b, 0.0).sum()
        gam = np.exp(F[:, None] + G[None, :] + L).sum()
    return float(eps * (fa + gb - gam) + eps * (a.sum() + b.sum()) / 2)


def primal_objective(F, G, *, n, m=1, h1, h2=0.0, eps):
    """sum gamma C + eps sum gamma ln gamma at gamma = exp(F_k + G_l - C_kl/eps)
    (Eq. 2.3's objective), dense."""
    L = log_gibbs(n, m, h1, h2, eps)
    lg = np.asarray(F, np.float64)[:, None] + np.asarray(G, np.float64)[None, :] + L
    gam = np.exp(lg)
    with np.errstate(invalid="ignore"):
        ent = np.where(gam > 0, gam * lg, 0.0).sum()
    return float((gam * (-L * eps)).sum() + eps * ent)


def eps_schedule(eps, eps0, factor):
    """eps_k = max(eps, eps0 factor^k), k = 0, 1, ... down to eps (factor in (0, 1),
    eps0 >= eps): the stages of the eps-scaling continuation."""
    assert 0.0 < factor < 1.0 and eps0 >= eps > 0.0
    out = []
    e = eps0
    while e > eps * (1.0 + 1e-12):
        out.append(e)
        e *= factor
    out.append(eps)
    return out


def solve_eps_scaling(a, b, *, n, m=1, h1, h2=0.0, eps, eps0, factor, stage_iters, itr_max,
                      tol=0.0, check_interval=1, input_is_log=False, apply="dense"):
    """eps-scaling continuation in the log domain: run Algorithm 1 / 2 at eps_0 > eps_1 >
    ... > eps, each stage warm-started from the previous stage's dual potentials f = eps F,
    g = eps G held fixed (F <- F eps_{k-1}/eps_k), the intermediate stages for
    `stage_iters` fixed iterations, the last with itr_max / tol.  Returns the last stage's
    result (plus 'stages')."""
    sched = eps_schedule(eps, eps0, factor)
    u0 = v0 = None
    prev = None
    for k, ek in enumerate(sched):
        if prev is not None:
            u0 = r["F"] * (prev / ek)
            v0 = r["G"] * (prev / ek)
        final = k == len(sched) - 1
        r = solve(a, b, n=n, m=m, h1=h1, h2=h2, eps=ek, itr_max=itr_max if final else stage_iters,
                  tol=tol if final else 0.0, check_interval=check_interval, domain="log",
                  input_is_log=input_is_log, apply=apply, u0=u0, v0=v0)
        prev = ek
    r["stages"] = sched
    return r
