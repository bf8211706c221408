"""Dense fp64 kernel applies — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything here is the plain definition written out:

* lambda = e^{-h/eps}                                  PAPER.md:112 (§3)
* K_ij = lambda^{|i-j|}, powers formed by stepwise
  multiplication (never exp(-m h/eps) directly)        PAPER.md:80-89, 236-238 (Remark 3.3)
* (K x)_k = sum_j lambda^{|k-j|} x_j                   PAPER.md:113-122, Eq. (3.1)
* log form: (log K e^X)_k = LSE_j (X_j - c|k-j|), c = h/eps
* 2D kernel K = T_M(lambda2) (x) T_N(lambda1) on column-major
  flattened arrays (index j*N + i)                     PAPER.md:244-280 (§4)
* distance-weighted kernel W_ij = |i-j| h lambda^{|i-j|}
  whose bilinear form is the return line               PAPER.md:163 (Alg. 1 l.14), 339 (Alg. 2)
"""
from __future__ import annotations

import math

import numpy as np


def lam(h: float, eps: float) -> float:
    """lambda = e^{-h/eps}."""
    if eps <= 0:
        raise ValueError("eps must be > 0")
    return math.exp(-h / eps)


def powers(n: int, lam_: float) -> np.ndarray:
    """[1, lambda, lambda^2, ..., lambda^{n-1}] by stepwise multiplication (Remark 3.3)."""
    pw = np.empty(max(n, 1), dtype=np.float64)
    pw[0] = 1.0
    for k in range(1, n):
        pw[k] = pw[k - 1] * lam_
    return pw[:n]


def dist(n: int) -> np.ndarray:
    i = np.arange(n)
    return np.abs(i[:, None] - i[None, :])


def kernel(n: int, lam_: float) -> np.ndarray:
    """The N x N Toeplitz Gibbs kernel K_ij = lambda^{|i-j|} (Eq. 3.1)."""
    return powers(n, lam_)[dist(n)]


def weighted_kernel(n: int, lam_: float, h: float) -> np.ndarray:
    """W_ij = |i-j| h lambda^{|i-j|}: sum_ij phi_i psi_j W_ij is Alg. 1's return line."""
    d = dist(n)
    return d * h * powers(n, lam_)[d]


def apply(x: np.ndarray, lam_: float) -> np.ndarray:
    """K x (x of shape [N] or [N, B]) by the dense matrix product of Eq. (3.1)."""
    x = np.asarray(x, dtype=np.float64)
    return kernel(x.shape[0], lam_) @ x


def weighted_apply(x: np.ndarray, lam_: float, h: float) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return weighted_kernel(x.shape[0], lam_, h) @ x


def lse(v: np.ndarray, axis=-1) -> np.ndarray:
    """log sum exp with the max factored out; all -inf gives -inf."""
    mx = np.max(v, axis=axis, keepdims=True)
    safe = np.where(np.isfinite(mx), mx, 0.0)
    with np.errstate(divide="ignore"):
        out = safe + np.log(np.sum(np.exp(v - safe), axis=axis, keepdims=True))
    return np.squeeze(out, axis=axis)


def apply_log(X: np.ndarray, c: float) -> np.ndarray:
    """(log K e^X)_k = LSE_j (X_j - c|k-j|) for a single vector X (length N)."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    return lse(X[None, :] - c * dist(n), axis=1)


def weighted_apply_log(X: np.ndarray, c: float, h: float) -> np.ndarray:
    """log (W e^X)_k = LSE_{j != k} (X_j - c|k-j| + log(|k-j| h))."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    d = dist(n)
    with np.errstate(divide="ignore"):
        logw = np.log(d * h)
    return lse(X[None, :] - c * d + logw, axis=1)


# ------------------------------------------------------------------ 2D (§4)
def kernel_2d(n: int, m: int, lam1: float, lam2: float) -> np.ndarray:
    """The fully materialised (N M) x (N M) block kernel of PAPER.md:255-280:
    block (k, l) is lambda2^{|k-l|} K0 with K0 = T_N(lambda1); column-major order."""
    K0 = kernel(n, lam1)
    K2 = kernel(m, lam2)
    out = np.empty((n * m, n * m))
    for k in range(m):
        for l in range(m):
            out[k * n:(k + 1) * n, l * n:(l + 1) * n] = K2[k, l] * K0
    return out


def apply_2d(X: np.ndarray, lam1: float, lam2: float) -> np.ndarray:
    """K vec(X) for X of shape (N, M): K0 on every column, then the lambda2 mixing
    of columns, i.e. T_N X T_M (the two Toeplitz factors of the block kernel)."""
    X = np.asarray(X, dtype=np.float64)
    n, m = X.shape
    return kernel(n, lam1) @ X @ kernel(m, lam2)


def apply_2d_log(X: np.ndarray, c1: float, c2: float) -> np.ndarray:
    """LSE over (i', j') of X_{i'j'} - c1|i-i'| - c2|j-j'| (dense, small sizes only)."""
    X = np.asarray(X, dtype=np.float64)
    n, m = X.shape
    D1 = dist(n)
    D2 = dist(m)
    full = X[None, :, None, :] - c1 * D1[:, :, None, None] - c2 * D2[None, None, :, :]
    # full[i, i', j, j']
    return lse(lse(full, axis=3), axis=1)


def cost_2d_bruteforce(Phi, Psi, lam1, lam2, h1, h2) -> float:
    """Alg. 2 return line as the literal quadruple sum (tiny sizes)."""
    n, m = Phi.shape
    P1 = powers(n, lam1)
    P2 = powers(m, lam2)
    tot = 0.0
    for i1 in range(n):
        for j1 in range(m):
            for i2 in range(n):
                for j2 in range(m):
                    di, dj = abs(i1 - i2), abs(j1 - j2)
                    tot += Phi[i1, j1] * Psi[i2, j2] * P1[di] * P2[dj] * (di * h1 + dj * h2)
    return tot
