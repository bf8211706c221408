"""Seeded synthetic inputs for the five BASELINE.json configurations and the paper's
1D random-distribution workload (E1).

This module is shared by the oracle side (tests, golden scripts) and the CUDA
side (tests, bench).  It holds NO arithmetic of the method (no kernel, no
Sinkhorn step, no cost): it only draws histograms, following the recipe of
SURVEY.md §8(d) "Synthetic inputs" (recorded again in DESIGN.md §3).

Every pair p of config c draws from its own stream
``Generator(PCG64(SeedSequence(seed_c, spawn_key=(p,))))`` with
``seed_c = 22021004200 + c``; a is drawn before b.  Per-pair streams make the
inputs independent of batch slicing and of the number of ranks.

Grid: every axis is [0, 1] with spacing h = 1/n and cell centres
x_i = (i + 1/2) h (reading R12).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

SEED_BASE = 22021004200


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    ndim: int
    n: int            # points along axis 1
    m: int            # points along axis 2 (1 in 1D)
    batch: int
    dtype: str        # "f64" | "f32"
    domain: str       # "scaling" | "log"
    eps: float
    itr_max: int
    tol: float
    input_is_log: bool
    description: str
    h: float = 0.0        # axis-1 spacing when not 1/n (E1: 6/(N-1) on [-3, 3])
    seed_index: int = 0   # seed_c = SEED_BASE + seed_index (0: the digit of "cK")
    hh2: float = 0.0      # axis-2 spacing when not 1/m (E3: h2 = 1)

    @property
    def size(self) -> int:
        return self.n * self.m

    @property
    def h1(self) -> float:
        return self.h if self.h else 1.0 / self.n

    @property
    def h2(self) -> float:
        if self.hh2:
            return self.hh2
        return 1.0 / self.m if self.ndim == 2 else 0.0

    @property
    def np_dtype(self):
        return np.float64 if self.dtype == "f64" else np.float32


CONFIGS = {
    "c1": Config("c1", 1, 1000, 1, 1, "f64", "scaling", 1e-2, 2000, 1e-9, False,
                 "1D N=1000 on [0,1], h=1/N, one pair fp64, 2-component Gaussian mixtures "
                 "+1e-6 floor, eps=1e-2, 2000 iters or marginal L1 err <= 1e-9"),
    # domain: the fp32 scaling domain overflows on some pairs of this config (max |log phi|
    # reaches ~80 of fp32's 88.7 within 64 pairs), so it runs in the log domain (R14)
    "c2": Config("c2", 1, 1024, 1, 4096, "f32", "log", 5e-3, 500, 0.0, False,
                 "batch 4096 pairs, 1D N=1024 fp32, Dirichlet(1) smoothed by width-5 box, "
                 "eps=5e-3, 500 iters"),
    "c3": Config("c3", 1, 1 << 24, 1, 1, "f64", "log", 1e-4, 1000, 0.0, True,
                 "one pair 1D N=2^24 fp64 log domain, mixtures of 8 Gaussians (std 1e-3..1e-2), "
                 "eps=1e-4, 1000 iters"),
    "c4": Config("c4", 2, 2048, 2048, 1, "f32", "log", 1e-3, 300, 0.0, True,
                 "2D 2048x2048 l1 cost, fp32 log domain, sums of 16 anisotropic Gaussians, "
                 "eps=1e-3, 300 iters"),
    "c5": Config("c5", 1, 4096, 1, 65536, "f32", "log", 1e-3, 1000, 0.0, False,
                 "batch 65536 pairs (8192 per GPU at 8 GPUs), 1D N=4096 fp32 log domain, "
                 "lognormal(0,1) bin weights, eps=1e-3, 1000 iters"),
}

# The paper's 1D random distributions (Table 1 :361-378): grid
# x_i = (i-1) dx - 3, dx = 6/(N-1) on [-3, 3]; u_i, v_j iid U[0,1], normalised; eps = 1e-3;
# 1000 iterations; 100 trials (here: one batch of 100 pairs).  fp64 scaling domain, the
# paper's unstabilised FS-1 (its precision is unstated, fp64 implied, R20).
for _k, _n in enumerate((500, 2000, 8000)):
    CONFIGS[f"e1_{_n}"] = Config(
        f"e1_{_n}", 1, _n, 1, 100, "f64", "scaling", 1e-3, 1000, 0.0, False,
        f"paper E1 (Table 1): 100 trials, 1D N={_n} on [-3,3], dx=6/(N-1), u,v iid U[0,1] "
        f"normalised, eps=1e-3, 1000 iters, fp64 scaling domain", h=6.0 / (_n - 1), seed_index=11 + _k)

# The paper's Ricker-wavelet experiment (Table 2 :412-429): f = R(t),
# g = R(t - s), R(t) = (1 - 2 pi^2 t^2) exp(-pi^2 t^2) (f0 = A = 1), s = -1.2032, squared and
# normalised by Eq. (ricker) with delta = 1e-3 (L = N so that each sums to 1); eps = 1e-2,
# 500 iterations, repeated 100 times (one batch of 100 identical pairs).  The time interval
# is unstated: [-4, 4] (SPEC.md's reading, R28), dt = 8/(N-1).  fp64 scaling domain.
for _k, _n in enumerate((500, 2000, 8000)):
    CONFIGS[f"e2_{_n}"] = Config(
        f"e2_{_n}", 1, _n, 1, 100, "f64", "scaling", 1e-2, 500, 0.0, False,
        f"paper E2 (Table 2): Ricker wavelet R(t) vs R(t+1.2032) on [-4,4], N={_n}, squared, "
        f"normalised with delta=1e-3, eps=1e-2, 500 iters, 100 repetitions, fp64 scaling domain",
        h=8.0 / (_n - 1), seed_index=21 + _k)

# The paper's 2D random distributions (Table 3): N x N grids, h1 = h2 = 1,
# the 1D recipe's iid U[0,1] weights normalised over the N^2 points, eps = 0.01 (so
# lambda = e^{-100} on both axes), 1000 iterations, 100 trials (one batch of 100 pairs).
# fp64 scaling domain, the paper's unstabilised FS-1 (Algorithm 2).
for _k, _n in enumerate((10, 20, 40, 80, 160)):
    CONFIGS[f"e3_{_n}"] = Config(
        f"e3_{_n}", 2, _n, _n, 100, "f64", "scaling", 1e-2, 1000, 0.0, False,
        f"paper E3 (Table 3): 100 trials, 2D {_n}x{_n}, h1=h2=1, u,v iid U[0,1] normalised, "
        f"eps=1e-2, 1000 iters, fp64 scaling domain", h=1.0, seed_index=41 + _k, hh2=1.0)

# The paper's stabilisation study (Figure 1 right): the same Ricker pair at
# eps = 1e-3, where the unstabilised iteration terminates abnormally; run with the paper's
# own stabilisation (Remark 2.1 + 3.2, domain "stabilized", tau = 1e10) for 2000
# iterations, 100 repetitions.  fp64.
for _k, _n in enumerate((500, 2000, 8000)):
    CONFIGS[f"e2s_{_n}"] = Config(
        f"e2s_{_n}", 1, _n, 1, 100, "f64", "stabilized", 1e-3, 2000, 0.0, False,
        f"paper E2 stabilisation study (PAPER.md:410): Ricker pair on [-4,4], N={_n}, eps=1e-3, "
        f"2000 iters, 100 repetitions, the paper's stabilised FS-1 (absorption tau=1e10)",
        h=8.0 / (_n - 1), seed_index=31 + _k)

# the paper's FS-1 time per trial on its CPU (Xeon Gold 5117): Table 1 (PAPER.md:371-373,
# 1000 iterations) and Table 2 (PAPER.md:422-424, 500 iterations); context for the paper
# workload bench lines (updates/s = N x iterations / time)
PAPER_TABLE1_SECONDS = {"e1_500": 8.70e-3, "e1_2000": 4.25e-2, "e1_8000": 1.53e-1,
                        "e2_500": 4.90e-3, "e2_2000": 1.52e-2, "e2_8000": 5.96e-2}


def pair_rng(cfg_index: int, pair: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence(SEED_BASE + cfg_index,
                                                                       spawn_key=(pair,))))


def centres(n: int) -> np.ndarray:
    return (np.arange(n, dtype=np.float64) + 0.5) / n


def _logsumexp(x: np.ndarray, axis=None) -> np.ndarray:
    mx = np.max(x, axis=axis, keepdims=True)
    out = mx + np.log(np.sum(np.exp(x - mx), axis=axis, keepdims=True))
    return np.squeeze(out, axis=axis) if axis is not None else out.reshape(())


# ---------------------------------------------------------------- per-config draws
def _c1_hist(rng, n):
    x = centres(n)
    mu = rng.uniform(0.2, 0.8, size=2)
    sd = rng.uniform(0.05, 0.1, size=2)
    p = np.zeros(n)
    for k in range(2):
        p += np.exp(-0.5 * ((x - mu[k]) / sd[k]) ** 2) / (sd[k] * math.sqrt(2 * math.pi))
    p /= p.sum()
    p += 1e-6
    return p / p.sum()


def _c2_hist(rng, n):
    w = rng.exponential(1.0, size=n)          # Dirichlet(1) = iid Exp(1), normalised
    w /= w.sum()
    # width-5 box filter as a truncated-window mean (edges average the in-range cells)
    c = np.concatenate([[0.0], np.cumsum(w)])
    lo = np.clip(np.arange(n) - 2, 0, n)
    hi = np.clip(np.arange(n) + 3, 0, n)
    s = (c[hi] - c[lo]) / (hi - lo)
    return s / s.sum()


def _c3_loghist(rng, n):
    x = centres(n)
    mu = rng.uniform(0.0, 1.0, size=8)
    sd = rng.uniform(1e-3, 1e-2, size=8)
    comps = np.empty((8, n))
    for k in range(8):
        comps[k] = -0.5 * ((x - mu[k]) / sd[k]) ** 2 - math.log(sd[k])
    la = _logsumexp(comps, axis=0)
    return la - _logsumexp(la)


def _c4_loghist(rng, n, m):
    # column-major flattening: flat index j*n + i, i along axis 1 (h1), j along axis 2 (h2)
    xi = centres(n)[:, None]
    yj = centres(m)[None, :]
    cx = rng.uniform(0.1, 0.9, size=16)
    cy = rng.uniform(0.1, 0.9, size=16)
    s1 = rng.uniform(0.01, 0.1, size=16)
    s2 = rng.uniform(0.01, 0.1, size=16)
    th = rng.uniform(0.0, math.pi, size=16)
    acc = np.full((n, m), -np.inf)
    for k in range(16):
        dx, dy = xi - cx[k], yj - cy[k]
        u = math.cos(th[k]) * dx + math.sin(th[k]) * dy
        v = -math.sin(th[k]) * dx + math.cos(th[k]) * dy
        comp = -0.5 * ((u / s1[k]) ** 2 + (v / s2[k]) ** 2) - math.log(s1[k] * s2[k])
        acc = np.logaddexp(acc, comp)
    la = acc - _logsumexp(acc.ravel())
    return la.ravel(order="F")


def _c5_hist(rng, n):
    w = rng.lognormal(0.0, 1.0, size=n)
    return w / w.sum()


def _e1_hist(rng, n):
    w = rng.uniform(0.0, 1.0, size=n)
    return w / w.sum()


RICKER_SHIFT = -1.2032
RICKER_DELTA = 1e-3


def ricker(t):
    """R(t) = A (1 - 2 pi^2 f0^2 t^2) exp(-pi^2 f0^2 t^2), f0 = A = 1."""
    x = (math.pi * t) ** 2
    return (1.0 - 2.0 * x) * np.exp(-x)


def ricker_pair(n, lo=-4.0, hi=4.0, shift=RICKER_SHIFT, delta=RICKER_DELTA):
    """(u, v) of Eq. (ricker): (f^2/||f^2||_1 + delta) / (1 + N delta), f = R(t), g = R(t - s)."""
    t = np.linspace(lo, hi, n)
    out = []
    for f in (ricker(t), ricker(t - shift)):
        f2 = f * f
        out.append((f2 / f2.sum() + delta) / (1.0 + n * delta))
    return out[0], out[1]


_DRAW = {
    "c1": lambda rng, cfg: _c1_hist(rng, cfg.n),
    "c2": lambda rng, cfg: _c2_hist(rng, cfg.n),
    "c3": lambda rng, cfg: _c3_loghist(rng, cfg.n),
    "c4": lambda rng, cfg: _c4_loghist(rng, cfg.n, cfg.m),
    "c5": lambda rng, cfg: _c5_hist(rng, cfg.n),
    "e1": lambda rng, cfg: _e1_hist(rng, cfg.n),
    "e3": lambda rng, cfg: _e1_hist(rng, cfg.n * cfg.m),
}


def pair(cfg: Config | str, p: int, n: int | None = None):
    """(a, b) for pair p in fp64 before any cast.  Log-weights when cfg.input_is_log.

    ``n`` overrides the grid size (smaller parity cases with the same recipe)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    if n is not None and n != cfg.n:
        cfg = dataclasses.replace(cfg, n=n, m=(n if cfg.ndim == 2 else 1),
                                  h=(6.0 / (n - 1) if cfg.name.startswith("e1") and n > 1 else cfg.h))
    idx = cfg.seed_index or int(cfg.name[1:])
    rng = pair_rng(idx, p)
    if cfg.name.startswith("e2"):  # deterministic signals: every repetition is the same pair (e2, e2s)
        return ricker_pair(cfg.n)
    draw = _DRAW[cfg.name.split("_")[0]]
    a = draw(rng, cfg)
    b = draw(rng, cfg)
    return a, b


def batch(cfg: Config | str, pairs, n: int | None = None):
    """Arrays [len(pairs)][size] in the config dtype (the values both sides consume)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    A, B = [], []
    for p in pairs:
        a, b = pair(cfg, p, n)
        A.append(a)
        B.append(b)
    A = np.stack(A).astype(cfg.np_dtype)
    B = np.stack(B).astype(cfg.np_dtype)
    return A, B


def random_positive(rng: np.random.Generator, shape, lo=0.05, hi=1.0, normalise=True):
    """Generic strictly positive histograms for small edge-case tests."""
    x = rng.uniform(lo, hi, size=shape)
    if normalise:
        x = x / x.sum(axis=-1, keepdims=True)
    return x
