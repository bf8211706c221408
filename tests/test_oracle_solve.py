"""Pins for the oracle's Sinkhorn loop (Algorithm 1 / 2) on CPU.

Pinned against: the exact N=2 entropic plan, the exact W1 closed form (itself
checked against scipy and an LP), the eps -> 0 sandwich bound, the dual-ascent
property of Sinkhorn half-steps, the marginal invariant after each update,
reflection symmetry, the scale invariance of the iteration map, the identity
kernel case, and agreement between the independent dense / recursion and
scaling / log code paths.
"""
import math

import numpy as np
import pytest
import scipy.optimize
import scipy.stats

import fs1_inputs as gi
from oracle import dense, recur, sinkhorn, w1


def _solve(a, b, **kw):
    n = len(a)
    kw.setdefault("h1", 1.0 / n)
    return sinkhorn.solve(a, b, n=n, **kw)


# ------------------------------------------------------------------ closed forms
def test_w1_closed_form_vs_scipy_and_lp():
    rng = np.random.default_rng(0)
    for n in [2, 3, 6, 8]:
        a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
        h = 0.25
        x = np.arange(n) * h
        ref = scipy.stats.wasserstein_distance(x, x, a, b)
        assert w1.w1_exact(a, b, h) == pytest.approx(ref, rel=1e-12)
        C = np.abs(x[:, None] - x[None, :]).ravel()
        Aeq = np.vstack([np.kron(np.eye(n), np.ones(n)), np.kron(np.ones(n), np.eye(n))])
        lp = scipy.optimize.linprog(C, A_eq=Aeq, b_eq=np.concatenate([a, b]), method="highs")
        assert w1.w1_exact(a, b, h) == pytest.approx(lp.fun, rel=1e-9, abs=1e-12)


def test_w1_golden(golden_dir):
    import json, os
    g = json.load(open(os.path.join(golden_dir, "spec_examples.json")))
    for e in g["w1"]:
        assert w1.w1_exact(e["a"], e["b"], e["h"]) == pytest.approx(e["w1"], rel=1e-15)


@pytest.mark.parametrize("a1,b1,eps", [(0.3, 0.6, 0.5), (0.9, 0.2, 1.0), (0.5, 0.5, 0.1), (0.05, 0.7, 2.0)])
def test_n2_closed_form(a1, b1, eps):
    """Converged Sinkhorn on N=2 equals the exact entropic plan."""
    a, b = np.array([a1, 1 - a1]), np.array([b1, 1 - b1])
    h = 1.0
    lam = math.exp(-h / eps)
    x, c = w1.n2_plan(a1, b1, lam)
    r = sinkhorn.solve(a, b, n=2, h1=h, eps=eps, itr_max=100000, tol=1e-15)
    assert r["flags"][0] == sinkhorn.CONVERGED
    phi, psi = np.exp(r["F"][0]), np.exp(r["G"][0])
    assert phi[0] * psi[0] == pytest.approx(x, rel=1e-10)
    assert r["cost"][0] == pytest.approx(h * c, rel=1e-10, abs=1e-14)


def test_eps_limit_sandwich_and_monotone():
    """0 <= <C,gamma_eps> - W1 <= eps*min(H(a),H(b)) (+ marginal slack) at convergence,
    and the cost decreases toward W1 as eps decreases."""
    rng = np.random.default_rng(2)
    n = 64
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    h = 1.0 / n
    W = w1.w1_exact(a, b, h)
    costs = []
    for eps in [0.1, 0.03, 0.01, 0.003]:
        r = sinkhorn.solve(a, b, n=n, h1=h, eps=eps, itr_max=200000, tol=1e-13, domain="log")
        assert r["flags"][0] == sinkhorn.CONVERGED
        gap = r["cost"][0] - W
        slack = (n - 1) * h * r["err"][0]
        assert -slack - 1e-13 <= gap <= eps * min(w1.entropy(a), w1.entropy(b)) + slack
        costs.append(r["cost"][0])
    assert all(costs[i] > costs[i + 1] for i in range(len(costs) - 1))


# ------------------------------------------------------------------ loop invariants
def _dual(F, G, a, b, c):
    n = len(a)
    D = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    return float(F @ a + G @ b - np.exp(F[:, None] + G[None, :] - c * D).sum())


def test_dual_ascent_and_marginals():
    """Each half-step maximises the dual over one block (G_j = log b_j - LSE_i(F_i - c|i-j|)
    is PAPER.md:154 in log form), so D(F,G) never decreases, and after each update the
    corresponding marginal of gamma is exact."""
    rng = np.random.default_rng(4)
    n, eps = 50, 0.05
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    h = 1.0 / n
    c = h / eps
    trace = []
    sinkhorn.solve(a, b, n=n, h1=h, eps=eps, itr_max=30, domain="log", trace=trace)
    vals = [_dual(F[:, 0], G[:, 0], a, b, c) for (_, _, F, G) in trace]
    assert all(vals[i + 1] >= vals[i] - 1e-13 for i in range(len(vals) - 1))
    D = np.abs(np.arange(n)[:, None] - np.arange(n)[None, :])
    for (_, half, F, G) in trace:
        gam = np.exp(F[:, 0][:, None] + G[:, 0][None, :] - c * D)
        if half == 0:
            np.testing.assert_allclose(gam.sum(0), b, rtol=1e-12)
        else:
            np.testing.assert_allclose(gam.sum(1), a, rtol=1e-12)


def test_identity_kernel_converges_at_one():
    """lambda = 0 (eps << h) and a = b: converges at iteration 1, err 0, cost 0."""
    rng = np.random.default_rng(5)
    a = gi.random_positive(rng, 16)
    r = sinkhorn.solve(a, a, n=16, h1=1.0, eps=1e-4, itr_max=50, tol=1e-14)
    assert r["iters"][0] == 1 and r["flags"][0] == sinkhorn.CONVERGED
    assert r["err"][0] == 0.0 and r["cost"][0] == 0.0


def test_n1():
    r = sinkhorn.solve([1.0], [1.0], n=1, h1=1.0, eps=0.1, itr_max=5)
    assert r["cost"][0] == 0.0 and r["iters"][0] == 5
    assert r["F"][0, 0] + r["G"][0, 0] == pytest.approx(0.0, abs=1e-15)


def test_reflection_symmetry():
    rng = np.random.default_rng(6)
    n = 40
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    r1 = _solve(a, b, eps=0.02, itr_max=25)
    r2 = _solve(a[::-1], b[::-1], eps=0.02, itr_max=25)
    np.testing.assert_allclose(r2["F"][0][::-1], r1["F"][0], rtol=1e-12)
    np.testing.assert_allclose(r2["G"][0][::-1], r1["G"][0], rtol=1e-12)
    assert r2["cost"][0] == pytest.approx(r1["cost"][0], rel=1e-12)


def test_scale_invariance_of_iteration_map():
    """phi0 -> c phi0 leaves the plan after one full iteration unchanged."""
    rng = np.random.default_rng(7)
    n = 30
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    base = np.full(n, 1.0 / n)
    r1 = _solve(a, b, eps=0.05, itr_max=1, u0=base, v0=base)
    r2 = _solve(a, b, eps=0.05, itr_max=1, u0=37.0 * base, v0=base)
    g1 = r1["F"][0][:, None] + r1["G"][0][None, :]
    g2 = r2["F"][0][:, None] + r2["G"][0][None, :]
    np.testing.assert_allclose(g1, g2, rtol=1e-12, atol=1e-12)


# ------------------------------------------------------------------ path agreement
@pytest.mark.parametrize("cfg", ["c1", "c2", "c5"])
def test_dense_recur_scaling_log_agree(cfg):
    c = gi.CONFIGS[cfg]
    n = 96
    a, b = gi.pair(c, 0, n=n)
    kw = dict(n=n, h1=1.0 / n, eps=0.02, itr_max=40)
    rd = sinkhorn.solve(a, b, **kw)
    rr = sinkhorn.solve(a, b, apply="recur", **kw)
    rl = sinkhorn.solve(a, b, domain="log", **kw)
    rlr = sinkhorn.solve(a, b, domain="log", apply="recur", **kw)
    for r in (rr, rl, rlr):
        np.testing.assert_allclose(r["F"], rd["F"], rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(r["G"], rd["G"], rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(r["cost"], rd["cost"], rtol=1e-12)
        np.testing.assert_allclose(r["err"], rd["err"], rtol=1e-9)


def test_batched_equals_single():
    rng = np.random.default_rng(9)
    n = 32
    A, B = gi.random_positive(rng, (5, n)), gi.random_positive(rng, (5, n))
    rb = sinkhorn.solve(A, B, n=n, h1=1.0 / n, eps=0.03, itr_max=20)
    for p in range(5):
        r = sinkhorn.solve(A[p], B[p], n=n, h1=1.0 / n, eps=0.03, itr_max=20)
        np.testing.assert_allclose(rb["F"][p], r["F"][0], rtol=1e-14)
        assert rb["cost"][p] == pytest.approx(r["cost"][0], rel=1e-14)


def test_tolerance_stop_and_fixed_iteration_replay():
    """A tol-stopped run equals the fixed-iteration run with itr_max = its l* (Q6)."""
    c = gi.CONFIGS["c1"]
    a, b = gi.pair(c, 0, n=200)
    kw = dict(n=200, h1=1 / 200, eps=0.02)
    r1 = sinkhorn.solve(a, b, itr_max=5000, tol=1e-9, **kw)
    assert r1["flags"][0] == sinkhorn.CONVERGED and r1["err"][0] <= 1e-9
    r2 = sinkhorn.solve(a, b, itr_max=int(r1["iters"][0]), **kw)
    assert r2["flags"][0] == sinkhorn.ITR_MAX
    np.testing.assert_array_equal(r1["F"], r2["F"])
    assert r1["cost"][0] == r2["cost"][0] and r1["err"][0] == r2["err"][0]


def test_check_interval():
    c = gi.CONFIGS["c1"]
    a, b = gi.pair(c, 0, n=100)
    r = sinkhorn.solve(a, b, n=100, h1=0.01, eps=0.02, itr_max=5000, tol=1e-8, check_interval=7)
    assert r["iters"][0] % 7 == 0 and r["flags"][0] == sinkhorn.CONVERGED


def test_nonfinite_flag_scaling_vs_log():
    """Unstabilised scaling-domain Sinkhorn terminates abnormally at small eps
    (PAPER.md:410); the log domain does not."""
    n = 200
    x = (np.arange(n) + 0.5) / n
    a = np.exp(-((x - 0.2) / 0.05) ** 2) + 1e-3
    b = np.exp(-((x - 0.8) / 0.05) ** 2) + 1e-3
    a, b = a / a.sum(), b / b.sum()
    r = sinkhorn.solve(a, b, n=n, h1=1.0 / n, eps=5e-4, itr_max=200)
    assert r["flags"][0] == sinkhorn.NONFINITE and 1 <= r["iters"][0] < 200
    rl = sinkhorn.solve(a, b, n=n, h1=1.0 / n, eps=5e-4, itr_max=200, domain="log", apply="recur")
    assert rl["flags"][0] == sinkhorn.ITR_MAX and np.isfinite(rl["cost"][0])


def test_2d_dense_recur_and_log_agree():
    c = gi.CONFIGS["c4"]
    n, m = 12, 10
    rng = np.random.default_rng(11)
    a = gi.random_positive(rng, n * m)
    b = gi.random_positive(rng, n * m)
    kw = dict(n=n, m=m, h1=1 / n, h2=1 / m, eps=0.05, itr_max=15)
    rd = sinkhorn.solve(a, b, **kw)
    for extra in [dict(apply="recur"), dict(domain="log"), dict(domain="log", apply="recur")]:
        r = sinkhorn.solve(a, b, **kw, **extra)
        np.testing.assert_allclose(r["F"], rd["F"], rtol=1e-11, atol=1e-11)
        np.testing.assert_allclose(r["cost"], rd["cost"], rtol=1e-12)


def test_2d_reduces_to_1d():
    """An N x 1 grid is the 1D problem along axis 1."""
    rng = np.random.default_rng(12)
    n = 20
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    r2 = sinkhorn.solve(a, b, n=n, m=1, h1=0.05, h2=0.0, eps=0.04, itr_max=10)
    r1 = sinkhorn.solve(a, b, n=n, h1=0.05, eps=0.04, itr_max=10)
    np.testing.assert_allclose(r2["F"], r1["F"], rtol=1e-14)


def test_2d_separable_converged_cost_sandwich():
    """At convergence the 2D entropic cost is >= the exact l1 OT cost (LP) and
    within eps*min(H) of it."""
    rng = np.random.default_rng(13)
    n, m = 4, 3
    a, b = gi.random_positive(rng, n * m), gi.random_positive(rng, n * m)
    h1, h2 = 0.3, 0.2
    ii, jj = np.meshgrid(np.arange(n), np.arange(m), indexing="xy")
    # column-major flat index j*n + i
    I = np.tile(np.arange(n), m)
    J = np.repeat(np.arange(m), n)
    C = (np.abs(I[:, None] - I[None, :]) * h1 + np.abs(J[:, None] - J[None, :]) * h2).ravel()
    N = n * m
    Aeq = np.vstack([np.kron(np.eye(N), np.ones(N)), np.kron(np.ones(N), np.eye(N))])
    lp = scipy.optimize.linprog(C, A_eq=Aeq, b_eq=np.concatenate([a, b]), method="highs").fun
    eps = 0.02
    r = sinkhorn.solve(a, b, n=n, m=m, h1=h1, h2=h2, eps=eps, itr_max=100000, tol=1e-13, domain="log")
    assert r["flags"][0] == sinkhorn.CONVERGED
    gap = r["cost"][0] - lp
    assert -1e-9 <= gap <= eps * min(w1.entropy(a), w1.entropy(b)) + 1e-9


# ------------------------------------------------------------------ log-weight inputs
@pytest.mark.parametrize("apply", ["dense", "recur"])
def test_input_is_log_equals_linear_input(apply):
    """solve(log a, log b, input_is_log=True) is the run on a, b (the branch that feeds
    every C3/C4 reference, oracle/sinkhorn.py): log domain against the log domain at
    1e-13, and against the independent scaling-domain path (plain K @ x) at 1e-11."""
    n = 150
    x = (np.arange(n) + 0.5) / n
    rng = np.random.default_rng(20)
    # smooth log-weights spanning ~200 nats (finite after exp: the linear paths can run)
    la = -((x - 0.3) / 0.07) ** 2 + 0.1 * rng.standard_normal(n)
    lb = -((x - 0.6) / 0.05) ** 2 + 0.1 * rng.standard_normal(n)
    la -= np.log(np.sum(np.exp(la)))
    lb -= np.log(np.sum(np.exp(lb)))
    kw = dict(n=n, h1=1.0 / n, eps=0.02, itr_max=60, apply=apply)
    rl = sinkhorn.solve(la, lb, domain="log", input_is_log=True, **kw)
    rlin = sinkhorn.solve(np.exp(la), np.exp(lb), domain="log", **kw)
    rs = sinkhorn.solve(np.exp(la), np.exp(lb), domain="scaling", **kw)
    for k in ("F", "G"):
        np.testing.assert_allclose(rl[k], rlin[k], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(rl[k], rs[k], rtol=1e-11, atol=1e-11)
    assert rl["cost"][0] == pytest.approx(rlin["cost"][0], rel=1e-13)
    assert rl["cost"][0] == pytest.approx(rs["cost"][0], rel=1e-12)
    assert rl["err"][0] == pytest.approx(rs["err"][0], rel=1e-9)


def test_input_is_log_minus_inf_weights():
    """-inf log-weights (zero mass) in the log domain give F = -inf (G = -inf) exactly
    there and equal the scaling-domain run with exact zeros elsewhere (the scaling
    path divides a_i = 0 by K psi > 0 and never forms a logarithm of the weights)."""
    rng = np.random.default_rng(21)
    n = 64
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    a[[0, 7, 8, 40]] = 0.0
    b[[3, 63]] = 0.0
    a, b = a / a.sum(), b / b.sum()
    with np.errstate(divide="ignore"):
        la, lb = np.log(a), np.log(b)
    kw = dict(n=n, h1=1.0 / n, eps=0.05, itr_max=30)
    rl = sinkhorn.solve(la, lb, domain="log", input_is_log=True, apply="recur", **kw)
    rs = sinkhorn.solve(a, b, domain="scaling", **kw)
    assert np.array_equal(np.isneginf(rl["F"][0]), a == 0)
    assert np.array_equal(np.isneginf(rl["G"][0]), b == 0)
    for k in ("F", "G"):
        m = np.isfinite(rs[k][0])
        np.testing.assert_allclose(rl[k][0][m], rs[k][0][m], rtol=1e-11, atol=1e-11)
    assert rl["cost"][0] == pytest.approx(rs["cost"][0], rel=1e-12)


# ------------------------------------------------------------------ dual objective, eps-scaling
def test_dual_objective_weak_and_strong_duality():
    """D <= the primal objective of every feasible plan (weak duality, checked against the
    exact LP-free N=2 entropic plan of oracle.w1) and D = primal at convergence."""
    for (a1, b1, eps) in [(0.3, 0.6, 0.5), (0.8, 0.2, 0.2)]:
        a, b = np.array([a1, 1 - a1]), np.array([b1, 1 - b1])
        r = sinkhorn.solve(a, b, n=2, h1=1.0, eps=eps, itr_max=100000, tol=1e-15, domain="log")
        D = sinkhorn.dual_objective(a, b, r["F"][0], r["G"][0], n=2, h1=1.0, eps=eps)
        # the exact entropic plan: gamma_11 = x (w1.n2_plan), the rest by the marginals
        x, _ = w1.n2_plan(a1, b1, math.exp(-1.0 / eps))
        g = np.array([[x, a1 - x], [b1 - x, 1 - a1 - b1 + x]])
        C = np.array([[0.0, 1.0], [1.0, 0.0]])
        primal = float((g * C).sum() + eps * (g * np.log(g)).sum())
        assert D == pytest.approx(primal, rel=1e-9, abs=1e-12)
        # any other feasible plan has a larger primal value
        for t in (0.5 * x, x + 0.5 * (min(a1, b1) - x)):
            g2 = np.array([[t, a1 - t], [b1 - t, 1 - a1 - b1 + t]])
            p2 = float((g2 * C).sum() + eps * (g2 * np.log(g2)).sum())
            assert D <= p2 + 1e-12


def test_dual_objective_monotone_and_converges_to_primal():
    rng = np.random.default_rng(40)
    n, eps = 30, 0.04
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    trace = []
    sinkhorn.solve(a, b, n=n, h1=1.0 / n, eps=eps, itr_max=40, domain="log", trace=trace)
    vals = [sinkhorn.dual_objective(a, b, F[:, 0], G[:, 0], n=n, h1=1.0 / n, eps=eps) for (_, _, F, G) in trace]
    assert all(vals[i + 1] >= vals[i] - 1e-14 for i in range(len(vals) - 1))
    r = sinkhorn.solve(a, b, n=n, h1=1.0 / n, eps=eps, itr_max=100000, tol=1e-14, domain="log")
    D = sinkhorn.dual_objective(a, b, r["F"][0], r["G"][0], n=n, h1=1.0 / n, eps=eps)
    P = sinkhorn.primal_objective(r["F"][0], r["G"][0], n=n, h1=1.0 / n, eps=eps)
    assert D == pytest.approx(P, rel=1e-10) and D >= vals[-1] - 1e-14
    # 2D: the same identity on a 4 x 3 grid
    n2, m2 = 4, 3
    a2, b2 = gi.random_positive(rng, n2 * m2), gi.random_positive(rng, n2 * m2)
    kw = dict(n=n2, m=m2, h1=0.3, h2=0.2, eps=0.1)
    r2 = sinkhorn.solve(a2, b2, itr_max=100000, tol=1e-14, domain="log", **kw)
    assert sinkhorn.dual_objective(a2, b2, r2["F"][0], r2["G"][0], **kw) == pytest.approx(
        sinkhorn.primal_objective(r2["F"][0], r2["G"][0], **kw), rel=1e-10)


def test_eps_scaling_single_stage_is_plain_solve():
    rng = np.random.default_rng(41)
    n = 40
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    kw = dict(n=n, h1=1.0 / n, eps=0.02, itr_max=50)
    r1 = sinkhorn.solve_eps_scaling(a, b, eps0=0.02, factor=0.5, stage_iters=7, **kw)
    r2 = sinkhorn.solve(a, b, domain="log", **kw)
    np.testing.assert_array_equal(r1["F"], r2["F"])
    assert r1["stages"] == [0.02]


def test_eps_scaling_reaches_the_same_fixed_point():
    """Continuation changes the path, not the limit: converged to tol, the plan equals the
    direct solve's (the entropic optimum is unique) and the dual objectives agree."""
    rng = np.random.default_rng(42)
    n = 60
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    kw = dict(n=n, h1=1.0 / n, eps=0.005, itr_max=200000, tol=1e-12)
    rs = sinkhorn.solve_eps_scaling(a, b, eps0=0.16, factor=0.5, stage_iters=30, **kw)
    rd = sinkhorn.solve(a, b, domain="log", **kw)
    assert rs["stages"] == [0.16, 0.08, 0.04, 0.02, 0.01, 0.005]
    assert rs["flags"][0] == sinkhorn.CONVERGED and rd["flags"][0] == sinkhorn.CONVERGED
    D = dense.dist(n)
    gs = np.exp(rs["F"][0][:, None] + rs["G"][0][None, :] - D * (1.0 / n) / 0.005)
    gd = np.exp(rd["F"][0][:, None] + rd["G"][0][None, :] - D * (1.0 / n) / 0.005)
    np.testing.assert_allclose(gs, gd, atol=1e-10)
    assert rs["cost"][0] == pytest.approx(rd["cost"][0], rel=1e-8)
    # ... and needs fewer iterations at the target eps than the cold start
    assert rs["iters"][0] < rd["iters"][0]


# ------------------------------------------------------------------ 3D extension
def _grid3(n, m, l):
    k = np.arange(n * m * l)
    return k % n, (k // n) % m, k // (n * m)


def test_3d_apply_equals_materialised_kernel_and_brute_force():
    n, m, l = 3, 4, 2
    h1, h2, h3, eps = 0.5, 0.3, 0.7, 0.4
    ops = sinkhorn._Ops3D(n, m, l, h1, h2, h3, eps, "dense")
    rng = np.random.default_rng(30)
    x = rng.uniform(0, 1, (n * m * l, 1))
    i, j, z = _grid3(n, m, l)
    C = (np.abs(i[:, None] - i[None, :]) * h1 + np.abs(j[:, None] - j[None, :]) * h2 +
         np.abs(z[:, None] - z[None, :]) * h3)
    Kfull = np.exp(-C / eps)
    np.testing.assert_allclose(ops.K_(x)[:, 0], Kfull @ x[:, 0], rtol=1e-13)
    # Kronecker form (column-major flattening: axis 1 fastest)
    Kk = np.kron(dense.kernel(l, dense.lam(h3, eps)), np.kron(dense.kernel(m, dense.lam(h2, eps)),
                                                              dense.kernel(n, dense.lam(h1, eps))))
    np.testing.assert_allclose(Kk, Kfull, rtol=1e-13)
    phi, psi = rng.uniform(0.1, 1, (n * m * l, 1)), rng.uniform(0.1, 1, (n * m * l, 1))
    cost_bf = float(phi[:, 0] @ ((Kfull * C) @ psi[:, 0]))
    assert ops.cost(phi, psi)[0] == pytest.approx(cost_bf, rel=1e-13)


def test_3d_with_one_layer_is_2d():
    rng = np.random.default_rng(31)
    n, m = 5, 4
    a, b = gi.random_positive(rng, n * m), gi.random_positive(rng, n * m)
    kw = dict(n=n, m=m, h1=0.2, h2=0.3, eps=0.1, itr_max=15)
    r2 = sinkhorn.solve(a, b, **kw)
    r3 = sinkhorn.solve(a, b, l=1, h3=0.9, **kw)
    np.testing.assert_array_equal(r2["F"], r3["F"])
    # a genuinely 3D grid whose third axis is decoupled (h3 huge: lambda3 = 0) is a
    # stack of independent 2D problems only in the kernel; with both layers carrying the
    # same mass pattern the plan is block-diagonal and the cost is the 2D cost
    r3b = sinkhorn.solve(np.concatenate([a, a]) / 2, np.concatenate([b, b]) / 2, l=2, h3=1e6, **kw)
    assert r3b["cost"][0] == pytest.approx(r2["cost"][0], rel=1e-10)


def test_3d_converged_cost_sandwich():
    """At convergence the 3D entropic cost is >= the exact l1 OT cost (LP on the 8-point
    grid) and within eps * min(H) of it."""
    rng = np.random.default_rng(32)
    n, m, l = 2, 2, 2
    N = n * m * l
    a, b = gi.random_positive(rng, N), gi.random_positive(rng, N)
    h1, h2, h3, eps = 0.3, 0.2, 0.4, 0.02
    i, j, z = _grid3(n, m, l)
    C = (np.abs(i[:, None] - i[None, :]) * h1 + np.abs(j[:, None] - j[None, :]) * h2 +
         np.abs(z[:, None] - z[None, :]) * h3).ravel()
    Aeq = np.vstack([np.kron(np.eye(N), np.ones(N)), np.kron(np.ones(N), np.eye(N))])
    lp = scipy.optimize.linprog(C, A_eq=Aeq, b_eq=np.concatenate([a, b]), method="highs").fun
    r = sinkhorn.solve(a, b, n=n, m=m, l=l, h1=h1, h2=h2, h3=h3, eps=eps, itr_max=200000, tol=1e-13)
    assert r["flags"][0] == sinkhorn.CONVERGED
    gap = r["cost"][0] - lp
    assert -1e-9 <= gap <= eps * min(w1.entropy(a), w1.entropy(b)) + 1e-9
