"""Pins for the oracle of the paper's stabilised FS-1 (Remark 2.1 + Remark 3.2,
PAPER.md:100-108, 217-232; oracle/stabilized.py, oracle/recur.c fs1o_stab_sweep).

Pinned against: the materialised rescaled kernel diag(e^A) K diag(e^B) (the definition
Remark 3.2's recursions rewrite), the plain recursion when nothing is absorbed, absorption
transparency (SPEC.md:541-style: absorbing at arbitrary iterations changes no plan entry),
the unstabilised scaling-domain oracle when no absorption fires, and the independent
log-sum-exp log-domain oracle on the paper's Ricker workload at eps = 1e-3, where the
unstabilised iteration terminates abnormally.
"""
import numpy as np
import pytest

import fs1_inputs as gi
from oracle import dense, recur, sinkhorn
from oracle import stabilized as st


@pytest.mark.parametrize("n", [1, 2, 3, 17, 64])
@pytest.mark.parametrize("lam", [0.0, 0.1, 0.5, 0.9, 0.999])
def test_stab_sweep_equals_rescaled_kernel(n, lam):
    """Remark 3.2's lines 5-6 / 10-11 compute diag(e^own) K diag(e^other) x (R8)."""
    rng = np.random.default_rng(100 + n)
    x = rng.uniform(0.1, 2.0, n)
    own, other = rng.uniform(-3, 3, n), rng.uniform(-3, 3, n)
    y = recur.stab_sweep(x, own, other, lam)
    ref = st.stab_apply_dense(x, own, other, lam)
    np.testing.assert_allclose(y, ref, rtol=1e-12, atol=0)
    # pure-Python brute force of the same sum
    bf = np.array([sum(np.exp(own[k]) * lam ** abs(k - j) * np.exp(other[j]) * x[j] for j in range(n))
                   for k in range(n)])
    np.testing.assert_allclose(y, bf, rtol=1e-12, atol=0)


def test_stab_sweep_reduces_to_plain_recursion():
    """alpha = beta = 0: every factor is exactly 1 (SPEC.md stabilized_fast_apply_1d example)."""
    rng = np.random.default_rng(7)
    for n in (1, 5, 300):
        x = rng.uniform(0, 1, n)
        z = np.zeros(n)
        np.testing.assert_array_equal(recur.stab_sweep(x, z, z, 0.83), recur.sweep(x, 0.83))


def test_stab_sweep_n1():
    assert recur.stab_sweep(np.array([0.7]), np.array([0.3]), np.array([-1.1]), 0.5)[0] == \
        pytest.approx(np.exp(0.3 - 1.1) * 0.7, rel=1e-15)


def test_stab_sweep_transposes():
    """The psi side (own = B, other = A) is the transpose of the phi side (own = A,
    other = B): <y, K~ x> = <K~^T y, x>."""
    rng = np.random.default_rng(8)
    n = 50
    A, B = rng.uniform(-2, 2, n), rng.uniform(-2, 2, n)
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    lhs = y @ recur.stab_sweep(x, A, B, 0.7)
    rhs = recur.stab_sweep(y, B, A, 0.7) @ x
    assert lhs == pytest.approx(rhs, rel=1e-13)


def _pair(n, seed):
    rng = np.random.default_rng(seed)
    return gi.random_positive(rng, n), gi.random_positive(rng, n)


def test_no_absorption_equals_plain_oracle():
    """tau = inf: the stabilised loop is Algorithm 1 itself (every factor = 1)."""
    n = 80
    a, b = _pair(n, 1)
    kw = dict(n=n, eps=0.02, itr_max=60)
    r = st.solve_stab(a, b, h=1.0 / n, tau=np.inf, **kw)
    ref = sinkhorn.solve(a, b, h1=1.0 / n, **kw)
    assert r["absorptions"] == [] and r["flags"][0] == sinkhorn.ITR_MAX
    np.testing.assert_allclose(r["F"], ref["F"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(r["G"], ref["G"], rtol=1e-12, atol=1e-12)
    assert r["cost"][0] == pytest.approx(ref["cost"][0], rel=1e-12)
    assert r["err"][0] == pytest.approx(ref["err"][0], rel=1e-10)


@pytest.mark.parametrize("trial", range(20))
def test_absorption_transparency(trial):
    """Absorbing at arbitrary iterations leaves every plan entry and the cost unchanged
    (SPEC.md:541 criterion 8: N = 64, 50 iterations, 1e-10)."""
    n = 64
    a, b = _pair(n, 1000 + trial)
    rng = np.random.default_rng(trial)
    at = set(rng.choice(np.arange(1, 50), size=rng.integers(1, 12), replace=False).tolist())
    kw = dict(n=n, h=1.0 / n, eps=0.03, itr_max=50)
    r0 = st.solve_stab(a, b, tau=np.inf, **kw)
    r1 = st.solve_stab(a, b, tau=np.inf, absorb_at=at, **kw)
    assert sorted(r1["absorptions"]) == sorted(at)
    g0 = r0["F"][0][:, None] + r0["G"][0][None, :]
    g1 = r1["F"][0][:, None] + r1["G"][0][None, :]
    np.testing.assert_allclose(np.exp(g1), np.exp(g0), rtol=1e-10, atol=0)
    assert r1["cost"][0] == pytest.approx(r0["cost"][0], rel=1e-10)
    assert r1["err"][0] == pytest.approx(r0["err"][0], rel=1e-8, abs=1e-14)


def test_absorb_keeps_plan():
    rng = np.random.default_rng(3)
    n = 10
    A, B = rng.uniform(-5, 5, n), rng.uniform(-5, 5, n)
    phi, psi = rng.uniform(0.1, 1e6, n), rng.uniform(1e-3, 10, n)
    A2, B2, p2, q2 = st.absorb(A, B, phi, psi)
    assert np.all(p2 == 1) and np.all(q2 == 1)
    np.testing.assert_allclose(np.exp(A2), np.exp(A) * phi, rtol=1e-14)
    np.testing.assert_allclose(np.exp(B2), np.exp(B) * psi, rtol=1e-14)


@pytest.mark.parametrize("n", [500, 2000])
def test_ricker_eps_1e3_stabilised_vs_log_domain(n):
    """at eps = 1e-3 the unstabilised iteration terminates abnormally; the
    stabilised one runs all iterations (absorbing repeatedly) and is the same iteration as
    the independent log-sum-exp oracle."""
    a, b = gi.ricker_pair(n)
    h, eps, itr = 8.0 / (n - 1), 1e-3, 2000
    un = sinkhorn.solve(a, b, n=n, h1=h, eps=eps, itr_max=itr, apply="recur")
    assert un["flags"][0] == sinkhorn.NONFINITE and un["iters"][0] < itr
    r = st.solve_stab(a, b, n=n, h=h, eps=eps, itr_max=itr)
    assert r["flags"][0] == sinkhorn.ITR_MAX and r["iters"][0] == itr and len(r["absorptions"]) > 10
    ref = sinkhorn.solve(a, b, n=n, h1=h, eps=eps, itr_max=itr, domain="log", apply="recur")
    for k in ("F", "G"):
        e = np.max(np.abs(r[k] - ref[k])) / max(np.max(np.abs(ref[k])), 1.0)
        assert e <= 1e-12, (k, e)
    assert r["cost"][0] == pytest.approx(ref["cost"][0], rel=1e-12)
    assert r["err"][0] == pytest.approx(ref["err"][0], rel=1e-9)


def test_stabilised_tolerance_stop():
    """err <= tol stops the stabilised loop (line 2 with the rescaled kernel) and the run
    replays at the same l* with tol = 0."""
    n = 120
    a, b = _pair(n, 5)
    kw = dict(n=n, h=1.0 / n, eps=0.01)
    r1 = st.solve_stab(a, b, itr_max=20000, tol=1e-9, tau=1e3, **kw)
    assert r1["flags"][0] == sinkhorn.CONVERGED and r1["err"][0] <= 1e-9 and r1["absorptions"]
    r2 = st.solve_stab(a, b, itr_max=int(r1["iters"][0]), tau=1e3, **kw)
    np.testing.assert_array_equal(r1["F"], r2["F"])
    assert r1["cost"][0] == r2["cost"][0]
