"""Pins for the oracle's kernel applies (CPU only).

Each test checks the oracle against something other than itself: worked
examples (tests/golden/spec_examples.json), brute force, a second algorithm
(the paper's recursion vs the dense product), the stability bound the paper
derives, calculus identities, and symmetry/linearity.
"""
import json
import math
import os

import numpy as np
import pytest

from oracle import dense, recur

LAMS = [0.0, 0.1, 0.5, 0.9, 0.999]


@pytest.fixture(scope="module")
def gold(golden_dir):
    with open(os.path.join(golden_dir, "spec_examples.json")) as f:
        return json.load(f)


def test_lambda_examples(gold):
    for e in gold["lambda"]:
        assert dense.lam(e["h"], e["eps"]) == pytest.approx(e["lam"], rel=1e-15)
    with pytest.raises(ValueError):
        dense.lam(1.0, 0.0)


def test_apply_examples(gold):
    for e in gold["apply_1d"]:
        x = np.array(e["x"], float)
        np.testing.assert_allclose(dense.apply(x, e["lam"]), e["y"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(recur.sweep(x, e["lam"]), e["y"], rtol=0, atol=1e-15)


def test_weighted_examples(gold):
    for e in gold["weighted_1d"]:
        x = np.array(e["x"], float)
        np.testing.assert_allclose(dense.weighted_apply(x, e["lam"], e["h"]), e["y"], atol=1e-15)
        if e["lam"] > 0:
            with np.errstate(divide="ignore"):
                y = np.exp(recur.wsweep_log(np.log(x), -math.log(e["lam"]), e["h"]))
            np.testing.assert_allclose(y, e["y"], atol=1e-15)


def test_2d_examples(gold):
    for e in gold["apply_2d"]:
        X = np.array(e["X"], float)
        np.testing.assert_allclose(dense.apply_2d(X, e["lam1"], e["lam2"]), e["Y"], atol=1e-15)
        Y = recur.sweep(recur.sweep(X, e["lam1"], axis=1), e["lam2"], axis=2)
        np.testing.assert_allclose(Y, e["Y"], atol=1e-15)


def test_dense_vs_bruteforce_python_loops():
    rng = np.random.default_rng(1)
    for n in [1, 2, 5, 13]:
        x = rng.standard_normal(n)
        for lam in LAMS:
            y = [sum(x[j] * lam ** abs(k - j) for j in range(n)) for k in range(n)]
            np.testing.assert_allclose(dense.apply(x, lam), y, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("n", [1, 2, 3, 17, 256, 1024])
@pytest.mark.parametrize("lam", LAMS)
def test_recursion_equals_dense(n, lam):
    """Eq. (recursion) PAPER.md:129-137 == Eq. (3.1) PAPER.md:113-122."""
    rng = np.random.default_rng(n)
    x = rng.uniform(0, 1, n)
    yd = dense.apply(x, lam)
    yr = recur.sweep(x, lam)
    assert np.max(np.abs(yr - yd)) <= 1e-12 * np.max(np.abs(yd))


@pytest.mark.parametrize("n", [1, 2, 9, 300])
@pytest.mark.parametrize("c", [0.01, 0.5, 3.0, 40.0])
def test_log_apply(n, c):
    rng = np.random.default_rng(7 + n)
    X = rng.uniform(-20, 5, n)
    ref = np.log(dense.apply(np.exp(X), math.exp(-c)))
    np.testing.assert_allclose(dense.apply_log(X, c), ref, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(recur.sweep_log(X, c), ref, rtol=1e-13, atol=1e-13)


def test_log_apply_with_zero_mass():
    X = np.array([-np.inf, 0.0, -np.inf, -np.inf, 1.0])
    c = 0.7
    ref = np.log(dense.apply(np.exp(X), math.exp(-c)))
    np.testing.assert_allclose(dense.apply_log(X, c), ref, rtol=1e-14)
    np.testing.assert_allclose(recur.sweep_log(X, c), ref, rtol=1e-14)
    assert np.all(np.isneginf(recur.sweep_log(np.full(4, -np.inf), c)))


@pytest.mark.parametrize("lam", [0.1, 0.5, 0.9, 0.99])
@pytest.mark.parametrize("delta", [1e-6, 1e-3])
def test_stability_bound(lam, delta):
    """|Delta(Kx)_k| <= ((2 - lam^k - lam^{N-k+1})/(1-lam) - 1) delta;
    equality when every perturbation is +delta (the bound is (K 1)_k delta)."""
    n = 64
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, n)
    k = np.arange(1, n + 1)
    bound = ((2 - lam ** k - lam ** (n - k + 1)) / (1 - lam) - 1) * delta
    d_same = recur.sweep(x + delta, lam) - recur.sweep(x, lam)
    np.testing.assert_allclose(d_same, bound, rtol=1e-6)
    for _ in range(5):
        d = rng.uniform(-delta, delta, n)
        diff = np.abs(recur.sweep(x + d, lam) - recur.sweep(x, lam))
        assert np.all(diff <= bound * (1 + 1e-9) + 1e-15)


def test_symmetry_and_linearity():
    rng = np.random.default_rng(11)
    x, z = rng.uniform(0, 1, 200), rng.uniform(0, 1, 200)
    lam = 0.83
    np.testing.assert_allclose(recur.sweep(x[::-1], lam)[::-1], recur.sweep(x, lam), rtol=1e-13)
    np.testing.assert_allclose(recur.sweep(2 * x - 3 * z, lam),
                               2 * recur.sweep(x, lam) - 3 * recur.sweep(z, lam), rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("lam", [0.2, 0.7, 0.95])
def test_weighted_kernel_is_lambda_derivative(lam):
    """W = h lam dK/dlam (d/dlam lam^d = d lam^{d-1}): pins the weighted kernel of the
    return line by a central difference of the plain kernel."""
    n, h = 40, 0.01
    dl = 1e-6
    dK = (dense.kernel(n, lam + dl) - dense.kernel(n, lam - dl)) / (2 * dl)
    np.testing.assert_allclose(dense.weighted_kernel(n, lam, h), h * lam * dK, rtol=1e-7, atol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 7, 100])
def test_weighted_recursion_equals_dense(n):
    rng = np.random.default_rng(n)
    x = rng.uniform(0.1, 1, n)
    c, h = 0.3, 0.01
    ref = dense.weighted_apply(x, math.exp(-c), h)
    got = np.exp(recur.wsweep_log(np.log(x), c, h))
    np.testing.assert_allclose(got, ref, rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(np.exp(dense.weighted_apply_log(np.log(x), c, h)), ref, rtol=1e-13)


def test_2d_kronecker_identity():
    """K = [lam2^{|k-l|} K0] on column-major vectors equals T_N X T_M."""
    rng = np.random.default_rng(5)
    for n, m in [(1, 1), (1, 6), (5, 1), (8, 7), (16, 16)]:
        X = rng.uniform(0, 1, (n, m))
        l1, l2 = 0.6, 0.3
        full = dense.kernel_2d(n, m, l1, l2) @ X.T.ravel()
        np.testing.assert_allclose(dense.apply_2d(X, l1, l2).T.ravel(), full, rtol=1e-13)
        Y = recur.sweep(recur.sweep(X, l1, axis=1), l2, axis=2)
        np.testing.assert_allclose(Y.T.ravel(), full, rtol=1e-13)


def test_2d_degenerate_axes():
    rng = np.random.default_rng(6)
    X = rng.uniform(0, 1, (9, 4))
    # lam2 = 0: columns independent
    Y = dense.apply_2d(X, 0.4, 0.0)
    for j in range(4):
        np.testing.assert_allclose(Y[:, j], dense.apply(X[:, j], 0.4), rtol=1e-14)
    # N = 1: 1D along the row
    R = rng.uniform(0, 1, (1, 11))
    np.testing.assert_allclose(dense.apply_2d(R, 0.4, 0.8)[0], dense.apply(R[0], 0.8), rtol=1e-14)


def test_2d_log_apply():
    rng = np.random.default_rng(8)
    X = rng.uniform(-5, 0, (6, 5))
    c1, c2 = 0.4, 1.3
    ref = np.log(dense.apply_2d(np.exp(X), math.exp(-c1), math.exp(-c2)))
    np.testing.assert_allclose(dense.apply_2d_log(X, c1, c2), ref, rtol=1e-13)
    Y = recur.sweep_log(recur.sweep_log(X, c1, axis=1), c2, axis=2)
    np.testing.assert_allclose(Y, ref, rtol=1e-13)


def test_2d_cost_separable_equals_quadruple_sum():
    """Alg. 2 return line: the separable evaluation used by the oracle
    equals the literal quadruple sum."""
    from oracle.sinkhorn import _Ops2D
    rng = np.random.default_rng(9)
    n, m = 6, 5
    P, S = rng.uniform(0, 1, (n, m)), rng.uniform(0, 1, (n, m))
    eps, h1, h2 = 0.7, 0.3, 0.2
    l1, l2 = math.exp(-h1 / eps), math.exp(-h2 / eps)
    ref = dense.cost_2d_bruteforce(P, S, l1, l2, h1, h2)
    for mode in ["dense", "recur"]:
        ops = _Ops2D(n, m, h1, h2, eps, mode)
        got = ops.cost(P.T.ravel()[:, None], S.T.ravel()[:, None])[0]
        assert got == pytest.approx(ref, rel=1e-13)
        got = ops.cost_log(np.log(P.T.ravel())[:, None], np.log(S.T.ravel())[:, None])[0]
        assert got == pytest.approx(ref, rel=1e-13)
    # h1 = h2 = 0 -> 0
    assert dense.cost_2d_bruteforce(P, S, 1.0, 1.0, 0.0, 0.0) == 0.0


def test_log_recursion_accumulator_precision():
    """The LSE recursion oracle at config-3-like magnitudes (|X| ~ 5e3, c ~ 6e-4, memory
    1/(1 - lambda) ~ 1700) stays within a few ulp of |y| of the dense definition: its
    extended-precision accumulator removes the fp64 drift (R24)."""
    n = 6000
    x = np.linspace(0.0, 1.0, n)
    X = 5000.0 * np.sin(3.0 * x) - 2000.0 * x
    c = 6e-4
    y = recur.sweep_log(X, c)
    ref = dense.apply_log(X, c)
    assert np.max(np.abs(y - ref)) / np.max(np.abs(ref)) <= 2e-15
