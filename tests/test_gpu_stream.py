"""GPU parity of the multi-CTA streaming kernel (K2) against the oracle.

K2 is the fp64 path for one large 1D problem (config C3, N = 2^24).  The plan
picks it automatically above the persistent kernel's capacity; here the
test-only plan override (kernel=2) also drives it at small and ragged sizes:
one tile, one tile per CTA, ragged last tiles, fewer tiles than SMs, and the
full C3 size.  The oracle is the dense definition where it is feasible and the
plain-C recursion (itself pinned equal to dense, test_oracle_apply.py) above.
"""
import math

import numpy as np
import pytest

import fs1_inputs as gi
from oracle import dense, recur, sinkhorn
from tests.gpu_util import assert_solve_parity, rel, rel_norm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402

K2 = 2
TOL64 = 1e-10


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def _ref_log_apply(X, c):
    """(reference, tolerance): dense LSE, or the recursion oracle (extended-precision
    accumulator, R24) where dense is infeasible."""
    if X.size <= 8192:
        return dense.apply_log(X, c), 1e-13
    return recur.sweep_log(X, c), 1e-13


# ------------------------------------------------------------------ kernel apply
APPLY_N = [1, 2, 255, 256, 257, 1000, 4109, 40000, 300001]


@pytest.mark.parametrize("n", APPLY_N)
@pytest.mark.parametrize("c", [6e-4, 0.1, 3.0])
def test_stream_apply_log(n, c):
    rng = np.random.default_rng(n + int(c * 1e4))
    X = np.cumsum(rng.normal(scale=0.3, size=n)) + rng.normal(size=n)
    y = fs1.apply(_cuda(X[None]), h=c, eps=1.0, domain="log", kernel=K2).cpu().numpy()[0]
    ref, tol = _ref_log_apply(X, c)
    assert rel_norm(y, ref) <= tol


@pytest.mark.parametrize("n", [3, 256, 1000, 4109])
def test_stream_apply_scaling(n):
    rng = np.random.default_rng(n)
    x = rng.uniform(0.1, 1.0, size=n)
    for c in [0.01, 0.5, 2.0]:
        lam = math.exp(-c)
        y = fs1.apply(_cuda(x[None]), h=c, eps=1.0, domain="scaling", kernel=K2).cpu().numpy()[0]
        ref = dense.kernel(n, lam) @ x
        assert np.max(np.abs(y / ref - 1.0)) <= 1e-13


def test_stream_apply_wide_range_and_zeros():
    """Log inputs spanning 1e4 nats with -inf runs: the extended-range carries keep
    every term (Remark 3.3) and -inf stays -inf only where the whole row is empty."""
    n = 70000
    x = np.linspace(0, 1, n)
    X = 4000 * np.sin(7 * x) - 3000 * x
    X[1000:5000] = -np.inf
    c = 2e-3
    y = fs1.apply(_cuda(X[None]), h=c, eps=1.0, domain="log", kernel=K2).cpu().numpy()[0]
    ref = recur.sweep_log(X, c)
    assert np.all(np.isfinite(y))
    assert rel_norm(y, ref) <= 1e-13


# ------------------------------------------------------------------ solve
SOLVE = [  # n, eps, itr, input_is_log
    (1, 0.01, 5, False),
    (3, 0.05, 20, False),
    (257, 1e-2, 40, False),
    (1000, 2e-3, 60, True),
    (3001, 1e-3, 30, True),
    (20000, 1e-4, 25, True),
]


def _pair(n, log):
    rng = np.random.default_rng(n)
    x = (np.arange(n) + 0.5) / n
    mu = rng.uniform(0.1, 0.9, size=(2, 3))
    sd = rng.uniform(0.02, 0.1, size=(2, 3))
    out = []
    for k in range(2):
        comp = -0.5 * ((x[None] - mu[k][:, None]) / sd[k][:, None]) ** 2 - np.log(sd[k])[:, None]
        la = np.logaddexp.reduce(comp, axis=0)
        la = la - np.logaddexp.reduce(la)
        out.append(la if log else np.exp(la))
    return out


@pytest.mark.parametrize("n,eps,itr,lg", SOLVE)
def test_stream_solve_parity(n, eps, itr, lg):
    a, b = _pair(n, lg)
    out = fs1.solve(_cuda(a[None]), _cuda(b[None]), h=1 / n, eps=eps, itr_max=itr, domain="log",
                    input_is_log=lg, kernel=K2)
    ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=eps, itr_max=itr, domain="log", input_is_log=lg,
                         apply="dense" if n <= 3001 else "recur")
    assert_solve_parity(out, ref, "log", "f64", tol=TOL64)


def test_stream_equals_persistent_kernel():
    """Both fp64 log-domain kernels on the same problem (n = 8192 fits both)."""
    n = 8192
    a, b = _pair(n, True)
    kw = dict(h=1 / n, eps=5e-4, itr_max=50, domain="log", input_is_log=True)
    o2 = fs1.solve(_cuda(a[None]), _cuda(b[None]), kernel=K2, **kw)
    o1 = fs1.solve(_cuda(a[None]), _cuda(b[None]), kernel=1, **kw)
    F1, F2 = o1["u"].cpu().numpy(), o2["u"].cpu().numpy()
    assert rel_norm(F2[0], F1[0]) <= 1e-12
    assert rel(o2["cost"].item(), o1["cost"].item()) <= 1e-12


def test_stream_tolerance_stop_and_replay():
    n = 2000
    a, b = _pair(n, False)
    for ci in (1, 7):
        out = fs1.solve(_cuda(a[None]), _cuda(b[None]), h=1 / n, eps=1e-2, itr_max=5000, tol=1e-9,
                        check_interval=ci, domain="log", kernel=K2)
        ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=1e-2, itr_max=5000, tol=1e-9, check_interval=ci,
                             domain="log")
        assert abs(int(out["iters"].item()) - int(ref["iters"][0])) <= ci
        assert out["flags"].item() == 1 and out["err"].item() <= 1e-9
    # fixed-iteration replay at the oracle's l* (R22)
    ls = int(ref["iters"][0])
    out = fs1.solve(_cuda(a[None]), _cuda(b[None]), h=1 / n, eps=1e-2, itr_max=ls, domain="log", kernel=K2)
    r2 = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=1e-2, itr_max=ls, domain="log")
    assert_solve_parity(out, r2, "log", "f64", tol=TOL64)


def test_stream_cost_entry_point():
    n = 3000
    rng = np.random.default_rng(3)
    F = np.cumsum(rng.normal(scale=0.2, size=n)) - 8
    G = np.cumsum(rng.normal(scale=0.2, size=n)) - 8
    eps = 3e-3
    c = fs1.cost(_cuda(F[None]), _cuda(G[None]), h=1 / n, eps=eps, domain="log", kernel=K2).item()
    D = dense.dist(n)
    ref = float(np.sum(np.exp(F[:, None] + G[None, :] - (1 / n / eps) * D) * D * (1 / n)))
    assert rel(c, ref) <= 1e-12


def test_stream_warm_start_resume_and_batch():
    n = 5000
    a, b = _pair(n, True)
    kw = dict(h=1 / n, eps=1e-3, domain="log", input_is_log=True, kernel=K2)
    full = fs1.solve(_cuda(a[None]), _cuda(b[None]), itr_max=30, **kw)
    part = fs1.solve(_cuda(a[None]), _cuda(b[None]), itr_max=12, **kw)
    rest = fs1.solve(_cuda(a[None]), _cuda(b[None]), itr_max=18, u0=part["u"], v0=part["v"], **kw)
    assert rel_norm(rest["u"].cpu().numpy()[0], full["u"].cpu().numpy()[0]) <= 1e-13
    # two problems in one call == one at a time
    A = np.stack([a, b])
    B = np.stack([b, a])
    two = fs1.solve(_cuda(A), _cuda(B), itr_max=30, **kw)
    assert np.array_equal(two["u"].cpu().numpy()[0], full["u"].cpu().numpy()[0])
    assert two["cost"].cpu().numpy()[0] == full["cost"].item()


def test_stream_determinism():
    n = 100000
    a, b = _pair(n, True)
    kw = dict(h=1 / n, eps=1e-4, itr_max=20, domain="log", input_is_log=True, kernel=K2)
    o1 = fs1.solve(_cuda(a[None]), _cuda(b[None]), **kw)
    o2 = fs1.solve(_cuda(a[None]), _cuda(b[None]), **kw)
    assert np.array_equal(o1["u"].cpu().numpy(), o2["u"].cpu().numpy())
    assert o1["cost"].item() == o2["cost"].item() and o1["err"].item() == o2["err"].item()


# ------------------------------------------------------------------ config 3 at full size
def _c3_inputs():
    cfg = gi.CONFIGS["c3"]
    a, b = gi.pair(cfg, 0)
    return cfg, a, b


def test_config3_trajectory_full_size():
    """N = 2^24 for 3 iterations: every potential against the recursion oracle."""
    cfg, a, b = _c3_inputs()
    out = fs1.solve(_cuda(a[None]), _cuda(b[None]), h=cfg.h1, eps=cfg.eps, itr_max=3, domain="log",
                    input_is_log=True)
    assert fs1.plan(fs1.Spec(ndim=1, n=cfg.n, m=1, h1=cfg.h1, h2=0.0, eps=cfg.eps, batch=1,
                             dtype=torch.float64, domain="log", input_is_log=True, itr_max=3)
                    ).info()["kernel"].startswith("stream")
    ref = sinkhorn.solve(a, b, n=cfg.n, h1=cfg.h1, eps=cfg.eps, itr_max=3, domain="log", input_is_log=True,
                         apply="recur")
    assert_solve_parity(out, ref, "log", "f64", tol=TOL64)


def test_config3_full_run_properties():
    """The bench's launch (N = 2^24, 1000 iterations): the last phi half-step, the exit
    error and the cost are recomputed by the oracle from the GPU's final state."""
    cfg, a, b = _c3_inputs()
    out = fs1.solve(_cuda(a[None]), _cuda(b[None]), h=cfg.h1, eps=cfg.eps, itr_max=cfg.itr_max,
                    domain="log", input_is_log=True)
    F = out["u"].cpu().numpy()[0]
    G = out["v"].cpu().numpy()[0]
    c = cfg.h1 / cfg.eps
    assert out["iters"].item() == cfg.itr_max and out["flags"].item() == 4
    # line 12: F = log a - log K e^G, elementwise over all 2^24 points
    Fr = a - recur.sweep_log(G, c)
    assert rel_norm(F, Fr) <= 1e-12
    # line 2 at exit: err = sum |e^{G + log K e^F} - b|
    T = recur.sweep_log(F, c)
    err = float(np.sum(np.abs(np.exp(G + T) - np.exp(b))))
    assert abs(out["err"].item() - err) <= 1e-10 * max(1.0, err)
    # line 14: cost
    ref = recur.sum_exp2(F, recur.wsweep_log(G, c, cfg.h1))
    assert rel(out["cost"].item(), ref) <= TOL64
