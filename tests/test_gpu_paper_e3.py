"""The paper's 2D random-distribution workload (E3, Table 3) on the GPU:
K5, Algorithm 2 in fp64 (scaling domain, the paper's unstabilised FS-1), against the
oracle's dense Algorithm 2 (oracle/sinkhorn.py, K = T_M (x) T_N applied per axis).

N x N for N = 10 ... 160, h1 = h2 = 1, eps = 0.01 (lambda = e^{-100}: fp32 cannot hold it),
u, v iid U[0,1] normalised, the full 1000 iterations.  Column 5 of Table 3 (the Frobenius
norm between the FS-1 and the dense Sinkhorn transport plans, 1e-17 .. 1e-18 there) is
reproduced as the Frobenius norm between the GPU's plan (fs1_transport_plan) and the
oracle's dense-Sinkhorn plan.
"""
import numpy as np
import pytest

import fs1_inputs as gi
from oracle import dense, sinkhorn
from tests.gpu_util import assert_solve_parity, rel, rel_norm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402


def _solve(cfg, A, B, itr=None, **kw):
    return fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), h=cfg.h1, h2=cfg.h2,
                     shape=(cfg.n, cfg.m), eps=cfg.eps, itr_max=cfg.itr_max if itr is None else itr,
                     domain="scaling", **kw)


def _ref(cfg, A, B, itr=None, **kw):
    return sinkhorn.solve(A, B, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps,
                          itr_max=cfg.itr_max if itr is None else itr, **kw)


@pytest.mark.parametrize("name", ["e3_10", "e3_20", "e3_40", "e3_80", "e3_160"])
def test_e3_full_protocol(name):
    cfg = gi.CONFIGS[name]
    A, B = gi.batch(cfg, range(2))
    out = _solve(cfg, A, B)
    ref = _ref(cfg, A, B)
    assert fs1.plan(fs1.Spec(ndim=2, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, batch=2,
                             dtype=torch.float64, itr_max=cfg.itr_max)).info()["kernel"].startswith("sep2d64")
    assert_solve_parity(out, ref, "scaling", "f64")


@pytest.mark.parametrize("name", ["e3_10", "e3_20", "e3_40", "e3_80"])
def test_e3_plan_frobenius(name):
    """Table 3 column 5: ||P_FS1 - P_Sinkhorn||_F at rounding level (the paper: 1.2e-17 at
    10x10 down to 7.7e-19 at 160x160)."""
    cfg = gi.CONFIGS[name]
    A, B = gi.batch(cfg, range(1))
    out = _solve(cfg, A, B)
    ref = _ref(cfg, A, B)
    g = fs1.transport_plan(out["u"], out["v"], h=cfg.h1, h2=cfg.h2, eps=cfg.eps, shape=(cfg.n, cfg.m))
    Pg = g[0].cpu().numpy()
    # the oracle's dense plan gamma = diag(phi) K diag(psi), K = T_M (x) T_N (column-major)
    K = np.kron(dense.kernel(cfg.m, dense.lam(cfg.h2, cfg.eps)), dense.kernel(cfg.n, dense.lam(cfg.h1, cfg.eps)))
    phi, psi = np.exp(ref["F"][0]), np.exp(ref["G"][0])
    Po = phi[:, None] * K * psi[None, :]
    d = np.linalg.norm(Pg - Po)
    assert d <= 1e-14, d
    # marginals of the plan: the u-marginal is exact after the phi update
    np.testing.assert_allclose(Po.sum(1), A[0], rtol=1e-9, atol=1e-15)


def test_tolerance_stop_and_apply():
    """tol-stopped 2D fp64 run (R22) on a smaller-c case that converges, and the plain K x."""
    cfg = gi.CONFIGS["e3_20"]
    A, B = gi.batch(cfg, range(1))
    kw = dict(h=0.05, h2=0.05, shape=(20, 20), eps=0.02, domain="scaling")
    ref = sinkhorn.solve(A, B, n=20, m=20, h1=0.05, h2=0.05, eps=0.02, itr_max=20000, tol=1e-10)
    assert ref["flags"][0] == 1
    out = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), itr_max=20000, tol=1e-10, **kw)
    assert out["flags"].item() == 1 and abs(out["iters"].item() - ref["iters"][0]) <= 1
    x = np.random.default_rng(3).uniform(0, 1, (3, 20 * 20))
    y = fs1.apply(torch.from_numpy(x).cuda(), h=0.05, h2=0.05, shape=(20, 20), eps=0.02).cpu().numpy()
    K = np.kron(dense.kernel(20, dense.lam(0.05, 0.02)), dense.kernel(20, dense.lam(0.05, 0.02)))
    np.testing.assert_allclose(y, x @ K.T, rtol=1e-13)
    c = fs1.cost(out["u"], out["v"], h=0.05, h2=0.05, shape=(20, 20), eps=0.02)
    assert rel(c.item(), out["cost"].item()) <= 1e-13


@pytest.mark.parametrize("shape", [(1, 1), (1, 7), (7, 1), (31, 33), (33, 64), (100, 3)])
def test_ragged_shapes(shape):
    n, m = shape
    rng = np.random.default_rng(n * 100 + m)
    A, B = gi.random_positive(rng, (3, n * m)), gi.random_positive(rng, (3, n * m))
    kw = dict(h=1.0 / n, h2=1.0 / m, shape=(n, m), eps=0.03, itr_max=60, domain="scaling")
    out = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), **kw)
    ref = sinkhorn.solve(A, B, n=n, m=m, h1=1.0 / n, h2=1.0 / m, eps=0.03, itr_max=60)
    assert_solve_parity(out, ref, "scaling", "f64")


@pytest.mark.parametrize("shape", [(10, 10), (33, 64), (160, 160), (64, 200), (1, 256), (256, 3)])
def test_warp_line_variant_equals_thread_line_kernel(shape):
    """K5w (one warp per line, chunked scan with two-factor multipliers) against K5's
    sequential thread-per-line recursion (test-only kind 5) and the oracle, at E3's
    lambda = e^{-100} and at a moderate lambda."""
    n, m = shape
    rng = np.random.default_rng(n + 7 * m)
    A, B = gi.random_positive(rng, (2, n * m)), gi.random_positive(rng, (2, n * m))
    for h, eps, itr in ((1.0, 0.01, 200), (1.0 / max(n, m), 0.05, 60)):
        kw = dict(h=h, h2=h, shape=(n, m), eps=eps, itr_max=itr, domain="scaling")
        w = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), **kw)
        t = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), kernel=5, **kw)
        ref = sinkhorn.solve(A, B, n=n, m=m, h1=h, h2=h, eps=eps, itr_max=itr)
        assert_solve_parity(w, ref, "scaling", "f64")
        assert_solve_parity(t, ref, "scaling", "f64")
    info = fs1.plan(fs1.Spec(ndim=2, n=n, m=m, h1=h, h2=h, eps=eps, batch=2, dtype=torch.float64,
                             itr_max=itr)).info()
    assert info["kernel"].startswith("sep2d64w")


def test_nonfinite_returns_the_stopping_state():
    """K5w stores phi, psi only before checks; a problem that overflows replays from the
    last stored state so that u, v still hold the state at which it stopped (fs1.h).
    h = 1, eps = 2e-3: the unstabilised iteration overflows after a few hundred
    iterations; NONFINITE at the oracle's iteration (as the thread-per-line kernel), and
    the returned state is the one that tripped the check: a non-finite phi or psi entry
    in every problem (the last state stored before the replay, the initial one, is
    finite).  Which entries are inf and which NaN is not compared: past an overflow the
    chunked scan forms inf * 0 (an underflowed lambda^L) where the sequential
    recursion keeps inf, and the dense oracle 0 * inf for every lambda^|i-j| that
    underflows."""
    n, m = 24, 40
    rng = np.random.default_rng(11)
    A, B = gi.random_positive(rng, (2, n * m)), gi.random_positive(rng, (2, n * m))
    kw = dict(h=1.0, h2=1.0, shape=(n, m), eps=0.002, itr_max=3000, domain="scaling")
    ref = sinkhorn.solve(A, B, n=n, m=m, h1=1.0, h2=1.0, eps=0.002, itr_max=3000)
    assert np.all(ref["flags"] == 2)
    w = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), **kw)
    t = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), kernel=5, **kw)
    assert np.all(w["flags"].cpu().numpy() == 2)
    np.testing.assert_array_equal(w["iters"].cpu().numpy(), ref["iters"])
    np.testing.assert_array_equal(t["iters"].cpu().numpy(), ref["iters"])
    assert np.isnan(w["cost"].cpu().numpy()).all() and np.isnan(w["err"].cpu().numpy()).all()
    u, v = w["u"].cpu().numpy(), w["v"].cpu().numpy()
    assert np.all((~np.isfinite(u)).any(1) | (~np.isfinite(v)).any(1))


@pytest.mark.parametrize("ci", [1, 7])
def test_check_interval_stop_state(ci):
    """tol-stopped run with checks every ci iterations: the stored state at the stopping
    check is the oracle's (the kernel stores phi, psi only before checks)."""
    n, m = 24, 40
    rng = np.random.default_rng(11)
    A, B = gi.random_positive(rng, (2, n * m)), gi.random_positive(rng, (2, n * m))
    h1, h2, eps = 1.0 / n, 1.0 / m, 0.05
    kw = dict(h=h1, h2=h2, shape=(n, m), eps=eps, domain="scaling")
    ref = sinkhorn.solve(A, B, n=n, m=m, h1=h1, h2=h2, eps=eps, itr_max=20000, tol=1e-9, check_interval=ci)
    out = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), itr_max=20000, tol=1e-9,
                    check_interval=ci, **kw)
    assert fs1.plan(fs1.Spec(ndim=2, n=n, m=m, h1=h1, h2=h2, eps=eps, batch=2, dtype=torch.float64,
                             itr_max=20000, tol=1e-9, check_interval=ci)).info()["kernel"].startswith("sep2d64w")
    it = out["iters"].cpu().numpy()
    assert np.all(out["flags"].cpu().numpy() == 1) and np.all(it % ci == 0)
    assert np.all(np.abs(it - ref["iters"]) <= ci)
    for p in range(2):
        fixed = sinkhorn.solve(A[p:p + 1], B[p:p + 1], n=n, m=m, h1=h1, h2=h2, eps=eps, itr_max=int(it[p]))
        one = {k: out[k][p:p + 1] for k in ("u", "v", "cost")}
        assert rel_norm(np.log(one["u"].cpu().numpy()[0]), fixed["F"][0]) <= 1e-10
        assert rel_norm(np.log(one["v"].cpu().numpy()[0]), fixed["G"][0]) <= 1e-10
        assert rel(one["cost"].item(), fixed["cost"][0]) <= 1e-10
