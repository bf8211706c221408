"""GPU parity of the separable 2D kernel (K3) against the oracle.

Algorithm 2 on n x m grids, fp32 log domain (config C4:
2048 x 2048).  Arrays are column-major, flat index j*n + i.
Tolerances: fp32 north_star 1e-4, read norm-wise (R17); the kernel
apply alone is held to 2e-6.
"""
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

TOL32 = 1e-4


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()


def _mat(flat, n, m):
    return flat.reshape(m, n).T


def _flat(M):
    return M.T.ravel()


def _field(n, m, seed, scale=3.0):
    rng = np.random.default_rng(seed)
    x = (np.arange(n) + 0.5) / n
    y = (np.arange(m) + 0.5) / m
    F = np.zeros((n, m))
    for _ in range(4):
        cx, cy = rng.uniform(0.2, 0.8, 2)
        s = rng.uniform(0.05, 0.3)
        F = np.logaddexp(F, -((x[:, None] - cx) ** 2 + (y[None, :] - cy) ** 2) / (2 * s * s))
    return scale * F + rng.normal(scale=0.1, size=(n, m))


def _ref_apply_log(X, c1, c2):
    n, m = X.shape
    if n * m <= 64 * 64:
        return dense.apply_2d_log(X, c1, c2)
    return recur.sweep_log(recur.sweep_log(X, c1, axis=1), c2, axis=2)


@pytest.mark.parametrize("n,m", [(1, 1), (1, 9), (9, 1), (5, 7), (37, 53), (64, 64), (128, 200), (300, 1000),
                                 (2048, 33)])
def test_sep2d_apply_log(n, m):
    X = _field(n, m, n * 1000 + m)
    c1, c2 = 0.3, 0.7
    y = fs1.apply(_cuda(_flat(X)[None]), h=c1, h2=c2, eps=1.0, domain="log", shape=(n, m))
    Y = _mat(y.double().cpu().numpy()[0], n, m)
    ref = _ref_apply_log(X.astype(np.float32).astype(np.float64), c1, c2)
    assert rel_norm(Y, ref) <= 2e-6


SOLVE = [  # n, m, eps, itr
    (1, 1, 1.0, 3),
    (6, 9, 0.05, 20),
    (40, 30, 0.01, 30),
    (64, 64, 5e-3, 40),
    (200, 120, 2e-3, 25),
]


def _pair2d(n, m, seed):
    la = _field(n, m, seed, 1.0)
    lb = _field(n, m, seed + 1, 1.0)
    la -= np.logaddexp.reduce(la.ravel())
    lb -= np.logaddexp.reduce(lb.ravel())
    return _flat(la), _flat(lb)


@pytest.mark.parametrize("n,m,eps,itr", SOLVE)
def test_sep2d_solve_parity(n, m, eps, itr):
    la, lb = _pair2d(n, m, n + m)
    A, B = la.astype(np.float32), lb.astype(np.float32)
    out = fs1.solve(_cuda(A[None]), _cuda(B[None]), h=1 / n, h2=1 / m, eps=eps, itr_max=itr, domain="log",
                    input_is_log=True, shape=(n, m))
    ref = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=n, m=m, h1=1 / n, h2=1 / m, eps=eps,
                         itr_max=itr, domain="log", input_is_log=True,
                         apply="dense" if n * m <= 64 * 64 else "recur")
    assert_solve_parity(out, ref, "log", "f32", tol=TOL32)


@pytest.mark.parametrize("n,m,eps", [(37, 53, 0.02), (256, 200, 2e-3), (600, 900, 2e-3)])
def test_sep2d_warp_line_kernel_equals_cta_line_kernel(n, m, eps):
    """K3w (warp per line, the solve default) and K3 (CTA per line, kernel=3) on the same
    problem: independent scan schedules of the same recursions agree to fp32 rounding."""
    la, lb = _pair2d(n, m, 5 * n + m)
    A, B = _cuda(la[None]), _cuda(lb[None])
    kw = dict(h=1 / n, h2=1 / m, eps=eps, itr_max=15, domain="log", input_is_log=True, shape=(n, m))
    assert fs1.plan(fs1.Spec(ndim=2, n=n, m=m, h1=1 / n, h2=1 / m, eps=eps, batch=1, dtype=torch.float32,
                             domain="log", input_is_log=True, itr_max=15)).info()["kernel"].startswith("sep2dw")
    ow = fs1.solve(A, B, **kw)
    oc = fs1.solve(A, B, kernel=3, **kw)
    assert rel_norm(ow["u"].double().cpu().numpy()[0], oc["u"].double().cpu().numpy()[0]) <= 2e-6
    assert rel_norm(ow["v"].double().cpu().numpy()[0], oc["v"].double().cpu().numpy()[0]) <= 2e-6
    assert rel(ow["cost"].item(), oc["cost"].item()) <= 1e-5
    assert abs(ow["err"].item() - oc["err"].item()) <= 1e-5 * max(1.0, oc["err"].item())


def test_sep2d_linear_weights_and_tolerance_stop():
    n, m = 48, 40
    la, lb = _pair2d(n, m, 7)
    A, B = np.exp(la).astype(np.float32), np.exp(lb).astype(np.float32)
    out = fs1.solve(_cuda(A[None]), _cuda(B[None]), h=1 / n, h2=1 / m, eps=0.05, itr_max=3000, tol=1e-5,
                    domain="log", shape=(n, m))
    ref = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=n, m=m, h1=1 / n, h2=1 / m, eps=0.05,
                         itr_max=3000, tol=1e-5, domain="log")
    assert out["flags"].item() == 1 and out["err"].item() <= 1e-5
    assert abs(int(out["iters"].item()) - int(ref["iters"][0])) <= 2
    ls = int(ref["iters"][0])
    o2 = fs1.solve(_cuda(A[None]), _cuda(B[None]), h=1 / n, h2=1 / m, eps=0.05, itr_max=ls, domain="log",
                   shape=(n, m))
    r2 = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=n, m=m, h1=1 / n, h2=1 / m, eps=0.05,
                        itr_max=ls, domain="log")
    assert_solve_parity(o2, r2, "log", "f32", tol=TOL32, check_err=False)


@pytest.mark.parametrize("ci", [2, 5])
def test_sep2d_check_interval(ci):
    """Checks every ci iterations (the solve keeps F, G only ahead of check iterations,
    DESIGN.md R26): the stop lands within ci of the oracle's, and the replay at the
    oracle's own stop is its state."""
    n, m = 96, 80
    la, lb = _pair2d(n, m, 13)
    A, B = la.astype(np.float32), lb.astype(np.float32)
    kw = dict(h=1 / n, h2=1 / m, eps=0.02, domain="log", input_is_log=True, shape=(n, m))
    out = fs1.solve(_cuda(A[None]), _cuda(B[None]), itr_max=4000, tol=1e-5, check_interval=ci, **kw)
    ref = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=n, m=m, h1=1 / n, h2=1 / m, eps=0.02,
                         itr_max=4000, tol=1e-5, check_interval=ci, domain="log", input_is_log=True, apply="recur")
    assert out["flags"].item() == 1 and out["err"].item() <= 1e-5
    assert out["iters"].item() % ci == 0
    assert abs(int(out["iters"].item()) - int(ref["iters"][0])) <= ci
    it = int(out["iters"].item())
    r2 = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=n, m=m, h1=1 / n, h2=1 / m, eps=0.02,
                        itr_max=it, domain="log", input_is_log=True, apply="recur")
    o2 = fs1.solve(_cuda(A[None]), _cuda(B[None]), itr_max=it, **kw)
    assert_solve_parity(o2, r2, "log", "f32", tol=TOL32, check_err=False)
    # the tol-stopped state is the fixed-iteration state at the same iteration
    assert rel_norm(out["u"].double().cpu().numpy()[0], o2["u"].double().cpu().numpy()[0]) <= 1e-6
    assert rel_norm(out["v"].double().cpu().numpy()[0], o2["v"].double().cpu().numpy()[0]) <= 1e-6


def test_sep2d_batch_of_problems():
    """Several 2D problems in one fs1_solve (one launch each, shared workspace): each equals
    its own single-problem solve, and the apply / cost entry points handle batches too."""
    n, m = 72, 56
    pairs = [_pair2d(n, m, 30 + k) for k in range(3)]
    A = np.stack([p[0] for p in pairs]).astype(np.float32)
    B = np.stack([p[1] for p in pairs]).astype(np.float32)
    kw = dict(h=1 / n, h2=1 / m, eps=0.01, itr_max=25, domain="log", input_is_log=True, shape=(n, m))
    out = fs1.solve(_cuda(A), _cuda(B), **kw)
    for k in range(3):
        one = fs1.solve(_cuda(A[k:k + 1]), _cuda(B[k:k + 1]), **kw)
        assert np.array_equal(out["u"][k].cpu().numpy(), one["u"][0].cpu().numpy())
        assert np.array_equal(out["v"][k].cpu().numpy(), one["v"][0].cpu().numpy())
        assert out["cost"][k].item() == one["cost"].item()
    cb = fs1.cost(out["u"], out["v"], h=1 / n, h2=1 / m, eps=0.01, domain="log", shape=(n, m))
    assert np.allclose(cb.cpu().numpy(), out["cost"].cpu().numpy(), rtol=1e-5)
    ref = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=n, m=m, h1=1 / n, h2=1 / m, eps=0.01,
                         itr_max=25, domain="log", input_is_log=True, apply="recur")
    assert_solve_parity(out, ref, "log", "f32", tol=TOL32)


def test_sep2d_cost_entry_point():
    n, m = 30, 45
    F = _field(n, m, 3, 2.0) - 9
    G = _field(n, m, 4, 2.0) - 9
    eps = 0.02
    c = fs1.cost(_cuda(_flat(F)[None]), _cuda(_flat(G)[None]), h=1 / n, h2=1 / m, eps=eps, domain="log",
                 shape=(n, m)).item()
    Ff, Gf = F.astype(np.float32).astype(np.float64), G.astype(np.float32).astype(np.float64)
    ref = dense.cost_2d_bruteforce(np.exp(Ff), np.exp(Gf), np.exp(-1 / n / eps), np.exp(-1 / m / eps), 1 / n, 1 / m)
    assert rel(c, ref) <= 1e-5


def test_sep2d_determinism_and_warm_start():
    n, m = 256, 192
    la, lb = _pair2d(n, m, 11)
    A, B = _cuda(la[None]), _cuda(lb[None])
    kw = dict(h=1 / n, h2=1 / m, eps=2e-3, domain="log", input_is_log=True, shape=(n, m))
    o1 = fs1.solve(A, B, itr_max=20, **kw)
    o2 = fs1.solve(A, B, itr_max=20, **kw)
    assert np.array_equal(o1["u"].cpu().numpy(), o2["u"].cpu().numpy())
    assert o1["cost"].item() == o2["cost"].item()
    p = fs1.solve(A, B, itr_max=8, **kw)
    r = fs1.solve(A, B, itr_max=12, u0=p["u"], v0=p["v"], **kw)
    assert rel_norm(r["u"].double().cpu().numpy()[0], o1["u"].double().cpu().numpy()[0]) <= 1e-6


# ------------------------------------------------------------------ config 4 at full size
def _c4():
    cfg = gi.CONFIGS["c4"]
    A, B = gi.batch(cfg, [0])
    return cfg, A, B


def test_config4_trajectory_full_size():
    """2048 x 2048 for 3 iterations against the recursion oracle (all 4.2M potentials)."""
    cfg, A, B = _c4()
    out = fs1.solve(_cuda(A), _cuda(B), h=cfg.h1, h2=cfg.h2, eps=cfg.eps, itr_max=3, domain="log",
                    input_is_log=True, shape=(cfg.n, cfg.m))
    ref = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2,
                         eps=cfg.eps, itr_max=3, domain="log", input_is_log=True, apply="recur")
    assert_solve_parity(out, ref, "log", "f32", tol=TOL32)


def test_config4_full_run_properties():
    """The bench's launch (300 iterations): the last phi half-step, the exit error and the
    cost are recomputed by the oracle from the GPU's final state."""
    cfg, A, B = _c4()
    n, m = cfg.n, cfg.m
    out = fs1.solve(_cuda(A), _cuda(B), h=cfg.h1, h2=cfg.h2, eps=cfg.eps, itr_max=cfg.itr_max, domain="log",
                    input_is_log=True, shape=(n, m))
    assert out["iters"].item() == cfg.itr_max and out["flags"].item() == 4
    F = _mat(out["u"].double().cpu().numpy()[0], n, m)
    G = _mat(out["v"].double().cpu().numpy()[0], n, m)
    la = _mat(A[0].astype(np.float64), n, m)
    lb = _mat(B[0].astype(np.float64), n, m)
    c1, c2 = cfg.h1 / cfg.eps, cfg.h2 / cfg.eps
    KG = recur.sweep_log(recur.sweep_log(G, c1, axis=1), c2, axis=2)
    assert rel_norm(F, la - KG) <= TOL32
    KF = recur.sweep_log(recur.sweep_log(F, c1, axis=1), c2, axis=2)
    err = float(np.sum(np.abs(np.exp(G + KF) - np.exp(lb))))
    assert abs(out["err"].item() - err) <= TOL32 * max(1.0, err)
    L1 = recur.sweep_log(recur.wsweep_log(G, c1, cfg.h1, axis=1), c2, axis=2)
    L2 = recur.wsweep_log(recur.sweep_log(G, c1, axis=1), c2, cfg.h2, axis=2)
    ref = recur.sum_exp2(F, L1) + recur.sum_exp2(F, L2)
    assert rel(out["cost"].item(), ref) <= TOL32


@pytest.mark.parametrize("side", ["a", "b"])
@pytest.mark.parametrize("n,m", [(256, 200), (1500, 1100)])
def test_sep2d_warp_line_nonfinite_weight(side, n, m):
    """K3w: a +inf log-weight poisons the problem in the first half-step that divides by
    it (phi^(1) = a / K psi for a, psi^(1) = b / K^T phi for b): the solve stops NONFINITE
    with l = 1 and NaN cost / err (S7, PAPER.md:148 has no finite error then); a NaN does
    the same."""
    for bad in (np.inf, np.nan):
        la, lb = _pair2d(n, m, 7 * n + m)
        (la if side == "a" else lb)[(m // 2) * n + n // 3] = bad  # column-major flat index
        kw = dict(h=1 / n, h2=1 / m, eps=2e-3, itr_max=20, domain="log", input_is_log=True, shape=(n, m))
        assert fs1.plan(fs1.Spec(ndim=2, n=n, m=m, h1=1 / n, h2=1 / m, eps=2e-3, batch=1,
                                 dtype=torch.float32, domain="log", input_is_log=True,
                                 itr_max=20)).info()["kernel"].startswith("sep2dw")
        out = fs1.solve(_cuda(la[None]), _cuda(lb[None]), **kw)
        assert out["flags"].item() == 2 and out["iters"].item() == 1, (bad, out["flags"], out["iters"])
        assert np.isnan(out["cost"].item())
