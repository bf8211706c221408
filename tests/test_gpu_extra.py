"""GPU parity of the steps either side of the loop: the dual objective
of Eq. (2.3) (fs1_dual) and the eps-scaling continuation (fs1_solve_eps_scaling), against
oracle.sinkhorn.dual_objective / solve_eps_scaling (pinned in tests/test_oracle_solve.py),
and the eps-limit sandwich of the oracle tests reproduced on the GPU."""
import numpy as np
import pytest

import fs1_inputs as gi
from oracle import sinkhorn, w1
from tests.gpu_util import assert_solve_parity, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402


def _t(x, dt=np.float64):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=dt)).cuda()


@pytest.mark.parametrize("domain,dtype,n", [("log", np.float64, 300), ("scaling", np.float64, 300),
                                            ("log", np.float32, 512), ("scaling", np.float32, 100)])
def test_dual_1d(domain, dtype, n):
    rng = np.random.default_rng(n)
    A, B = gi.random_positive(rng, (3, n)).astype(dtype), gi.random_positive(rng, (3, n)).astype(dtype)
    kw = dict(h=1.0 / n, eps=0.02, domain=domain)
    out = fs1.solve(_t(A, dtype), _t(B, dtype), itr_max=25, **kw)
    D = fs1.dual(_t(A, dtype), _t(B, dtype), out["u"], out["v"], **kw).cpu().numpy()
    F = out["u"].double().cpu().numpy()
    G = out["v"].double().cpu().numpy()
    if domain == "scaling":
        F, G = np.log(F), np.log(G)
    tol = 1e-10 if dtype == np.float64 else 1e-5
    for p in range(3):
        ref = sinkhorn.dual_objective(A[p].astype(np.float64), B[p].astype(np.float64), F[p], G[p], n=n,
                                      h1=1.0 / n, eps=0.02)
        assert abs(D[p] - ref) <= tol * max(1.0, abs(ref)), (p, D[p], ref)


def test_dual_monotone_and_equals_primal_at_convergence():
    n = 200
    a, b = gi.pair("c1", 0, n=n)
    kw = dict(h=1.0 / n, eps=0.02, domain="log")
    vals = []
    for it in (1, 2, 5, 10, 40, 160):
        o = fs1.solve(_t(a[None]), _t(b[None]), itr_max=it, **kw)
        vals.append(fs1.dual(_t(a[None]), _t(b[None]), o["u"], o["v"], **kw).item())
    assert all(vals[i + 1] >= vals[i] - 1e-13 for i in range(len(vals) - 1))
    o = fs1.solve(_t(a[None]), _t(b[None]), itr_max=100000, tol=1e-13, **kw)
    D = fs1.dual(_t(a[None]), _t(b[None]), o["u"], o["v"], **kw).item()
    P = sinkhorn.primal_objective(o["u"].cpu().numpy()[0], o["v"].cpu().numpy()[0], n=n, h1=1.0 / n, eps=0.02)
    assert abs(D - P) <= 1e-10


@pytest.mark.parametrize("kind", ["k5_f64", "k3_f32log"])
def test_dual_2d(kind):
    n, m = 24, 20
    rng = np.random.default_rng(7)
    A, B = gi.random_positive(rng, (2, n * m)), gi.random_positive(rng, (2, n * m))
    if kind == "k5_f64":
        dt, domain, tol = np.float64, "scaling", 1e-10
    else:
        dt, domain, tol = np.float32, "log", 1e-5
    kw = dict(h=1.0 / n, h2=1.0 / m, shape=(n, m), eps=0.05, domain=domain)
    o = fs1.solve(_t(A, dt), _t(B, dt), itr_max=20, **kw)
    D = fs1.dual(_t(A, dt), _t(B, dt), o["u"], o["v"], **kw).cpu().numpy()
    F, G = o["u"].double().cpu().numpy(), o["v"].double().cpu().numpy()
    if domain == "scaling":
        F, G = np.log(F), np.log(G)
    for p in range(2):
        ref = sinkhorn.dual_objective(A[p].astype(dt).astype(np.float64), B[p].astype(dt).astype(np.float64),
                                      F[p], G[p], n=n, m=m, h1=1.0 / n, h2=1.0 / m, eps=0.05)
        assert abs(D[p] - ref) <= tol * max(1.0, abs(ref))


@pytest.mark.parametrize("n,dt", [(500, np.float64), (1000, np.float32), (300000, np.float64)])
def test_eps_scaling_parity(n, dt):
    """The continuation against the oracle's, stage for stage (fixed iterations): persistent
    kernels (fp64, fp32) and the streaming kernel K2 (n = 3e5)."""
    if n > 10000:
        cfg = gi.CONFIGS["c3"]
        a, b = gi.pair(cfg, 0, n=n)
        A, B = a[None], b[None]
        kw = dict(h=1.0 / n, eps=1e-4, input_is_log=True)
        sched = dict(eps0=8e-4, factor=0.5, stage_iters=4, itr_max=6)
        apply = "recur"
    else:
        rng = np.random.default_rng(n)
        A, B = gi.random_positive(rng, (2, n)), gi.random_positive(rng, (2, n))
        kw = dict(h=1.0 / n, eps=2e-3)
        sched = dict(eps0=3.2e-2, factor=0.5, stage_iters=10, itr_max=40)
        apply = "dense"
    A, B = A.astype(dt), B.astype(dt)
    out = fs1.solve_eps_scaling(_t(A, dt), _t(B, dt), **kw, **sched)
    ref = sinkhorn.solve_eps_scaling(A.astype(np.float64), B.astype(np.float64), n=n, h1=kw["h"], eps=kw["eps"],
                                     input_is_log=kw.get("input_is_log", False), apply=apply, **sched)
    assert out["stages"] == len(ref["stages"])
    assert_solve_parity(out, ref, "log", "f64" if dt == np.float64 else "f32")


def test_eps_scaling_converges_to_direct_solution():
    n = 400
    a, b = gi.pair("c1", 0, n=n)
    kw = dict(h=1.0 / n, eps=2e-3, itr_max=200000, tol=1e-10)
    s = fs1.solve_eps_scaling(_t(a[None]), _t(b[None]), eps0=0.064, factor=0.5, stage_iters=50, **kw)
    d = fs1.solve(_t(a[None]), _t(b[None]), domain="log", **kw)
    assert s["flags"].item() == 1 and d["flags"].item() == 1
    assert s["iters"].item() < d["iters"].item()
    assert rel(s["cost"].item(), d["cost"].item()) <= 1e-7


def test_eps_sandwich_on_gpu():
    """At convergence 0 <= <C,gamma_eps> - W1 <= eps min(H(a), H(b)) (+ marginal slack), the
    cost decreasing toward W1 as eps decreases (oracle test_eps_limit_sandwich_and_monotone,
    here on the GPU; small eps reached by eps-scaling)."""
    rng = np.random.default_rng(2)
    n = 64
    a, b = gi.random_positive(rng, n), gi.random_positive(rng, n)
    h = 1.0 / n
    W = w1.w1_exact(a, b, h)
    costs = []
    for eps in [0.1, 0.03, 0.01, 0.003]:
        r = fs1.solve_eps_scaling(_t(a[None]), _t(b[None]), h=h, eps=eps, eps0=max(eps, 0.1), factor=0.5,
                                  stage_iters=200, itr_max=400000, tol=1e-13)
        assert r["flags"].item() == 1
        gap = r["cost"].item() - W
        slack = (n - 1) * h * r["err"].item()
        assert -slack - 1e-13 <= gap <= eps * min(w1.entropy(a), w1.entropy(b)) + slack
        costs.append(r["cost"].item())
    assert all(costs[i] > costs[i + 1] for i in range(len(costs) - 1))
