"""The 3D separable extension ("easily extended to high-dimensional cases")
on the GPU: K5 with a third axis, fp64 scaling domain, against the oracle's dense 3D
Algorithm 2 (oracle.sinkhorn._Ops3D, pinned against the materialised kernel, brute force,
the 2D reduction and an LP in tests/test_oracle_solve.py).  Column-major flat index
(z m + j) n + i."""
import numpy as np
import pytest

import fs1_inputs as gi
from oracle import sinkhorn
from tests.gpu_util import assert_solve_parity, rel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402


def _t(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


@pytest.mark.parametrize("shape", [(8, 6, 5), (16, 16, 16), (1, 1, 7), (7, 1, 1), (33, 5, 3), (3, 40, 2)])
def test_3d_parity(shape):
    n, m, l = shape
    N = n * m * l
    rng = np.random.default_rng(N)
    A, B = gi.random_positive(rng, (2, N)), gi.random_positive(rng, (2, N))
    kw = dict(h=1.0 / n, h2=1.0 / m, h3=1.0 / l, eps=0.05)
    out = fs1.solve(_t(A), _t(B), shape=shape, itr_max=50, **kw)
    ref = sinkhorn.solve(A, B, n=n, m=m, l=l, h1=kw["h"], h2=kw["h2"], h3=kw["h3"], eps=kw["eps"], itr_max=50)
    assert_solve_parity(out, ref, "scaling", "f64")


@pytest.mark.parametrize("N", [10, 20])
def test_3d_random_h1_eps_001_full_protocol(N):
    """E3's recipe on an N^3 grid (h = 1 per axis, eps = 0.01: lambda = e^{-100} on every
    axis, u, v iid U[0,1] normalised), the full 1000 iterations."""
    rng = np.random.default_rng(100 + N)
    A = rng.uniform(0, 1, (1, N ** 3))
    B = rng.uniform(0, 1, (1, N ** 3))
    A /= A.sum()
    B /= B.sum()
    out = fs1.solve(_t(A), _t(B), shape=(N, N, N), h=1.0, h2=1.0, h3=1.0, eps=0.01, itr_max=1000)
    ref = sinkhorn.solve(A, B, n=N, m=N, l=N, h1=1.0, h2=1.0, h3=1.0, eps=0.01, itr_max=1000)
    assert_solve_parity(out, ref, "scaling", "f64")


def test_3d_apply_cost_dual_and_tolerance_stop():
    n, m, l = 9, 7, 5
    N = n * m * l
    rng = np.random.default_rng(3)
    A, B = gi.random_positive(rng, (1, N)), gi.random_positive(rng, (1, N))
    kw = dict(shape=(n, m, l), h=0.1, h2=0.15, h3=0.2, eps=0.05)
    ops = sinkhorn._Ops3D(n, m, l, 0.1, 0.15, 0.2, 0.05, "dense")
    x = rng.uniform(0, 1, (3, N))
    y = fs1.apply(_t(x), **kw).cpu().numpy()
    np.testing.assert_allclose(y, ops.K_(x.T).T, rtol=1e-13)
    ref = sinkhorn.solve(A, B, n=n, m=m, l=l, h1=0.1, h2=0.15, h3=0.2, eps=0.05, itr_max=50000, tol=1e-11)
    assert ref["flags"][0] == 1
    out = fs1.solve(_t(A), _t(B), itr_max=50000, tol=1e-11, **kw)
    assert out["flags"].item() == 1 and abs(out["iters"].item() - ref["iters"][0]) <= 1
    c = fs1.cost(out["u"], out["v"], **kw)
    assert rel(c.item(), out["cost"].item()) <= 1e-13
    D = fs1.dual(_t(A), _t(B), out["u"], out["v"], **kw).item()
    F, G = np.log(out["u"].cpu().numpy()[0]), np.log(out["v"].cpu().numpy()[0])
    i = np.arange(N) % n
    j = (np.arange(N) // n) % m
    z = np.arange(N) // (n * m)
    C = (np.abs(i[:, None] - i[None, :]) * 0.1 + np.abs(j[:, None] - j[None, :]) * 0.15 +
         np.abs(z[:, None] - z[None, :]) * 0.2)
    gam = np.exp(F[:, None] + G[None, :] - C / 0.05)
    Dref = 0.05 * (A[0] @ F + B[0] @ G - gam.sum()) + 0.05
    assert abs(D - Dref) <= 1e-10
