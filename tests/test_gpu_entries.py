"""GPU parity of fs1_plan_entries: single entries gamma_kl of the transport plan
diag(phi) K diag(psi) (SPEC's plan_entry) at index
triples, for problems of any size.

Oracle: the plan written out from its definition, diag(phi) K diag(psi) with K the dense
materialised kernel (oracle/dense.py: lambda^{|i-j|}, the 2D block kernel, the 3D
Kronecker product), on the ORACLE's own solve state (oracle/sinkhorn.py); at C3's full size
(N = 2^24, 1000 iterations) the committed oracle golden's F, G at its sampled points.
"""
import os

import numpy as np
import pytest

import fs1_inputs as gi
from oracle import dense, sinkhorn

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import _lib as L  # noqa: E402
from paper_2202_10042_b200 import fs1  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _triples(rng, batch, size, count):
    return np.stack([rng.integers(0, batch, count), rng.integers(0, size, count), rng.integers(0, size, count)], 1)


def _plan_ref(F, G, K):
    """gamma = diag(e^F) K diag(e^G) from the definition (fp64)."""
    return np.exp(F)[:, None] * K * np.exp(G)[None, :]


@pytest.mark.parametrize("dom,dt", [("scaling", "f64"), ("log", "f64"), ("log", "f32")])
def test_entries_1d_against_definition(dom, dt):
    n, eps, itr = 300, 0.01, 40
    A, B = gi.batch("c2", range(3), n=n)
    ref = sinkhorn.solve(A, B, n=n, h1=1 / n, eps=eps, itr_max=itr, domain="log")
    T = torch.float64 if dt == "f64" else torch.float32
    if dom == "scaling":
        u, v = torch.from_numpy(np.exp(ref["F"])), torch.from_numpy(np.exp(ref["G"]))
    else:
        u, v = torch.from_numpy(ref["F"]), torch.from_numpy(ref["G"])
    u, v = u.to(T).cuda(), v.to(T).cuda()
    rng = np.random.default_rng(5)
    idx = _triples(rng, 3, n, 4000)
    idx[:50, 2] = idx[:50, 1]  # diagonal entries (lambda^0)
    g = fs1.plan_entries(u, v, torch.from_numpy(idx).cuda(), h=1 / n, eps=eps, domain=dom).cpu().numpy()
    K = dense.kernel(n, dense.lam(1 / n, eps))
    # the state as the GPU read it (rounded to the plan dtype), the plan by its definition
    Fu = u.double().cpu().numpy() if dom != "scaling" else np.log(u.double().cpu().numpy())
    Gv = v.double().cpu().numpy() if dom != "scaling" else np.log(v.double().cpu().numpy())
    want = np.array([_plan_ref(Fu[p], Gv[p], K)[k, q] for p, k, q in idx])
    np.testing.assert_allclose(g, want, rtol=1e-12, atol=0)


def test_entries_of_gpu_solve_match_oracle_plan():
    """GPU solve -> GPU entries against the oracle's solve -> plan (the f3 path end to end)."""
    n, eps, itr = 500, 1e-3, 200
    A, B = gi.batch("e1_500", range(2), n=n)
    h = 6.0 / (n - 1)
    out = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), h=h, eps=eps, itr_max=itr)
    ref = sinkhorn.solve(A, B, n=n, h1=h, eps=eps, itr_max=itr)
    rng = np.random.default_rng(9)
    idx = _triples(rng, 2, n, 3000)
    idx[:, 2] = np.clip(idx[:, 1] + rng.integers(-3, 4, 3000), 0, n - 1)  # near the diagonal: not all 0
    g = fs1.plan_entries(out["u"], out["v"], torch.from_numpy(idx).cuda(), h=h, eps=eps).cpu().numpy()
    K = dense.kernel(n, dense.lam(h, eps))
    want = np.array([_plan_ref(ref["F"][p], ref["G"][p], K)[k, q] for p, k, q in idx])
    big = want > 1e-300
    assert big.sum() > 1000
    np.testing.assert_allclose(g[big], want[big], rtol=1e-9, atol=0)


def test_entries_2d_3d_against_dense_kernels():
    rng = np.random.default_rng(2)
    # 2D (column-major, l1 distance h1 |di| + h2 |dj|): the oracle's block kernel
    n, m, h1, h2, eps = 12, 9, 0.1, 0.15, 0.05
    F, G = rng.normal(size=(1, n * m)), rng.normal(size=(1, n * m))
    idx = _triples(rng, 1, n * m, 2000)
    # (2D plans: fp64 scaling (K5) or fp32 log (K3w); the entries need only the geometry)
    u2, v2 = torch.from_numpy(np.exp(F)).cuda(), torch.from_numpy(np.exp(G)).cuda()
    g = fs1.plan_entries(u2, v2, torch.from_numpy(idx).cuda(), h=h1, h2=h2, eps=eps, shape=(n, m)).cpu().numpy()
    K2 = dense.kernel_2d(n, m, dense.lam(h1, eps), dense.lam(h2, eps))
    want = _plan_ref(F[0], G[0], K2)[idx[:, 1], idx[:, 2]]
    np.testing.assert_allclose(g, want, rtol=1e-12, atol=0)
    gl = fs1.plan_entries(torch.from_numpy(F).float().cuda(), torch.from_numpy(G).float().cuda(),
                          torch.from_numpy(idx).cuda(), h=h1, h2=h2, eps=eps, domain="log", shape=(n, m)).cpu().numpy()
    np.testing.assert_allclose(gl, want, rtol=1e-5, atol=0)  # fp32 logs
    # equals the materialised plan of fs1_transport_plan entry for entry
    gam = fs1.transport_plan(u2, v2, h=h1, h2=h2, eps=eps, shape=(n, m)).cpu().numpy()[0]
    np.testing.assert_allclose(g, gam[idx[:, 1], idx[:, 2]], rtol=1e-15, atol=0)
    # 3D: K = T_L (x) T_M (x) T_N on the flat index (z m + j) n + i
    n, m, l, h3 = 5, 4, 3, 0.2
    phi, psi = rng.uniform(0.5, 2.0, size=(2, n * m * l)), rng.uniform(0.5, 2.0, size=(2, n * m * l))
    idx = _triples(rng, 2, n * m * l, 2000)
    g = fs1.plan_entries(torch.from_numpy(phi).cuda(), torch.from_numpy(psi).cuda(), torch.from_numpy(idx).cuda(),
                         h=h1, h2=h2, h3=h3, eps=eps, shape=(n, m, l)).cpu().numpy()
    K3 = np.kron(dense.kernel(l, dense.lam(h3, eps)),
                 np.kron(dense.kernel(m, dense.lam(h2, eps)), dense.kernel(n, dense.lam(h1, eps))))
    want = np.array([phi[p, k] * K3[k, q] * psi[p, q] for p, k, q in idx])
    np.testing.assert_allclose(g, want, rtol=1e-12, atol=0)


def test_entries_edge_cases():
    n = 64
    u = torch.zeros(2, n, dtype=torch.float64, device="cuda")
    v = torch.ones(2, n, dtype=torch.float64, device="cuda")
    u[0, 3] = 2.0
    idx = torch.tensor([[0, 3, 3], [0, 3, 5], [0, 4, 3], [1, 0, 0], [2, 0, 0], [0, -1, 0], [0, 0, n]],
                       dtype=torch.int64, device="cuda")
    g = fs1.plan_entries(u, v, idx, h=1.0, eps=1.0).cpu().numpy()  # scaling: phi = 0 except u[0, 3]
    assert g[0] == 2.0 and g[1] == pytest.approx(2.0 * np.exp(-2.0), rel=1e-15) and g[2] == 0.0 and g[3] == 0.0
    assert np.all(np.isnan(g[4:]))  # out of range: NaN
    empty = torch.empty(0, 3, dtype=torch.int64, device="cuda")
    assert fs1.plan_entries(u, v, empty, h=1.0, eps=1.0).numel() == 0
    lib = L.lib()
    assert lib.fs1_plan_entries(None, None, None, None, 0, None, None) == L.FS1_ERR_ARG
    with pytest.raises(ValueError):
        fs1.plan_entries(u, v, idx.int(), h=1.0, eps=1.0)


def test_entries_c3_full_size_against_golden():
    """C3 at its full protocol (N = 2^24, 1000 iterations, the launch bench.py times), then
    entries between neighbouring sampled points of the oracle golden: gamma from the GPU's
    state against exp(F_k + G_l - c |k - l|) from the golden's (oracle-written) F, G.  Two
    logs enter, each within the north_star 1e-10 norm-wise bar."""
    p = os.path.join(GOLDEN, "c3_full.npz")
    gld = np.load(p)
    cfg = gi.CONFIGS["c3"]
    a, b = gi.batch(cfg, [0])
    out = fs1.solve(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), h=cfg.h1, eps=cfg.eps,
                    itr_max=cfg.itr_max, domain="log", input_is_log=cfg.input_is_log)
    sidx, F, G = gld["idx"], gld["F"], gld["G"]
    k = np.arange(0, len(sidx) - 1, 7)
    pairs = np.stack([np.zeros_like(k), sidx[k], sidx[k + 1]], 1).astype(np.int64)
    pairs = np.concatenate([pairs, np.stack([np.zeros_like(k), sidx[k + 1], sidx[k]], 1)])
    fk = np.concatenate([F[k], F[k + 1]])
    gl = np.concatenate([G[k + 1], G[k]])
    c = cfg.h1 / cfg.eps
    logw = fk + gl - c * np.abs(pairs[:, 1] - pairs[:, 2])
    g = fs1.plan_entries(out["u"], out["v"], torch.from_numpy(pairs).cuda(), h=cfg.h1, eps=cfg.eps,
                         domain="log").cpu().numpy()
    ok = np.isfinite(logw) & (logw > -700)
    assert ok.sum() > 10000
    amax = max(float(gld["F_absmax"]), float(gld["G_absmax"]), 1.0)
    e = np.max(np.abs(np.log(g[ok]) - logw[ok]))
    assert e <= 2e-10 * amax, (e, amax)
    assert np.all(g[~np.isfinite(logw)] == 0.0)
