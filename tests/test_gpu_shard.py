"""GPU parity of the sharded single-problem path (include/fs1_shard.h, K2s).

One 1D problem split into `world` contiguous tile segments.
On one GPU the ranks run in lock step in one process (`shard.solve_segments`):
the per-rank kernels and the exchanged totals are exactly those of a
multi-GPU run; only the all-gather is a concatenation.  Checked against the
oracle (dense where feasible, else the plain-C recursion) at world sizes
1-8 with ragged last segments, against the single-GPU streaming kernel at
the full C3 size, and for the tolerance-stopped loop (R22).
"""
import numpy as np
import pytest

import fs1_inputs as gi
from oracle import sinkhorn
from tests.gpu_util import TOL, rel, rel_norm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1, shard  # noqa: E402

TOL64 = TOL["f64"]


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def _pair(n, seed, log=True):
    rng = np.random.default_rng(seed)
    x = (np.arange(n) + 0.5) / n
    out = []
    for _ in range(2):
        mu = rng.uniform(0.1, 0.9, 3)
        sd = rng.uniform(0.02, 0.1, 3)
        comp = -0.5 * ((x[None] - mu[:, None]) / sd[:, None]) ** 2 - np.log(sd)[:, None]
        la = np.logaddexp.reduce(comp, axis=0)
        la -= np.logaddexp.reduce(la)
        out.append(la if log else np.exp(la))
    return out


def _parity(o, ref):
    assert o["iters"] == ref["iters"][0] and o["flags"] == ref["flags"][0]
    F, G = o["u"].cpu().numpy(), o["v"].cpu().numpy()
    assert rel_norm(F, ref["F"][0]) <= TOL64
    assert rel_norm(G, ref["G"][0]) <= TOL64
    assert rel(o["cost"], ref["cost"][0]) <= TOL64
    assert abs(o["err"] - ref["err"][0]) <= TOL64 * max(1.0, ref["err"][0])


@pytest.mark.parametrize("n,world", [(1, 1), (255, 1), (256, 1), (700, 2), (1000, 3), (2049, 4), (3001, 8),
                                     (3001, 12)])
def test_segments_solve_parity(n, world):
    eps = max(2e-3, 0.5 / n)  # h/eps <= 2: within the per-tile range (h/eps x 256 <= 600)
    a, b = _pair(n, n + world)
    tiles = -(-n // 256)
    if world > tiles:
        with pytest.raises(Exception):
            shard.solve_segments(_cuda(a), _cuda(b), world, h=1 / n, eps=eps, itr_max=5, input_is_log=True)
        return
    o = shard.solve_segments(_cuda(a), _cuda(b), world, h=1 / n, eps=eps, itr_max=30, input_is_log=True)
    segs = o["segments"]
    assert segs[0][0] == 0 and sum(l for _, l in segs) == n
    assert all(segs[k][0] + segs[k][1] == segs[k + 1][0] for k in range(len(segs) - 1))
    assert [s for s in segs] == [shard.segment(n, world, r) for r in range(world)]
    ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=eps, itr_max=30, domain="log", input_is_log=True)
    _parity(o, ref)


def test_segments_linear_weights_recursion_oracle():
    n, world = 20000, 5
    a, b = _pair(n, 9, log=False)
    o = shard.solve_segments(_cuda(a), _cuda(b), world, h=1 / n, eps=1e-4, itr_max=12)
    ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=1e-4, itr_max=12, domain="log", apply="recur")
    _parity(o, ref)


@pytest.mark.parametrize("world", [2, 3])
def test_segments_short_last_block(world):
    """Segments of 21 / 14 tiles split into blocks of 8 (two-level tile scan): the short
    last block enters the rank totals the other ranks decay over their segments."""
    n = 42 * 256
    a, b = _pair(n, 17)
    kw = dict(h=1 / n, eps=1e-3, itr_max=20, input_is_log=True)
    o = shard.solve_segments(_cuda(a), _cuda(b), world, **kw)
    ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=1e-3, itr_max=20, domain="log", input_is_log=True,
                         apply="recur")
    _parity(o, ref)


def test_segments_independent_of_world_size():
    """Every world size gives the same state to rounding (the split only moves where
    the exchanged totals enter the recursions)."""
    n = 9000
    a, b = _pair(n, 3)
    kw = dict(h=1 / n, eps=5e-4, itr_max=40, input_is_log=True)
    base = shard.solve_segments(_cuda(a), _cuda(b), 1, **kw)
    for world in (2, 5, 8):
        o = shard.solve_segments(_cuda(a), _cuda(b), world, **kw)
        assert rel_norm(o["u"].cpu().numpy(), base["u"].cpu().numpy()) <= 1e-12
        assert rel_norm(o["v"].cpu().numpy(), base["v"].cpu().numpy()) <= 1e-12
        assert rel(o["cost"], base["cost"]) <= 1e-12


def test_segments_tolerance_stop_and_check_interval():
    n, world = 2000, 3
    a, b = _pair(n, 5)
    for ci in (1, 4):
        o = shard.solve_segments(_cuda(a), _cuda(b), world, h=1 / n, eps=1e-2, itr_max=5000, tol=1e-9,
                                 check_interval=ci, input_is_log=True)
        ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=1e-2, itr_max=5000, tol=1e-9, check_interval=ci,
                             domain="log", input_is_log=True)
        assert o["flags"] == 1 and o["err"] <= 1e-9
        assert abs(o["iters"] - int(ref["iters"][0])) <= ci
        ls = int(ref["iters"][0])
        o2 = shard.solve_segments(_cuda(a), _cuda(b), world, h=1 / n, eps=1e-2, itr_max=ls, input_is_log=True)
        r2 = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=1e-2, itr_max=ls, domain="log", input_is_log=True)
        _parity(o2, r2)


def test_segments_equal_streaming_kernel_at_config3_size():
    """N = 2^24 over 8 segments against the single-GPU streaming kernel (K2, itself
    pinned to the oracle at this size, test_gpu_stream.py) for 5 iterations."""
    cfg = gi.CONFIGS["c3"]
    a, b = gi.pair(cfg, 0)
    A, B = _cuda(a), _cuda(b)
    o = shard.solve_segments(A, B, 8, h=cfg.h1, eps=cfg.eps, itr_max=5, input_is_log=True)
    k2 = fs1.solve(A[None], B[None], h=cfg.h1, eps=cfg.eps, itr_max=5, domain="log", input_is_log=True)
    assert rel_norm(o["u"].cpu().numpy(), k2["u"].cpu().numpy()[0]) <= 1e-11
    assert rel_norm(o["v"].cpu().numpy(), k2["v"].cpu().numpy()[0]) <= 1e-11
    assert rel(o["cost"], k2["cost"].item()) <= 1e-11
    assert abs(o["err"] - k2["err"].item()) <= 1e-10 * max(1.0, k2["err"].item())


@pytest.mark.parametrize("world", [1, 3])
def test_graph_replay_equals_eager_loop(world):
    """The captured-iteration driver (CUDA graph replays) runs the same kernels in the same
    order as the eager loop: bitwise-equal state, error and cost."""
    n = 5000
    a, b = _pair(n, 21)
    kw = dict(h=1 / n, eps=1e-3, itr_max=25, input_is_log=True)
    og = shard.solve_segments(_cuda(a), _cuda(b), world, graph=True, **kw)
    oe = shard.solve_segments(_cuda(a), _cuda(b), world, graph=False, **kw)
    assert np.array_equal(og["u"].cpu().numpy(), oe["u"].cpu().numpy())
    assert np.array_equal(og["v"].cpu().numpy(), oe["v"].cpu().numpy())
    assert og["cost"] == oe["cost"] and og["err"] == oe["err"] and og["iters"] == oe["iters"] == 25


def test_graph_replay_nonfinite_iteration():
    """A +inf log-weight poisons the state at the first half-step: the device counter
    records iteration 1 through the graph replays, as the eager loop does."""
    n = 3000
    a, b = _pair(n, 22)
    a = a.copy()
    a[1234] = np.inf
    for graph in (True, False):
        o = shard.solve_segments(_cuda(a), _cuda(b), 2, h=1 / n, eps=1e-2, itr_max=10, input_is_log=True,
                                 graph=graph)
        assert o["flags"] == 2 and o["iters"] == 1 and np.isnan(o["cost"]) and np.isnan(o["err"])


def test_shard_plan_errors():
    import ctypes
    from paper_2202_10042_b200 import _lib as L
    d = L.Desc(ndim=1, n=1000, m=1, h1=1e-3, h2=0.0, eps=1e-2, batch=1, dtype=L.FS1_F64, domain=L.FS1_LOG,
               input_is_log=0, itr_max=10, tol=0.0, check_interval=1, warm_start=0)
    h, ws, lo, ln = ctypes.c_void_p(), ctypes.c_size_t(), ctypes.c_int64(), ctypes.c_int64()
    args = (ctypes.byref(h), ctypes.byref(ws), ctypes.byref(lo), ctypes.byref(ln))
    assert L.lib().fs1_shard_plan(ctypes.byref(d), 2, 2, 0, *args) == L.FS1_ERR_ARG      # rank >= world
    assert L.lib().fs1_shard_plan(ctypes.byref(d), 5, 0, 0, *args) == L.FS1_ERR_ARG      # world > tiles
    d.dtype = L.FS1_F32
    assert L.lib().fs1_shard_plan(ctypes.byref(d), 2, 0, 0, *args) == L.FS1_ERR_UNSUPPORTED
    d.dtype, d.eps = L.FS1_F64, 1e-6                                                     # c x 256 > 600
    assert L.lib().fs1_shard_plan(ctypes.byref(d), 2, 0, 0, *args) == L.FS1_ERR_UNSUPPORTED
    d.eps = 0.0
    assert L.lib().fs1_shard_plan(ctypes.byref(d), 2, 0, 0, *args) == L.FS1_ERR_EPS


# ---- fused exchange (mailboxes over peer memory, include/fs1_shard.h) ----------------
@pytest.mark.parametrize("world,graph,tol", [(1, True, 0.0), (2, True, 0.0), (5, True, 0.0), (8, False, 0.0),
                                             (3, False, 1e-9), (16, True, 0.0)])
def test_fused_exchange_equals_gathered(world, graph, tol):
    """The kernels deliver the totals into every rank's mailbox (row `rank` of slot
    e & 1, flag release / acquire) instead of the host all-gather: the same values
    reach the same kernels, so state, error, cost and iteration count are bitwise
    those of the gathered exchange — over graph replays, the eager loop with the
    tolerance stop (check steps), and the largest fused world (16)."""
    n = 8000
    a, b = _pair(n, 31 + world)
    kw = dict(h=1 / n, eps=2e-3, itr_max=40 if tol == 0.0 else 3000, tol=tol, check_interval=3,
              input_is_log=True, graph=graph)
    of = shard.solve_segments(_cuda(a), _cuda(b), world, fused=True, **kw)
    og = shard.solve_segments(_cuda(a), _cuda(b), world, fused=False, **kw)
    assert np.array_equal(of["u"].cpu().numpy(), og["u"].cpu().numpy())
    assert np.array_equal(of["v"].cpu().numpy(), og["v"].cpu().numpy())
    assert of["cost"] == og["cost"] and of["err"] == og["err"]
    assert of["iters"] == og["iters"] and of["flags"] == og["flags"]
    if tol > 0.0:
        assert of["flags"] == 1 and of["err"] <= tol


def test_fused_exchange_oracle_parity_and_repeat():
    """Fused exchange against the oracle, twice in a row (fresh mailboxes per solve:
    flags and epochs start at zero), and the mailbox ABI's argument checks."""
    import ctypes
    from paper_2202_10042_b200 import _lib as L
    n, world = 3001, 4
    a, b = _pair(n, 41)
    ref = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=2e-3, itr_max=30, domain="log", input_is_log=True)
    for _ in range(2):
        o = shard.solve_segments(_cuda(a), _cuda(b), world, h=1 / n, eps=2e-3, itr_max=30, input_is_log=True,
                                 fused=True)
        _parity(o, ref)
    lib = L.lib()
    assert lib.fs1_shard_mailbox_bytes(0) == 0 and lib.fs1_shard_mailbox_bytes(17) == 0
    assert lib.fs1_shard_mailbox_bytes(16) >= 16 * 8 * 8 + 17 * 4
    p = ctypes.c_void_p()
    assert lib.fs1_shard_mailbox_alloc(0, 0, ctypes.byref(p), None) == L.FS1_ERR_ARG
    assert lib.fs1_shard_mailbox_alloc(2, 0, None, None) == L.FS1_ERR_ARG
    assert lib.fs1_shard_set_mailboxes(None, None) == L.FS1_ERR_ARG
    r = shard.ShardRank(n, 2, 0, h=1 / n, eps=2e-3, itr_max=1, input_is_log=True)
    with pytest.raises(L.FS1Error):
        r.set_mailboxes([0, 0])  # NULL mailbox


def test_shard_decide_and_sum_on_device():
    """fs1_shard_decide / fs1_shard_sum: the loop-top rule and the rank-ordered sums run on
    the device; they equal the host-side rank-ordered fp64 sums bitwise."""
    n = 5000
    r = shard.ShardRank(n, 3, 0, h=1.0 / n, eps=1e-2, itr_max=10, tol=1e-9, device=0)
    dev = torch.device("cuda:0")
    rows = torch.tensor([[0.1, 0.0], [1e-17, 0.0], [0.3, 0.0]], dtype=torch.float64, device=dev)
    err, f, ls = r.decide(rows, 4)
    host = 0.0
    for k in range(3):
        host += rows[k, 0].item()
    assert err == host and f == 0 and ls == 4
    small = torch.tensor([[4e-10, 0.0], [5e-10, 0.0], [0.0, 0.0]], dtype=torch.float64, device=dev)
    assert r.decide(small, 6)[1] == 1                      # err <= tol: CONVERGED
    assert r.decide(rows, 10)[1] == 4                      # l >= itr_max: ITR_MAX
    bad = torch.tensor([[0.1, 0.0], [0.2, 7.0], [0.3, 5.0]], dtype=torch.float64, device=dev)
    e2, f2, l2 = r.decide(bad, 8)
    assert f2 == 2 and l2 == 5                             # the first non-finite iteration
    parts = torch.tensor([[1.0 / 3.0], [1e-20], [2.0 / 7.0]], dtype=torch.float64, device=dev)
    s = r.rank_sum(parts).item()
    assert s == (0.0 + 1.0 / 3.0) + 1e-20 + 2.0 / 7.0
