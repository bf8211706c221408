"""GPU parity of K4, the paper's own stabilised FS-1 (Remark 2.1 absorption + Remark 3.2
recursions; R8, R29, R30), against the oracle
oracle/stabilized.py (pinned in tests/test_oracle_stabilized.py).

fp64: potentials norm-wise at 1e-10 (R17), cost and err at 1e-10, iterations
and flags exact.  The headline case is the paper's stabilisation study: the Ricker pair
at eps = 1e-3, where the unstabilised iteration terminates abnormally and
the stabilised one runs all 2000 iterations.
"""
import math
import sys

import numpy as np
import pytest

import fs1_inputs as gi
from oracle import recur, sinkhorn
from oracle import stabilized as st
from tests.gpu_util import assert_solve_parity, rel, rel_norm

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402

TOL = 1e-10


def _cuda(x):
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()


def _stab(a, b, *, h, eps, itr_max, tol=0.0, tau=0.0, input_is_log=False):
    return fs1.solve(_cuda(a), _cuda(b), h=h, eps=eps, itr_max=itr_max, tol=tol, domain="stabilized",
                     tau=tau, input_is_log=input_is_log)


def _ref(a, b, **kw):
    """Oracle, one pair at a time, stacked like a batched result."""
    A, B = np.atleast_2d(a), np.atleast_2d(b)
    rs = [st.solve_stab(A[p], B[p], n=A.shape[1], **kw) for p in range(A.shape[0])]
    out = {k: np.concatenate([r[k] for r in rs]) for k in ("F", "G", "iters", "err", "flags", "cost")}
    out["absorptions"] = [r["absorptions"] for r in rs]
    return out


@pytest.mark.parametrize("n", [500, 2000, 8000])
def test_ricker_eps_1e3_full_protocol(n):
    """2000 iterations at eps = 1e-3 complete (the unstabilised run aborts)."""
    a, b = gi.ricker_pair(n)
    h, eps, itr = 8.0 / (n - 1), 1e-3, 2000
    A, B = np.stack([a, a]), np.stack([b, b])
    out = _stab(A, B, h=h, eps=eps, itr_max=itr)
    ref = _ref(a, b, h=h, eps=eps, itr_max=itr)
    assert len(ref["absorptions"][0]) > 10
    assert np.all(out["flags"].cpu().numpy() == 4) and np.all(out["iters"].cpu().numpy() == itr)
    assert_solve_parity(out, ref, "log", "f64", tol=TOL, pairs=[0])
    # both rows of the batch are the same problem: bitwise the same result
    u = out["u"].cpu().numpy()
    assert np.array_equal(u[0], u[1]) and out["cost"][0].item() == out["cost"][1].item()
    # the unstabilised iteration of the same problem terminates abnormally
    un = fs1.solve(_cuda(A[:1]), _cuda(B[:1]), h=h, eps=eps, itr_max=itr, domain="scaling")
    assert un["flags"].item() == 2


@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 100, 513, 1000, 2049, 4097, 8192])
def test_random_pairs_forced_absorptions(n):
    """Random positive pairs, tau = 1e3 (absorbing every few iterations), every size class
    of the instantiation table including ragged tails."""
    rng = np.random.default_rng(n)
    A, B = gi.random_positive(rng, (2, n)), gi.random_positive(rng, (2, n))
    h, eps, itr = 1.0 / n, 0.004, 120
    out = _stab(A, B, h=h, eps=eps, itr_max=itr, tau=1e3)
    ref = _ref(A, B, h=h, eps=eps, itr_max=itr, tau=1e3)
    assert_solve_parity(out, ref, "log", "f64", tol=TOL)


def test_tau_infinite_equals_plain_scaling_until_overflow():
    """With tau above any value the state reaches, nothing is absorbed and K4 is the plain
    scaling-domain Algorithm 1 (every Remark 3.2 factor is exactly lambda)."""
    rng = np.random.default_rng(5)
    n = 300
    A, B = gi.random_positive(rng, (1, n)), gi.random_positive(rng, (1, n))
    kw = dict(h=1.0 / n, eps=0.05, itr_max=80)
    out = _stab(A, B, tau=sys.float_info.max, **kw)
    ref = sinkhorn.solve(A, B, n=n, h1=kw["h"], eps=kw["eps"], itr_max=kw["itr_max"])
    assert_solve_parity(out, ref, "log", "f64", tol=TOL)


def test_tolerance_stop():
    """err <= tol stops the loop (line 2 with the rescaled kernel); the iteration lands within
    +-1 of the oracle's (R22), and the fixed-iteration replay at the oracle's l* matches."""
    n = 700
    a, b = gi.pair("c1", 0, n=n)        # C1's recipe (converges at eps = 1e-2)
    h, eps, tau = 1.0 / n, 1e-2, 1e3     # tau = 1e3: absorptions along the way
    ref = _ref(a, b, h=h, eps=eps, itr_max=20000, tol=1e-9, tau=tau)
    assert ref["flags"][0] == 1 and ref["absorptions"][0]
    out = _stab(a[None], b[None], h=h, eps=eps, itr_max=20000, tol=1e-9, tau=tau)
    assert out["flags"].item() == 1 and abs(out["iters"].item() - ref["iters"][0]) <= 1
    assert out["err"].item() <= 1e-9
    ls = int(ref["iters"][0])
    fixed = _stab(a[None], b[None], h=h, eps=eps, itr_max=ls, tau=tau)
    ref_fixed = _ref(a, b, h=h, eps=eps, itr_max=ls, tau=tau)
    assert_solve_parity(fixed, ref_fixed, "log", "f64", tol=TOL)


def test_input_is_log():
    n = 900
    a, b = gi.ricker_pair(n)
    h, eps = 8.0 / (n - 1), 1e-3
    out = _stab(np.log(a)[None], np.log(b)[None], h=h, eps=eps, itr_max=300, input_is_log=True)
    ref = _ref(a, b, h=h, eps=eps, itr_max=300)
    assert_solve_parity(out, ref, "log", "f64", tol=TOL)


def test_nonfinite_when_never_absorbing():
    """tau = DBL_MAX at eps = 1e-3 (nothing finite exceeds it: never absorbed): the
    iteration overflows like the paper's unstabilised runs, NONFINITE within
    a couple of iterations of the oracle (oracle tau = inf)."""
    n = 500
    a, b = gi.ricker_pair(n)
    h, eps = 8.0 / (n - 1), 1e-3
    out = _stab(a[None], b[None], h=h, eps=eps, itr_max=2000, tau=sys.float_info.max)
    ref = _ref(a, b, h=h, eps=eps, itr_max=2000, tau=math.inf)
    assert ref["flags"][0] == 2 and out["flags"].item() == 2
    assert abs(out["iters"].item() - ref["iters"][0]) <= 2
    assert math.isnan(out["cost"].item()) and math.isnan(out["err"].item())


def test_cost_entry_point():
    """fs1_cost on a stabilised plan: the return line of a given (F, G), equal to the
    oracle's log-sum-exp cost and to the cost the solve fused."""
    n = 2000
    a, b = gi.ricker_pair(n)
    h, eps = 8.0 / (n - 1), 1e-3
    out = _stab(a[None], b[None], h=h, eps=eps, itr_max=500)
    c = fs1.cost(out["u"], out["v"], h=h, eps=eps, domain="stabilized")
    F, G = out["u"].cpu().numpy()[0], out["v"].cpu().numpy()[0]
    ref = recur.sum_exp2(F, recur.wsweep_log(G, h / eps, h))
    assert rel(c.item(), ref) <= TOL and rel(out["cost"].item(), ref) <= TOL


def test_batch_members_independent():
    rng = np.random.default_rng(9)
    n = 777
    A, B = gi.random_positive(rng, (5, n)), gi.random_positive(rng, (5, n))
    kw = dict(h=1.0 / n, eps=0.002, itr_max=90, tau=1e4)
    out = _stab(A, B, **kw)
    for p in (0, 3):
        one = _stab(A[p:p + 1], B[p:p + 1], **kw)
        assert np.array_equal(one["u"].cpu().numpy()[0], out["u"].cpu().numpy()[p])
        assert one["cost"].item() == out["cost"][p].item()


def test_stabilised_equals_log_domain_kernel():
    """Two GPU methods, one iteration: K4 (the paper's stabilisation) and K1's log domain
    agree at eps = 1e-3 on the Ricker pair (N = 8000, 300 iterations)."""
    n = 8000
    a, b = gi.ricker_pair(n)
    h, eps = 8.0 / (n - 1), 1e-3
    s = _stab(a[None], b[None], h=h, eps=eps, itr_max=300)
    lg = fs1.solve(_cuda(a[None]), _cuda(b[None]), h=h, eps=eps, itr_max=300, domain="log")
    assert rel_norm(s["u"].cpu().numpy()[0], lg["u"].cpu().numpy()[0]) <= TOL
    assert rel(s["cost"].item(), lg["cost"].item()) <= TOL
