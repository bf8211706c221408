"""The Python face's argument checks and per-stream workspaces (paper_2202_10042_b200/fs1.py):
mismatched batch sizes, half-given warm starts and non-contiguous state are refused before
any launch; two streams running the same multi-CTA plan concurrently each use their own
workspace and give the serial results bitwise; the plan cache is bounded."""
import numpy as np
import pytest

import fs1_inputs as gi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402


def _t(x, dt=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(x)).to(device="cuda", dtype=dt)


def test_argument_checks():
    rng = np.random.default_rng(0)
    A, B = gi.random_positive(rng, (4, 64)), gi.random_positive(rng, (4, 64))
    a, b = _t(A), _t(B)
    kw = dict(h=1 / 64, eps=0.02, itr_max=5)
    with pytest.raises(ValueError):
        fs1.solve(a, b[:1], **kw)                       # b has fewer pairs than a
    with pytest.raises(ValueError):
        fs1.solve(a, b, u0=torch.zeros_like(a), **kw)   # u0 without v0
    with pytest.raises(ValueError):
        fs1.solve(a, b, u0=torch.zeros(8, 64, dtype=torch.float64, device="cuda")[::2],
                  v0=torch.zeros_like(a), **kw)         # non-contiguous u0
    with pytest.raises(ValueError):
        fs1.solve(a, b.float(), **kw)                   # dtype mismatch
    with pytest.raises(ValueError):
        fs1.cost(a, b[:2], h=1 / 64, eps=0.02)          # v with fewer pairs than u
    with pytest.raises(ValueError):
        fs1.solve(a.cpu(), b.cpu(), **kw)               # host tensors: no CPU path
    out = fs1.solve(a, b, **kw)                         # and the valid call runs
    assert out["iters"].shape == (4,)


def test_two_streams_same_plan_concurrently():
    """K2 (cooperative grid with its barrier counter in the workspace) on two streams at
    once: each stream gets its own workspace, both results equal the serial one bitwise."""
    cfg = gi.CONFIGS["c3"]
    n = 200000
    a, b = gi.pair(cfg, 0, n=n)
    A, B = _t(a[None]), _t(b[None])
    kw = dict(h=1.0 / n, eps=cfg.eps, itr_max=8, domain="log", input_is_log=True)
    ref = fs1.solve(A, B, **kw)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(s1):
        o1 = fs1.solve(A, B, **kw)
    with torch.cuda.stream(s2):
        o2 = fs1.solve(A, B, **kw)
    torch.cuda.synchronize()
    for o in (o1, o2):
        assert np.array_equal(o["u"].cpu().numpy(), ref["u"].cpu().numpy())
        assert o["cost"].item() == ref["cost"].item()


def test_plan_cache_is_bounded():
    rng = np.random.default_rng(1)
    A, B = gi.random_positive(rng, (1, 32)), gi.random_positive(rng, (1, 32))
    for k in range(fs1.CACHE_PLANS + 8):
        fs1.solve(_t(A), _t(B), h=1 / 32, eps=0.01 + 1e-4 * k, itr_max=2)
    assert len(fs1._CACHE) <= fs1.CACHE_PLANS
