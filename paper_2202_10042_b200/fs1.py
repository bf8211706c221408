"""Thin Python face of libfs1 (include/fs1.h): the same entry points, with
PyTorch tensors for device memory and the current CUDA stream.

Nothing here computes any part of the method; every step runs in the CUDA
kernels behind the C ABI.  See DESIGN.md §1 for the boundary.
"""
from __future__ import annotations

import collections
import ctypes
import dataclasses

import torch

from . import _lib as L

_DT = {torch.float32: L.FS1_F32, torch.float64: L.FS1_F64}
_DOMAIN = {"scaling": L.FS1_SCALING, "log": L.FS1_LOG, "stabilized": L.FS1_STABILIZED}


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


@dataclasses.dataclass(frozen=True)
class Spec:
    ndim: int
    n: int
    m: int
    h1: float
    h2: float
    eps: float
    batch: int
    dtype: torch.dtype
    domain: str = "scaling"
    input_is_log: bool = False
    itr_max: int = 1000
    tol: float = 0.0
    check_interval: int = 1
    warm_start: bool = False
    tau: float = 0.0         # "stabilized": absorption threshold (0 = the library default 1e10)
    kernel: int = 0          # 0 auto; test-only overrides (fs1__plan_kind in fs1_api.cu)
    l: int = 1               # 3D: points along axis 3
    h3: float = 0.0          # 3D: axis-3 spacing

    def desc(self) -> L.Desc:
        return L.Desc(ndim=self.ndim, n=self.n, m=self.m, h1=self.h1, h2=self.h2, eps=self.eps,
                      batch=self.batch, dtype=_DT[self.dtype],
                      domain=_DOMAIN[self.domain],
                      input_is_log=int(self.input_is_log), itr_max=self.itr_max, tol=self.tol,
                      check_interval=self.check_interval, warm_start=int(self.warm_start),
                      tau=float(self.tau), l=int(self.l) if self.ndim == 3 else 1,
                      h3=float(self.h3) if self.ndim == 3 else 0.0)


class Plan:
    """fs1_plan / fs1_plan_destroy around one problem description."""

    def __init__(self, spec: Spec, device: int = 0):
        self.spec = spec
        self.device = device
        self._h = ctypes.c_void_p()
        ws = ctypes.c_size_t()
        d = spec.desc()
        if spec.kernel:
            s = L.lib().fs1__plan_kind(ctypes.byref(d), device, spec.kernel, ctypes.byref(self._h),
                                       ctypes.byref(ws))
        else:
            s = L.lib().fs1_plan(ctypes.byref(d), device, ctypes.byref(self._h), ctypes.byref(ws))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_plan")
        self.workspace_bytes = ws.value
        self._ws = {}            # one workspace per CUDA stream (solves on two streams never share one)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().fs1_plan_destroy(h)
            except Exception:  # interpreter shutdown: module globals already torn down
                pass
            self._h = None

    def info(self) -> dict:
        pi = L.PlanInfo()
        s = L.lib().fs1_plan_info(self._h, ctypes.byref(pi))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_plan_info")
        return {"kernel": pi.kernel.decode(), "chunk": pi.chunk, "threads": pi.threads,
                "ctas_per_problem": pi.ctas_per_problem, "grid": pi.grid,
                "smem_bytes": pi.smem_bytes, "workspace_bytes": pi.workspace_bytes}

    def workspace(self):
        """This plan's workspace for the current stream of its device (allocated on first
        use).  The grid-barrier counters and scratch vectors of the multi-CTA kernels live
        there, so two streams running the same plan concurrently each get their own."""
        if not self.workspace_bytes:
            return None
        sid = torch.cuda.current_stream(self.device).cuda_stream
        ws = self._ws.get(sid)
        if ws is None:
            ws = self._ws[sid] = torch.empty(self.workspace_bytes + 256, dtype=torch.uint8,
                                             device=f"cuda:{self.device}")
        off = (-ws.data_ptr()) % 256
        return ws[off:]

    # raw entry points (tensors must be on this plan's device, contiguous)
    def solve_into(self, a, b, u, v, iters, err, flags, cost):
        s = L.lib().fs1_solve(self._h, _ptr(a), _ptr(b), _ptr(u), _ptr(v), _ptr(iters), _ptr(err),
                              _ptr(flags), _ptr(cost), _ptr(self.workspace()), _stream(self.device))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_solve")

    def cost_into(self, u, v, cost):
        s = L.lib().fs1_cost(self._h, _ptr(u), _ptr(v), _ptr(cost), _ptr(self.workspace()),
                             _stream(self.device))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_cost")

    def apply_into(self, x, y):
        s = L.lib().fs1_apply(self._h, _ptr(x), _ptr(y), _ptr(self.workspace()), _stream(self.device))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_apply")


_CACHE: "collections.OrderedDict" = collections.OrderedDict()
CACHE_PLANS = 16          # least-recently-used plans (and their workspaces) kept alive


def plan(spec: Spec, device: int = 0) -> Plan:
    key = (spec, device)
    p = _CACHE.get(key)
    if p is None:
        p = _CACHE[key] = Plan(spec, device)
        while len(_CACHE) > CACHE_PLANS:
            _CACHE.popitem(last=False)
    else:
        _CACHE.move_to_end(key)
    return p


def _check(t, name, dtype, device, size, numel=None):
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype or t.device.index != device or not t.is_contiguous():
        raise ValueError(f"{name}: expected contiguous {dtype} on cuda:{device}")
    if t.numel() == 0 or t.numel() % size:
        raise ValueError(f"{name}: numel {t.numel()} is not a positive multiple of {size}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name}: numel {t.numel()} != {numel} (one row per pair of a)")


def _geom(t, shape, h, h2, h3):
    """(ndim, n, m, l, size, h1, h2, h3) from a tensor's last axis (1D) or shape=(n, m) /
    (n, m, l) (2D / 3D, column-major flat index (z m + j) n + i); h2, h3 default to h."""
    if shape is None:
        return 1, t.shape[-1], 1, 1, t.shape[-1], float(h), 0.0, 0.0
    shape = tuple(int(x) for x in shape)
    if len(shape) == 2:
        n, m = shape
        return 2, n, m, 1, n * m, float(h), float(h if h2 is None else h2), 0.0
    if len(shape) == 3:
        n, m, l = shape
        return (3, n, m, l, n * m * l, float(h), float(h if h2 is None else h2),
                float(h if h3 is None else h3))
    raise ValueError(f"shape must have 2 or 3 axes, got {shape}")


def _spec(t, shape, h, h2, h3, eps, batch, **kw):
    ndim, n, m, l, size, h1, hh2, hh3 = _geom(t, shape, h, h2, h3)
    return Spec(ndim=ndim, n=n, m=m, h1=h1, h2=hh2, eps=float(eps), batch=batch, dtype=t.dtype, l=l, h3=hh3, **kw)


def solve(a, b, *, h, eps, itr_max, tol=0.0, domain="scaling", input_is_log=False,
          check_interval=1, u0=None, v0=None, shape=None, h2=None, h3=None, want_cost=True, kernel=0,
          tau=0.0):
    """Batched FS-1 solve.  a, b: CUDA tensors [batch, n] (1D) or [batch, n*m(*l)] with
    shape=(n, m) / (n, m, l) (2D / 3D, column-major).  domain: "scaling" | "log" |
    "stabilized" (the paper's Remark 2.1 / 3.2 stabilisation, absorption threshold tau).
    Returns dict u, v, iters, err, flags, cost."""
    dev = a.device.index
    size = _geom(a, shape, h, h2, h3)[4]
    _check(a, "a", a.dtype, dev, size)
    _check(b, "b", a.dtype, dev, size, a.numel())
    if (u0 is None) != (v0 is None):
        raise ValueError("warm start needs both u0 and v0 (or neither)")
    if u0 is not None:
        _check(u0, "u0", a.dtype, dev, size, a.numel())
        _check(v0, "v0", a.dtype, dev, size, a.numel())
    batch = a.numel() // size
    spec = _spec(a, shape, h, h2, h3, eps, batch, domain=domain, input_is_log=bool(input_is_log),
                 itr_max=int(itr_max), tol=float(tol), check_interval=int(check_interval),
                 warm_start=u0 is not None, kernel=int(kernel), tau=float(tau))
    p = plan(spec, dev)
    if u0 is not None:
        u = u0.clone(memory_format=torch.contiguous_format)
        v = v0.clone(memory_format=torch.contiguous_format)
    else:
        u, v = torch.empty_like(a), torch.empty_like(b)
    iters = torch.empty(batch, dtype=torch.int32, device=a.device)
    err = torch.empty(batch, dtype=torch.float64, device=a.device)
    flags = torch.empty(batch, dtype=torch.int32, device=a.device)
    cost = torch.empty(batch, dtype=torch.float64, device=a.device) if want_cost else None
    p.solve_into(a, b, u, v, iters, err, flags, cost)
    return {"u": u, "v": v, "iters": iters, "err": err, "flags": flags, "cost": cost}


def cost(u, v, *, h, eps, domain="scaling", shape=None, h2=None, h3=None, kernel=0):
    """The return line (PAPER.md:163 / 339) on a given state."""
    dev = u.device.index
    size = _geom(u, shape, h, h2, h3)[4]
    _check(u, "u", u.dtype, dev, size)
    _check(v, "v", u.dtype, dev, size, u.numel())
    batch = u.numel() // size
    spec = _spec(u, shape, h, h2, h3, eps, batch, domain=domain, itr_max=0, kernel=int(kernel))
    out = torch.empty(batch, dtype=torch.float64, device=u.device)
    plan(spec, dev).cost_into(u, v, out)
    return out


def apply(x, *, h, eps, domain="scaling", shape=None, h2=None, h3=None, kernel=0):
    """y = K x (scaling) or log K e^x (log) for every vector of x."""
    dev = x.device.index
    size = _geom(x, shape, h, h2, h3)[4]
    _check(x, "x", x.dtype, dev, size)
    batch = x.numel() // size
    spec = _spec(x, shape, h, h2, h3, eps, batch, domain=domain, itr_max=0, kernel=int(kernel))
    y = torch.empty_like(x)
    plan(spec, dev).apply_into(x, y)
    return y


def transport_plan(u, v, *, h, eps, domain="scaling", shape=None, h2=None):
    """gamma = diag(phi) K diag(psi) per problem: [batch, n*m, n*m] (fs1_transport_plan)."""
    dev = u.device.index
    size = _geom(u, shape, h, h2, None)[4]
    _check(u, "u", u.dtype, dev, size)
    _check(v, "v", u.dtype, dev, size, u.numel())
    batch = u.numel() // size
    spec = _spec(u, shape, h, h2, None, eps, batch, domain=domain, itr_max=0)
    g = torch.empty(batch, size, size, dtype=u.dtype, device=u.device)
    p = plan(spec, dev)
    s = L.lib().fs1_transport_plan(p._h, _ptr(u), _ptr(v), _ptr(g), _stream(dev))
    if s != L.FS1_OK:
        raise L.FS1Error(s, "fs1_transport_plan")
    return g


def plan_entries(u, v, idx, *, h, eps, domain="scaling", shape=None, h2=None, h3=None):
    """gamma_kl of the transport plan at index triples idx = [count, 3] int64 (problem,
    source flat index, target flat index) for problems of any size: [count] fp64
    (fs1_plan_entries; NaN for a triple out of range)."""
    dev = u.device.index
    size = _geom(u, shape, h, h2, h3)[4]
    _check(u, "u", u.dtype, dev, size)
    _check(v, "v", u.dtype, dev, size, u.numel())
    if idx.dtype != torch.int64 or idx.dim() != 2 or idx.shape[1] != 3 or idx.device != u.device:
        raise ValueError("idx must be an int64 [count, 3] tensor on u's device")
    idx = idx.contiguous()
    batch = u.numel() // size
    spec = _spec(u, shape, h, h2, h3, eps, batch, domain=domain, itr_max=0)
    p = plan(spec, dev)
    out = torch.empty(idx.shape[0], dtype=torch.float64, device=u.device)
    s = L.lib().fs1_plan_entries(p._h, _ptr(u), _ptr(v), _ptr(idx), idx.shape[0], _ptr(out), _stream(dev))
    if s != L.FS1_OK:
        raise L.FS1Error(s, "fs1_plan_entries")
    return out


def dual(a, b, u, v, *, h, eps, domain="scaling", input_is_log=False, shape=None, h2=None, h3=None, kernel=0):
    """fs1_dual: the dual objective of Eq. (2.3) at the state (u, v) for every pair ([batch] fp64)."""
    dev = u.device.index
    size = _geom(u, shape, h, h2, h3)[4]
    _check(u, "u", u.dtype, dev, size)
    for t, nm in ((a, "a"), (b, "b"), (v, "v")):
        _check(t, nm, u.dtype, dev, size, u.numel())
    batch = u.numel() // size
    spec = _spec(u, shape, h, h2, h3, eps, batch, domain=domain, input_is_log=bool(input_is_log), itr_max=0,
                 kernel=int(kernel))
    p = plan(spec, dev)
    scratch = torch.empty_like(u)
    out = torch.empty(batch, dtype=torch.float64, device=u.device)
    s = L.lib().fs1_dual(p._h, _ptr(a), _ptr(b), _ptr(u), _ptr(v), _ptr(scratch), _ptr(out),
                         _ptr(p.workspace()), _stream(dev))
    if s != L.FS1_OK:
        raise L.FS1Error(s, "fs1_dual")
    return out


def solve_eps_scaling(a, b, *, h, eps, eps0, factor, stage_iters, itr_max, tol=0.0, input_is_log=False,
                      check_interval=1, shape=None, h2=None, u0=None, v0=None):
    """fs1_solve_eps_scaling (log domain): the eps-scaling continuation eps0 -> eps; outputs as
    solve() for the last stage, plus 'stages'."""
    dev = a.device.index
    size = _geom(a, shape, h, h2, None)[4]
    _check(a, "a", a.dtype, dev, size)
    _check(b, "b", a.dtype, dev, size, a.numel())
    if (u0 is None) != (v0 is None):
        raise ValueError("warm start needs both u0 and v0 (or neither)")
    batch = a.numel() // size
    spec = _spec(a, shape, h, h2, None, eps, batch, domain="log", input_is_log=bool(input_is_log),
                 itr_max=int(itr_max), tol=float(tol), check_interval=int(check_interval),
                 warm_start=u0 is not None)
    d = spec.desc()
    ns = ctypes.c_int32()
    wsb = ctypes.c_size_t()
    s = L.lib().fs1_eps_scaling_plan(ctypes.byref(d), dev, float(eps0), float(factor), ctypes.byref(ns),
                                     ctypes.byref(wsb))
    if s != L.FS1_OK:
        raise L.FS1Error(s, "fs1_eps_scaling_plan")
    ws = torch.empty(wsb.value + 256, dtype=torch.uint8, device=a.device) if wsb.value else None
    wsp = None if ws is None else ctypes.c_void_p(ws.data_ptr() + (-ws.data_ptr()) % 256)
    if u0 is not None:
        _check(u0, "u0", a.dtype, dev, size, a.numel())
        _check(v0, "v0", a.dtype, dev, size, a.numel())
        u = u0.clone(memory_format=torch.contiguous_format)
        v = v0.clone(memory_format=torch.contiguous_format)
    else:
        u, v = torch.empty_like(a), torch.empty_like(b)
    iters = torch.empty(batch, dtype=torch.int32, device=a.device)
    err = torch.empty(batch, dtype=torch.float64, device=a.device)
    flags = torch.empty(batch, dtype=torch.int32, device=a.device)
    cost = torch.empty(batch, dtype=torch.float64, device=a.device)
    s = L.lib().fs1_solve_eps_scaling(ctypes.byref(d), dev, float(eps0), float(factor), int(stage_iters),
                                      _ptr(a), _ptr(b), _ptr(u), _ptr(v), _ptr(iters), _ptr(err), _ptr(flags),
                                      _ptr(cost), wsp, wsb.value, _stream(dev))
    if s != L.FS1_OK:
        raise L.FS1Error(s, "fs1_solve_eps_scaling")
    # (ws is returned to torch's caching allocator stream-ordered: safe while the launches run)
    return {"u": u, "v": v, "iters": iters, "err": err, "flags": flags, "cost": cost, "stages": int(ns.value)}
