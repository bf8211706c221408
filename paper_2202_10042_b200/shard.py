"""One 1D FS-1 problem sharded over ranks (include/fs1_shard.h).

Every rank (one GPU) owns a contiguous segment of whole 256-point tiles.  Per
half-step the ranks exchange the totals of the consumed vector (4 doubles each,
the recursion values a segment passes to its neighbours) with
one all-gather, then each rank runs `fs1_shard_half` on its segment.  This module
is marshalling and loop control only (Algorithm 1's while, with the
readings of DESIGN.md R2-R6); every arithmetic step runs in the CUDA kernels.

With tol = 0 (fixed iterations) one iteration — both half-steps of every local rank and
both exchanges — is captured once as a CUDA graph and replayed (`_run_graph`).

Two drivers share `ShardRank`:
  * `solve_sharded`    one rank per process, totals moved by torch.distributed
                       (NCCL over NVLink on the GPU box; gloo in CPU tests);
  * `solve_segments`   all ranks in one process on one device, in lock step, the
                       all-gather done by concatenation (single-GPU tests and
                       world-size sweeps: the per-rank work is identical).
"""
from __future__ import annotations

import ctypes
import math

import torch

from . import _lib as L
from .fs1 import _ptr, _stream


class ShardRank:
    """fs1_shard_* state of one rank: plan, workspace and the small device scratch."""

    def __init__(self, n, world, rank, *, h, eps, itr_max, tol=0.0, check_interval=1,
                 input_is_log=False, device=0):
        self.device = device
        self.world, self.rank = world, rank
        d = L.Desc(ndim=1, n=n, m=1, h1=h, h2=0.0, eps=eps, batch=1, dtype=L.FS1_F64,
                   domain=L.FS1_LOG, input_is_log=int(input_is_log), itr_max=itr_max, tol=tol,
                   check_interval=check_interval, warm_start=0)
        self._h = ctypes.c_void_p()
        ws = ctypes.c_size_t()
        lo, ln = ctypes.c_int64(), ctypes.c_int64()
        s = L.lib().fs1_shard_plan(ctypes.byref(d), world, rank, device, ctypes.byref(self._h),
                                   ctypes.byref(ws), ctypes.byref(lo), ctypes.byref(ln))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_shard_plan")
        self.lo, self.len = lo.value, ln.value
        dev = torch.device(f"cuda:{device}")
        raw = torch.empty(ws.value + 256, dtype=torch.uint8, device=dev)
        self._raw = raw
        self.ws = raw[(-raw.data_ptr()) % 256:]
        self.tot = torch.zeros(4, dtype=torch.float64, device=dev)
        self.errflag = torch.zeros(2, dtype=torch.float64, device=dev)
        self.tot8 = torch.zeros(8, dtype=torch.float64, device=dev)
        self.cost = torch.zeros(1, dtype=torch.float64, device=dev)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            try:
                L.lib().fs1_shard_destroy(h)
            except Exception:
                pass
            self._h = None

    def _ok(self, s, what):
        if s != L.FS1_OK:
            raise L.FS1Error(s, what)

    def init(self, a_seg, b_seg):
        self._ok(L.lib().fs1_shard_init(self._h, _ptr(a_seg), _ptr(b_seg), _ptr(self.tot), _ptr(self.ws),
                                        _stream(self.device)), "fs1_shard_init")
        return self.tot

    def half(self, which, hs, check, write, l1, psi_in, psi_out, all_tot):
        self._ok(L.lib().fs1_shard_half(self._h, which, hs, int(check), int(write), l1, psi_in, psi_out,
                                        _ptr(all_tot), _ptr(self.tot), _ptr(self.errflag), _ptr(self.ws),
                                        _stream(self.device)), "fs1_shard_half")
        return self.tot, self.errflag

    def cost_totals(self, psi):
        self._ok(L.lib().fs1_shard_cost_totals(self._h, psi, _ptr(self.tot8), _ptr(self.ws),
                                               _stream(self.device)), "fs1_shard_cost_totals")
        return self.tot8

    def finish(self, psi, all_tot8, u_seg, v_seg, want_cost=True):
        self._ok(L.lib().fs1_shard_finish(self._h, psi, _ptr(all_tot8) if want_cost else None, _ptr(u_seg),
                                          _ptr(v_seg), _ptr(self.cost) if want_cost else None, _ptr(self.ws),
                                          _stream(self.device)), "fs1_shard_finish")
        return self.cost


def _run(ranks, segs_a, segs_b, gather, itr_max, tol, check_interval, want_cost):
    """Algorithm 1's loop over lock-stepped ranks.  gather(list of per-local-rank tensors)
    -> [world, k] tensor of every rank's values in rank order (the one exchange)."""
    tots = [r.init(a, b) for r, a, b in zip(ranks, segs_a, segs_b)]
    use_tol = tol > 0.0
    l, qi, hs, flag, err = 0, 0, 0, 4, float("nan")
    while True:
        check = l >= itr_max or (use_tol and l % check_interval == 0)
        last = l >= itr_max
        qo = qi ^ 1 if check else qi
        allT = gather(tots)
        outs = [r.half(0, hs, check, not last, l + 1, qi, qo, allT) for r in ranks]
        if check:
            ef = gather([o[1] for o in outs]).cpu()  # one host sync per check
            err = float(sum(ef[k, 0].item() for k in range(ef.shape[0])))  # fixed rank order
            bad = [int(ef[k, 1].item()) for k in range(ef.shape[0]) if ef[k, 1].item() > 0]
            if bad:  # "terminates abnormally": the first non-finite iteration
                l, flag = min(bad), 2
                break
            if last or err <= tol:
                flag = 1 if (use_tol and err <= tol) else 4
                break
            qi = qo
        hs += 1
        allT = gather([o[0].clone() for o in outs])
        tots = [r.half(1, hs, False, True, l + 1, qi, qi, allT)[0].clone() for r in ranks]
        hs += 1
        l += 1
    return l, qi, flag, err


def _run_graph(ranks, segs_a, segs_b, gather, itr_max):
    """The fixed-iteration loop (tol = 0) with one iteration captured as a
    CUDA graph — both half-steps of every local rank and both exchanges — and replayed:
    no host round trip or per-kernel launch cost per half-step.  The non-finite record
    uses the plan's device iteration counter (l1 = -1).  Same kernels, same order, same
    results as `_run`."""
    for r, a, b in zip(ranks, segs_a, segs_b):
        r.init(a, b)

    def iteration():
        allT = gather([r.tot for r in ranks])
        outs = [r.half(0, 0, False, True, -1, 0, 0, allT) for r in ranks]
        allT2 = gather([o[0].clone() for o in outs])
        for r in ranks:
            r.half(1, 1, False, True, -1, 0, 0, allT2)

    if itr_max >= 1:
        iteration()                      # l = 0, eager (also warms the capture path)
    if itr_max >= 2:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            iteration()
        for _ in range(itr_max - 1):     # l = 1 .. itr_max - 1
            g.replay()
    # loop top at l = itr_max: the exit check, psi^(l) kept in buffer 0
    allT = gather([r.tot for r in ranks])
    outs = [r.half(0, 0, True, False, itr_max + 1, 0, 1, allT) for r in ranks]
    ef = gather([o[1] for o in outs]).cpu()
    err = float(sum(ef[k, 0].item() for k in range(ef.shape[0])))
    bad = [int(ef[k, 1].item()) for k in range(ef.shape[0]) if ef[k, 1].item() > 0]
    if bad:
        return min(bad), 0, 2, err
    return itr_max, 0, 4, err


def _finish(ranks, qi, gather, flag, want_cost, dtype_dev):
    us, vs = [], []
    all8 = gather([r.cost_totals(qi).clone() for r in ranks]) if want_cost else None
    parts = []
    for r in ranks:
        u = torch.empty(r.len, dtype=torch.float64, device=dtype_dev(r))
        v = torch.empty_like(u)
        c = r.finish(qi, all8, u, v, want_cost=want_cost)
        parts.append(c.clone())
        us.append(u)
        vs.append(v)
    return us, vs, parts


def solve_segments(a, b, world, *, h, eps, itr_max, tol=0.0, check_interval=1, input_is_log=False,
                   want_cost=True, graph=True):
    """All `world` ranks in this process on a's device (lock step); a, b: [N] fp64 CUDA.
    Returns {u, v (full F, G), iters, err, flags, cost} like fs1.solve for batch 1."""
    n = a.numel()
    dev = a.device.index
    ranks = [ShardRank(n, world, r, h=h, eps=eps, itr_max=itr_max, tol=tol, check_interval=check_interval,
                       input_is_log=input_is_log, device=dev) for r in range(world)]
    sa = [a[r.lo:r.lo + r.len].contiguous() for r in ranks]
    sb = [b[r.lo:r.lo + r.len].contiguous() for r in ranks]
    gather = lambda ts: torch.stack([t.clone() for t in ts])  # noqa: E731
    if graph and tol == 0.0:
        l, qi, flag, err = _run_graph(ranks, sa, sb, gather, itr_max)
    else:
        l, qi, flag, err = _run(ranks, sa, sb, gather, itr_max, tol, check_interval, want_cost)
    ok = flag != 2
    us, vs, parts = _finish(ranks, qi, gather, flag, want_cost and ok, lambda r: a.device)
    cost = float(sum(p.item() for p in parts)) if (want_cost and ok) else float("nan")
    return {"u": torch.cat(us), "v": torch.cat(vs), "iters": l, "err": err if ok else float("nan"),
            "flags": flag, "cost": cost, "segments": [(r.lo, r.len) for r in ranks]}


def solve_sharded(a_seg, b_seg, n, *, h, eps, itr_max, tol=0.0, check_interval=1, input_is_log=False,
                  want_cost=True, group=None, graph=True):
    """This process's rank of a torch.distributed job: a_seg, b_seg are its segment
    [lo, lo+len) of the N-point problem (see `segment`).  Collectives: one all-gather of
    4 doubles per half-step, of 2 per check, of 8 for the cost, one all-reduce at exit."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = a_seg.device.index
    r = ShardRank(n, world, rank, h=h, eps=eps, itr_max=itr_max, tol=tol, check_interval=check_interval,
                  input_is_log=input_is_log, device=dev)
    if a_seg.numel() != r.len or b_seg.numel() != r.len:
        raise ValueError(f"rank {rank}: segment length {r.len} expected, got {a_seg.numel()}")

    def gather(ts):
        (t,) = ts
        return gather_totals(t, group)

    if graph and tol == 0.0:
        l, qi, flag, err = _run_graph([r], [a_seg], [b_seg], gather, itr_max)
    else:
        l, qi, flag, err = _run([r], [a_seg], [b_seg], gather, itr_max, tol, check_interval, want_cost)
    ok = flag != 2
    us, vs, parts = _finish([r], qi, gather, flag, want_cost and ok, lambda _: a_seg.device)
    cost = float("nan")
    if want_cost and ok:
        allc = gather([parts[0]]).cpu()
        cost = float(sum(allc[k, 0].item() for k in range(world)))
    return {"u": us[0], "v": vs[0], "iters": l, "err": err if ok else float("nan"), "flags": flag,
            "cost": cost, "segment": (r.lo, r.len)}


def gather_totals(t, group=None):
    """[world, k] = every rank's k values in rank order (the per-half-step exchange):
    one all_gather_into_tensor over NCCL; a list all_gather on other backends (gloo)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = t.contiguous().reshape(-1)
    out = torch.empty(world, t.numel(), dtype=t.dtype, device=t.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, t, group=group)
    else:
        dist.all_gather(list(out.unbind(0)), t, group=group)
    return out


def segment(n, world, rank):
    """[lo, lo + len) of rank's segment: whole 256-point tiles split as evenly as possible."""
    tiles = -(-n // 256)
    t0, t1 = rank * tiles // world, (rank + 1) * tiles // world
    lo = t0 * 256
    return lo, min(t1 * 256, n) - lo
