"""One 1D FS-1 problem sharded over ranks (include/fs1_shard.h).

Every rank (one GPU) owns a contiguous segment of whole 256-point tiles.  Per
half-step the ranks exchange the totals of the consumed vector (4 doubles each,
the recursion values a segment passes to its neighbours) with
one all-gather, then each rank runs `fs1_shard_half` on its segment.  This module
is marshalling and loop control only (Algorithm 1's while, with the
readings of DESIGN.md R2-R6); every arithmetic step runs in the CUDA kernels.

With tol = 0 (fixed iterations) one iteration — both half-steps of every local rank and
both exchanges — is captured once as a CUDA graph and replayed (`_run_graph`).

`fused=True` replaces the per-half-step all-gather of the totals by the fused
exchange of include/fs1_shard.h: the kernel producing a rank's totals stores them
into every rank's mailbox over peer memory (CUDA IPC mappings of the peers'
mailboxes on the NVLink box) and the next half-step's kernel waits on the flags —
no collective and no host step per half-step.  The check-step error sum and the
cost still go through torch.distributed.

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
        self.decision = torch.zeros(4, dtype=torch.float64, device=dev)
        self.total = torch.zeros(1, dtype=torch.float64, device=dev)

    def set_mailboxes(self, boxes):
        """boxes: every rank's mailbox pointer (int) as seen from this device; None = off."""
        arr = None if boxes is None else (ctypes.c_void_p * len(boxes))(*boxes)
        self._ok(L.lib().fs1_shard_set_mailboxes(self._h, arr), "fs1_shard_set_mailboxes")

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

    def decide(self, all_errflag, l):
        """fs1_shard_decide: (err, flag, l at stop) of the loop top, computed on the device
        from every rank's errflag row; the host reads the result only."""
        self._ok(L.lib().fs1_shard_decide(self._h, _ptr(all_errflag.contiguous()), l, _ptr(self.decision),
                                          _stream(self.device)), "fs1_shard_decide")
        d = self.decision.cpu()  # one host read per check
        return float(d[0]), int(d[1]), int(d[2])

    def rank_sum(self, rows, col=0):
        """fs1_shard_sum: the rank-ordered sum of column `col` of [world][k] rows (device)."""
        rows = rows.contiguous()
        self._ok(L.lib().fs1_shard_sum(self._h, _ptr(rows), rows.shape[1], col, _ptr(self.total),
                                       _stream(self.device)), "fs1_shard_sum")
        return self.total

    def cost_totals(self, psi):
        self._ok(L.lib().fs1_shard_cost_totals(self._h, psi, _ptr(self.tot8), _ptr(self.ws),
                                               _stream(self.device)), "fs1_shard_cost_totals")
        return self.tot8

    def finish(self, psi, all_tot8, u_seg, v_seg, want_cost=True):
        self._ok(L.lib().fs1_shard_finish(self._h, psi, _ptr(all_tot8) if want_cost else None, _ptr(u_seg),
                                          _ptr(v_seg), _ptr(self.cost) if want_cost else None, _ptr(self.ws),
                                          _stream(self.device)), "fs1_shard_finish")
        return self.cost


def _run(ranks, segs_a, segs_b, gather, itr_max, tol, check_interval, want_cost, tgather=None):
    """Algorithm 1's loop over lock-stepped ranks.  gather(list of per-local-rank tensors)
    -> [world, k] tensor of every rank's values in rank order (the one exchange);
    tgather: the same for the totals (None: `gather`; fused exchange: returns None)."""
    tgather = tgather or gather
    tots = [r.init(a, b) for r, a, b in zip(ranks, segs_a, segs_b)]
    use_tol = tol > 0.0
    l, qi, hs, flag, err = 0, 0, 0, 4, float("nan")
    while True:
        check = l >= itr_max or (use_tol and l % check_interval == 0)
        last = l >= itr_max
        qo = qi ^ 1 if check else qi
        allT = tgather(tots)
        outs = [r.half(0, hs, check, not last, l + 1, qi, qo, allT) for r in ranks]
        if check:
            # the stop rule of line 2 on the device (rank-ordered error sum, first non-finite
            # iteration); one host read of the decision per check
            err, f, lstop = ranks[0].decide(gather([o[1] for o in outs]), l)
            if f:
                l, flag = (lstop if f == 2 else l), f
                break
            qi = qo
        hs += 1
        allT = tgather([o[0].clone() for o in outs])
        tots = [r.half(1, hs, False, True, l + 1, qi, qi, allT)[0].clone() for r in ranks]
        hs += 1
        l += 1
    return l, qi, flag, err


def _run_graph(ranks, segs_a, segs_b, gather, itr_max, tgather=None):
    """The fixed-iteration loop (tol = 0) with one iteration captured as a
    CUDA graph — both half-steps of every local rank and both exchanges — and replayed:
    no host round trip or per-kernel launch cost per half-step.  The non-finite record
    uses the plan's device iteration counter (l1 = -1).  Same kernels, same order, same
    results as `_run`."""
    tgather = tgather or gather
    for r, a, b in zip(ranks, segs_a, segs_b):
        r.init(a, b)

    def iteration():
        allT = tgather([r.tot for r in ranks])
        outs = [r.half(0, 0, False, True, -1, 0, 0, allT) for r in ranks]
        allT2 = tgather([o[0].clone() for o in outs])
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
    allT = tgather([r.tot for r in ranks])
    outs = [r.half(0, 0, True, False, itr_max + 1, 0, 1, allT) for r in ranks]
    err, f, lstop = ranks[0].decide(gather([o[1] for o in outs]), itr_max)
    if f == 2:
        return lstop, 0, 2, err
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


class Mailbox:
    """One rank's mailbox of the fused exchange (fs1_shard_mailbox_*): device memory
    its peers write into, with the CUDA IPC handle that maps it in their processes."""

    def __init__(self, world, device):
        self.ptr = ctypes.c_void_p()
        h = (ctypes.c_ubyte * 64)()
        s = L.lib().fs1_shard_mailbox_alloc(world, device, ctypes.byref(self.ptr), h)
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_shard_mailbox_alloc")
        self.handle = bytes(h)
        self.opened = []

    def open_peer(self, handle, device):
        p = ctypes.c_void_p()
        s = L.lib().fs1_shard_mailbox_open(handle, device, ctypes.byref(p))
        if s != L.FS1_OK:
            raise L.FS1Error(s, "fs1_shard_mailbox_open")
        self.opened.append(p)
        return p.value

    def free(self):
        torch.cuda.synchronize()
        for p in self.opened:
            L.lib().fs1_shard_mailbox_close(p)
        self.opened = []
        if self.ptr.value:
            L.lib().fs1_shard_mailbox_free(self.ptr)
            self.ptr = ctypes.c_void_p()


def solve_segments(a, b, world, *, h, eps, itr_max, tol=0.0, check_interval=1, input_is_log=False,
                   want_cost=True, graph=True, fused=False):
    """All `world` ranks in this process on a's device (lock step); a, b: [N] fp64 CUDA.
    Returns {u, v (full F, G), iters, err, flags, cost} like fs1.solve for batch 1.
    fused: the totals move through the ranks' mailboxes (here all on one device, so the
    kernels' flag waits are already satisfied when they run: the lock step issues
    every rank's producer before any consumer)."""
    n = a.numel()
    dev = a.device.index
    ranks = [ShardRank(n, world, r, h=h, eps=eps, itr_max=itr_max, tol=tol, check_interval=check_interval,
                       input_is_log=input_is_log, device=dev) for r in range(world)]
    sa = [a[r.lo:r.lo + r.len].contiguous() for r in ranks]
    sb = [b[r.lo:r.lo + r.len].contiguous() for r in ranks]
    gather = lambda ts: torch.stack([t.clone() for t in ts])  # noqa: E731
    tgather, boxes = None, []
    if fused:
        boxes = [Mailbox(world, dev) for _ in range(world)]
        for r in ranks:
            r.set_mailboxes([bx.ptr.value for bx in boxes])
        tgather = lambda ts: None  # noqa: E731
    try:
        if graph and tol == 0.0:
            l, qi, flag, err = _run_graph(ranks, sa, sb, gather, itr_max, tgather)
        else:
            l, qi, flag, err = _run(ranks, sa, sb, gather, itr_max, tol, check_interval, want_cost, tgather)
    finally:
        for bx in boxes:
            bx.free()
        if fused:
            for r in ranks:
                r.set_mailboxes(None)
    ok = flag != 2
    us, vs, parts = _finish(ranks, qi, gather, flag, want_cost and ok, lambda r: a.device)
    cost = ranks[0].rank_sum(gather(parts)).item() if (want_cost and ok) else float("nan")
    return {"u": torch.cat(us), "v": torch.cat(vs), "iters": l, "err": err if ok else float("nan"),
            "flags": flag, "cost": cost, "segments": [(r.lo, r.len) for r in ranks]}


def solve_sharded(a_seg, b_seg, n, *, h, eps, itr_max, tol=0.0, check_interval=1, input_is_log=False,
                  want_cost=True, group=None, graph=True, fused=False):
    """This process's rank of a torch.distributed job: a_seg, b_seg are its segment
    [lo, lo+len) of the N-point problem (see `segment`).  Collectives: one all-gather of
    4 doubles per half-step (none with fused=True: the kernels deliver the totals into
    the peers' IPC-mapped mailboxes), of 2 per check, of 8 for the cost."""
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

    tgather, box = None, None
    if fused:
        box = Mailbox(world, dev)
        handles = exchange_handles(box.handle, group)
        ptrs = [box.ptr.value if k == rank else box.open_peer(handles[k], dev) for k in range(world)]
        r.set_mailboxes(ptrs)
        tgather = lambda ts: None  # noqa: E731
        dist.barrier(group)  # every mailbox mapped before any rank's first delivery
    try:
        if graph and tol == 0.0:
            l, qi, flag, err = _run_graph([r], [a_seg], [b_seg], gather, itr_max, tgather)
        else:
            l, qi, flag, err = _run([r], [a_seg], [b_seg], gather, itr_max, tol, check_interval, want_cost,
                                    tgather)
    finally:
        if box is not None:
            torch.cuda.synchronize()
            dist.barrier(group)  # no peer still writes into this mailbox
            box.free()
            r.set_mailboxes(None)
    ok = flag != 2
    us, vs, parts = _finish([r], qi, gather, flag, want_cost and ok, lambda _: a_seg.device)
    cost = float("nan")
    if want_cost and ok:
        cost = r.rank_sum(gather([parts[0]])).item()
    return {"u": us[0], "v": vs[0], "iters": l, "err": err if ok else float("nan"), "flags": flag,
            "cost": cost, "segment": (r.lo, r.len)}


def exchange_handles(handle, group=None):
    """Every rank's mailbox IPC handle (bytes) in rank order: one all_gather_object, once
    per solve (host-side, any backend)."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, handle, group=group)
    if any(not isinstance(h, bytes) or len(h) != len(handle) for h in handles):
        raise RuntimeError("mailbox handle exchange: malformed handle")
    return handles


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
