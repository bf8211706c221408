"""Host logic of the sharded single-problem path (paper_2202_10042_b200/shard.py), on CPU.

* the segment split: whole 256-point tiles, contiguous, covering [0, N), balanced;
* the exchange: `gather_totals` under torch.distributed (gloo, world size 2) returns
  every rank's totals in rank order — the all-gather each half-step performs over
  NCCL on the GPU box;
* the loop control `_run` (Algorithm 1's while, readings DESIGN.md
  R2-R6) driven with stand-in ranks that record the calls: paper order (psi step,
  then phi step), the check on the psi half-step at the loop top, psi^(l) kept in
  its buffer when a check stops the loop, the half-step counter, the first
  non-finite iteration, and the fixed rank order of the error sum.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2202_10042_b200 import shard


@pytest.mark.parametrize("n,world", [(1, 1), (256, 1), (257, 2), (1000, 3), (2 ** 24, 8), (5000, 19)])
def test_segment_split(n, world):
    segs = [shard.segment(n, world, r) for r in range(world)]
    assert segs[0][0] == 0 and sum(l for _, l in segs) == n
    for k in range(world - 1):
        assert segs[k][0] + segs[k][1] == segs[k + 1][0]
        assert segs[k][1] % 256 == 0  # whole tiles except the last segment
    tiles = [-(-l // 256) for _, l in segs]
    assert max(tiles) - min(tiles) <= 1


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = torch.tensor([rank + 0.5, -1.0 * rank, 2.0 ** (rank + 3), float(rank)], dtype=torch.float64)
    out = shard.gather_totals(t)
    hs = shard.exchange_handles(bytes([rank + 7]) * 64)  # the fused exchange's IPC handles
    if rank == 0:
        q.put(out.numpy())
        q.put(hs)
    dist.barrier()
    dist.destroy_process_group()


def test_gather_totals_gloo_world2():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = q.get(timeout=120)
    hs = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out.shape == (2, 4)
    for r in range(2):
        assert list(out[r]) == [r + 0.5, -1.0 * r, 2.0 ** (r + 3), float(r)]
    assert hs == [bytes([7]) * 64, bytes([8]) * 64]  # every rank's handle, in rank order


class FakeRank:
    """Stands in for ShardRank: records calls; errors follow `errs` (per check).  `decide`
    stands in for fs1_shard_decide (the device rule, tested on the GPU in
    tests/test_gpu_shard.py) with the same rule written out here."""

    def __init__(self, rank, errs, bad_at=None, fused=False, itr_max=None, tol=None):
        self.rank, self.errs, self.bad_at, self.fused = rank, list(errs), bad_at, fused
        self.itr_max, self.tol = itr_max, tol
        self.calls = []
        self.tot = torch.zeros(4, dtype=torch.float64)
        self.ef = torch.zeros(2, dtype=torch.float64)

    def init(self, a, b):
        self.calls.append(("init",))
        return self.tot

    def half(self, which, hs, check, write, l1, psi_in, psi_out, all_tot):
        assert (all_tot is None) if self.fused else (all_tot.shape[1] == 4)
        self.calls.append(("half", which, hs, check, write, l1, psi_in, psi_out))
        if check:
            e = self.errs.pop(0) if self.errs else 1.0
            bad = self.bad_at if (self.bad_at is not None and l1 - 1 >= self.bad_at) else 0
            self.ef = torch.tensor([e, float(bad)], dtype=torch.float64)
        return self.tot, self.ef

    def decide(self, all_ef, l):
        self.calls.append(("decide", l))
        err = 0.0
        for k in range(all_ef.shape[0]):       # rank order
            err += float(all_ef[k, 0])
        bad = [int(all_ef[k, 1]) for k in range(all_ef.shape[0]) if all_ef[k, 1] > 0]
        if bad:
            return err, 2, min(bad)
        if l >= self.itr_max or err <= self.tol:
            return err, (1 if (self.tol > 0 and err <= self.tol) else 4), l
        return err, 0, l


def _gather(ts):
    return torch.stack([t.clone() for t in ts])


def test_loop_fixed_iterations():
    ranks = [FakeRank(0, [], itr_max=3, tol=0.0), FakeRank(1, [], itr_max=3, tol=0.0)]
    l, qi, flag, err = shard._run(ranks, [None] * 2, [None] * 2, _gather, 3, 0.0, 1, True)
    assert (l, qi, flag) == (3, 0, 4)
    expect = [("init",)]
    hs = 0
    for it in range(3):  # psi step then phi step, no check (tol = 0), psi in place
        expect += [("half", 0, hs, False, True, it + 1, 0, 0), ("half", 1, hs + 1, False, True, it + 1, 0, 0)]
        hs += 2
    expect += [("half", 0, hs, True, False, 4, 0, 1)]  # exit check at l = itr_max, no write
    assert ranks[0].calls == expect + [("decide", 3)]  # the decision is taken once, by rank 0's plan
    assert ranks[1].calls == expect
    assert err == 2.0  # 1.0 + 1.0 in rank order


def test_loop_tolerance_keeps_psi_of_the_stopping_check():
    # rank errors per check at l = 0, 2, 4: sums 3e-9 + ..., stop when <= 1e-9
    r0 = FakeRank(0, [1.0, 1e-6, 4e-10], itr_max=100, tol=1e-9)
    r1 = FakeRank(1, [1.0, 1e-6, 5e-10], itr_max=100, tol=1e-9)
    l, qi, flag, err = shard._run([r0, r1], [None] * 2, [None] * 2, _gather, 100, 1e-9, 2, True)
    assert flag == 1 and l == 4 and err == 4e-10 + 5e-10
    checks = [c for c in r0.calls if c[0] == "half" and c[3]]
    assert [c[5] - 1 for c in checks] == [0, 2, 4]           # loop tops that check
    assert all(c[6] != c[7] for c in checks)                 # psi^(l) survives every check
    # the stopping check wrote into the other buffer; the returned psi is the kept one
    assert qi == checks[-1][6]
    phi_steps = [c for c in r0.calls if c[0] == "half" and c[1] == 1]
    assert all(c[6] == c[7] for c in phi_steps)


def test_loop_nonfinite_reports_first_iteration():
    r0 = FakeRank(0, [1.0] * 10, bad_at=None, itr_max=50, tol=1e-12)
    r1 = FakeRank(1, [1.0] * 10, bad_at=3, itr_max=50, tol=1e-12)
    l, qi, flag, err = shard._run([r0, r1], [None] * 2, [None] * 2, _gather, 50, 1e-12, 5, True)
    assert flag == 2
    assert l == 3  # the device-recorded first non-finite iteration, seen at the check at l = 5


def test_loop_fused_exchange_same_calls_no_totals():
    """fused exchange: the loop passes no totals (the kernels deliver them) and issues
    exactly the gathered loop's calls; the check-step errors still use `gather`."""
    for tol, errs in ((0.0, []), (1e-9, [1.0, 1e-6, 4e-10])):
        kw = dict(itr_max=6, tol=tol)
        g = [FakeRank(0, errs, **kw), FakeRank(1, errs, **kw)]
        f = [FakeRank(0, errs, fused=True, **kw), FakeRank(1, errs, fused=True, **kw)]
        rg = shard._run(g, [None] * 2, [None] * 2, _gather, 6, tol, 2, True)
        rf = shard._run(f, [None] * 2, [None] * 2, _gather, 6, tol, 2, True, tgather=lambda ts: None)
        assert rg == rf
        assert [r.calls for r in g] == [r.calls for r in f]
