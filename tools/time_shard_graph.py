"""Device time of one captured iteration (both half-steps of every lock-stepped rank and
both exchanges) of the sharded path, gathered vs fused exchange, CUDA events around
graph replays.  usage: python tools/time_shard_graph.py [log2 N] [replays]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import fs1_inputs as gi
from paper_2202_10042_b200 import shard

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = gi.CONFIGS["c3"]
n = 1 << lg
eps = cfg.eps * (1 << 24) / n
a, b = gi.pair(cfg, 0, n=n)
A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()


def per_iteration(world, fused):
    ranks = [shard.ShardRank(n, world, r, h=1.0 / n, eps=eps, itr_max=10 ** 6, input_is_log=True, device=0)
             for r in range(world)]
    boxes = []
    if fused:
        boxes = [shard.Mailbox(world, 0) for _ in range(world)]
        for r in ranks:
            r.set_mailboxes([bx.ptr.value for bx in boxes])
    gather = (lambda ts: None) if fused else (lambda ts: torch.stack([t.clone() for t in ts]))
    for r in ranks:
        r.init(A[r.lo:r.lo + r.len].contiguous(), B[r.lo:r.lo + r.len].contiguous())

    def iteration():
        allT = gather([r.tot for r in ranks])
        outs = [r.half(0, 0, False, True, -1, 0, 0, allT) for r in ranks]
        allT2 = gather([o[0].clone() for o in outs])
        for r in ranks:
            r.half(1, 1, False, True, -1, 0, 0, allT2)

    iteration()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        iteration()
    for _ in range(5):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    for bx in boxes:
        bx.free()
    return e0.elapsed_time(e1) * 1e3 / reps


for world in (1, 2, 4, 8):
    tg = per_iteration(world, False)
    tf = per_iteration(world, True)
    print(f"N=2^{lg} world {world}: per iteration (2 half-steps, all ranks on one GPU) gathered {tg:.1f} us, "
          f"fused {tf:.1f} us; per rank-half-step {tg / (2 * world):.1f} / {tf / (2 * world):.1f} us", flush=True)
