"""Per-half-step time of the sharded path (lock-step ranks on one GPU) vs K2 at N = 2^k."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1, shard
lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
itr = int(sys.argv[2]) if len(sys.argv) > 2 else 50
cfg = gi.CONFIGS["c3"]
n = 1 << lg
eps = cfg.eps * (1 << 24) / n
a, b = gi.pair(cfg, 0, n=n)
A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
def tk2():
    torch.cuda.synchronize(); t = time.perf_counter()
    fs1.solve(A[None], B[None], h=1.0 / n, eps=eps, itr_max=itr, domain="log", input_is_log=True)
    torch.cuda.synchronize(); return time.perf_counter() - t
def tsh(world, it=None, graph=True, fused=False):
    torch.cuda.synchronize(); t = time.perf_counter()
    shard.solve_segments(A, B, world, h=1.0 / n, eps=eps, itr_max=it or itr, input_is_log=True, graph=graph,
                         fused=fused)
    torch.cuda.synchronize(); return time.perf_counter() - t
tk2(); tsh(1)
k2 = min(tk2() for _ in range(3))
for world in (1, 2, 8):
    for graph, fused in ((True, False), (True, True), (False, False), (False, True)):
        t1 = min(tsh(world, itr, graph, fused) for _ in range(2))
        t2 = min(tsh(world, 3 * itr, graph, fused) for _ in range(2))
        per = (t2 - t1) / (4 * itr)  # steady state: marginal cost of a half-step
        print(f"N=2^{lg} world {world} graph {graph} fused {fused}: {per * 1e6:.1f} us per half-step "
              f"(all ranks on one GPU) "
              f"vs K2 {k2 / (2 * itr) * 1e6:.1f} us", flush=True)
