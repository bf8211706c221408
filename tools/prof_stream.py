"""Run the C3 problem (N=2^24, fp64 log) for a given number of iterations (profiling)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1
itr = int(sys.argv[1]) if len(sys.argv) > 1 else 50
kern = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = gi.CONFIGS["c3"]
a, b = gi.pair(cfg, 0)
A = torch.from_numpy(a[None]).cuda(); B = torch.from_numpy(b[None]).cuda()
for _ in range(2):
    o = fs1.solve(A, B, h=cfg.h1, eps=cfg.eps, itr_max=itr, domain="log", input_is_log=True, kernel=kern)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); o = fs1.solve(A, B, h=cfg.h1, eps=cfg.eps, itr_max=itr, domain="log", input_is_log=True, kernel=kern); e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(f"kernel {kern} itr {itr}: {ms:.3f} ms, {ms/itr*1e3/2:.1f} us per half-step, {48*cfg.n*itr/ms/1e6:.0f} GB/s algorithmic", flush=True)
