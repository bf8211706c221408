import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from oracle import sinkhorn
from paper_2202_10042_b200 import fs1
np.set_printoptions(precision=4, linewidth=200)
for n, dt in [(64, torch.float32), (64, torch.float64), (1024, torch.float32)]:
    A, B = gi.batch("c5", [0], n=n)
    a = torch.from_numpy(A).to(dt).cuda(); b = torch.from_numpy(B).to(dt).cuda()
    for it in [0, 1, 2, 3]:
        o = fs1.solve(a, b, h=1/n, eps=(0.02 if n == 64 else 0.005), itr_max=it, domain="log")
        r = sinkhorn.solve(a.double().cpu().numpy(), b.double().cpu().numpy(), n=n, h1=1/n, eps=(0.02 if n == 64 else 0.005), itr_max=it, domain="log")
        print(n, dt, it, "flags", o["flags"].item(), "iters", o["iters"].item(), "cost", o["cost"].item(), r["cost"][0], "err", o["err"].item(), r["err"][0])
        print("  F gpu", o["u"][0, :8].cpu().numpy(), " ref", r["F"][0, :8])
        print("  G gpu", o["v"][0, :8].cpu().numpy(), " ref", r["G"][0, :8])
        print("  maxdiff F", np.nanmax(np.abs(o["u"][0].double().cpu().numpy() - r["F"][0])), "G", np.nanmax(np.abs(o["v"][0].double().cpu().numpy() - r["G"][0])))
