import numpy as np, torch, sys
sys.path.insert(0, '.')
import fs1_inputs as gi
from oracle import sinkhorn
from paper_2202_10042_b200 import fs1
for n in [500, 2000, 8000]:
    a, b = gi.ricker_pair(n); h = 8.0 / (n - 1); eps = 1e-3
    A, B = torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda()
    un = fs1.solve(A, B, h=h, eps=eps, itr_max=3000, domain="scaling")
    rr = sinkhorn.solve(a[None], b[None], n=n, h1=h, eps=eps, itr_max=3000, domain="scaling", apply="recur")
    rd = sinkhorn.solve(a[None], b[None], n=n, h1=h, eps=eps, itr_max=3000, domain="scaling", apply="dense") if n <= 2000 else None
    # max |log phi| just before the abort
    k = int(rr["iters"][0]) - 1
    rk = sinkhorn.solve(a[None], b[None], n=n, h1=h, eps=eps, itr_max=k, domain="scaling", apply="recur")
    print(n, "gpu", un["iters"].item(), un["flags"].item(), "recur", rr["iters"][0], rr["flags"][0],
          "dense", None if rd is None else (rd["iters"][0], rd["flags"][0]),
          "max|F| at l*-1", np.max(np.abs(rk["F"])), np.max(np.abs(rk["G"])), flush=True)
