import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import dense, recur, sinkhorn
from paper_2202_10042_b200 import fs1
def cu(x): return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).cuda()
for n in [1, 300, 5000]:
    X = np.random.default_rng(n).normal(size=n)
    y = fs1.apply(cu(X[None]), h=0.1, eps=1.0, domain="log", kernel=2); torch.cuda.synchronize()
    ref = dense.apply_log(X, 0.1)
    print("apply", n, np.max(np.abs(y.cpu().numpy()[0] - ref)), flush=True)
n = 1000
rng = np.random.default_rng(0)
a = rng.uniform(0.1, 1, n); a /= a.sum(); b = rng.uniform(0.1, 1, n); b /= b.sum()
for itr in [0, 1, 5]:
    o = fs1.solve(cu(a[None]), cu(b[None]), h=1/n, eps=1e-2, itr_max=itr, domain="log", kernel=2); torch.cuda.synchronize()
    r = sinkhorn.solve(a, b, n=n, h1=1/n, eps=1e-2, itr_max=itr, domain="log")
    print("solve", itr, np.max(np.abs(o["u"].cpu().numpy()[0] - r["F"][0])), np.max(np.abs(o["v"].cpu().numpy()[0] - r["G"][0])),
          o["cost"].item(), r["cost"][0], o["err"].item(), r["err"][0], o["iters"].item(), o["flags"].item(), flush=True)
