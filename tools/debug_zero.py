import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from oracle import sinkhorn
from paper_2202_10042_b200 import fs1
np.set_printoptions(precision=6, linewidth=200)
n, eps = 256, 0.01
A, B = gi.batch("c5", range(1), n=n)
A[0, 40:90] = 0.0
A /= A.sum()
for it in [1, 2, 5, 40]:
    o = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), h=1/n, eps=eps, itr_max=it, domain="log")
    with np.errstate(divide="ignore"):
        r = sinkhorn.solve(np.log(A), np.log(B), n=n, h1=1/n, eps=eps, itr_max=it, domain="log", input_is_log=True)
    F = o["u"][0].cpu().numpy(); G = o["v"][0].cpu().numpy()
    m = np.isfinite(r["F"][0])
    dF = np.where(m, np.abs(F - r["F"][0]), 0); dG = np.abs(G - r["G"][0])
    print(it, "maxdF", dF.max(), "at", np.argsort(-dF)[:8], "maxdG", dG.max(), "at", np.argsort(-dG)[:8], "plan", fs1.plan(fs1.Spec(ndim=1,n=n,m=1,h1=1/n,h2=0.0,eps=eps,batch=1,dtype=torch.float64,domain="log",itr_max=it)).info()["kernel"])
