import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from oracle import sinkhorn
from paper_2202_10042_b200 import fs1
np.set_printoptions(precision=5, linewidth=220)
n = 1024
A, B = gi.batch("c5", [0], n=n)
a = torch.from_numpy(A).float().cuda(); b = torch.from_numpy(B).float().cuda()
for it in [2, 3]:
    o = fs1.solve(a, b, h=1/n, eps=0.005, itr_max=it, domain="log")
    r = sinkhorn.solve(a.double().cpu().numpy(), b.double().cpu().numpy(), n=n, h1=1/n, eps=0.005, itr_max=it, domain="log")
    F = o["u"][0].double().cpu().numpy(); G = o["v"][0].double().cpu().numpy()
    bad = np.nonzero(~np.isfinite(F))[0]
    print(it, "bad F idx", bad[:40], len(bad))
    dF = np.abs(F - r["F"][0]); dG = np.abs(G - r["G"][0])
    print(" worst F idx", np.argsort(-np.nan_to_num(dF, nan=1e9, posinf=1e9))[:10], "worst G", np.argsort(-dG)[:10])
    if len(bad):
        i = bad[0]; s = max(0, i - 3)
        print(" F", F[s:i+4]); print(" Fr", r["F"][0][s:i+4]); print(" G", G[s:i+4]); print(" Gr", r["G"][0][s:i+4])
        print(" a", A[0][s:i+4], " b", B[0][s:i+4])
    if it == 2:
        print(" F range", F.min(), F.max(), " G range", G.min(), G.max())
        ch = (np.arange(n) // 32)
        for t in range(32):
            m = ch == t
            print(t, "Fmax %.3f Fmin %.3f Gmax %.3f Gmin %.3f" % (F[m].max(), F[m].min(), G[m].max(), G[m].min()))
