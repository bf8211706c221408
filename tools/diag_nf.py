import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import sinkhorn, dense
from paper_2202_10042_b200 import fs1
n = 200
x = (np.arange(n) + 0.5) / n
a = np.exp(-((x - 0.2) / 0.05) ** 2) + 1e-3
b = np.exp(-((x - 0.8) / 0.05) ** 2) + 1e-3
a, b = a / a.sum(), b / b.sum()
ag = torch.from_numpy(a[None]).cuda(); bg = torch.from_numpy(b[None]).cuda()
for k in [1, 2, 5, 10, 20, 40, 60, 70, 80, 90, 97]:
    o = fs1.solve(ag, bg, h=1 / n, eps=5e-4, itr_max=k)
    r = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=5e-4, itr_max=k)
    F = np.log(o["u"].cpu().numpy()[0]); G = np.log(o["v"].cpu().numpy()[0])
    dF = np.abs(F - r["F"][0]); dG = np.abs(G - r["G"][0])
    i = int(np.argmax(dF))
    print(k, "dF", dF.max(), "at", i, F[i], r["F"][0][i], "dG", dG.max(), int(np.argmax(dG)), flush=True)
# apply on the oracle's state at k=90
r = sinkhorn.solve(a, b, n=n, h1=1 / n, eps=5e-4, itr_max=90)
phi = np.exp(r["F"][0]); K = dense.kernel(n, dense.lam(1 / n, 5e-4))
y = fs1.apply(torch.from_numpy(phi[None]).cuda(), h=1 / n, eps=5e-4).cpu().numpy()[0]
yr = K @ phi
d = np.abs(y / yr - 1)
print("apply rel", d.max(), int(np.argmax(d)), y[np.argmax(d)], yr[np.argmax(d)])
print("plan", fs1.plan(fs1.Spec(ndim=1, n=n, m=1, h1=1/n, h2=0.0, eps=5e-4, batch=1, dtype=torch.float64, itr_max=90)).info())
