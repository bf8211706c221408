import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, math
import fs1_inputs as gi
from oracle import sinkhorn, dense
from paper_2202_10042_b200 import fs1
for dt in [torch.float64, torch.float32]:
  for n in [100, 128, 129, 200, 256, 300, 512, 513, 1000]:
    eps = 0.01
    A, B = gi.batch("c5", range(1), n=n)
    a = torch.from_numpy(A).to(dt).cuda(); b = torch.from_numpy(B).to(dt).cuda()
    o = fs1.solve(a, b, h=1/n, eps=eps, itr_max=1, domain="log")
    r = sinkhorn.solve(a.double().cpu().numpy(), b.double().cpu().numpy(), n=n, h1=1/n, eps=eps, itr_max=1)
    y = fs1.apply(a, h=1/n, eps=eps, domain="log").double().cpu().numpy()[0]
    yr = dense.apply_log(a.double().cpu().numpy()[0], (1/n)/eps)
    k = fs1.plan(fs1.Spec(ndim=1,n=n,m=1,h1=1/n,h2=0.0,eps=eps,batch=1,dtype=dt,domain="log",itr_max=1)).info()["kernel"]
    print(dt, n, k, "G err %.2e F err %.2e apply err %.2e" % (np.abs(o["v"][0].double().cpu().numpy()-r["G"][0]).max(), np.abs(o["u"][0].double().cpu().numpy()-r["F"][0]).max(), np.abs(y-yr).max()))
