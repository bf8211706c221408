import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1
cfg = gi.CONFIGS["c2"]
A, B = gi.batch(cfg, range(cfg.batch))
a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
for dom in ("scaling", "log"):
    kw = dict(h=cfg.h1, eps=cfg.eps, itr_max=cfg.itr_max, domain=dom)
    for _ in range(5): o = fs1.solve(a, b, **kw)
    torch.cuda.synchronize(); ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); o = fs1.solve(a, b, **kw); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    fl = o["flags"].cpu().numpy()
    print(dom, min(ts), "nonfinite pairs", int((fl == 2).sum()))
