"""Time one persistent-kernel variant on a C2-recipe batch at another N (test-only override)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1
n, batch, kern = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
cfg = gi.CONFIGS["c2"]
A, B = gi.batch(cfg, range(batch), n=n)
a, b = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
kw = dict(h=1.0 / n, eps=cfg.eps * 1024 / n, itr_max=cfg.itr_max, domain="log", kernel=kern)
for _ in range(5):  # warm-up (clocks ramp)
    o = fs1.solve(a, b, **kw)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); o = fs1.solve(a, b, **kw); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
spec = fs1.Spec(ndim=1, n=n, m=1, h1=1.0 / n, h2=0.0, eps=kw["eps"], batch=batch, dtype=torch.float32,
                domain="log", itr_max=cfg.itr_max, kernel=kern)
ms = min(ts)
print(n, batch, fs1.plan(spec).info()["kernel"], f"{ms:.3f} ms", f"{n * batch * cfg.itr_max / ms / 1e9:.3f} Gupd/ms")
