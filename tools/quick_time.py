import sys, time, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1

def run(cfgname, batch=None, itr=None, domain=None, reps=3):
    cfg = gi.CONFIGS[cfgname]
    B = batch or cfg.batch
    itr = itr or cfg.itr_max
    dom = domain or cfg.domain
    rng = np.random.default_rng(0)
    # quick synthetic of the right shape (bench uses the real generator)
    A = rng.lognormal(0, 1, (B, cfg.n)); A /= A.sum(1, keepdims=True)
    Bm = rng.lognormal(0, 1, (B, cfg.n)); Bm /= Bm.sum(1, keepdims=True)
    dt = torch.float32 if cfg.dtype == "f32" else torch.float64
    a = torch.from_numpy(A).to(dt).cuda(); b = torch.from_numpy(Bm).to(dt).cuda()
    out = fs1.solve(a, b, h=cfg.h1, eps=cfg.eps, itr_max=itr, domain=dom)
    torch.cuda.synchronize()
    p = fs1.plan(fs1.Spec(ndim=1, n=cfg.n, m=1, h1=cfg.h1, h2=0.0, eps=cfg.eps, batch=B, dtype=dt, domain=dom, itr_max=itr))
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); p.solve_into(a, b, out["u"], out["v"], out["iters"], out["err"], out["flags"], out["cost"]); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    t = min(ts) / 1e3
    ups = cfg.n * itr * B / t
    print(json.dumps({"cfg": cfgname, "B": B, "itr": itr, "dom": dom, "info": p.info(), "ms": t * 1e3, "updates_per_s": ups,
                      "flags": int(out["flags"][0]), "cost0": float(out["cost"][0])}), flush=True)

if __name__ == "__main__":
    run("c2")
    run("c2", domain="log")
    run("c5", batch=8192)
    run("c1", itr=2000)
