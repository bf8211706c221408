"""Achieved parity of the full-protocol runs against the committed goldens (C3, C4):
norm-wise potential errors, cost and err differences (tests/test_gpu_golden.py gates them)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fs1_inputs as gi  # noqa: E402
from paper_2202_10042_b200 import fs1  # noqa: E402

for name in ("c3", "c4"):
    g = np.load(os.path.join(ROOT, "tests", "golden", f"{name}_full.npz"))
    cfg = gi.CONFIGS[name]
    a, b = gi.batch(cfg, [0])
    kw = dict(h=cfg.h1, eps=cfg.eps, itr_max=cfg.itr_max, tol=cfg.tol, domain=cfg.domain,
              input_is_log=cfg.input_is_log)
    if cfg.ndim == 2:
        kw.update(shape=(cfg.n, cfg.m), h2=cfg.h2)
    out = fs1.solve(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), **kw)
    F = out["u"][0].double().cpu().numpy()
    G = out["v"][0].double().cpu().numpy()
    idx = g["idx"]
    eF = np.max(np.abs(F[idx] - g["F"])) / max(float(g["F_absmax"]), 1.0)
    eG = np.max(np.abs(G[idx] - g["G"])) / max(float(g["G_absmax"]), 1.0)
    ec = abs(out["cost"].item() - float(g["cost"])) / abs(float(g["cost"]))
    ee = abs(out["err"].item() - float(g["err"]))
    print(f"{name}: {cfg.itr_max} iterations, {idx.size} sampled points; norm-wise F {eF:.3e} G {eG:.3e}; "
          f"cost rel {ec:.3e} (gpu {out['cost'].item()!r} oracle {float(g['cost'])!r}); err abs {ee:.3e}; "
          f"kernel {fs1.plan(fs1.Spec(ndim=cfg.ndim, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, batch=1, dtype=torch.float64 if cfg.dtype == 'f64' else torch.float32, domain=cfg.domain, input_is_log=cfg.input_is_log, itr_max=cfg.itr_max)).info()['kernel']}")
