"""K2s (segments) vs K2 (single-GPU streaming) at growing N on the C3 recipe."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1, shard
cfg = gi.CONFIGS["c3"]
for lg in [int(x) for x in (sys.argv[1:] or ['16', '18', '20', '22'])]:
    n = 1 << lg
    a, b = gi.pair(cfg, 0, n=n)
    A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    eps = cfg.eps * (1 << 24) / n
    k2 = fs1.solve(A[None], B[None], h=1.0 / n, eps=eps, itr_max=5, domain="log", input_is_log=True)
    F2 = k2["u"].cpu().numpy()[0]
    for world in (1, 2, 8):
        o = shard.solve_segments(A, B, world, h=1.0 / n, eps=eps, itr_max=5, input_is_log=True)
        F = o["u"].cpu().numpy()
        d = np.max(np.abs(F - F2)) / max(1.0, np.max(np.abs(F2)))
        bad = np.nonzero(np.abs(F - F2) > 1e-9 * max(1.0, np.max(np.abs(F2))))[0]
        print(n, world, "tiles", n // 256, f"{d:.2e}", o["cost"], k2["cost"].item(),
              "bad tiles", np.unique(bad // 256)[:12], len(bad), flush=True)
