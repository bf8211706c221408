"""Per-phase timing of the K2 psi half-step on C3 (globaltimer stamps, CTA 0 and median)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1, _lib
cfg = gi.CONFIGS["c3"]
a, b = gi.pair(cfg, 0)
A = torch.from_numpy(a[None]).cuda(); B = torch.from_numpy(b[None]).cuda()
kern = int(sys.argv[1]) if len(sys.argv) > 1 else 0
kw = dict(h=cfg.h1, eps=cfg.eps, itr_max=60, domain="log", input_is_log=True, kernel=kern)
o = fs1.solve(A, B, **kw)
spec = fs1.Spec(ndim=1, n=cfg.n, m=1, h1=cfg.h1, h2=0.0, eps=cfg.eps, batch=1, dtype=torch.float64,
                domain="log", input_is_log=True, itr_max=60, kernel=kern)
p = fs1.plan(spec, 0)
G = p.info()["grid"]
buf = torch.zeros(G * 64 * 8, dtype=torch.int64, device="cuda")
lib = _lib.lib()
lib.fs1__set_stream_timers.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.fs1__set_stream_timers(p._h, ctypes.c_void_p(buf.data_ptr()))
o = fs1.solve(A, B, **kw); torch.cuda.synchronize()
t = buf.cpu().numpy().reshape(G, 64, 8).astype(np.float64)
t = t[:, 5:59]  # steady state
# stamps (thread 0): [0] loop top, [1] stream done (block synced), [3] tile scan + publish
# done, [4] grid barrier passed + warp 0's fold and tile carries done
stream = t[:, :, 1] - t[:, :, 0]
scan = t[:, :, 3] - t[:, :, 1]
wait_fold = t[:, :, 4] - t[:, :, 3]
step = t[:, 1:, 0] - t[:, :-1, 0]   # psi-start to next psi-start = full iteration
med = lambda x: np.median(x) / 1e3
print(f"CTAs {G}; psi half-step (us): stream med {med(stream):.2f} max {med(stream.max(0)):.2f} "
      f"min {med(stream.min(0)):.2f} | tile scan+publish {med(scan):.2f} | barrier+fold {med(wait_fold):.2f} "
      f"| iteration {med(step):.2f}")
print("  per-CTA stream (us): p10 %.2f p50 %.2f p90 %.2f" % tuple(np.percentile(stream, [10, 50, 90]) / 1e3))
scan_only = t[:, :, 5] - t[:, :, 1]
sync_or = t[:, :, 6] - t[:, :, 5]
pub = t[:, :, 3] - t[:, :, 6]
bar = t[:, :, 7] - t[:, :, 3]
fold = t[:, :, 4] - t[:, :, 7]
print(f"  tile scan {med(scan_only):.2f} | sync_or {med(sync_or):.2f} | publish {med(pub):.2f} | barrier wait "
      f"{med(bar):.2f} (slowest-arriving CTA: {np.median(bar.min(0))/1e3:.2f}) | fold+carries {med(fold):.2f}")
