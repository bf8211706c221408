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
carries = t[:, :, 1] - t[:, :, 0]
stream = t[:, :, 2] - t[:, :, 1]
scan = t[:, :, 3] - t[:, :, 2]
step = t[:, 1:, 0] - t[:, :-1, 0]   # psi-start to next psi-start = full iteration
waitb = t[:, :, 0] - 0
# barrier wait: from my publish to the next psi start is phi step + barrier; report slowest CTA stream
print(f"CTAs {G}; per psi half-step (us): carries {np.median(carries)/1e3:.2f}  stream med {np.median(stream)/1e3:.2f} "
      f"max {np.median(stream.max(0))/1e3:.2f} min {np.median(stream.min(0))/1e3:.2f}  scan+publish {np.median(scan)/1e3:.2f}  "
      f"iteration {np.median(step)/1e3:.2f}")
ext = t[:, :, 4] - t[:, :, 0]
sync1 = t[:, :, 5] - t[:, :, 4]
tiles = t[:, :, 1] - t[:, :, 5]
print(f"  carries split (us): ext fold {np.median(ext)/1e3:.2f}  first sync {np.median(sync1)/1e3:.2f}  per-tile {np.median(tiles)/1e3:.2f}")
