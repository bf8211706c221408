"""Per-phase timing of the K3w pass R at iteration 5 on C4 (globaltimer stamps per warp).
The stamps are compiled in only in probe builds: bash tools/variant.sh probe -DFS1_K3W_PROBE=1,
then run with FS1_LIB=gpurun_var/lib_probe.so."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1, _lib
cfg = gi.CONFIGS["c4"]
A, B = gi.batch(cfg, [0])
a = torch.from_numpy(A).cuda(); b = torch.from_numpy(B).cuda()
kern = int(sys.argv[1]) if len(sys.argv) > 1 else 0
kw = dict(h=cfg.h1, h2=cfg.h2, eps=cfg.eps, itr_max=10, domain="log", input_is_log=True, shape=(cfg.n, cfg.m), kernel=kern)
o = fs1.solve(a, b, **kw)
spec = fs1.Spec(ndim=2, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, batch=1, dtype=torch.float32,
                domain="log", input_is_log=True, itr_max=10, kernel=kern)
p = fs1.plan(spec, 0)
G = p.info()["grid"]
buf = torch.zeros(G * 8 * 16 + G, dtype=torch.int64, device="cuda")
lib = _lib.lib()
lib.fs1__set_sep_timers.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
lib.fs1__set_sep_timers(p._h, ctypes.c_void_p(buf.data_ptr()))
o = fs1.solve(a, b, **kw); torch.cuda.synchronize()
raw = buf.cpu().numpy().astype(np.float64)
t = raw[:G * 128].reshape(G, 8, 2, 8)
bar = raw[G * 128:]
t0 = t[:, :, 0, 0].min()
names = ["start", "X loaded", "apply1", "LT wait", "update", "apply2", "CTA sync", "T-write"]
for g in range(2):
    tg = t[:, :, g, :]
    ok = tg[:, :, 0] > 0
    if not ok.any():
        continue
    d = np.diff(tg, axis=2)[ok] / 1e3
    print(f"group round {g}: warps {ok.sum()}; start offset med {np.median(tg[:, :, 0][ok] - t0)/1e3:.2f} us")
    for k in range(7):
        print(f"   {names[k]:>9s} -> {names[k+1]:<9s} med {np.median(d[:, k]):7.2f}  max {np.max(d[:, k]):7.2f} us")
print(f"grid barrier exit (pass R end): med {np.median(bar - t0)/1e3:.2f}  max {np.max(bar - t0)/1e3:.2f} us after the first start")
end = t[:, :, 0, 7].max(axis=1)
st = t[:, :, 0, 0].min(axis=1)
for lo, hi, name in [(0, min(G, 148), "CTAs 0-147"), (148, G, "CTAs 148+")]:
    if hi > lo:
        print(f"{name}: start med {np.median(st[lo:hi]-t0)/1e3:.2f}  end med {np.median(end[lo:hi]-t0)/1e3:.2f} max {np.max(end[lo:hi]-t0)/1e3:.2f} us")
