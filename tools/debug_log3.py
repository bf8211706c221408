import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import fs1_inputs as gi
from paper_2202_10042_b200 import fs1, _lib
np.set_printoptions(precision=4, linewidth=220, suppress=True)
n = 1024; itr = 3
A, B = gi.batch("c5", [0], n=n)
a = torch.from_numpy(A).float().cuda(); b = torch.from_numpy(B).float().cuda()
spec = fs1.Spec(ndim=1, n=n, m=1, h1=1/n, h2=0.0, eps=0.005, batch=1, dtype=torch.float32, domain="log", itr_max=itr)
p = fs1.Plan(spec)
buf = torch.zeros((2*itr+2, 32, 10), dtype=torch.float64, device="cuda")
_lib.lib().fs1__set_debug.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
_lib.lib().fs1__set_debug(p._h, ctypes.c_void_p(buf.data_ptr()))
u = torch.empty_like(a); v = torch.empty_like(b)
it = torch.empty(1, dtype=torch.int32, device="cuda"); er = torch.empty(1, dtype=torch.float64, device="cuda"); fl = torch.empty(1, dtype=torch.int32, device="cuda"); co = torch.empty(1, dtype=torch.float64, device="cuda")
p.solve_into(a, b, u, v, it, er, fl, co)
torch.cuda.synchronize()
d = buf.cpu().numpy()
print("flags", fl.item(), "iters", it.item())
for s in range(2*itr+1):
    print("slot", s, " cols: xe R kexp ye slow f cf cb y0 x0")
    print(d[s][:6]); print(d[s][-2:])
