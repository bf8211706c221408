"""One N-point problem over the ranks of a torch.distributed job (NCCL): each rank solves
its segment with shard.solve_sharded; rank 0 compares with the single-GPU kernel.

  python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 \\
      tools/shard_dist_demo.py [log2 N] [iterations] [fused 0/1]

fused = 1: the totals move through the ranks' IPC-mapped mailboxes (fused exchange).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import torch.distributed as dist

import fs1_inputs as gi
from paper_2202_10042_b200 import fs1, shard

lg = int(sys.argv[1]) if len(sys.argv) > 1 else 20
itr = int(sys.argv[2]) if len(sys.argv) > 2 else 20
fused = bool(int(sys.argv[3])) if len(sys.argv) > 3 else False
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
rank, world = dist.get_rank(), dist.get_world_size()
cfg = gi.CONFIGS["c3"]
n = 1 << lg
eps = cfg.eps * (1 << 24) / n
a, b = gi.pair(cfg, 0, n=n)
lo, ln = shard.segment(n, world, rank)
A = torch.from_numpy(a[lo:lo + ln].copy()).cuda()
B = torch.from_numpy(b[lo:lo + ln].copy()).cuda()
o = shard.solve_sharded(A, B, n, h=1.0 / n, eps=eps, itr_max=itr, input_is_log=True, fused=fused)
F = torch.empty(n, dtype=torch.float64, device="cuda")
parts = [torch.empty(shard.segment(n, world, r)[1], dtype=torch.float64, device="cuda") for r in range(world)]
dist.all_gather(parts, o["u"])
if rank == 0:
    Fs = torch.cat(parts).cpu().numpy()
    k2 = fs1.solve(torch.from_numpy(a[None]).cuda(), torch.from_numpy(b[None]).cuda(), h=1.0 / n, eps=eps,
                   itr_max=itr, domain="log", input_is_log=True)
    Fk = k2["u"].cpu().numpy()[0]
    d = np.max(np.abs(Fs - Fk)) / max(1.0, np.max(np.abs(Fk)))
    print(f"world {world} fused {int(fused)} N 2^{lg}: F rel {d:.2e}, cost {o['cost']:.15g} vs {k2['cost'].item():.15g}, "
          f"iters {o['iters']} flags {o['flags']}", flush=True)
dist.barrier()
dist.destroy_process_group()
