import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import fs1_inputs as gi
from paper_2202_10042_b200 import shard
cfg = gi.CONFIGS["c3"]
a, b = gi.pair(cfg, 0)
A, B = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
shard.solve_segments(A, B, int(sys.argv[1]), h=cfg.h1, eps=cfg.eps, itr_max=4, input_is_log=True, graph=False)
torch.cuda.synchronize()
