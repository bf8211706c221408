"""Multi-process (world size 2, gloo, CPU) test of the batch-sharding path: each rank
solves its contiguous block of pairs, results are all-gathered in pair order, and every
pair's result equals the single-process result bitwise (per-pair seeds).
The per-rank compute here is the oracle (no GPU in this container); on the GPU box the
same sharding and gather run around fs1_solve with NCCL (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fs1_inputs as gi
from oracle import sinkhorn
from paper_2202_10042_b200 import dist as fdist

TOTAL, N, ITR = 7, 64, 15


def _solve_pairs(pairs):
    cfg = gi.CONFIGS["c5"]
    A, B = gi.batch(cfg, pairs, n=N)
    r = sinkhorn.solve(A.astype(np.float64), B.astype(np.float64), n=N, h1=1 / N, eps=cfg.eps * 40,
                       itr_max=ITR, domain="log")
    return fdist.pack_results(torch.from_numpy(r["cost"]), torch.from_numpy(r["err"]),
                              torch.from_numpy(r["iters"]), torch.from_numpy(r["flags"]))


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = fdist.shard(TOTAL, rank, world)
    res = _solve_pairs(list(mine))
    full = fdist.gather_results(res, TOTAL)
    if rank == 0:
        q.put(full.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_blocks_cover_pairs_once():
    for total in (1, 7, 8, 65536):
        for world in (1, 2, 3, 8):
            ids = [i for r in range(world) for i in fdist.shard(total, r, world)]
            assert ids == list(range(total))


@pytest.mark.timeout(300)
def test_two_rank_gather_equals_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=240)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    ref = _solve_pairs(list(range(TOTAL))).numpy()
    assert full.shape == (TOTAL, 4)
    assert np.array_equal(full, ref)
