"""Batch sharding across GPUs: host-side plumbing only.

Pairs are independent, so each rank solves a contiguous block of pair ids with
no communication during the iterations; the one collective of the path is an
all-gather of the per-pair results {cost, err, iters, flags} after the solve
(NCCL over NVLink on the GPU box; gloo in the CPU tests).  Per-pair inputs come
from per-pair seeds, so every pair's result is independent of the rank count.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(total: int, rank: int, world: int) -> range:
    """Contiguous block of pair ids of `rank` (sizes differ by at most one)."""
    lo = total * rank // world
    hi = total * (rank + 1) // world
    return range(lo, hi)


def pack_results(cost, err, iters, flags) -> torch.Tensor:
    """[B, 4] fp64 rows {cost, err, iters, flags} (iters/flags are exact in fp64)."""
    return torch.stack([cost.double(), err.double(), iters.double(), flags.double()], 1)


def gather_results(res: torch.Tensor, total: int, group=None) -> torch.Tensor:
    """All-gather the [B_rank, 4] result rows of every rank into [total, 4], ordered by
    global pair id.  Equal shard sizes use one all_gather_into_tensor; unequal ones
    are padded to the largest shard."""
    world = dist.get_world_size(group)
    sizes = [len(shard(total, r, world)) for r in range(world)]
    bmax = max(sizes)
    if res.shape[0] < bmax:
        res = torch.cat([res, res.new_zeros(bmax - res.shape[0], res.shape[1])])
    out = res.new_empty(world * bmax, res.shape[1])
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, res.contiguous(), group=group)
    else:
        dist.all_gather(list(out.chunk(world)), res.contiguous(), group=group)
    return torch.cat([out[r * bmax:r * bmax + sizes[r]] for r in range(world)])
