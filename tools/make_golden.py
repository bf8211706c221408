"""Write the full-protocol oracle goldens of configs C3 and C4 (tests/golden/*_full.npz).

Calls ONLY ``oracle/`` (the fp64 Algorithm 1 / 2 loops with the paper's O(N)
recursion, pinned equal to the dense definition in tests/test_oracle_*.py) and
``fs1_inputs`` (the seeded generators).  Nothing here touches the CUDA path.

  C3: Algorithm 1, N = 2^24, eps = 1e-4, log domain,
      itr_max = 1000, tol = 0 (fixed iterations, R5).  ~2 h on 2 cores.
  C4: Algorithm 2, 2048 x 2048, eps = 1e-3, log domain,
      itr_max = 300, tol = 0.  ~10 min on 8 cores.

The full potentials are too large to commit (C3: 2 x 128 MiB), so each golden
keeps a deterministic subsample (a fixed stride plus both ends of the vector,
where the recursions start) together with the full-vector max |F|, max |G|
(the denominators of the norm-wise gate, R17), the exit error, the
cost, the iteration count and the flags, plus the sha256 of this script and of
every oracle source it ran.

Usage:  python tools/make_golden.py c3|c4 [--out tests/golden]
"""
from __future__ import annotations

import argparse
import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import fs1_inputs as gi  # noqa: E402
from oracle import sinkhorn  # noqa: E402

# subsample: every STRIDE-th point + the first and last EDGE points
SAMPLE = {"c3": (64, 4096), "c4": (67, 4096)}


def sample_index(size: int, stride: int, edge: int) -> np.ndarray:
    idx = np.concatenate([np.arange(0, size, stride), np.arange(min(edge, size)),
                          np.arange(max(size - edge, 0), size)])
    return np.unique(idx)


def _sha(path):
    with open(path, "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(SAMPLE))
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden"))
    ap.add_argument("--itr-max", type=int, default=None, help="override (smoke runs only)")
    args = ap.parse_args()
    cfg = gi.CONFIGS[args.config]
    itr = cfg.itr_max if args.itr_max is None else args.itr_max
    a, b = gi.pair(cfg, 0)
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    t0 = time.time()
    ref = sinkhorn.solve(a, b, n=cfg.n, m=cfg.m, h1=cfg.h1, h2=cfg.h2, eps=cfg.eps, itr_max=itr,
                         tol=cfg.tol, domain=cfg.domain, input_is_log=cfg.input_is_log,
                         apply="recur")
    secs = time.time() - t0
    F, G = ref["F"][0], ref["G"][0]
    stride, edge = SAMPLE[args.config]
    idx = sample_index(F.size, stride, edge)
    fin = np.isfinite(F)
    srcs = ["oracle/sinkhorn.py", "oracle/recur.py", "oracle/recur.c", "oracle/dense.py",
            "fs1_inputs/__init__.py", "tools/make_golden.py"]
    name = f"{args.config}_full.npz" if args.itr_max is None else f"{args.config}_it{itr}.npz"
    out = os.path.join(args.out, name)
    np.savez_compressed(
        out, idx=idx.astype(np.int64), F=F[idx], G=G[idx],
        F_absmax=np.max(np.abs(F[fin])), G_absmax=np.max(np.abs(G[np.isfinite(G)])),
        F_nfinite=int(fin.sum()), G_nfinite=int(np.isfinite(G).sum()),
        cost=ref["cost"][0], err=ref["err"][0], iters=int(ref["iters"][0]),
        flags=int(ref["flags"][0]), itr_max=itr, oracle_seconds=secs,
        config=args.config, pair=0,
        sources=np.array(srcs), sha256=np.array([_sha(os.path.join(ROOT, s)) for s in srcs]))
    print(f"{out}: {itr} iterations in {secs:.0f} s; cost {ref['cost'][0]!r} err {ref['err'][0]!r}")


if __name__ == "__main__":
    main()
