"""B200-native FS-1 (arXiv 2202.10042) hot path: Sinkhorn iterations for the
Wasserstein-1 metric on uniform grids with O(N) kernel applies, as sm_100a CUDA
kernels behind the C ABI of include/fs1.h.

    from paper_2202_10042_b200 import fs1
    out = fs1.solve(a, b, h=1/N, eps=1e-3, itr_max=1000, domain="log")
"""
from . import _lib  # noqa: F401  (loads nothing until first use)
from .fs1 import Plan, Spec, apply, cost, plan, solve  # noqa: F401

__all__ = ["Plan", "Spec", "solve", "cost", "apply", "plan"]
