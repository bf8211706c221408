"""The paper's 1D random-distribution experiment (E1, Table 1) on the GPU.

u_i, v_j iid U[0,1] on N grid points of [-3, 3] (dx = 6/(N-1)), normalised;
eps = 1e-3; the paper's unstabilised FS-1 (fp64 scaling domain here); 1000
iterations.  Parity against the oracle on the same seeded
trials at the paper's three sizes, including the full 1000-iteration protocol at
N = 500, and the paper's column-5 quantity: the Frobenius distance between the
transport plan of dense Sinkhorn (the oracle) and of FS-1 (PAPER.md:371-373
prints 6.54e-15, 4.98e-18, 3.92e-18).
"""
import numpy as np
import pytest

import fs1_inputs as gi
from oracle import dense, sinkhorn
from tests.gpu_util import assert_solve_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2202_10042_b200 import fs1  # noqa: E402


@pytest.mark.parametrize("name,pairs,itr,apply", [("e1_500", 4, 1000, "dense"), ("e1_2000", 2, 100, "dense"),
                                                  ("e1_8000", 2, 20, "recur")])
def test_e1_parity(name, pairs, itr, apply):
    cfg = gi.CONFIGS[name]
    A, B = gi.batch(cfg, range(pairs))
    out = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), h=cfg.h1, eps=cfg.eps, itr_max=itr,
                    domain="scaling")
    ref = sinkhorn.solve(A, B, n=cfg.n, h1=cfg.h1, eps=cfg.eps, itr_max=itr, domain="scaling", apply=apply)
    assert_solve_parity(out, ref, "scaling", "f64")


def test_e1_plan_difference_table1_column5():
    """||P_FS1 - P_Sinkhorn||_F after the full protocol at N = 500, P = diag(phi) K diag(psi):
    at rounding level, as in the paper (6.54e-15 there, on its own trials)."""
    cfg = gi.CONFIGS["e1_500"]
    A, B = gi.batch(cfg, [0])
    out = fs1.solve(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), h=cfg.h1, eps=cfg.eps,
                    itr_max=cfg.itr_max, domain="scaling")
    ref = sinkhorn.solve(A, B, n=cfg.n, h1=cfg.h1, eps=cfg.eps, itr_max=cfg.itr_max, domain="scaling")
    K = dense.kernel(cfg.n, np.exp(-cfg.h1 / cfg.eps))
    P_gpu = fs1.transport_plan(out["u"], out["v"], h=cfg.h1, eps=cfg.eps, domain="scaling").cpu().numpy()[0]
    P_ref = np.exp(ref["F"][0])[:, None] * K * np.exp(ref["G"][0])[None, :]
    d = np.linalg.norm(P_gpu - P_ref)
    assert d <= 1e-12 * np.linalg.norm(P_ref), d
