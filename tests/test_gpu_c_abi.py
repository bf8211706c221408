"""The library from plain C (examples/c_abi_demo.c): built with gcc against include/fs1.h and
libfs1.so only (no Python, no PyTorch in the process), its results equal the oracle's."""
import os
import subprocess

import numpy as np
import pytest

from oracle import sinkhorn

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_solves_through_the_abi(tmp_path):
    exe = str(tmp_path / "c_abi_demo")
    pkg = os.path.join(ROOT, "paper_2202_10042_b200")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "c_abi_demo.c"),
                    "-L", pkg, "-lfs1", "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{pkg}",
                    "-Wl,-rpath,/usr/local/cuda/lib64", "-lm", "-o", exe], check=True)
    n, batch, itr = 300, 3, 120
    out = subprocess.run([exe, str(n), str(batch), str(itr)], check=True, capture_output=True, text=True).stdout
    rows = [l.split() for l in out.splitlines() if l.startswith("pair")]
    assert len(rows) == batch
    x = (np.arange(n) + 0.5) / n
    for p, r in enumerate(rows):
        a = 1.0 + 0.5 * np.sin(2 * np.pi * (p + 1) * x)
        b = 1.0 + 0.5 * np.sin(2 * np.pi * (p + 1) * (1.0 - x))
        a, b = a / a.sum(), b / b.sum()
        ref = sinkhorn.solve(a[None], b[None], n=n, h1=1 / n, eps=1e-2, itr_max=itr, domain="log")
        cost, err, iters, flags = float(r[3]), float(r[5]), int(r[7]), int(r[9])
        assert iters == itr and flags == 4
        assert abs(cost - ref["cost"][0]) <= 1e-10 * abs(ref["cost"][0])
        assert abs(err - ref["err"][0]) <= 1e-10 * max(1.0, abs(ref["err"][0]))
