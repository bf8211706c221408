"""Shared helpers for the GPU parity tests (compare the CUDA path with the oracle)."""
import math

import numpy as np

TOL = {"f64": 1e-10, "f32": 1e-4}   # BASELINE.json north_star tolerances (relative)


def rel_norm(Fg, Fo):
    """max |F_gpu - F_orc| / max(max|F_orc|, 1) over bins where the oracle is finite
    (R17: norm-wise relative error of the log-scalings)."""
    Fg = np.asarray(Fg, np.float64)
    Fo = np.asarray(Fo, np.float64)
    m = np.isfinite(Fo)
    assert np.array_equal(np.isfinite(Fg), m), "finite pattern differs"
    if not m.any():
        return 0.0
    return float(np.max(np.abs(Fg[m] - Fo[m])) / max(np.max(np.abs(Fo[m])), 1.0))


def rel(a, b):
    a, b = float(a), float(b)
    if b == 0.0:
        return abs(a)
    return abs(a - b) / abs(b)


def gpu_F(out, domain):
    """log-scalings F, G from fs1.solve outputs (scaling: log of phi, psi)."""
    u = out["u"].double().cpu().numpy()
    v = out["v"].double().cpu().numpy()
    if domain == "scaling":
        with np.errstate(divide="ignore"):
            return np.log(u), np.log(v)
    return u, v


def assert_solve_parity(out, ref, domain, dtype, tol=None, check_err=True, pairs=None):
    t = TOL[dtype] if tol is None else tol
    F, G = gpu_F(out, domain)
    it = out["iters"].cpu().numpy()
    fl = out["flags"].cpu().numpy()
    cost = out["cost"].cpu().numpy()
    err = out["err"].cpu().numpy()
    idx = range(F.shape[0]) if pairs is None else pairs
    for j, p in enumerate(idx):
        assert it[p] == ref["iters"][j], (p, it[p], ref["iters"][j])
        assert fl[p] == ref["flags"][j], (p, fl[p], ref["flags"][j])
        eF = rel_norm(F[p], ref["F"][j])
        eG = rel_norm(G[p], ref["G"][j])
        ec = rel(cost[p], ref["cost"][j])
        assert eF <= t and eG <= t and ec <= t, (p, eF, eG, ec)
        if check_err and math.isfinite(ref["err"][j]):
            assert abs(err[p] - ref["err"][j]) <= t * max(1.0, abs(ref["err"][j])), (p, err[p], ref["err"][j])
