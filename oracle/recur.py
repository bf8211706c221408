"""ctypes face of oracle/recur.c — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The shared object is compiled with plain gcc on first use (or by
``__graft_entry__.build()``); it is never linked into the product library.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "recur.c")
_SO = os.path.join(_HERE, "_recur.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99",
                               "-fno-fast-math", _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        d, l, p = ctypes.c_double, ctypes.c_long, ctypes.c_void_p
        _lib.fs1o_sweep_scaling.argtypes = [p, l, l, l, l, d, p]
        _lib.fs1o_sweep_log.argtypes = [p, l, l, l, l, d, p]
        _lib.fs1o_wsweep_log.argtypes = [p, l, l, l, l, d, d, p]
        _lib.fs1o_stab_sweep.argtypes = [p, p, p, l, d, p]
        _lib.fs1o_sum_exp2.argtypes = [p, p, l]
        _lib.fs1o_sum_exp2.restype = d
    return _lib


def _c(x):
    return np.ascontiguousarray(x, dtype=np.float64)


def _lines(x, axis):
    """(n, stride, lines, lstride) for a 1D vector or a column-major (N, M) array
    stored as a flat vector.  axis 1 = along i (contiguous), axis 2 = along j."""
    if x.ndim == 1:
        return x.shape[0], 1, 1, x.shape[0]
    n, m = x.shape
    if axis == 1:
        return n, 1, m, n
    return m, n, n, 1


def _run(fn, x, axis, *args):
    xf = _c(x.T.ravel() if x.ndim == 2 else x)   # column-major flat buffer
    y = np.empty_like(xf)
    n, st, ln, lst = _lines(x, axis)
    fn(xf.ctypes.data, n, st, ln, lst, *args, y.ctypes.data)
    return y.reshape(x.shape[::-1]).T if x.ndim == 2 else y


def sweep(x, lam, axis=1):
    """K x along one axis by Algorithm 1's forward/backward recursion."""
    return _run(lib().fs1o_sweep_scaling, np.asarray(x, np.float64), axis, float(lam))


def sweep_log(X, c, axis=1):
    """log(K e^X) along one axis by the LSE form of the recursion."""
    return _run(lib().fs1o_sweep_log, np.asarray(X, np.float64), axis, float(c))


def wsweep_log(X, c, h, axis=1):
    """log(W e^X) along one axis, W_kj = |k-j| h lam^{|k-j|}."""
    return _run(lib().fs1o_wsweep_log, np.asarray(X, np.float64), axis, float(c), float(h))


def sum_exp2(A, B) -> float:
    A, B = _c(A).ravel(), _c(B).ravel()
    return float(lib().fs1o_sum_exp2(A.ctypes.data, B.ctypes.data, A.size))


def stab_sweep(x, own, other, lam):
    """Remark 3.2's recursions: diag(e^own) K diag(e^other) x with only
    neighbour-difference exponentials; own/other are the absorbed potentials divided by eps."""
    x, own, other = _c(x), _c(own), _c(other)
    y = np.empty_like(x)
    lib().fs1o_stab_sweep(x.ctypes.data, own.ctypes.data, other.ctypes.data, x.size, float(lam),
                          y.ctypes.data)
    return y
