"""CPU-side checks of the C ABI: the library loads, exports every symbol
include/*.h declares, and rejects invalid descriptions before touching CUDA."""
import ctypes
import os
import re

import pytest

from paper_2202_10042_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            names |= set(re.findall(r"^\s*(?:fs1_status|void|const char\*|int|size_t)\s+(fs1_\w+)\s*\(", src, re.M))
    return sorted(names)


def test_library_exports_every_header_symbol():
    lib = L.lib()
    names = _header_functions()
    assert set(names) == set(L.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n
    assert lib.fs1_abi_version() == 2


def test_status_strings():
    lib = L.lib()
    for s in range(6):
        assert lib.fs1_status_string(s).decode().startswith("FS1_")


def _desc(**kw):
    d = dict(ndim=1, n=64, m=1, h1=1 / 64, h2=0.0, eps=0.01, batch=2, dtype=L.FS1_F32,
             domain=L.FS1_SCALING, input_is_log=0, itr_max=10, tol=0.0, check_interval=1,
             warm_start=0)
    d.update(kw)
    return L.Desc(**d)


@pytest.mark.parametrize("kw,status", [
    (dict(n=0), L.FS1_ERR_ARG),
    (dict(batch=0), L.FS1_ERR_ARG),
    (dict(ndim=3), L.FS1_ERR_ARG),
    (dict(m=5), L.FS1_ERR_ARG),            # 1D with m != 1
    (dict(itr_max=-1), L.FS1_ERR_ARG),
    (dict(tol=-1.0), L.FS1_ERR_ARG),
    (dict(check_interval=0), L.FS1_ERR_ARG),
    (dict(dtype=7), L.FS1_ERR_ARG),
    (dict(eps=0.0), L.FS1_ERR_EPS),
    (dict(eps=-1.0), L.FS1_ERR_EPS),
    (dict(h1=0.0), L.FS1_ERR_EPS),
    (dict(eps=float("inf")), L.FS1_ERR_EPS),
    (dict(ndim=2, m=4, h2=0.0), L.FS1_ERR_EPS),
    (dict(domain=3), L.FS1_ERR_ARG),
    (dict(domain=L.FS1_STABILIZED, dtype=L.FS1_F64, tau=0.5), L.FS1_ERR_ARG),      # tau must exceed 1
    (dict(domain=L.FS1_STABILIZED, dtype=L.FS1_F64, tau=float("inf")), L.FS1_ERR_ARG),
    (dict(domain=L.FS1_STABILIZED), L.FS1_ERR_UNSUPPORTED),                        # fp32
    (dict(domain=L.FS1_STABILIZED, dtype=L.FS1_F64, ndim=2, m=4, h2=0.25), L.FS1_ERR_UNSUPPORTED),
    (dict(domain=L.FS1_STABILIZED, dtype=L.FS1_F64, warm_start=1), L.FS1_ERR_UNSUPPORTED),
    (dict(domain=L.FS1_STABILIZED, dtype=L.FS1_F64, n=8193), L.FS1_ERR_UNSUPPORTED),  # > FS1_MAX_STAB
])
def test_plan_rejects_invalid(kw, status):
    lib = L.lib()
    d = _desc(**kw)
    h = ctypes.c_void_p()
    ws = ctypes.c_size_t()
    assert lib.fs1_plan(ctypes.byref(d), 0, ctypes.byref(h), ctypes.byref(ws)) == status
    assert not h.value


def test_null_arguments():
    lib = L.lib()
    assert lib.fs1_plan(None, 0, None, None) == L.FS1_ERR_ARG
    assert lib.fs1_solve(None, None, None, None, None, None, None, None, None, None, None) == L.FS1_ERR_ARG
    assert lib.fs1_cost(None, None, None, None, None, None) == L.FS1_ERR_ARG
    assert lib.fs1_apply(None, None, None, None, None) == L.FS1_ERR_ARG
    assert lib.fs1_plan_entries(None, None, None, None, 0, None, None) == L.FS1_ERR_ARG
    lib.fs1_plan_destroy(None)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2202_10042_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
                assert "oracle/" not in txt or f.endswith(".py") is False, f
