"""ctypes declarations of include/fs1.h (argument marshalling only).

The library is loaded from this package directory.  There is no fallback: if
libfs1.so is missing or cannot be loaded, importing raises immediately.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FS1_LIB") or os.path.join(HERE, "libfs1.so")  # FS1_LIB: variant builds (tools)

FS1_OK, FS1_ERR_ARG, FS1_ERR_EPS, FS1_ERR_UNSUPPORTED, FS1_ERR_CUDA, FS1_ERR_WORKSPACE = range(6)
FS1_F32, FS1_F64 = 0, 1
FS1_SCALING, FS1_LOG, FS1_STABILIZED = 0, 1, 2
FLAG_CONVERGED, FLAG_NONFINITE, FLAG_ITR_MAX = 1, 2, 4

EXPORTS = ["fs1_plan", "fs1_solve", "fs1_cost", "fs1_apply", "fs1_transport_plan", "fs1_plan_entries", "fs1_dual",
           "fs1_eps_scaling_plan", "fs1_solve_eps_scaling", "fs1_plan_info",
           "fs1_plan_destroy", "fs1_status_string", "fs1_abi_version",
           # include/fs1_shard.h
           "fs1_shard_plan", "fs1_shard_init", "fs1_shard_half", "fs1_shard_cost_totals",
           "fs1_shard_finish", "fs1_shard_destroy", "fs1_shard_mailbox_bytes", "fs1_shard_mailbox_alloc",
           "fs1_shard_mailbox_open", "fs1_shard_mailbox_close", "fs1_shard_mailbox_free",
           "fs1_shard_set_mailboxes", "fs1_shard_decide", "fs1_shard_sum"]


class Desc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("m", ctypes.c_int64),
        ("h1", ctypes.c_double),
        ("h2", ctypes.c_double),
        ("eps", ctypes.c_double),
        ("batch", ctypes.c_int64),
        ("dtype", ctypes.c_int32),
        ("domain", ctypes.c_int32),
        ("input_is_log", ctypes.c_int32),
        ("itr_max", ctypes.c_int32),
        ("tol", ctypes.c_double),
        ("check_interval", ctypes.c_int32),
        ("warm_start", ctypes.c_int32),
        ("tau", ctypes.c_double),
        ("l", ctypes.c_int64),
        ("h3", ctypes.c_double),
    ]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("kernel", ctypes.c_char * 48),
        ("chunk", ctypes.c_int32),
        ("threads", ctypes.c_int32),
        ("ctas_per_problem", ctypes.c_int32),
        ("grid", ctypes.c_int64),
        ("smem_bytes", ctypes.c_size_t),
        ("workspace_bytes", ctypes.c_size_t),
    ]


class FS1Error(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{what}: {lib().fs1_status_string(status).decode()} ({status})")


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`python -m paper_2202_10042_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, st = ctypes.c_void_p, ctypes.c_int
        L.fs1_plan.argtypes = [ctypes.POINTER(Desc), ctypes.c_int, ctypes.POINTER(vp),
                               ctypes.POINTER(ctypes.c_size_t)]
        L.fs1_plan.restype = st
        L.fs1_solve.argtypes = [vp] * 11
        L.fs1_solve.restype = st
        L.fs1_cost.argtypes = [vp] * 6
        L.fs1_cost.restype = st
        L.fs1_apply.argtypes = [vp] * 5
        L.fs1_apply.restype = st
        L.fs1_transport_plan.argtypes = [vp] * 5
        L.fs1_transport_plan.restype = st
        L.fs1_plan_entries.argtypes = [vp, vp, vp, vp, ctypes.c_longlong, vp, vp]
        L.fs1_plan_entries.restype = st
        L.fs1_dual.argtypes = [vp] * 9
        L.fs1_dual.restype = st
        dd = ctypes.c_double
        L.fs1_eps_scaling_plan.argtypes = [ctypes.POINTER(Desc), st, dd, dd, ctypes.POINTER(ctypes.c_int32),
                                           ctypes.POINTER(ctypes.c_size_t)]
        L.fs1_eps_scaling_plan.restype = st
        L.fs1_solve_eps_scaling.argtypes = [ctypes.POINTER(Desc), st, dd, dd, ctypes.c_int32] + [vp] * 9 + \
            [ctypes.c_size_t, vp]
        L.fs1_solve_eps_scaling.restype = st
        L.fs1_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
        L.fs1_plan_info.restype = st
        L.fs1_plan_destroy.argtypes = [vp]
        L.fs1_plan_destroy.restype = None
        L.fs1_status_string.argtypes = [st]
        L.fs1_status_string.restype = ctypes.c_char_p
        L.fs1_abi_version.restype = ctypes.c_int
        # test-only: plan with a forced kernel family (1 persistent, 2 streaming)
        L.fs1__plan_kind.argtypes = [ctypes.POINTER(Desc), ctypes.c_int, ctypes.c_int, ctypes.POINTER(vp),
                                     ctypes.POINTER(ctypes.c_size_t)]
        L.fs1__plan_kind.restype = st
        # include/fs1_shard.h
        i64p = ctypes.POINTER(ctypes.c_int64)
        L.fs1_shard_plan.argtypes = [ctypes.POINTER(Desc), st, st, st, ctypes.POINTER(vp),
                                     ctypes.POINTER(ctypes.c_size_t), i64p, i64p]
        L.fs1_shard_plan.restype = st
        L.fs1_shard_init.argtypes = [vp] * 6
        L.fs1_shard_init.restype = st
        L.fs1_shard_half.argtypes = [vp, st, st, st, st, st, st, st, vp, vp, vp, vp, vp]
        L.fs1_shard_half.restype = st
        L.fs1_shard_cost_totals.argtypes = [vp, st, vp, vp, vp]
        L.fs1_shard_cost_totals.restype = st
        L.fs1_shard_finish.argtypes = [vp, st, vp, vp, vp, vp, vp, vp]
        L.fs1_shard_finish.restype = st
        L.fs1_shard_destroy.argtypes = [vp]
        L.fs1_shard_destroy.restype = None
        L.fs1_shard_mailbox_bytes.argtypes = [st]
        L.fs1_shard_mailbox_bytes.restype = ctypes.c_size_t
        L.fs1_shard_mailbox_alloc.argtypes = [st, st, ctypes.POINTER(vp), vp]
        L.fs1_shard_mailbox_alloc.restype = st
        L.fs1_shard_mailbox_open.argtypes = [vp, st, ctypes.POINTER(vp)]
        L.fs1_shard_mailbox_open.restype = st
        L.fs1_shard_mailbox_close.argtypes = [vp]
        L.fs1_shard_mailbox_close.restype = st
        L.fs1_shard_mailbox_free.argtypes = [vp]
        L.fs1_shard_mailbox_free.restype = st
        L.fs1_shard_set_mailboxes.argtypes = [vp, vp]
        L.fs1_shard_set_mailboxes.restype = st
        L.fs1_shard_decide.argtypes = [vp, vp, st, vp, vp]
        L.fs1_shard_decide.restype = st
        L.fs1_shard_sum.argtypes = [vp, vp, st, st, vp, vp]
        L.fs1_shard_sum.restype = st
        _lib = L
    return _lib
