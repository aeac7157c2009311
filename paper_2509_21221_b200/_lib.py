"""ctypes declarations of the C-ABI in include/gwtf.h (libgwtf.so, built in-tree).

There is no fallback: if the native library is missing or cannot load, importing the
binding raises.  The product path never touches oracle/.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgwtf.so")

GWTF_ABI_VERSION = 1
GWTF_HOST_PTRS = 1 << 0
GWTF_WARM_REPAIR_ALL = 1 << 1  # warm_reroute repairs every instance (no triage)
GWTF_FORCE_GLOBAL_TIER = 1 << 30  # testing: exact solve through the global-memory tier
GWTF_FORCE_CLUSTER_TIER = 1 << 29  # testing: exact solve through the cluster tier
OBJ_SUM, OBJ_MINIMAX = 0, 1
STATUS = {0: "OK", 1: "E_INVALID", 2: "E_NOMEM", 3: "E_CUDA", 4: "E_OVERFLOW", 5: "E_STATE", 6: "E_UNSUPPORTED"}

P = ctypes.c_void_p
I32, I64, U32, U64, DBL = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double


class ProblemDesc(ctypes.Structure):
    _fields_ = [
        ("abi_version", U32), ("num_instances", I32), ("num_stages", I32), ("clients_per_stage", I32),
        ("max_cap", I32), ("cap", P), ("alive", P), ("src_cost", P), ("snk_cost", P), ("link_cost", P),
        ("supply", P), ("seed", U64), ("inst_base", I64), ("T0", DBL), ("alpha", DBL), ("objective", I32),
        ("steady_window", I32), ("deny_after", I32), ("device", I32), ("stream", P), ("flags", U32),
    ]


class GwtfError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__(f"{fn} -> {STATUS.get(status, status)}: {msg}")
        self.status = status


EXPORTS = {
    "gwtf_eq1_cost_tiles": ([I32, I32, I32, I32, P, P, P, P, P, I64, P, P, P, P], I32),
    "gwtf_addition_build": ([I32, I32, P, P, P, P, P, P, P, P, I64, I64, P, P, P, P, P], I32),
    "gwtf_addition_select": ([I64, P, P, P, P], I32),
    "gwtf_flow_create": ([ctypes.POINTER(ProblemDesc), ctypes.POINTER(P)], I32),
    "gwtf_flow_solve_batch": ([P, P, P, P, P], I32),
    "gwtf_flow_decentralized_rounds": ([P, I32, P, P, P, P, P], I32),
    "gwtf_flow_solve_and_rounds": ([P, I32, P, P, P, P, P, P, P, P], I32),
    "gwtf_flow_apply_churn": ([P, P, P, I64], I32),
    "gwtf_flow_get_assignment": ([P, P, P, P, P], I32),
    "gwtf_flow_residual_caps": ([P, P], I32),
    "gwtf_flow_export_round_state": ([P, P, P, P, P, P, P, P, P], I32),
    "gwtf_flow_import_round_state": ([P, P, P, P, P, P, P, P, P], I32),
    "gwtf_mc_rounds": ([I32, I32, I32, I32, I32, P, P, P, P, P, P, U64, I64, DBL, DBL, I32, I32, I32, I32,
                        P, P, P, P, P, P, P, P, P, P, I32, I64, P], I32),
    "gwtf_flow_snapshot": ([P], I32),
    "gwtf_flow_restore": ([P], I32),
    "gwtf_flow_set_profiling": ([P, I32], I32),
    "gwtf_flow_kernel_times": ([P, ctypes.POINTER(ctypes.c_char_p), P, P, I32, P], I32),
    "gwtf_flow_stats": ([P, P, I32], I32),
    "gwtf_flow_greedy_baseline": ([P, P, P], I32),
    "gwtf_flow_warm_reroute": ([P, P, P, P, P, P, P, P, P], I32),
    "gwtf_flow_destroy": ([P], I32),
    "gwtf_last_error": ([], ctypes.c_char_p),
    "gwtf_abi_version": ([], I32),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"native library {LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in EXPORTS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        if L.gwtf_abi_version() != GWTF_ABI_VERSION:
            raise RuntimeError("libgwtf.so ABI version mismatch")
        _lib = L
    return _lib


def check(fn_name, status):
    if status != 0:
        raise GwtfError(fn_name, status, lib().gwtf_last_error().decode(errors="replace"))
