"""ctypes declarations of libspion.so (include/spion.h).  Marshalling only."""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# SPION_LIB: an alternative build of the same library (A/B experiments, tools/build_variant.py)
SO_PATH = os.environ.get("SPION_LIB") or os.path.join(PKG, "lib", "libspion.so")

OK = 0
STATUS = {0: "ok", 1: "shape", 2: "param", 3: "data", 4: "align", 5: "workspace", 6: "cuda", 7: "unsupported"}
F32, BF16 = 0, 1
PATH_CUDA_CORE, PATH_TCGEN05 = 0, 1  # spion_attn_path
BWD_DETERMINISTIC, BWD_FUSED = 1, 2  # spion_attn_bwd_ex flags
GEMM_ROWMAJOR, GEMM_HEADS = 0, 1  # spion_gemm_bf16 layouts
SOFTMAX = {"paper": 0, "masked": 1}
THRESH = {"linear": 0, "nearest": 1, "absolute": 2}
# spion_pattern_flags (include/spion.h): SPION-C, prose recursion, all-cells seeding
PATTERN_VARIANTS = {"noflood": 1, "prose": 2, "all_seeds": 4}


class SpionError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        super().__init__(f"{what}: {STATUS.get(status, status)} ({status})")


class BSR(ctypes.Structure):
    _fields_ = [
        ("L", ctypes.c_int32), ("block", ctypes.c_int32), ("nblk", ctypes.c_int32), ("nnzb_cap", ctypes.c_int32),
        ("brow_ptr", ctypes.c_void_p), ("bcol_idx", ctypes.c_void_p), ("bcol_ptr", ctypes.c_void_p),
        ("brow_idx", ctypes.c_void_p), ("mask", ctypes.c_void_p), ("nnzb", ctypes.c_void_p),
        ("plan", ctypes.c_void_p), ("plan_bytes", ctypes.c_size_t),
    ]


EXPORTS = {
    "spion_bsr_plan_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "spion_pattern_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32]),
    "spion_pattern": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(BSR),
                                     ctypes.c_void_p, ctypes.c_void_p]),
    "spion_pattern_variant": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                             ctypes.c_double, ctypes.c_int, ctypes.c_uint32, ctypes.c_void_p,
                                             ctypes.c_size_t, ctypes.POINTER(BSR), ctypes.c_void_p, ctypes.c_void_p]),
    "spion_pattern_check": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "spion_mha_heads": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]),
    "spion_gemm_bf16": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_int32, ctypes.c_float, ctypes.c_void_p]),
    "spion_dropout_residual": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_float, ctypes.c_uint64, ctypes.c_void_p]),
    "spion_score_mean_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]),
    "spion_score_mean": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_int64, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "spion_bsr_from_mask": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(BSR),
                                           ctypes.c_void_p, ctypes.c_void_p]),
    "spion_attn_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int]),
    "spion_attn_fwd_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                                         ctypes.c_int]),
    "spion_attn_path": (ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                         ctypes.c_int64, ctypes.c_int, ctypes.POINTER(BSR)]),
    "spion_attn_fwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int, ctypes.POINTER(BSR), ctypes.c_int, ctypes.c_float,
                                      ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "spion_attn_bwd": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int, ctypes.POINTER(BSR), ctypes.c_int, ctypes.c_float,
                                      ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]),
    "spion_attn_bwd_ex": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(BSR),
                                         ctypes.c_int, ctypes.c_float, ctypes.c_uint32, ctypes.c_void_p,
                                         ctypes.c_size_t, ctypes.c_void_p]),
    "spion_step_arena_bytes": (ctypes.c_size_t, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                 ctypes.c_int]),
    "spion_step_host": (ctypes.c_int, [ctypes.c_void_p] * 10 + [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                                                ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                                                ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                                ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t,
                                                                ctypes.c_void_p, ctypes.c_void_p]),
    "spion_pattern_pool_region": (ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_size_t)]),
    "spion_pattern_pool": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t,
                                          ctypes.c_void_p]),
    "spion_pattern_finalize": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_int,
                                              ctypes.c_uint32, ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(BSR),
                                              ctypes.c_void_p, ctypes.c_void_p]),
    "spion_launch_count": (ctypes.c_int64, []),
    "spion_tc_launch_count": (ctypes.c_int64, []),
    "spion_transition": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]),
    "spion_status_str": (ctypes.c_char_p, [ctypes.c_int]),
}

_lib = None


def lib():
    """Load libspion.so (fails loudly if the extension has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"libspion.so not found at {SO_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(SO_PATH)
        for name, (res, args) in EXPORTS.items():
            if os.environ.get("SPION_LIB") and not hasattr(L, name):
                continue  # an older A/B build may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int, what: str):
    if status != OK:
        raise SpionError(status, what)
