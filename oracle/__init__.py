"""CPU oracle for SPION's block-sparse attention hot path (arXiv 2309.12578).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
the ``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import
this package.  The product package ``paper_2309_12578_b200`` never imports
it, and the two share no code.

This module is argument marshalling (numpy <-> ctypes) around
``spion_oracle.c``; every step of the arithmetic is in that file, each
function citing the passage of the paper it follows.  Parity status of each
function is listed in the header of ``spion_oracle.c`` and in DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spion_oracle.c")
_SO = os.path.join(_HERE, "libspion_oracle.so")

TH_QUANTILE_LINEAR = 0
TH_QUANTILE_NEAREST = 1
TH_ABSOLUTE = 2
SOFTMAX_PAPER = 0
SOFTMAX_MASKED = 1

_MODES = {"paper": SOFTMAX_PAPER, "masked": SOFTMAX_MASKED}
_KINDS = {"linear": TH_QUANTILE_LINEAR, "nearest": TH_QUANTILE_NEAREST, "absolute": TH_ABSOLUTE}


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc -O2 (no fast-math, no vector intrinsics)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math", "-o", _SO, _SRC, "-lm"]
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i32, i64, f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        sigs = {
            "spion_oracle_quantize": (ctypes.c_int, [P, i64, P]),
            "spion_oracle_diag_conv": (ctypes.c_int, [P, i32, i32, P]),
            "spion_oracle_pool_sum": (ctypes.c_int, [P, i32, i32, P]),
            "spion_oracle_threshold_gt": (ctypes.c_int, [P, i64, i32, f64, i32, P, P]),
            "spion_oracle_flood_fill": (ctypes.c_int, [P, i32, P, P]),
            "spion_oracle_mask_to_bsr": (i64, [P, i32, P, P, P, P]),
            "spion_oracle_pattern": (ctypes.c_int, [P, i32, i32, i32, f64, i32, P, P, P]),
            "spion_oracle_flood_fill_variant": (ctypes.c_int, [P, i32, P, i32, P]),
            "spion_oracle_score_mean": (ctypes.c_int, [P, P, i64, i32, i32, f64, P, P]),
            "spion_oracle_transition": (ctypes.c_int, [f64, f64, f64, f64, P, P]),
            "spion_oracle_pattern_variant": (ctypes.c_int, [P, i32, i32, i32, f64, i32, i32, P, P, P]),
            "spion_oracle_attn_fwd": (ctypes.c_int, [P, P, P, i32, i32, i32, P, f64, i32, P, P, P]),
            "spion_oracle_attn_bwd": (ctypes.c_int, [P, P, P, P, i32, i32, i32, P, f64, i32, P, P, P]),
        }
        for name, (res, args) in sigs.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class OracleError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(f"{what}: oracle status {rc}")


# ---------------------------------------------------------------- pattern
def quantize(A: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float32)
    q = np.empty(A.shape, dtype=np.int64)
    _check(lib().spion_oracle_quantize(_ptr(A), A.size, _ptr(q)), "quantize")
    return q


def diag_conv(q: np.ndarray, F: int) -> np.ndarray:
    q = np.ascontiguousarray(q, dtype=np.int64)
    L = q.shape[0]
    out = np.empty_like(q)
    _check(lib().spion_oracle_diag_conv(_ptr(q), L, F, _ptr(out)), "diag_conv")
    return out


def pool_sum(conv: np.ndarray, B: int) -> np.ndarray:
    conv = np.ascontiguousarray(conv, dtype=np.int64)
    L = conv.shape[0]
    if B <= 0 or L % B:
        raise OracleError("pool_sum: L % B != 0")
    n = L // B
    out = np.empty((n, n), dtype=np.int64)
    _check(lib().spion_oracle_pool_sum(_ptr(conv), L, B, _ptr(out)), "pool_sum")
    return out


def threshold_gt(pool: np.ndarray, B: int, theta: float, kind: str = "linear"):
    pool = np.ascontiguousarray(pool, dtype=np.int64)
    gt = np.empty(pool.shape, dtype=np.uint8)
    t = ctypes.c_double(0.0)
    _check(
        lib().spion_oracle_threshold_gt(_ptr(pool), pool.size, B, float(theta), _KINDS[kind], _ptr(gt),
                                        ctypes.byref(t)),
        "threshold_gt",
    )
    return gt, t.value


# pattern variants: SPION-C, prose recursion (R2), all-cells seeding
VARIANTS = {"noflood": 1, "prose": 2, "all_seeds": 4}


def variant_bits(variant) -> int:
    """'noflood' / 'prose' / 'all_seeds' (or a '+'-joined combination, or an int) -> flag bits."""
    if isinstance(variant, int):
        return variant
    return sum(VARIANTS[v] for v in variant.split("+")) if variant else 0


def flood_fill(pool: np.ndarray, gt: np.ndarray, variant=0) -> np.ndarray:
    pool = np.ascontiguousarray(pool, dtype=np.int64)
    gt = np.ascontiguousarray(gt, dtype=np.uint8)
    n = pool.shape[0]
    fl = np.empty((n, n), dtype=np.uint8)
    _check(lib().spion_oracle_flood_fill_variant(_ptr(pool), n, _ptr(gt), variant_bits(variant), _ptr(fl)),
           "flood_fill")
    return fl


def mask_to_bsr(fl: np.ndarray):
    fl = np.ascontiguousarray(fl, dtype=np.uint8)
    n = fl.shape[0]
    cap = max(1, int(fl.astype(bool).sum()))
    brow_ptr = np.empty(n + 1, np.int32)
    bcol_idx = np.empty(cap, np.int32)
    bcol_ptr = np.empty(n + 1, np.int32)
    brow_idx = np.empty(cap, np.int32)
    nnz = lib().spion_oracle_mask_to_bsr(_ptr(fl), n, _ptr(brow_ptr), _ptr(bcol_idx), _ptr(bcol_ptr),
                                         _ptr(brow_idx))
    return {
        "brow_ptr": brow_ptr,
        "bcol_idx": bcol_idx[:nnz].copy(),
        "bcol_ptr": bcol_ptr,
        "brow_idx": brow_idx[:nnz].copy(),
        "nnzb": int(nnz),
    }


def pattern(A: np.ndarray, B: int, F: int = 31, theta: float = 96.0, kind: str = "linear", variant=0):
    """Alg. 3 end to end (variant: see VARIANTS). Returns (fl_out uint8 [n][n], pool int64 [n][n], t)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    L = A.shape[0]
    if A.shape != (L, L) or B <= 0 or L % B:
        raise OracleError("pattern: bad shape")
    n = L // B
    pool = np.empty((n, n), np.int64)
    fl = np.empty((n, n), np.uint8)
    t = ctypes.c_double(0.0)
    _check(
        lib().spion_oracle_pattern_variant(_ptr(A), L, B, F, float(theta), _KINDS[kind], variant_bits(variant),
                                           _ptr(pool), _ptr(fl), ctypes.byref(t)),
        "pattern",
    )
    return fl, pool, t.value


# -------------------------------------------------------------- attention
def attn_fwd(Q, K, V, fl, B: int, scale: float, mode: str = "paper", want_P: bool = False):
    """One (batch, head): Q,K,V [L][d] -> O [L][d] fp64, lse [L] fp64 (, P [L][L])."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    fl = np.ascontiguousarray(fl, dtype=np.uint8)
    L, d = Q.shape
    O = np.empty((L, d), np.float64)
    lse = np.empty(L, np.float64)
    P = np.empty((L, L), np.float64) if want_P else None
    _check(
        lib().spion_oracle_attn_fwd(_ptr(Q), _ptr(K), _ptr(V), L, d, B, _ptr(fl), float(scale), _MODES[mode],
                                    _ptr(O), _ptr(lse), _ptr(P) if want_P else None),
        "attn_fwd",
    )
    return (O, lse, P) if want_P else (O, lse)


def attn_bwd(Q, K, V, dO, fl, B: int, scale: float, mode: str = "paper"):
    """One (batch, head): -> dQ, dK, dV [L][d] fp64."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    V = np.ascontiguousarray(V, dtype=np.float64)
    dO = np.ascontiguousarray(dO, dtype=np.float64)
    fl = np.ascontiguousarray(fl, dtype=np.uint8)
    L, d = Q.shape
    dQ = np.empty((L, d), np.float64)
    dK = np.empty((L, d), np.float64)
    dV = np.empty((L, d), np.float64)
    _check(
        lib().spion_oracle_attn_bwd(_ptr(Q), _ptr(K), _ptr(V), _ptr(dO), L, d, B, _ptr(fl), float(scale),
                                    _MODES[mode], _ptr(dQ), _ptr(dK), _ptr(dV)),
        "attn_bwd",
    )
    return dQ, dK, dV


# -------------------------------------------------------------- NEXT-1: dense-phase scores
def score_mean(Q, K, scale: float):
    """A^s = mean over (batch, head) of softmax(scale Q K^T), fp64; Q, K [bh][L][d].
    Returns (A [L][L], sum of A^2)."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    K = np.ascontiguousarray(K, dtype=np.float64)
    bh, L, d = Q.shape
    A = np.empty((L, L), np.float64)
    ss = ctypes.c_double(0.0)
    _check(lib().spion_oracle_score_mean(_ptr(Q), _ptr(K), bh, L, d, float(scale), _ptr(A), ctypes.byref(ss)),
           "score_mean")
    return A, ss.value


def transition(sumsq_im2: float, sumsq_im1: float, sumsq_i: float, alpha: float):
    """Alg. 2 / Eq. 2 transition test from three consecutive sums of squares -> (bool, d_{i-1}, d_i)."""
    d1, d2 = ctypes.c_double(0.0), ctypes.c_double(0.0)
    r = lib().spion_oracle_transition(float(sumsq_im2), float(sumsq_im1), float(sumsq_i), float(alpha),
                                      ctypes.byref(d1), ctypes.byref(d2))
    return bool(r), d1.value, d2.value

