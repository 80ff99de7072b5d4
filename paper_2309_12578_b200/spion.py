"""PyTorch-facing API of the SPION hot path (argument marshalling only).

Every step of the computation runs in libspion.so's CUDA kernels; this module
owns device memory (torch tensors), picks the current CUDA stream and passes
plain pointers through the C ABI (include/spion.h).  There is no CPU or
PyTorch fallback: a missing library or a non-CUDA tensor raises.

    bsr = pattern(scores, block=64, filter=31, alpha=99.0)     # Alg. 3/4
    o, lse = attn_fwd(q, k, v, bsr)                            # Alg. 5/6, Eq. 5
    dq, dk, dv = attn_bwd(q, k, v, o, do, lse, bsr)            # custom autograd
    o = attention(q, k, v, bsr)                                # autograd.Function
    attn_path(q, bsr) -> "tcgen05" | "cuda_core"               # which kernels run
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import torch

from . import _native as N


def _stream(dev: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _p(t: Optional[torch.Tensor]):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _require_cuda(*ts):
    for t in ts:
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("spion kernels need CUDA tensors (there is no CPU path)")


@dataclass
class BlockPattern:
    """Block-CSR + block-CSC of a layer's pattern, and the kernels' work plan (device tensors)."""
    L: int
    block: int
    nblk: int
    brow_ptr: torch.Tensor
    bcol_idx: torch.Tensor
    bcol_ptr: torch.Tensor
    brow_idx: torch.Tensor
    mask: torch.Tensor
    nnzb_dev: torch.Tensor
    plan: torch.Tensor
    workspace: Optional[torch.Tensor] = None
    flat: Optional[torch.Tensor] = None

    def c_struct(self) -> N.BSR:
        s = N.BSR()
        s.L, s.block, s.nblk = self.L, self.block, self.nblk
        s.nnzb_cap = self.bcol_idx.numel()
        s.brow_ptr, s.bcol_idx = self.brow_ptr.data_ptr(), self.bcol_idx.data_ptr()
        s.bcol_ptr, s.brow_idx = self.bcol_ptr.data_ptr(), self.brow_idx.data_ptr()
        s.mask, s.nnzb = self.mask.data_ptr(), self.nnzb_dev.data_ptr()
        s.plan, s.plan_bytes = self.plan.data_ptr(), self.plan.numel()
        return s

    @property
    def nnzb(self) -> int:
        return int(self.nnzb_dev[0].item())

    def csr(self):
        k = self.nnzb
        return self.brow_ptr, self.bcol_idx[:k]

    def csc(self):
        k = self.nnzb
        return self.bcol_ptr, self.brow_idx[:k]


def empty_pattern(L: int, block: int, device) -> BlockPattern:
    """Allocate a pattern as views into ONE int32 buffer (``.flat``), so a rank can
    broadcast a whole pattern with a single collective."""
    lib = N.lib()
    n = L // block
    plan_bytes = lib.spion_bsr_plan_bytes(L, block)
    sizes = [n + 1, n * n, n + 1, n * n, (n * n + 3) // 4, 4, (plan_bytes + 3) // 4]
    offs = [0]
    for sz in sizes:
        offs.append(offs[-1] + ((sz + 3) // 4) * 4)  # 16-byte aligned views
    flat = torch.zeros(offs[-1], dtype=torch.int32, device=device)
    v = [flat[offs[i]:offs[i] + sizes[i]] for i in range(len(sizes))]
    bp = BlockPattern(
        L=L, block=block, nblk=n, brow_ptr=v[0], bcol_idx=v[1], bcol_ptr=v[2], brow_idx=v[3],
        mask=v[4].view(torch.uint8)[: n * n], nnzb_dev=v[5], plan=v[6].view(torch.uint8)[:plan_bytes],
    )
    bp.flat = flat
    return bp


def pattern(scores: torch.Tensor, block: int, filter: int = 31, alpha: Optional[float] = None,
            t: Optional[float] = None, kind: str = "linear", out: Optional[BlockPattern] = None,
            sync: bool = False, variant: str = "") -> BlockPattern:
    """Alg. 3: scores [L][L] fp32 in [0,1] -> block pattern.

    Give ``alpha`` (percent, quantile threshold, ``kind`` linear|nearest) or ``t``
    (absolute threshold in pool-mean units).  ``variant``: "" (Alg. 3/4, SPION-CF) or a
    '+'-joined subset of noflood (SPION-C), prose (reading R2), all_seeds; SPION-F is filter=1."""
    _require_cuda(scores)
    if scores.dtype != torch.float32 or scores.dim() != 2 or scores.shape[0] != scores.shape[1]:
        raise ValueError("scores must be a square fp32 matrix")
    scores = scores.contiguous()
    L = scores.shape[0]
    lib = N.lib()
    if t is not None:
        kind, theta = "absolute", float(t)
    else:
        if alpha is None:
            raise ValueError("give alpha or t")
        theta = float(alpha)
    bp = out if out is not None else empty_pattern(L, block, scores.device)
    ws_bytes = lib.spion_pattern_workspace_bytes(L, block)
    if bp.workspace is None or bp.workspace.numel() < ws_bytes:
        bp.workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=scores.device)
    s = bp.c_struct()
    nnz = ctypes.c_int32(0)
    bits = sum(N.PATTERN_VARIANTS[v] for v in variant.split("+")) if variant else 0
    st = lib.spion_pattern_variant(_p(scores), L, block, filter, theta, N.THRESH[kind], bits, _p(bp.workspace),
                                   ws_bytes, ctypes.byref(s), ctypes.byref(nnz) if sync else None,
                                   _stream(scores.device))
    N.check(st, "spion_pattern")
    return bp


def _pattern_ws(bp: BlockPattern, device) -> int:
    ws_bytes = N.lib().spion_pattern_workspace_bytes(bp.L, bp.block)
    if bp.workspace is None or bp.workspace.numel() < ws_bytes:
        bp.workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=device)
    return ws_bytes


def pattern_pool(scores_rows: torch.Tensor, L: int, block: int, filter: int = 31, row_begin: int = 0,
                 out: Optional[BlockPattern] = None) -> BlockPattern:
    """Eq. 3-4 over source rows [row_begin, row_begin + rows) of an L x L score
    matrix, given as those rows only (``scores_rows``: [rows][L] fp32), into the pool region of
    ``out.workspace`` (zero-filled first).  Pools of a row partition add up to the whole matrix's
    pool: sum ``pool_region(bp)`` over the devices (one all-reduce), then ``pattern_finalize``."""
    _require_cuda(scores_rows)
    if scores_rows.dtype != torch.float32 or scores_rows.dim() != 2 or scores_rows.shape[1] != L:
        raise ValueError("scores_rows must be fp32 [rows][L]")
    scores_rows = scores_rows.contiguous()
    bp = out if out is not None else empty_pattern(L, block, scores_rows.device)
    ws_bytes = _pattern_ws(bp, scores_rows.device)
    rows = scores_rows.shape[0]
    st = N.lib().spion_pattern_pool(_p(scores_rows) if rows else None, L, block, filter, row_begin, row_begin + rows,
                                    _p(bp.workspace), ws_bytes, _stream(scores_rows.device))
    N.check(st, "spion_pattern_pool")
    return bp


def pool_region(bp: BlockPattern) -> torch.Tensor:
    """int64 view of the part of ``bp.workspace`` that devices sum (pool sums + bad-score count)."""
    off = ctypes.c_size_t(0)
    cnt = N.lib().spion_pattern_pool_region(bp.L, bp.block, ctypes.byref(off))
    return bp.workspace[off.value: off.value + 8 * cnt].view(torch.int64)


def pattern_finalize(bp: BlockPattern, alpha: Optional[float] = None, t: Optional[float] = None,
                     kind: str = "linear", variant: str = "", sync: bool = False) -> BlockPattern:
    """Threshold, flood fill, diagonal, CSR/CSC and plan (Alg. 3 l.4-end) from the pool in
    ``bp.workspace`` (after ``pattern_pool`` and, on several devices, the sum of ``pool_region``)."""
    if t is not None:
        kind, theta = "absolute", float(t)
    else:
        if alpha is None:
            raise ValueError("give alpha or t")
        theta = float(alpha)
    if bp.workspace is None:
        raise ValueError("pattern_finalize needs the workspace pattern_pool filled")
    s = bp.c_struct()
    nnz = ctypes.c_int32(0)
    bits = sum(N.PATTERN_VARIANTS[v] for v in variant.split("+")) if variant else 0
    st = N.lib().spion_pattern_finalize(bp.L, bp.block, theta, N.THRESH[kind], bits, _p(bp.workspace),
                                        bp.workspace.numel(), ctypes.byref(s), ctypes.byref(nnz) if sync else None,
                                        _stream(bp.workspace.device))
    N.check(st, "spion_pattern_finalize")
    return bp


def bsr_from_mask(mask: torch.Tensor, L: int, block: int, out: Optional[BlockPattern] = None) -> BlockPattern:
    """Block pattern from a caller-supplied [nblk][nblk] {0,1} uint8 mask (device)."""
    _require_cuda(mask)
    mask = mask.to(torch.uint8).contiguous()
    bp = out if out is not None else empty_pattern(L, block, mask.device)
    s = bp.c_struct()
    nnz = ctypes.c_int32(0)
    st = N.lib().spion_bsr_from_mask(_p(mask), L, block, ctypes.byref(s), ctypes.byref(nnz), _stream(mask.device))
    N.check(st, "spion_bsr_from_mask")
    return bp


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return N.BF16
    if t.dtype == torch.float32:
        return N.F32
    raise ValueError("Q/K/V must be bf16 or fp32")


def _layout(q: torch.Tensor):
    if q.dim() != 3 or q.stride(2) != 1:
        raise ValueError("expected [bh][L][d] with d contiguous")
    return q.shape[0], q.shape[1], q.shape[2], q.stride(0), q.stride(1)


def attn_fwd(q, k, v, bp: BlockPattern, mode: str = "paper", scale: Optional[float] = None,
             out: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
             workspace: Optional[torch.Tensor] = None):
    """O, lse of block-sparse attention (Eq. 5 / Alg. 6).  q,k,v: [bh][L][d], same strides.
    ``workspace``: >= spion_attn_fwd_workspace_bytes (the kernels' work-item counters); one per
    concurrently running call (allocated per call when omitted)."""
    _require_cuda(q, k, v)
    bh, L, d, sb, sl = _layout(q)
    if k.stride() != q.stride() or v.stride() != q.stride() or k.shape != q.shape or v.shape != q.shape:
        raise ValueError("q, k, v must share shape and strides")
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if out is None:
        out = torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=q.device)
    if lse is None:
        lse = torch.empty((bh, L), dtype=torch.float32, device=q.device)
    lib = N.lib()
    if workspace is None:
        nb = lib.spion_attn_fwd_workspace_bytes(bh, L, d, _dtype_code(q))
        workspace = torch.empty(max(nb, 16), dtype=torch.uint8, device=q.device)
    s = bp.c_struct()
    st = lib.spion_attn_fwd(_p(q), _p(k), _p(v), _p(out), _p(lse), bh, L, d, sb, sl, _dtype_code(q),
                            ctypes.byref(s), N.SOFTMAX[mode], float(scale), _p(workspace), workspace.numel(),
                            _stream(q.device))
    N.check(st, "spion_attn_fwd")
    return out, lse


def attn_path(q: torch.Tensor, bp: BlockPattern) -> str:
    """Which kernels attn_fwd / attn_bwd run for q's shape and layout and this pattern:
    "tcgen05" (tensor cores), "cuda_core", or raises if the call would be rejected."""
    bh, L, d, sb, sl = _layout(q)
    s = bp.c_struct()
    r = N.lib().spion_attn_path(bh, L, d, sb, sl, _dtype_code(q), ctypes.byref(s))
    if r < 0:
        N.check(-r, "spion_attn_path")
    return "tcgen05" if r == N.PATH_TCGEN05 else "cuda_core"


def tc_launch_count() -> int:
    """Tensor-core attention kernels launched by this process (host counter)."""
    return int(N.lib().spion_tc_launch_count())


def attn_workspace(bh: int, L: int, d: int, dtype, device) -> torch.Tensor:
    nb = N.lib().spion_attn_workspace_bytes(bh, L, d, N.BF16 if dtype == torch.bfloat16 else N.F32)
    return torch.empty(nb, dtype=torch.uint8, device=device)


def attn_bwd(q, k, v, o, do, lse, bp: BlockPattern, mode: str = "paper", scale: Optional[float] = None,
             workspace: Optional[torch.Tensor] = None, dq=None, dk=None, dv=None, deterministic: bool = False,
             fused: bool = False):
    """dQ, dK, dV of block-sparse attention (reading Q17).  Default: the two-pass tensor-core backward
    (bitwise reproducible; ``deterministic`` asks for it explicitly).  ``fused``: block 64 runs ONE
    pass over the column tiles (dQ summed by L2 reduce-adds in scheduling order)."""
    _require_cuda(q, k, v, o, do, lse)
    bh, L, d, sb, sl = _layout(q)
    for t in (k, v, o, do):
        if t.stride() != q.stride() or t.shape != q.shape:
            raise ValueError("q, k, v, o, do must share shape and strides")
    if scale is None:
        scale = 1.0 / math.sqrt(d)
    if workspace is None:
        workspace = attn_workspace(bh, L, d, q.dtype, q.device)
    mk = lambda: torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=q.device)
    dq = mk() if dq is None else dq
    dk = mk() if dk is None else dk
    dv = mk() if dv is None else dv
    s = bp.c_struct()
    flags = (N.BWD_DETERMINISTIC if deterministic else 0) | (N.BWD_FUSED if fused else 0)
    if flags:
        st = N.lib().spion_attn_bwd_ex(_p(q), _p(k), _p(v), _p(o), _p(do), _p(lse), _p(dq), _p(dk), _p(dv), bh, L, d,
                                       sb, sl, _dtype_code(q), ctypes.byref(s), N.SOFTMAX[mode], float(scale), flags,
                                       _p(workspace), workspace.numel(), _stream(q.device))
    else:
        st = N.lib().spion_attn_bwd(_p(q), _p(k), _p(v), _p(o), _p(do), _p(lse), _p(dq), _p(dk), _p(dv), bh, L, d, sb,
                                    sl, _dtype_code(q), ctypes.byref(s), N.SOFTMAX[mode], float(scale), _p(workspace),
                                    workspace.numel(), _stream(q.device))
    N.check(st, "spion_attn_bwd")
    return dq, dk, dv


class _SparseAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, bp, mode, scale):
        o, lse = attn_fwd(q, k, v, bp, mode, scale)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.bp, ctx.mode, ctx.scale = bp, mode, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        if do.stride() != q.stride():  # the kernels take one layout for every tensor: materialise q's
            do = torch.empty_strided(q.shape, q.stride(), dtype=q.dtype, device=q.device).copy_(do)
        if q.is_contiguous():  # dQ, dK, dV as slices of one buffer (a zero-copy [3][bh][L][d] for the QKV GEMM)
            g = torch.empty((3,) + tuple(q.shape), dtype=q.dtype, device=q.device)
            dq, dk, dv = attn_bwd(q, k, v, o, do, lse, ctx.bp, ctx.mode, ctx.scale, dq=g[0], dk=g[1], dv=g[2])
        else:
            dq, dk, dv = attn_bwd(q, k, v, o, do, lse, ctx.bp, ctx.mode, ctx.scale)
        return dq, dk, dv, None, None, None


def attention(q, k, v, bp: BlockPattern, mode: str = "paper", scale: Optional[float] = None):
    """Differentiable block-sparse attention (the paper's sparseMHA core, Alg. 5 l.4-8)."""
    return _SparseAttention.apply(q, k, v, bp, mode, scale)


def launch_count() -> int:
    return int(N.lib().spion_launch_count())


# ------------------------------------------------------------------ NEXT-1: dense-phase scores
def score_mean(q: torch.Tensor, k: torch.Tensor, scale: Optional[float] = None, out: Optional[torch.Tensor] = None,
               sumsq: Optional[torch.Tensor] = None):
    """A^s = mean over (batch, head) of softmax(scale q k^T) as fp32 [L][L], and sum(A^2)
    (Eq. 2's squared norm) as a python float.  q, k: [bh][L][64] bf16 (device).  With ``sumsq`` (a
    one-element device float64 tensor, e.g. a slot of transition()'s input) the sum is written
    there and returned as that tensor, without a host sync."""
    _require_cuda(q, k)
    bh, L, d = q.shape
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    lib = N.lib()
    nb = lib.spion_score_mean_workspace_bytes(bh, L, d)
    ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=q.device)
    A = out if out is not None else torch.empty((L, L), dtype=torch.float32, device=q.device)
    ss = sumsq if sumsq is not None else torch.zeros(1, dtype=torch.float64, device=q.device)
    if ss.dtype != torch.float64 or not ss.is_cuda:
        raise ValueError("sumsq must be a device float64 tensor")
    st = lib.spion_score_mean(_p(q), _p(k), bh, L, d, q.stride(0), q.stride(1), scale, _p(ws), nb, _p(A), _p(ss),
                              _stream(q.device))
    N.check(st, "spion_score_mean")
    return A, (ss if sumsq is not None else float(ss.item()))


def transition(sumsq: torch.Tensor, alpha: float, sync: bool = True):
    """Alg. 2 with Eq. 2 through spion_transition: ``sumsq`` is a device fp64
    tensor [3] of sum((A^s)^2) for dense-phase steps i-2, i-1, i (from score_mean).  Returns
    (switch, distances) — switch is a python bool when ``sync`` else a device int32 [1]; distances a
    device fp64 [2] = (distance_{i-1}, distance_i)."""
    _require_cuda(sumsq)
    if sumsq.dtype != torch.float64 or sumsq.numel() != 3:
        raise ValueError("sumsq must be a device float64 tensor of 3 sums of squares")
    sumsq = sumsq.contiguous()
    flag = torch.zeros(1, dtype=torch.int32, device=sumsq.device)
    dist = torch.empty(2, dtype=torch.float64, device=sumsq.device)
    host = ctypes.c_int32(0)
    st = N.lib().spion_transition(_p(sumsq), float(alpha), _p(flag), _p(dist), ctypes.byref(host) if sync else None,
                                  _stream(sumsq.device))
    N.check(st, "spion_transition")
    return (bool(host.value) if sync else flag), dist
