"""the sparse-MHA sub-layer of Alg. 5 around the SPION kernels.

    S = concat_h( SparseAttention(Q_h, K_h, V_h, P) ),  Q|K|V = X W^{QKV}      (Alg. 5 l.2-8)
    O = dropout(S W^O) + E                                                      (Alg. 5 l.9)

The projections run on this library's tcgen05 GEMM (`spion_gemm_bf16`) with the head split /
concatenation folded into its addressing: Q|K|V = X W^{QKV}^T stores the attention inputs
[3][batch*H][L][64] straight from the GEMM epilogue (l.2-3), and S W^O^T reads the attention output
[batch*H][L][64] straight into the GEMM (l.8-9); their backward activation GEMMs (dS = dY W^O and
dX = dQKV W^{QKV}) use the same layouts.  The weight gradients are cuBLAS GEMMs over the
concatenated activations (one head-merge pass each).  The dropout + residual of l.9 is one kernel
(`spion_dropout_residual`), the attention the tcgen05 SPION kernels.  Weights in nn.Linear layout
(out x in).  Alg. 5 l.1 (LayerNorm) belongs to the encoder around it and is not part of this
sub-layer.  bf16 throughout; autograd-complete.
"""
from __future__ import annotations

import math
from typing import Optional

import torch

from . import _native as N
from . import spion


def _heads(packed: torch.Tensor, heads: torch.Tensor, batch: int, L: int, W: int, H: int, d: int, to_heads: bool):
    lib = N.lib()
    st = lib.spion_mha_heads(spion._p(packed), spion._p(heads), batch, L, W, H, d, 1 if to_heads else 0,
                             spion._stream(packed.device))
    N.check(st, "spion_mha_heads")


class _SplitHeads(torch.autograd.Function):
    """[batch][L][3][H][d] projection output -> (Q, K, V) [batch*H][L][d] (Alg. 5 l.3)."""

    @staticmethod
    def forward(ctx, qkv, H: int):
        batch, L, three_hd = qkv.shape
        d = three_hd // (3 * H)
        out = torch.empty((3, batch * H, L, d), dtype=qkv.dtype, device=qkv.device)
        _heads(qkv.contiguous(), out, batch, L, 3, H, d, True)
        ctx.shape = (batch, L, H, d)
        return out[0], out[1], out[2]

    @staticmethod
    def backward(ctx, dq, dk, dv):
        batch, L, H, d = ctx.shape
        g = torch.stack([x if x is not None else torch.zeros((batch * H, L, d), dtype=torch.bfloat16, device=dq.device)
                         for x in (dq, dk, dv)]).contiguous()
        out = torch.empty((batch, L, 3 * H * d), dtype=g.dtype, device=g.device)
        _heads(out, g, batch, L, 3, H, d, False)
        return out, None


class _MergeHeads(torch.autograd.Function):
    """[batch*H][L][d] -> [batch][L][H*d] (Alg. 5 l.8, concatenate)."""

    @staticmethod
    def forward(ctx, o, batch: int, H: int):
        bh, L, d = o.shape
        out = torch.empty((batch, L, H * d), dtype=o.dtype, device=o.device)
        _heads(out, o.contiguous(), batch, L, 1, H, d, False)
        ctx.shape = (batch, L, H, d)
        return out

    @staticmethod
    def backward(ctx, g):
        batch, L, H, d = ctx.shape
        out = torch.empty((batch * H, L, d), dtype=g.dtype, device=g.device)
        _heads(g.contiguous(), out, batch, L, 1, H, d, True)
        return out, None, None


class _DropoutResidual(torch.autograd.Function):
    """out = e + dropout(y, p) with a counter-based mask (seed), regenerated in the backward."""

    @staticmethod
    def forward(ctx, y, e, p: float, seed: int):
        if y.dtype != torch.bfloat16 or e.dtype != torch.bfloat16 or y.numel() != e.numel():
            raise ValueError("dropout_residual: y and e must be bf16 with the same number of elements")
        # bind the contiguous copies to locals: they must outlive the (asynchronous) kernel launch
        yc, ec = y.contiguous(), e.contiguous()
        out = torch.empty_like(ec)
        st = N.lib().spion_dropout_residual(spion._p(yc), spion._p(ec), spion._p(out), out.numel(),
                                            float(p), int(seed), spion._stream(y.device))
        N.check(st, "spion_dropout_residual")
        ctx.p, ctx.seed = p, seed
        return out

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        dy = torch.empty_like(g)
        st = N.lib().spion_dropout_residual(spion._p(g), None, spion._p(dy), g.numel(), float(ctx.p), int(ctx.seed),
                                            spion._stream(g.device))
        N.check(st, "spion_dropout_residual")
        return dy, g, None, None


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, m: int, n: int, k: int, a_heads: bool = False,
         c_heads: bool = False, L: int = 0, H: int = 0, batch: int = 0, alpha: float = 1.0) -> torch.Tensor:
    """out = alpha * A B^T on the tcgen05 GEMM (spion_gemm_bf16); A / out row-major or in the attention
    layout [W][batch*H][L][64] (a_heads / c_heads); b: [N][K] row-major."""
    spion._require_cuda(a, b, out)
    for t in (a, b, out):
        if t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise ValueError("gemm: contiguous bf16 tensors")
    lay = lambda heads: N.GEMM_HEADS if heads else N.GEMM_ROWMAJOR
    st = N.lib().spion_gemm_bf16(spion._p(a), spion._p(b), spion._p(out), m, n, k, lay(a_heads), lay(c_heads), L, H,
                                 batch, float(alpha), spion._stream(a.device))
    N.check(st, "spion_gemm_bf16")
    return out


def _stacked(dq, dk, dv):
    """(dQ, dK, dV) as one [3][bh][L][d] tensor: a zero-copy view when they are consecutive slices of
    one buffer (the attention backward allocates them that way), else a copy."""
    sz = dq.numel() * dq.element_size()
    if (dq.is_contiguous() and dk.is_contiguous() and dv.is_contiguous() and dq.shape == dk.shape == dv.shape
            and dk.data_ptr() == dq.data_ptr() + sz and dv.data_ptr() == dk.data_ptr() + sz):
        return dq.as_strided((3,) + tuple(dq.shape), (dq.numel(),) + tuple(dq.stride()))
    return torch.stack([dq, dk, dv]).contiguous()


class _QKVProjection(torch.autograd.Function):
    """Alg. 5 l.2-3: E [batch][L][D] -> Q, K, V [batch*H][L][d] = heads of E W_qkv^T (W_qkv [3D][D])."""

    @staticmethod
    def forward(ctx, e, w_qkv, H: int):
        batch, L, D = e.shape
        d = D // H
        ec = e.contiguous()
        qkv = torch.empty((3, batch * H, L, d), dtype=e.dtype, device=e.device)
        gemm(ec, w_qkv.contiguous(), qkv, batch * L, 3 * D, D, c_heads=True, L=L, H=H, batch=batch)
        ctx.save_for_backward(ec, w_qkv)
        ctx.dims = (batch, L, D, H)
        return qkv[0], qkv[1], qkv[2]

    @staticmethod
    def backward(ctx, dq, dk, dv):
        e, w_qkv = ctx.saved_tensors
        batch, L, D, H = ctx.dims
        d = D // H
        z = lambda x: x if x is not None else torch.zeros((batch * H, L, d), dtype=e.dtype, device=e.device)
        g = _stacked(z(dq), z(dk), z(dv))
        de = torch.empty((batch, L, D), dtype=e.dtype, device=e.device)
        gemm(g, w_qkv.t().contiguous(), de, batch * L, D, 3 * D, a_heads=True, L=L, H=H, batch=batch)
        packed = torch.empty((batch, L, 3 * D), dtype=e.dtype, device=e.device)
        _heads(packed, g, batch, L, 3, H, d, False)
        dw = packed.view(batch * L, 3 * D).t() @ e.view(batch * L, D)  # weight gradient (cuBLAS)
        return de, dw, None


class _OutProjection(torch.autograd.Function):
    """Alg. 5 l.8-9: heads S [batch*H][L][d] -> concat_h(S) W_o^T [batch][L][D] (W_o [D][D])."""

    @staticmethod
    def forward(ctx, s, w_o, batch: int, H: int):
        bh, L, d = s.shape
        D = H * d
        sc = s.contiguous()
        y = torch.empty((batch, L, D), dtype=s.dtype, device=s.device)
        gemm(sc, w_o.contiguous(), y, batch * L, D, D, a_heads=True, L=L, H=H, batch=batch)
        ctx.save_for_backward(sc, w_o)
        ctx.dims = (batch, L, D, H)
        return y

    @staticmethod
    def backward(ctx, dy):
        s, w_o = ctx.saved_tensors
        batch, L, D, H = ctx.dims
        d = D // H
        dyc = dy.contiguous()
        ds = torch.empty((batch * H, L, d), dtype=s.dtype, device=s.device)
        gemm(dyc, w_o.t().contiguous(), ds, batch * L, D, D, c_heads=True, L=L, H=H, batch=batch)
        packed = torch.empty((batch, L, D), dtype=s.dtype, device=s.device)
        _heads(packed, s, batch, L, 1, H, d, False)
        dw = dyc.view(batch * L, D).t() @ packed.view(batch * L, D)  # weight gradient (cuBLAS)
        return ds, dw, None, None


def qkv_projection(e: torch.Tensor, w_qkv: torch.Tensor, H: int):
    return _QKVProjection.apply(e, w_qkv, H)


def out_projection(s: torch.Tensor, w_o: torch.Tensor, batch: int, H: int):
    return _OutProjection.apply(s, w_o, batch, H)


def split_heads(qkv: torch.Tensor, H: int):
    return _SplitHeads.apply(qkv, H)


def merge_heads(o: torch.Tensor, batch: int, H: int):
    return _MergeHeads.apply(o, batch, H)


def dropout_residual(y: torch.Tensor, e: torch.Tensor, p: float, seed: int):
    return _DropoutResidual.apply(y, e, p, seed)


class SparseMHA(torch.nn.Module):
    """Alg. 5 on the SPION kernels: E [batch][L][D] bf16 -> dropout(S W^O) + E.

    The block pattern is a `spion.BlockPattern` (from `spion.pattern` at the transition, Alg. 2),
    shared by every head and batch item (reading Q16)."""

    def __init__(self, D: int, H: int, dropout: float = 0.1, mode: str = "paper", device=None,
                 dtype=torch.bfloat16, seed: int = 0):
        super().__init__()
        if D % H or (D // H) % 8:
            raise ValueError("D must split into H heads of a multiple of 8")
        self.D, self.H, self.d, self.p, self.mode = D, H, D // H, dropout, mode
        g = torch.Generator(device="cpu").manual_seed(seed)
        s = 1.0 / math.sqrt(D)
        # nn.Linear layout (out x in): Q|K|V = E W_qkv^T, Y = S W_o^T
        self.w_qkv = torch.nn.Parameter((torch.randn(3 * D, D, generator=g) * s).to(device=device, dtype=dtype))
        self.w_o = torch.nn.Parameter((torch.randn(D, D, generator=g) * s).to(device=device, dtype=dtype))
        self.step = 0

    def forward(self, e: torch.Tensor, bp: spion.BlockPattern, seed: Optional[int] = None) -> torch.Tensor:
        batch, L, D = e.shape
        q, k, v = qkv_projection(e, self.w_qkv, self.H)               # l.2-3 (tcgen05 GEMM -> heads)
        s = spion.attention(q, k, v, bp, self.mode)                   # l.4-7 (tcgen05 kernels)
        y = out_projection(s, self.w_o, batch, self.H)                # l.8-9 (heads -> tcgen05 GEMM)
        if seed is None:
            seed, self.step = self.step, self.step + 1
        p = self.p if self.training else 0.0
        return dropout_residual(y, e, p, seed)                        # l.9
