"""the sparse-MHA sub-layer of Alg. 5 around the SPION kernels.

    S = concat_h( SparseAttention(Q_h, K_h, V_h, P) ),  Q|K|V = X W^{QKV}      (Alg. 5 l.2-8)
    O = dropout(S W^O) + E                                                      (Alg. 5 l.9)

The head split / concatenation and the dropout + residual run in this library's kernels
(`spion_mha_heads`, `spion_dropout_residual`), the attention in the tcgen05 kernels; the two
projections are plain GEMMs (torch.matmul -> cuBLAS).  Alg. 5 l.1 (LayerNorm) belongs to the
encoder around it and is not part of this sub-layer.  bf16 throughout; autograd-complete.
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
        self.w_qkv = torch.nn.Parameter((torch.randn(D, 3 * D, generator=g) * s).to(device=device, dtype=dtype))
        self.w_o = torch.nn.Parameter((torch.randn(D, D, generator=g) * s).to(device=device, dtype=dtype))
        self.step = 0

    def forward(self, e: torch.Tensor, bp: spion.BlockPattern, seed: Optional[int] = None) -> torch.Tensor:
        batch, L, D = e.shape
        qkv = e @ self.w_qkv                                          # l.2 (cuBLAS)
        q, k, v = split_heads(qkv, self.H)                            # l.3
        s = spion.attention(q, k, v, bp, self.mode)                   # l.4-7 (tcgen05 kernels)
        y = merge_heads(s, batch, self.H) @ self.w_o                  # l.8-9 (cuBLAS)
        if seed is None:
            seed, self.step = self.step, self.step + 1
        p = self.p if self.training else 0.0
        return dropout_residual(y, e, p, seed)                        # l.9
