"""Work and traffic accounting for the bench and the roofline.

Paper formulas: operations for one head's attention matrix,
with D read as the per-head dimension d (reading Q22):
    dense  = 2 L^2 (2D+1) - L (D+1)
    sparse = 2 C (2D+1) - L (D+1),   C = number of stored scores
Graded metric: useful tensor-core FLOPs = 12 B^2 d per stored
block per (batch*head) for fwd+bwd (fwd QK^T and PV: 4 B^2 d; bwd dV, dP, dQ,
dK: 8 B^2 d); recomputation is not credited.
"""
from __future__ import annotations


def paper_dense_ops(L: int, D: int) -> int:
    return 2 * L * L * (2 * D + 1) - L * (D + 1)


def paper_sparse_ops(L: int, D: int, C: int) -> int:
    return 2 * C * (2 * D + 1) - L * (D + 1)


def useful_flops(B: int, d: int, nnzb: int, bh: int, fwd: bool = True, bwd: bool = True) -> int:
    per = (4 if fwd else 0) + (8 if bwd else 0)
    return per * B * B * d * nnzb * bh


def attn_bytes(L: int, d: int, bh: int, elt: int = 2) -> int:
    """Algorithmic HBM bytes for fwd+bwd (each tensor touched once):
    fwd reads Q,K,V and writes O (elt bytes) + lse (fp32);
    bwd reads Q,K,V,O,dO,lse and writes dQ,dK,dV.  = (12*elt*d + 8) L bh."""
    return (12 * elt * d + 8) * L * bh


def pattern_bytes(L: int, n: int) -> int:
    """Pattern stencil: the L x L fp32 score matrix read once, n x n int64 pool written."""
    return 4 * L * L + 8 * n * n
