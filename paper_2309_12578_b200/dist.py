"""Multi-GPU plumbing of the hot path: one process per GPU.

The path partitions over (batch x head): every (batch, head) slice is an
independent problem, so ranks share no data-path tensors.  The one exchange is
the per-layer block pattern (P:653 — one pattern per layer, shared by all heads
and batch items), in one of two ways:
  * allreduce (default): Eq. 3-4 are sums over the source rows of the
    score matrix, so each rank pools its own contiguous slab of rows
    (`pattern_rows`, spion_pattern_pool), ONE all-reduce (int64 sum: exact and
    order-independent) adds the pool regions, and every rank finalises the
    identical pattern itself (spion_pattern_finalize): the stencil's work is
    split N ways and no rank is special;
  * broadcast: rank 0 generates the whole pattern and broadcasts the packed
    BlockPattern (block-CSR, block-CSC, mask and work plan in ONE int32 buffer).
One collective either way (NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous equal shard [start, stop) of `total` (batch x head) slices for `rank`."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    per, rem = divmod(total, world)
    start = rank * per + min(rank, rem)
    return start, start + per + (1 if rank < rem else 0)


def broadcast_pattern(flat: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """Broadcast a packed pattern buffer (BlockPattern.flat) from `src` in place."""
    if flat.dtype != torch.int32 or not flat.is_contiguous():
        raise ValueError("expected the contiguous int32 BlockPattern.flat buffer")
    dist.broadcast(flat, src=src, group=group)
    return flat


def pattern_rows(L: int, block: int, rank: int, world: int) -> tuple[int, int]:
    """Source rows [r0, r1) of the L x L score matrix that `rank` pools: a contiguous shard of the
    L / block block rows (block-aligned, so spion_pattern_pool accepts it)."""
    if L % block:
        raise ValueError("L % block != 0")
    b0, b1 = shard(L // block, rank, world)
    return b0 * block, b1 * block


def allreduce_pool(region: torch.Tensor, group=None) -> torch.Tensor:
    """Sum the ranks' pool regions (spion.pool_region: int64) in place."""
    if region.dtype != torch.int64 or not region.is_contiguous():
        raise ValueError("expected the contiguous int64 pool region of a pattern workspace")
    dist.all_reduce(region, op=dist.ReduceOp.SUM, group=group)
    return region
