"""Multi-GPU plumbing of the hot path: one process per GPU.

The path partitions over (batch x head): every (batch, head) slice is an
independent problem, so ranks share no data-path tensors.  The one exchange is
the per-layer block pattern (P:653 — one pattern per layer, shared by all heads
and batch items): rank 0 generates it and broadcasts the whole BlockPattern
(block-CSR, block-CSC, mask and work plan packed in ONE int32 buffer) with a
single collective (NCCL over NVLink on the GPU box, gloo in the CPU tests).
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
