"""SPION (arXiv 2309.12578) block-sparse attention hot path for B200 (sm_100a).

Pattern generation (Alg. 3/4) and block-sparse attention forward/backward
(Alg. 5/6, Eq. 5) in hand-written CUDA behind the C ABI of include/spion.h.
"""
from .spion import (BlockPattern, attention, attn_bwd, attn_fwd, attn_path, attn_workspace, bsr_from_mask,
                    empty_pattern, launch_count, pattern, tc_launch_count)

__all__ = ["BlockPattern", "attention", "attn_bwd", "attn_fwd", "attn_path", "attn_workspace", "bsr_from_mask",
           "empty_pattern", "launch_count", "pattern", "tc_launch_count"]
