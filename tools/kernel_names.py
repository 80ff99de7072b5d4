"""List the CUDA kernels one bench-like step launches (torch.profiler), to show which path ran."""
import math
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2309_12578_b200 import spion  # noqa: E402

L, B, bh, d = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (1024, 32, 256, 64)))
dev = torch.device("cuda:0")
A = synth.syn_scores(L, B, heads=2, seed=1, device=dev)
q, k, v, do = synth.qkvdo(bh, L, d, seed=3, dtype=torch.bfloat16, device=dev)
bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
o, lse = spion.attn_fwd(q, k, v, bp)
spion.attn_bwd(q, k, v, o, do, lse, bp)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    bp = spion.pattern(A, B, filter=31, alpha=75.0)
    o, lse = spion.attn_fwd(q, k, v, bp)
    spion.attn_bwd(q, k, v, o, do, lse, bp)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=20))
