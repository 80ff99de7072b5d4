"""Profiling helper: run spion.pattern a few times at one shape (python tools/pattern_once.py L B [reps])."""
import sys
sys.path.insert(0, ".")
import torch
import synth
from paper_2309_12578_b200 import spion

L, B = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
A = synth.syn_scores(L, B, heads=2, seed=1, device="cuda")
bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
for _ in range(reps):
    spion.pattern(A, B, filter=31, alpha=75.0, out=bp)
torch.cuda.synchronize()
print("ok", bp.nnzb)
