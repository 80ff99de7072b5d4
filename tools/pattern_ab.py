"""Time spion.pattern at the LRA shapes (CUDA events, 50 calls); SPION_LIB selects a library variant."""
import sys, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion
for L, B in [(1024, 32), (2048, 64), (4096, 64)]:
    A = synth.lra_scores(L, B, seed=1, device="cuda")
    bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
    for _ in range(5):
        spion.pattern(A, B, filter=31, alpha=75.0, out=bp)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50):
        spion.pattern(A, B, filter=31, alpha=75.0, out=bp)
    e1.record(); torch.cuda.synchronize()
    print(f"L={L} B={B} pattern us {e0.elapsed_time(e1) / 50 * 1000:.1f}")
