"""Time the NEXT-1 dense-phase score capture (spion.score_mean) at the LRA shapes; CUDA events,
3 warm-up + 10 timed calls.  Work: the dense lse forward (QK^T and PV on every block) plus one
QK^T pass and L^2*bh exponentials for A^s."""
import sys, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion
for name, L, bh in [("image", 1024, 256), ("listops", 2048, 256), ("text", 4096, 128)]:
    q, k, _, _ = synth.qkvdo(bh, L, 64, seed=1, dtype=torch.bfloat16, device="cuda")
    A = torch.empty((L, L), dtype=torch.float32, device="cuda")
    for _ in range(3):
        spion.score_mean(q, k, out=A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10):
        spion.score_mean(q, k, out=A)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    fl = 2 * L * L * 64 * bh * 3  # fwd QK^T + PV, then QK^T again
    print(f"{name}: L={L} bh={bh}  {ms:.3f} ms  {fl / ms / 1e9:.0f} TF/s (MMA)  {L * L * bh / ms / 1e6:.0f} G exp/s")
