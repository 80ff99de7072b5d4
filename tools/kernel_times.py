"""Per-kernel mean device time (torch.profiler / CUPTI activity records) of this library's kernels
over one config's pattern + fwd + bwd, repeated on rotating inputs: A/B diagnostics only (never a
bench number).  usage: [SPION_LIB=...] python tools/kernel_times.py [config] [reps] [E: bh / E]"""
import collections, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2309_12578_b200 import spion
cfg = sys.argv[1] if len(sys.argv) > 1 else "text"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
L, B, H, batch, towers, alpha = {"image": (1024, 32, 4, 64, 1, 75.0), "listops": (2048, 64, 8, 32, 1, 75.0),
                                 "text": (4096, 64, 8, 16, 1, 55.0), "retrieval": (4096, 64, 8, 16, 2, 55.0)}[cfg]
bh, d = batch * towers * H, 64
if len(sys.argv) > 3:  # rank 0's share of an E-rank job: bh / E slices
    bh //= int(sys.argv[3])
dev = torch.device("cuda:0")
sets = []
for s in range(3):
    A = synth.lra_scores(L, B, seed=(1, 1001)[s % 2], device=dev)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=7 + s, dtype=torch.bfloat16, device=dev)
    sets.append((A, q, k, v, do, spion.empty_pattern(L, B, dev), spion.attn_workspace(bh, L, d, torch.bfloat16, dev)))
def step(i):
    A, q, k, v, do, bp, ws = sets[i % len(sets)]
    spion.pattern(A, B, filter=31, alpha=alpha, out=bp)
    o, lse = spion.attn_fwd(q, k, v, bp, "paper", 1 / math.sqrt(d), workspace=ws)
    spion.attn_bwd(q, k, v, o, do, lse, bp, "paper", 1 / math.sqrt(d), workspace=ws)
for i in range(6):
    step(i)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for i in range(reps):
        step(i)
    torch.cuda.synchronize()
acc = collections.defaultdict(list)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA and ("spion" in e.name or "kernel" in e.name):
        acc[e.name].append(e.device_time)
for name, ts in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    if "elementwise" in name or "vectorized" in name:
        continue
    print(f"{cfg:9s} {name[:60]:60s} n={len(ts):3d} mean_us={sum(ts) / len(ts):8.2f}")
