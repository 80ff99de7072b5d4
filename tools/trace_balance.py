"""Debug: per-CTA start/end (globaltimer) of the last attention kernel launched with SPION_TRACE=1:
load balance of the persistent tile scheduler.  usage: python tools/trace_balance.py <config> <fwd|dq|dkdv>"""
import ctypes, os, sys
os.environ["SPION_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion, _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "text"
which = sys.argv[2] if len(sys.argv) > 2 else "dkdv"
L, B, bh = {"image": (1024, 32, 256), "text": (4096, 64, 128), "listops": (2048, 64, 256)}[cfg]
dev = torch.device("cuda:0")
A = synth.lra_scores(L, B, seed=1, device=dev)
q, k, v, do = synth.qkvdo(bh, L, 64, seed=3, dtype=torch.bfloat16, device=dev)
bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
o, lse = spion.attn_fwd(q, k, v, bp)
spion.attn_bwd(q, k, v, o, do, lse, bp)
torch.cuda.synchronize()
lib = N.lib()
lib.spion_debug_trace.restype = ctypes.c_int64
def grab():
    buf = (ctypes.c_ulonglong * (8 * 2048 + 4096))()
    n = lib.spion_debug_trace(buf, 8 * 2048 + 4096)
    a = np.array(buf[:n], dtype=np.uint64)[8 * 2048:].reshape(-1, 2).astype(np.int64)
    return a[a[:, 1] > 0]
if which == "fwd":
    spion.attn_fwd(q, k, v, bp)
    a = grab()
else:
    spion.attn_bwd(q, k, v, o, do, lse, bp)  # trace holds the last launch: dkdv
    a = grab()
t0 = a[:, 0].min()
s, e = (a[:, 0] - t0) / 1000, (a[:, 1] - t0) / 1000
print(f"{cfg} {which}: CTAs {len(a)}  kernel span {e.max():.1f} us  start max {s.max():.2f} us")
print(f"  CTA end: min {e.min():.1f} p10 {np.percentile(e, 10):.1f} median {np.median(e):.1f} p90 {np.percentile(e, 90):.1f} max {e.max():.1f}")
print(f"  mean busy fraction {np.mean(e - s) / e.max():.3f}")
