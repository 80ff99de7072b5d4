"""Debug: event trace of CTA 0 of the dK/dV kernel (SPION_TRACE=1)."""
import ctypes, os, sys
os.environ["SPION_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion, _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "image"
L, B, bh = {"image": (1024, 32, 256), "text": (4096, 64, 128)}[cfg]
d = 64
dev = torch.device("cuda:0")
A = synth.syn_scores(L, B, heads=2, seed=1, device=dev)
q, k, v, do = synth.qkvdo(bh, L, d, seed=3, dtype=torch.bfloat16, device=dev)
bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
o, lse = spion.attn_fwd(q, k, v, bp)
for _ in range(2):
    spion.attn_bwd(q, k, v, o, do, lse, bp)
torch.cuda.synchronize()
lib = N.lib()
lib.spion_debug_trace.restype = ctypes.c_int64
buf = (ctypes.c_ulonglong * (3 * 2048))()
n = lib.spion_debug_trace(buf, 3 * 2048)
a = np.array(buf[:n], dtype=np.uint64).reshape(3, 1024, 2)
names = {10: "P  q_empty ok", 20: "M  q_full ok", 21: "M  buf_free ok (S issue)", 22: "M  p_full ok (dVdK issue)", 30: "S  step start", 31: "S  s_full ok", 32: "S  p arrive"}
evs = []
for role in range(3):
    for e, t in a[role]:
        if t: evs.append((int(t), int(e)))
evs.sort()
t0 = evs[0][0]
for t, e in evs[:90]:
    print(f"{(t - t0) / 1000:9.3f} us  {names.get(e, e)}")
def times(code):
    return np.array([t for t, e in evs if e == code], dtype=np.int64)
a30, a31, a32 = times(30), times(31), times(32)
m = min(len(a30), len(a31), len(a32))
print("steps", m, "mean step us", np.diff(a32).mean() / 1000)
print("softmax: wait s_full", np.mean(a31[:m] - a30[:m]) / 1000, "compute", np.mean(a32[:m] - a31[:m]) / 1000)
a20, a21, a22 = times(20), times(21), times(22)
m2 = min(len(a20), len(a21), len(a22))
print("MMA: q_full->buf_free", np.mean(a21[:m2] - a20[:m2]) / 1000)
