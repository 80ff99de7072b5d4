"""Debug: event trace of CTA 0 of the dK/dV kernel (SPION_TRACE=1).

roles: 0 producer (1 item, 2 K/V issue, 3 Q stage issue), 1 MMA (10 item, 11 kv_full,
12 S issue, 13 dV/dK issue), 2/3 softmax warp 0 / warp 4 lane 0 (20 item, 21 s_full,
22 p arrive, 23 acc_full, 24 epilogue done)."""
import ctypes, os, sys
os.environ["SPION_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion, _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "text"
L, B, bh = {"image": (1024, 32, 256), "text": (4096, 64, 128), "listops": (2048, 64, 256)}[cfg]
d = 64
dev = torch.device("cuda:0")
A = synth.lra_scores(L, B, seed=1, device=dev)
q, k, v, do = synth.qkvdo(bh, L, d, seed=3, dtype=torch.bfloat16, device=dev)
bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
o, lse = spion.attn_fwd(q, k, v, bp)
for _ in range(3):
    spion.attn_bwd(q, k, v, o, do, lse, bp)
torch.cuda.synchronize()
lib = N.lib()
lib.spion_debug_trace.restype = ctypes.c_int64
R = 5
buf = (ctypes.c_ulonglong * (R * 2048))()
n = lib.spion_debug_trace(buf, R * 2048)
a = np.array(buf[:n], dtype=np.uint64).reshape(R, 1024, 2)
evs = []
names = {1: "P item", 2: "P KV issue", 3: "P Q issue", 10: "M item", 11: "M kv_full", 12: "M S issue", 13: "M dVdK issue", 14: "M S issued", 15: "M dVdK issued", 16: "m S0", 17: "m S4", 18: "m S8",
         20: "S item", 21: "S s_full", 22: "S p arrive", 23: "S acc_full", 24: "S epi done"}
clk = []
mm = []
for role in range(R):
    for e, t in a[role]:
        if t:
            evs.append((int(t), int(e) & 255, role))
            clk.append((int(t), int(e) >> 8))
            if role == 1 and (int(e) & 255) in (16, 17, 18): mm.append((int(e) & 255, int(e) >> 8))
clk.sort()
mm.sort(key=lambda x: x[1])
d1 = [b[1] - a[1] for a, b in zip(mm, mm[1:]) if a[0] == 16 and b[0] == 17]
d2 = [b[1] - a[1] for a, b in zip(mm, mm[1:]) if a[0] == 17 and b[0] == 18]
raw = sorted([(int(e) >> 8, int(e) & 255) for e, t in a[1] if t])
import os
if os.environ.get("RAW"):
    for c, e in raw[200:260]: print("   clk", c - raw[0][0], names.get(e, e))
if d1: print("issue cycles: first 4 SS MMAs median %d, next 4 median %d" % (sorted(d1)[len(d1) // 2], sorted(d2)[len(d2) // 2]))
print("SM clock during the trace: %.0f MHz" % ((clk[-1][1] - clk[0][1]) / (clk[-1][0] - clk[0][0]) * 1e3))
evs.sort()
t0 = evs[0][0]
names0 = {1: "P item", 2: "P KV issue", 3: "P Q issue", 10: "M item", 11: "M kv_full", 12: "M S issue", 13: "M dVdK issue", 14: "M S issued", 16: "m S0", 17: "m S4", 18: "m S8", 15: "M dVdK issued",
         20: "S item", 21: "S s_full", 22: "S p arrive", 23: "S acc_full", 24: "S epi done"}
lim = int(sys.argv[2]) if len(sys.argv) > 2 else 120
for t, e, r in evs[:lim]:
    print(f"{(t - t0) / 1000:9.3f} us  r{r} {names.get(e, e)}")
T = (evs[-1][0] - t0) / 1000
def times(code, role=None):
    return np.array([t for t, e, r in evs if e == code and (role is None or r == role)], dtype=np.int64)
print("span us", T, "items", len(times(10)), "entries", len(times(12)))
s21, s22 = times(21, 2), times(22, 2)
m = min(len(s21), len(s22))
print("softmax wg0: compute per entry us", np.mean(s22[:m] - s21[:m]) / 1000, " busy frac", np.sum(s22[:m] - s21[:m]) / 1000 / T)
e23, e24 = times(23, 2), times(24, 2)
m = min(len(e23), len(e24))
print("epilogue us", np.mean(e24[:m] - e23[:m]) / 1000, " total", np.sum(e24[:m] - e23[:m]) / 1000)
for a_, b_, nm in [(23, 25, "acc_full->staged"), (25, 26, "staged->barrier"), (26, 24, "barrier->done")]:
    for role in (2, 3):
        x, y = times(a_, role), times(b_, role)
        m = min(len(x), len(y))
        if m:
            print(f"  r{role} {nm}: {np.mean(y[:m] - x[:m]) / 1000:.3f} us")
# per item: acc_full wait duration (last p arrive -> acc_full)
x, y = times(22, 2), times(23, 2)
print("items", len(y))
