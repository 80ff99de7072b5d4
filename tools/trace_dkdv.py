"""Debug: event trace of CTA 0 of the dK/dV kernel (SPION_TRACE=1); each event = SM clock << 8 | id.
Needs a build with the events compiled in: python tools/build_variant.py trev -DSPION_TRACE_EVENTS=1,
then SPION_LIB=build_variants/trev/libspion.so python tools/trace_dkdv.py.

roles: 0 producer, 1 S^T/dP^T MMA warp, 2/3 softmax thread 0 / 128, 4 dV/dK MMA warp.
Prints the median cycles between consecutive events of each role, and a raw window."""
import collections, ctypes, os, sys
os.environ["SPION_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion, _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "text"
L, B, bh = {"image": (1024, 32, 256), "text": (4096, 64, 128), "listops": (2048, 64, 256)}[cfg]
bh = int(os.environ.get("BH", bh))
d = 64
dev = torch.device("cuda:0")
A = synth.lra_scores(L, B, seed=1, device=dev)
q, k, v, do = synth.qkvdo(bh, L, d, seed=3, dtype=torch.bfloat16, device=dev)
bp = spion.pattern(A, B, filter=31, alpha=float(os.environ.get("ALPHA", "55")), sync=True)
o, lse = spion.attn_fwd(q, k, v, bp)
for _ in range(3):
    spion.attn_bwd(q, k, v, o, do, lse, bp)
torch.cuda.synchronize()
lib = N.lib()
lib.spion_debug_trace.restype = ctypes.c_int64
R = 5
buf = (ctypes.c_ulonglong * (8 * 2048))()
n = lib.spion_debug_trace(buf, 8 * 2048)
a = np.array(buf[:n], dtype=np.uint64).reshape(8, 2048)
names = {1: "P item", 2: "P KV issue", 3: "P Q issue", 5: "P sched slot free", 6: "P lists loaded", 7: "P kv_empty done", 10: "M item", 11: "M kv_full", 12: "S waits done",
         13: "dVdK p_full done", 14: "S syncwarp done", 15: "dVdK syncwarp done", 20: "sm item", 21: "sm s_full",
         22: "sm p arrive", 23: "sm acc_full", 24: "sm epi done", 30: "dVdK loop top", 31: "dVdK elect",
         32: "dVdK MMAs issued", 33: "dVdK commits done", 40: "S loop top", 41: "S commits done", 42: "S q_full done",
         43: "S MMAs issued"}
evs = []
for role in range(R):
    for w in a[role]:
        w = int(w)
        if w:
            evs.append((w >> 8, w & 255, role))
evs.sort()
c0 = evs[0][0]
for role in range(R):
    ev = [(c, e) for c, e, r in evs if r == role]
    dd = collections.defaultdict(list)
    for (x0, e0), (x1, e1) in zip(ev, ev[1:]):
        dd[(e0, e1)].append(x1 - x0)
    print("role", role, "events", len(ev), "span", (ev[-1][0] - ev[0][0]) if ev else 0, "median cycles between consecutive events:")
    for (e0, e1), vv in sorted(dd.items(), key=lambda kv: -len(kv[1]))[:10]:
        if len(vv) > 10:
            print("   %-20s -> %-20s n=%4d median %6d" % (names.get(e0, e0), names.get(e1, e1), len(vv), sorted(vv)[len(vv) // 2]))
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 300
WIN = int(os.environ.get("WIN", "80"))
for c, e, r in evs[lo:lo + WIN]:
    print(f"{c - c0:9d} r{r} {names.get(e, e)}")
# gaps in the dV/dK warp's issue stream (role 4, event 15 = a block's dV/dK MMAs issued)
iss = [c for c, e, r in evs if r == 4 and e == 15]
items = [c for c, e, r in evs if r == 1 and e == 10]
gaps = [(b - a, a - c0) for a, b in zip(iss, iss[1:])]
print("dVdK issues", len(iss), "median gap", sorted(g for g, _ in gaps)[len(gaps) // 2], "sum of gaps > 2000:",
      sum(g for g, _ in gaps if g > 2000), "of span", iss[-1] - iss[0])
print("largest gaps (cycles, at):", sorted(gaps, reverse=True)[:12])
print("item starts:", [c - c0 for c in items][:40])
print("first/last event of the CTA:", evs[0][0] - c0, evs[-1][0] - c0)
if len(sys.argv) > 3:  # dump every event: cycle role name
    with open(sys.argv[3], "w") as fo:
        for c, e, r in evs:
            fo.write(f"{c - c0} {r} {names.get(e, e)}\n")
