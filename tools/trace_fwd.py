"""Debug: event trace of CTA 0 of the forward kernel (SPION_TRACE=1); each event = SM clock << 8 | id.
Needs a build with the events compiled in: python tools/build_variant.py trev -DSPION_TRACE_EVENTS=1,
then SPION_LIB=build_variants/trev/libspion.so python tools/trace_fwd.py.

roles: 0 producer, 1 S-MMA warp, 2/3 softmax threads 0 / 64, 4 P.V MMA warp.
Prints the median cycles between consecutive events of each role, and a raw window."""
import collections, ctypes, os, sys
os.environ["SPION_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion, _native as N
cfg = sys.argv[1] if len(sys.argv) > 1 else "text"
L, B, bh, alpha = {"image": (1024, 32, 256, 75), "text": (4096, 64, 128, 55), "listops": (2048, 64, 256, 75)}[cfg]
d = 64
dev = torch.device("cuda:0")
A = synth.lra_scores(L, B, seed=1, device=dev)
q, k, v, do = synth.qkvdo(bh, L, d, seed=3, dtype=torch.bfloat16, device=dev)
bp = spion.pattern(A, B, filter=31, alpha=float(alpha), sync=True)
for _ in range(3):
    o, lse = spion.attn_fwd(q, k, v, bp)
torch.cuda.synchronize()
lib = N.lib()
lib.spion_debug_trace.restype = ctypes.c_int64
R = 5
buf = (ctypes.c_ulonglong * (8 * 2048))()
n = lib.spion_debug_trace(buf, 8 * 2048)
a = np.array(buf[:n], dtype=np.uint64).reshape(8, 2048)
names = {1: "P item", 3: "P kv_empty done", 10: "M item", 11: "M q_full", 44: "S kv_full", 42: "S freeb",
         43: "S MMAs issued", 41: "S commits done", 13: "PV p_full", 32: "PV MMAs issued", 33: "PV commits done",
         20: "sm item", 21: "sm s_full", 52: "sm max done", 53: "sm exp done", 22: "sm p arrive", 23: "sm epi waits",
         24: "sm epi done"}
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
        if len(vv) > 5:
            print("   %-20s -> %-20s n=%4d median %6d mean %6d" % (names.get(e0, e0), names.get(e1, e1), len(vv),
                                                                sorted(vv)[len(vv) // 2], sum(vv) / len(vv)))
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 300
for c, e, r in evs[lo:lo + 100]:
    print(f"{c - c0:9d} r{r} {names.get(e, e)}")
