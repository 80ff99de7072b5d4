"""Debug: K2 phase timestamps (SPION_TRACE=1) and K1/K2 durations for each LRA shape."""
import ctypes, os, sys
os.environ["SPION_TRACE"] = "1"
import numpy as np, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion, _native as N
lib = N.lib()
lib.spion_debug_k2_trace.restype = ctypes.c_int64
for L, B in [(1024, 32), (2048, 64), (4096, 64)]:
    A = synth.syn_scores(L, B, heads=2, seed=1, device="cuda")
    bp = spion.pattern(A, B, filter=31, alpha=75.0, sync=True)
    for _ in range(3):
        spion.pattern(A, B, filter=31, alpha=75.0, out=bp, sync=True)
    buf = (ctypes.c_ulonglong * 16)()
    lib.spion_debug_k2_trace(buf)
    t = np.array(buf[:12], dtype=np.int64)
    d = np.diff(t[:7]) / 1000
    print(L, B, "K2 phases us: load %.2f thresh %.2f edges %.2f flood %.2f fl %.2f bsr+plan %.2f total %.2f" % (*d, (t[6] - t[0]) / 1000))
    seq = [t[5], t[7], t[8], t[9], t[10], t[11], t[6]]
    print("   thresh: or %.2f select %.2f tie %.2f" % tuple(np.diff([buf[1], buf[12], buf[13], buf[2]]) / 1000))
    print("   bsr+plan: colw %.2f cnt+scan %.2f ptr+idx %.2f mask %.2f plan-cnt+scan %.2f plan-lists %.2f" % tuple(np.diff(seq) / 1000))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        spion.pattern(A, B, filter=31, alpha=75.0, out=bp)
    e1.record(); torch.cuda.synchronize()
    print("   pattern call avg us", e0.elapsed_time(e1) / 20 * 1000)
