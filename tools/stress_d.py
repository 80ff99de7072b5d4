"""Debug: after each backward, compare the D = rowsum(dO * O) and -lse*log2(e) the dQ kernel stored in
the workspace against torch, to localise a rare run-to-run difference.
usage: python tools/stress_d.py <L> <B> <bh> <reps>"""
import sys
import torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion
L, B, bh, reps = (int(x) for x in sys.argv[1:5])
dev = torch.device("cuda:0")
A = synth.lra_scores(L, B, seed=4)
bp = spion.pattern(A.to(dev), B, filter=31, alpha=75.0, sync=True)
q, k, v, do = (x.to(dev) for x in synth.qkvdo(bh, L, 64, seed=2, dtype=torch.bfloat16))
ws = spion.attn_workspace(bh, L, 64, torch.bfloat16, dev)
o, lse = spion.attn_fwd(q, k, v, bp)
D_ref = None
nbad = 0
for rep in range(reps):
    o2, lse2 = spion.attn_fwd(q, k, v, bp)
    g = spion.attn_bwd(q, k, v, o2, do, lse2, bp, workspace=ws)
    torch.cuda.synchronize()
    Dk = ws[256:256 + bh * L * 4].view(torch.float32).view(bh, L)
    off = 256 + ((bh * L * 4 + 255) // 256) * 256
    nl = ws[off:off + bh * L * 4].view(torch.float32).view(bh, L)
    if D_ref is None:
        D_ref = Dk.clone()
        D_t = (o2.float() * do.float()).sum(-1)
        print("D vs torch max", float((Dk - D_t).abs().max()), "nl vs torch", float((nl + lse2 * 1.4426950408889634).abs().max()))
        g_ref = [x.clone() for x in g]
        continue
    dd = (Dk - D_ref).abs()
    if dd.max() > 0 or any(not torch.equal(a, b) for a, b in zip(g, g_ref)):
        nbad += 1
        if nbad <= 4:
            bb, rr = divmod(int(dd.argmax()), L)
            rows = torch.nonzero(dd[bb] > 0).flatten().tolist()
            gd = (g[0].float() - g_ref[0].float()).abs()
            gb = int(gd.flatten(1).amax(1).argmax())
            grows = torch.nonzero(gd[gb].amax(1) > 0).flatten().tolist()
            print(f"   dq diff max {float(gd.max()):.3g} bh {gb} rows {grows[:12]}..{grows[-4:]} ({len(grows)})")
            print(f"rep {rep}: D diff max {float(dd.max()):.3g} bh {bb} rows {rows[:16]} | o equal {torch.equal(o2, o)} "
                  f"lse equal {torch.equal(lse2, lse)} | grads equal {[torch.equal(a, b) for a, b in zip(g, g_ref)]}")
print("reps with differences:", nbad, "of", reps - 1)
