"""Debug: repeat fwd/bwd on fixed inputs and report any run-to-run difference (races).
usage: python tools/stress_repeat.py <L> <B> <bh> <reps> [concurrent]"""
import sys
import torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import spion
L, B, bh, reps = (int(x) for x in sys.argv[1:5])
conc = len(sys.argv) > 5
dev = torch.device("cuda:0")
A = synth.lra_scores(L, B, seed=4)
bp = spion.pattern(A.to(dev), B, filter=31, alpha=75.0, sync=True)
sets = [tuple(x.to(dev) for x in synth.qkvdo(bh, L, 64, seed=s, dtype=torch.bfloat16)) for s in (1, 2)]
ref = []
for q, k, v, do in sets:
    o, lse = spion.attn_fwd(q, k, v, bp)
    ref.append((o, lse) + spion.attn_bwd(q, k, v, o, do, lse, bp))
torch.cuda.synchronize()
streams = [torch.cuda.Stream() for _ in sets]
wss = [spion.attn_workspace(bh, L, 64, torch.bfloat16, dev) for _ in sets]
bad = {}
for rep in range(reps):
    got = [None, None]
    for i, ((q, k, v, do), st) in enumerate(zip(sets, streams)):
        with torch.cuda.stream(st if conc else torch.cuda.current_stream()):
            o, lse = spion.attn_fwd(q, k, v, bp, workspace=wss[i])
            got[i] = (o, lse) + spion.attn_bwd(q, k, v, o, do, lse, bp, workspace=wss[i])
    torch.cuda.synchronize()
    for i, (g, r) in enumerate(zip(got, ref)):
        for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), g, r):
            if not torch.equal(a, b):
                d = (a.float() - b.float()).abs()
                nbh = int((d.flatten(1).amax(1) > 0).sum()) if d.dim() > 1 else 0
                bad.setdefault(name, []).append((rep, i, float(d.max()), nbh))
                if d.dim() == 3 and len(bad[name]) <= 2:
                    bb = int(d.flatten(1).amax(1).argmax())
                    rows = torch.nonzero(d[bb].amax(1) > 0).flatten().tolist()
                    print(f"  {name} rep {rep} set {i} bh {bb}: rows {rows[:3]}..{rows[-3:]} ({len(rows)} rows), "
                          f"blocks {sorted(set(r // B for r in rows))}, max|ref| {float(b[bb].float().abs().max()):.3g}")
print("L", L, "B", B, "bh", bh, "concurrent" if conc else "sequential", "mismatches:",
      {k: (len(v), v[:3]) for k, v in bad.items()} or "none")
