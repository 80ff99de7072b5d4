import math, sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, oracle
from paper_2309_12578_b200 import spion
def run(L, B, bh, density, mode):
    d = 64
    fl = synth.syn_mask(L // B, density, seed=L + bh)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).cuda(), L, B)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=L + d, dtype=torch.bfloat16)
    qd, kd, vd, dod = (x.cuda() for x in (q, k, v, do))
    o, lse = spion.attn_fwd(qd, kd, vd, bp, mode, 1 / 8)
    torch.cuda.synchronize()
    o1 = o.float().cpu().numpy().copy()
    dq, dk, dv = spion.attn_bwd(qd, kd, vd, o, dod, lse, bp, mode, 1 / 8)
    torch.cuda.synchronize()
    o2 = o.float().cpu().numpy()
    for b in range(bh):
        O_r, _ = oracle.attn_fwd(q[b].double().numpy(), k[b].double().numpy(), v[b].double().numpy(), fl, B, 1 / 8, mode)
        e1 = np.abs(o1[b] - O_r).max(-1); e2 = np.abs(o2[b] - O_r).max(-1)
        print(L, B, bh, mode, "slice", b, "O err after fwd", e1.max(), "after bwd", e2.max(), "bad block rows", sorted(set((np.where(e1 > 0.02)[0] // B).tolist())))
run(512, 64, 3, 0.2, "paper")
run(512, 64, 2, 0.2, "masked")
run(512, 64, 2, 0.2, "masked")
run(512, 64, 2, 0.2, "paper")
