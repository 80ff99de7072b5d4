import math, sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, oracle
from paper_2309_12578_b200 import spion
def run(L, B, bh, density, mode, verbose=False):
    d = 64
    fl = synth.syn_mask(L // B, density, seed=L + bh)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).cuda(), L, B)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=L + d, dtype=torch.bfloat16)
    qd, kd, vd, dod = (x.cuda() for x in (q, k, v, do))
    o, lse = spion.attn_fwd(qd, kd, vd, bp, mode, 1 / 8)
    torch.cuda.synchronize()
    o1 = o.float().cpu().numpy(); l1 = lse.cpu().numpy()
    nbad = 0
    for b in range(bh):
        O_r, lse_r = oracle.attn_fwd(q[b].double().numpy(), k[b].double().numpy(), v[b].double().numpy(), fl, B, 1 / 8, mode)
        e1 = np.abs(o1[b] - O_r).max(-1)
        badr = np.where(e1 > 0.02)[0]
        if len(badr):
            nbad += 1
            r = badr[0]
            print(mode, "slice", b, "bad rows", len(badr), "block rows", sorted(set((badr // B).tolist())), "row", r,
                  "lse err", abs(l1[b][r] - lse_r[r]), "|O|", np.abs(o1[b][r]).max(), "|Oref|", np.abs(O_r[r]).max(),
                  "ratio", float(np.dot(o1[b][r], O_r[r]) / np.dot(O_r[r], O_r[r])))
    return nbad
tot = 0
for it in range(6):
    tot += run(512, 64, 3, 0.2, "paper")
    tot += run(512, 64, 2, 0.2, "masked")
    tot += run(1024, 64, 2, 0.3, "masked")
    tot += run(512, 32, 3, 0.15, "masked")
print("total bad slices", tot)
