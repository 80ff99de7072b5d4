import math, sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, oracle
from paper_2309_12578_b200 import spion
for (L, B, bh) in [(512, 64, 2), (512, 32, 2), (256, 64, 1)]:
    fl = synth.syn_mask(L // B, 0.2, seed=L + bh)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).cuda(), L, B)
    q, k, v, do = synth.qkvdo(bh, L, 64, seed=L + 64, dtype=torch.bfloat16)
    qd, kd, vd, dod = (x.cuda() for x in (q, k, v, do))
    o, lse = spion.attn_fwd(qd, kd, vd, bp)
    dq, dk, dv = spion.attn_bwd(qd, kd, vd, o, dod, lse, bp)
    torch.cuda.synchronize()
    dvn = dv.float().cpu().numpy()
    dkn = dk.float().cpu().numpy()
    bad_rows = np.where(~np.isfinite(dvn).all(-1))
    print(L, B, bh, "dV nan rows", len(bad_rows[0]), "of", bh * L, "first", list(zip(bad_rows[0][:8], bad_rows[1][:8])), "dK nan", (~np.isfinite(dkn)).sum())
    dQ_r, dK_r, dV_r = oracle.attn_bwd(q[0].double().numpy(), k[0].double().numpy(), v[0].double().numpy(), do[0].double().numpy(), fl, B, 1/8, "paper")
    fin = np.isfinite(dvn[0]).all(-1)
    print("   dV err (finite rows)", np.abs(dvn[0][fin] - dV_r[fin]).max() if fin.any() else None, "dK err", np.abs(dkn[0] - dK_r).max())
    print("   mask", fl.astype(int).tolist())
