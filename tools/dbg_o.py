import math, sys, numpy as np, torch
sys.path.insert(0, ".")
import synth, oracle
from paper_2309_12578_b200 import spion
L, B, d, bh, density, mode = 512, 64, 64, 2, 0.2, "masked"
fl = synth.syn_mask(L // B, density, seed=L + bh)
print(fl.astype(int))
bp = spion.bsr_from_mask(torch.from_numpy(fl).cuda(), L, B)
q, k, v, do = synth.qkvdo(bh, L, d, seed=L + d, dtype=torch.bfloat16)
for m in ("masked", "paper"):
    o, lse = spion.attn_fwd(q.cuda(), k.cuda(), v.cuda(), bp, m, 1 / 8)
    torch.cuda.synchronize()
    O_r, lse_r = oracle.attn_fwd(q[0].double().numpy(), k[0].double().numpy(), v[0].double().numpy(), fl, B, 1 / 8, m)
    err = np.abs(o[0].float().cpu().numpy() - O_r).max(-1)
    lerr = np.abs(lse[0].cpu().numpy() - lse_r)
    bad = np.where(err > 0.02)[0]
    print(m, "bad rows", len(bad), bad[:10], "max err", err.max(), "lse err max", lerr.max(), "at", lerr.argmax())
    print("  per block-row max err", [round(float(err[i*B:(i+1)*B].max()), 4) for i in range(L // B)])
    print("  per block-row lse err", [round(float(lerr[i*B:(i+1)*B].max()), 4) for i in range(L // B)])
print("plan fwd:", bp.plan.view(torch.int32)[:40].tolist())
