"""sparse attention fwd+bwd vs dense attention on B200, across block densities.

For each LRA shape: SPION fwd+bwd (tcgen05 kernels) on SYN(rho) block masks (synth.syn_mask: forced
diagonal, a stripe, band, random blocks) for rho in RHOS, and dense attention fwd+bwd through
torch SDPA (flash / cuDNN backends, library code) and flash_attn 2.8 — both bf16 [batch, heads, L, 64].
Device time with CUDA events, 3 warm-up + 20 timed iterations, two rotating input sets.  Prints
a markdown table and writes JSON (argv[1], default gpurun_out/density_sweep.json).  Context for the
paper's Fig. 6/7 claims (sparse vs dense speedups), not a bench line."""
import json, math, sys

import torch
import torch.nn.functional as F

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2309_12578_b200 import accounting, spion  # noqa: E402

SHAPES = [("image", 1024, 32, 4, 64), ("listops", 2048, 64, 8, 32), ("text", 4096, 64, 8, 16)]
RHOS = [0.02, 0.05, 0.10, 0.25, 0.50, 1.0]
dev = torch.device("cuda:0")


def timeit(fn, iters=20, warm=3):
    for i in range(warm):
        fn(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for i in range(iters):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


rows = []
for name, L, B, H, batch in SHAPES:
    bh, d = batch * H, 64
    n = L // B
    sets = [synth.qkvdo(bh, L, d, seed=11 + s, dtype=torch.bfloat16, device=dev) for s in range(2)]
    res = {"shape": name, "L": L, "block": B, "heads": H, "batch": batch}
    # dense references (4-D [batch, heads, L, d])
    dense = [[x.view(batch, H, L, d).requires_grad_(k < 3) for k, x in enumerate(st)] for st in sets]

    def sdpa(i, backend):
        q, k, v, do = dense[i % 2]
        with torch.nn.attention.sdpa_kernel(backend):
            o = F.scaled_dot_product_attention(q, k, v)
        torch.autograd.grad(o, (q, k, v), do)

    for label, be in (("sdpa_flash", torch.nn.attention.SDPBackend.FLASH_ATTENTION),
                      ("sdpa_cudnn", torch.nn.attention.SDPBackend.CUDNN_ATTENTION)):
        try:
            res[label + "_ms"] = timeit(lambda i: sdpa(i, be))
        except Exception as e:  # backend unavailable for this shape
            res[label + "_ms"] = None
            res[label + "_err"] = str(e)[:120]
    try:
        from flash_attn import flash_attn_func
        fa = [[x.view(batch, H, L, d).transpose(1, 2).contiguous().requires_grad_(k < 3) for k, x in enumerate(st)]
              for st in sets]

        def fa2(i):
            q, k, v, do = fa[i % 2]
            o = flash_attn_func(q, k, v)
            torch.autograd.grad(o, (q, k, v), do)

        res["flash_attn2_ms"] = timeit(fa2)
    except Exception as e:
        res["flash_attn2_ms"] = None
        res["flash_attn2_err"] = str(e)[:120]
    for rho in RHOS:
        m = synth.syn_mask(n, rho, seed=7)
        bp = spion.bsr_from_mask(torch.as_tensor(m, dtype=torch.uint8, device=dev), L, B)
        nnzb = bp.nnzb
        outs = [dict(o=torch.empty_like(st[0]), lse=torch.empty((bh, L), dtype=torch.float32, device=dev),
                     dq=torch.empty_like(st[0]), dk=torch.empty_like(st[0]), dv=torch.empty_like(st[0])) for st in sets]
        ws = spion.attn_workspace(bh, L, d, torch.bfloat16, dev)

        def sp(i):
            q, k, v, do = sets[i % 2]
            o = outs[i % 2]
            spion.attn_fwd(q, k, v, bp, "paper", 1 / math.sqrt(d), out=o["o"], lse=o["lse"])
            spion.attn_bwd(q, k, v, o["o"], do, o["lse"], bp, "paper", 1 / math.sqrt(d), workspace=ws,
                           dq=o["dq"], dk=o["dk"], dv=o["dv"])

        ms = timeit(sp)
        fl = accounting.useful_flops(B, d, nnzb, bh)
        res[f"rho_{rho}"] = {"nnzb": nnzb, "density": nnzb / n / n, "ms": ms, "useful_tflops": fl / ms / 1e9}
    rows.append(res)
    print(json.dumps(res), flush=True)

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/density_sweep.json"
json.dump(rows, open(out, "w"), indent=1)
print("\n| shape | dense flash_attn2 ms | SDPA flash ms | SDPA cuDNN ms | " + " | ".join(f"ρ={r} ms (TF/s)" for r in RHOS) + " |")
print("|" + "---|" * (4 + len(RHOS)))
f = lambda x: "n/a" if x is None else f"{x:.3f}"
for r in rows:
    cells = [f"{r[f'rho_{rho}']['ms']:.3f} ({r[f'rho_{rho}']['useful_tflops']:.0f})" for rho in RHOS]
    print(f"| {r['shape']} | {f(r['flash_attn2_ms'])} | {f(r['sdpa_flash_ms'])} | {f(r['sdpa_cudnn_ms'])} | " + " | ".join(cells) + " |")
