"""NEXT-4: time the sparse-MHA sub-layer (Alg. 5) fwd+bwd at LRA shapes, and its parts (CUDA events).
Pattern: the bench's synthetic score recipe at alpha = 75 (flood fill), computed once (the transition)."""
import sys, torch
sys.path.insert(0, ".")
import synth
from paper_2309_12578_b200 import mha, spion

def t(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it

for name, L, B, H, batch in [("image", 1024, 32, 4, 64), ("text", 4096, 64, 8, 16)]:
    D = 64 * H
    bp = spion.pattern(synth.lra_scores(L, B, seed=1, device="cuda"), B, filter=31, alpha=75.0, sync=True)
    m = mha.SparseMHA(D, H, dropout=0.1, device="cuda")
    e = torch.randn(batch, L, D, device="cuda").bfloat16().requires_grad_(True)
    g = torch.randn(batch, L, D, device="cuda").bfloat16()

    def step():
        out = m(e, bp, seed=1)
        out.backward(g)

    q, k, v = [x.contiguous() for x in mha.qkv_projection(e.detach(), m.w_qkv.detach(), H)]
    ed, wq = e.detach(), m.w_qkv.detach()
    parts = {
        "sub-layer fwd+bwd": t(step),
        "QKV projection (tcgen05 GEMM -> heads)": t(lambda: mha.qkv_projection(ed, wq, H)),
        "QKV GEMM (cuBLAS, packed; reference)": t(lambda: ed @ wq.t()),
        "out projection (heads -> tcgen05 GEMM)": t(lambda: mha.out_projection(q, m.w_o.detach(), batch, H)),
        "attention fwd": t(lambda: spion.attn_fwd(q, k, v, bp)),
        "merge heads": t(lambda: mha.merge_heads(q, batch, H)),
        "dropout+residual": t(lambda: mha.dropout_residual(q.view(batch, L, D), e.detach(), 0.1, 1)),
    }
    M = batch * L
    gf = 2 * M * 3 * D * D / parts["QKV projection (tcgen05 GEMM -> heads)"] / 1e9
    print(name, "QKV projection TFLOP/s", round(gf, 1))
    print(name, f"L={L} D={D} batch={batch} nnzb={bp.nnzb}", {k: round(v, 4) for k, v in parts.items()})
