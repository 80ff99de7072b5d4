"""NEXT-4: the sparse-MHA sub-layer (Alg. 5) on the SPION kernels — head split /
concatenation and dropout + residual kernels, and the module against a plain PyTorch reference
(dense masked attention built from the same block mask, fp32)."""
import math

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _mods():
    from paper_2309_12578_b200 import mha, spion
    return mha, spion


def test_split_merge_heads_exact():
    mha, _ = _mods()
    batch, L, H, d = 3, 96, 4, 64
    qkv = torch.randn(batch, L, 3 * H * d, device=DEV).bfloat16()
    q, k, v = mha.split_heads(qkv, H)
    ref = qkv.view(batch, L, 3, H, d).permute(2, 0, 3, 1, 4).reshape(3, batch * H, L, d)
    assert torch.equal(q, ref[0]) and torch.equal(k, ref[1]) and torch.equal(v, ref[2])
    s = mha.merge_heads(q.contiguous(), batch, H)
    assert torch.equal(s, ref[0].view(batch, H, L, d).permute(0, 2, 1, 3).reshape(batch, L, H * d))
    # backward of the split is the concatenation (and vice versa): autograd round trip
    x = qkv.clone().requires_grad_(True)
    a, b, c = mha.split_heads(x, H)
    (a.float().sum() + 2 * b.float().sum() + 3 * c.float().sum()).backward()
    g = x.grad.view(batch, L, 3, H, d)
    assert torch.equal(g[:, :, 0], torch.ones_like(g[:, :, 0])) and torch.equal(g[:, :, 2], 3 * torch.ones_like(g[:, :, 2]))


def test_dropout_residual():
    mha, _ = _mods()
    n = 1 << 20
    y = torch.randn(n, device=DEV).bfloat16()
    e = torch.randn(n, device=DEV).bfloat16()
    out = mha.dropout_residual(y, e, 0.0, 7)
    assert torch.equal(out, (e.float() + y.float()).bfloat16())
    p = 0.3
    o1, o2 = mha.dropout_residual(y, e, p, 11), mha.dropout_residual(y, e, p, 11)
    assert torch.equal(o1, o2)
    kept = mha.dropout_residual(torch.ones_like(y), torch.zeros_like(e), p, 11).float() != 0  # the seed-11 mask
    frac = kept.float().mean().item()
    assert abs(frac - (1 - p)) < 0.005, frac
    assert not torch.equal(o1, mha.dropout_residual(y, e, p, 12))
    # backward drops the same elements, scaled by 1/(1-p)
    yy = y.clone().requires_grad_(True)
    ee = e.clone().requires_grad_(True)
    mha.dropout_residual(yy, ee, p, 11).float().sum().backward()
    gy = yy.grad.float()
    assert torch.equal(gy != 0, kept) and torch.allclose(gy[kept], torch.full_like(gy[kept], 1 / (1 - p)), rtol=1e-2)
    assert torch.equal(ee.grad, torch.ones_like(e))


def _reference(e, w_qkv, w_o, fl, B, H, mode):
    """Alg. 5 with torch ops in fp32: dense masked attention from the block mask."""
    batch, L, D = e.shape
    d = D // H
    qkv = e @ w_qkv.t()  # nn.Linear layout (out x in)
    q, k, v = qkv.view(batch, L, 3, H, d).permute(2, 0, 3, 1, 4)
    allowed = torch.from_numpy(np.kron(fl, np.ones((B, B)))).bool().to(e.device)
    s = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    s = s.masked_fill(~allowed, float("-inf"))
    if mode == "paper":  # implicit zeros join the normaliser (reading Q1)
        m = s.amax(-1, keepdim=True)
        z = torch.exp(s - m).sum(-1, keepdim=True) + (~allowed).sum(-1, keepdim=True) * torch.exp(-m)
        p = torch.exp(s - m) / z
    else:
        p = torch.softmax(s, -1)
    o = (p @ v).permute(0, 2, 1, 3).reshape(batch, L, D)
    return o @ w_o.t() + e


@pytest.mark.parametrize("M,N,K,a_heads,c_heads,batch,L,H", [
    (256, 256, 128, False, False, 1, 256, 2),      # plain row-major
    (1024, 384, 192, False, False, 1, 1024, 1),    # several N tiles, K = 3 steps
    (2 * 512, 3 * 256, 256, False, True, 2, 512, 4),  # QKV: scatter into [3][batch*H][L][64]
    (2 * 512, 256, 256, True, False, 2, 512, 4),      # out-projection: gather from [batch*H][L][64]
    (3 * 256, 256, 3 * 128, True, False, 3, 256, 2),  # dX: gather from [3][batch*H][L][64]
    (4 * 128, 128, 128, False, True, 4, 128, 2),      # dS: scatter, L = 128 (one tile per batch item)
])
def test_gemm_bf16_layouts(M, N, K, a_heads, c_heads, batch, L, H):
    """spion_gemm_bf16 (tcgen05) against torch fp32 matmul, with the head-layout gather / scatter
    checked against explicit permutes."""
    mha, spion = _mods()
    torch.manual_seed(M + N + K)
    a2 = torch.randn(M, K, device=DEV).bfloat16()
    b = (torch.randn(N, K, device=DEV) / math.sqrt(K)).bfloat16()
    ref = a2.float() @ b.float().t()
    to_heads = lambda x, W: x.view(batch, L, W, H, 64).permute(2, 0, 3, 1, 4).contiguous()  # [W][batch][H][L][64]
    a = to_heads(a2, K // (64 * H)) if a_heads else a2
    out = torch.empty((N // (64 * H), batch * H, L, 64) if c_heads else (M, N), device=DEV, dtype=torch.bfloat16)
    c0 = spion.tc_launch_count()
    mha.gemm(a, b, out, M, N, K, a_heads=a_heads, c_heads=c_heads, L=L, H=H, batch=batch, alpha=1.0)
    torch.cuda.synchronize()
    assert spion.tc_launch_count() - c0 == 1
    got = out.view(N // (64 * H), batch, H, L, 64).permute(1, 3, 0, 2, 4).reshape(M, N) if c_heads else out
    err = (got.float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-2, err


@pytest.mark.parametrize("mode", ["paper", "masked"])
def test_sparse_mha_matches_reference(mode):
    mha, spion = _mods()
    batch, L, D, H, B = 2, 512, 256, 4, 64
    torch.manual_seed(0)
    m = mha.SparseMHA(D, H, dropout=0.0, mode=mode, device=DEV)
    fl = synth.syn_mask(L // B, 0.3, seed=3)
    bp = spion.bsr_from_mask(torch.as_tensor(fl, dtype=torch.uint8, device=DEV), L, B)
    e = (torch.randn(batch, L, D, device=DEV) * 0.5).bfloat16().requires_grad_(True)
    out = m(e, bp)
    g = torch.randn_like(out)
    out.backward(g)
    e32 = e.detach().float().requires_grad_(True)
    wq = m.w_qkv.detach().float().requires_grad_(True)
    wo = m.w_o.detach().float().requires_grad_(True)
    ref = _reference(e32, wq, wo, fl, B, H, mode)
    ref.backward(g.float())
    for name, got, want in (("out", out, ref), ("dE", e.grad, e32.grad), ("dWqkv", m.w_qkv.grad, wq.grad),
                            ("dWo", m.w_o.grad, wo.grad)):
        err = (got.float() - want).abs().max().item()
        scale = want.abs().max().item()
        assert err <= 2e-2 * scale + 1e-3, (name, err, scale)
