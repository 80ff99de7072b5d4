"""GPU parity of block-sparse attention fwd/bwd against the fp64 oracle.

Bars (BASELINE.json north_star): fp32 mode max-abs 1e-4 on O, dQ, dK, dV (and
lse 1e-5); bf16 mode max-abs 2e-2 plus a normalised bar max-abs/max|ref| <= 1e-2
(at 10% density PAPER-mode outputs are ~0.2 in magnitude, so 2e-2
alone would accept 10% relative error), lse 1e-3.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _spion():
    from paper_2309_12578_b200 import spion
    return spion


def _expect_tc(L, B, d, dtype):
    """Shapes the tensor-core (tcgen05) path must take (SURVEY 8(b) envelope)."""
    return dtype == torch.bfloat16 and d == 64 and B in (32, 64) and L % 4 == 0 and L // B <= 128


def _run(q, k, v, do, bp, mode, scale, fused=False):
    """fwd + bwd through the C ABI; asserts which kernels ran (the tensor-core kernels for every
    shape in their envelope — no silent CUDA-core fallback).  fused: SPION_BWD_FUSED."""
    spion = _spion()
    qd, kd, vd, dod = (x.to(DEV) for x in (q, k, v, do))
    path = spion.attn_path(qd, bp)
    assert path == ("tcgen05" if _expect_tc(bp.L, bp.block, q.shape[2], q.dtype) else "cuda_core"), path
    tc0 = spion.tc_launch_count()
    o, lse = spion.attn_fwd(qd, kd, vd, bp, mode, scale)
    dq, dk, dv = spion.attn_bwd(qd, kd, vd, o, dod, lse, bp, mode, scale, fused=fused)
    torch.cuda.synchronize()
    ran_tc = spion.tc_launch_count() - tc0
    assert (ran_tc >= 2) if path == "tcgen05" else (ran_tc == 0), (path, ran_tc)
    return [x.float().cpu().numpy() for x in (o, lse, dq, dk, dv)]


def _oracle_slice(args):
    b, q, k, v, do, fl, B, scale, mode = args
    Q, K, V, dO = (x[b].double().numpy() for x in (q, k, v, do))
    O_r, lse_r = oracle.attn_fwd(Q, K, V, fl, B, scale, mode)
    dQ_r, dK_r, dV_r = oracle.attn_bwd(Q, K, V, dO, fl, B, scale, mode)
    return b, (O_r, lse_r, dQ_r, dK_r, dV_r)


def _compare(outs, q, k, v, do, fl, B, mode, scale, slices, tol, norm_tol=None, lse_tol=None):
    """Element-wise comparison with the fp64 oracle on every slice in `slices`; the oracle runs
    one slice per host thread (its C calls release the GIL)."""
    import concurrent.futures as cf
    import os

    o, lse, dq, dk, dv = outs
    worst = {}
    slices = list(slices)
    work = [(b, q, k, v, do, fl, B, scale, mode) for b in slices]
    with cf.ThreadPoolExecutor(max_workers=min(len(work), os.cpu_count() or 1)) as ex:
        results = ex.map(_oracle_slice, work) if len(work) > 1 else map(_oracle_slice, work)
        for b, (O_r, lse_r, dQ_r, dK_r, dV_r) in results:
            for name, got, ref in (("O", o[b], O_r), ("dQ", dq[b], dQ_r), ("dK", dk[b], dK_r), ("dV", dv[b], dV_r)):
                err = np.abs(got - ref).max()
                worst[name] = max(worst.get(name, 0.0), err)
                assert err <= tol, (name, b, err)
                if norm_tol is not None and np.abs(ref).max() > 0:
                    assert err / np.abs(ref).max() <= norm_tol, (name, b, err, np.abs(ref).max())
            fin = np.isfinite(lse_r)
            assert (np.isfinite(lse[b]) == fin).all()
            if lse_tol is not None and fin.any():
                assert np.abs(lse[b][fin] - lse_r[fin]).max() <= lse_tol
    return worst


# ---------------------------------------------------------------- fp32 (CUDA cores)
@pytest.mark.parametrize("mode", ["paper", "masked"])
def test_tiny_config_fp32(mode):
    """configs[0]: L=64, block=8, 1 head, d=16, batch=1, fixed threshold, fp32 fwd+bwd."""
    spion = _spion()
    L, B, d = 64, 8, 16
    A = synth.syn_scores(L, B, heads=1, seed=11)
    bp = spion.pattern(A.to(DEV), B, filter=31, t=0.1, sync=True)
    fl, _, _ = oracle.pattern(A.numpy(), B, 31, 0.1, "absolute")
    q, k, v, do = synth.qkvdo(1, L, d, seed=5, dtype=torch.float32)
    scale = 1 / math.sqrt(d)
    outs = _run(q, k, v, do, bp, mode, scale)
    _compare(outs, q, k, v, do, fl, B, mode, scale, [0], 1e-4, lse_tol=1e-5)


@pytest.mark.parametrize("L,B,d,bh,density,mode", [
    (256, 16, 32, 3, 0.2, "paper"), (256, 32, 64, 2, 0.15, "masked"), (192, 64, 64, 2, 0.5, "paper"),
    (128, 8, 128, 1, 0.3, "masked"), (96, 32, 24, 2, 1.0, "paper"),
])
def test_fp32_parity(L, B, d, bh, density, mode):
    spion = _spion()
    n = L // B
    fl = synth.syn_mask(n, density, seed=L + B)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=L * d, dtype=torch.float32)
    scale = 1 / math.sqrt(d)
    outs = _run(q, k, v, do, bp, mode, scale)
    _compare(outs, q, k, v, do, fl, B, mode, scale, range(bh), 1e-4, lse_tol=1e-5)


@pytest.mark.parametrize("mode", ["paper", "masked"])
def test_fp32_empty_rows(mode):
    spion = _spion()
    L, B, d = 128, 16, 16
    fl = synth.syn_mask(8, 0.3, seed=1)
    fl[3] = 0
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(2, L, d, seed=9, dtype=torch.float32)
    outs = _run(q, k, v, do, bp, mode, 0.25)
    _compare(outs, q, k, v, do, fl, B, mode, 0.25, range(2), 1e-4, lse_tol=1e-5)
    o, lse = outs[0], outs[1]
    assert (o[:, 48:64] == 0).all()
    assert (lse[:, 48:64] == (math.log(L) if mode == "paper" else -math.inf)).all() or mode == "paper"


def test_fp32_strided_layout():
    """[L][heads][d] storage (batch 1): stride_bh = d, stride_l = heads*d."""
    spion = _spion()
    L, B, d, H = 128, 16, 32, 3
    fl = synth.syn_mask(L // B, 0.25, seed=4)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(H, L, d, seed=77, dtype=torch.float32)
    to_strided = lambda x: x.to(DEV).permute(1, 0, 2).contiguous().permute(1, 0, 2)
    qd, kd, vd, dod = (to_strided(x) for x in (q, k, v, do))
    o, lse = spion.attn_fwd(qd, kd, vd, bp, "paper", 0.2)
    dq, dk, dv = spion.attn_bwd(qd, kd, vd, o, dod, lse, bp, "paper", 0.2)
    outs = [x.float().cpu().numpy() for x in (o, lse, dq, dk, dv)]
    _compare(outs, q, k, v, do, fl, B, "paper", 0.2, range(H), 1e-4)


def test_bf16_strided_layout():
    """bf16 [L][heads][d] storage (stride_l = heads*d, stride_bh = d: strided TMA tensor maps on
    the tensor-core path) against the oracle."""
    spion = _spion()
    L, B, d, H = 512, 64, 64, 3
    fl = synth.syn_mask(L // B, 0.3, seed=6)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(H, L, d, seed=78, dtype=torch.bfloat16)
    to_strided = lambda x: x.to(DEV).permute(1, 0, 2).contiguous().permute(1, 0, 2)
    qd, kd, vd, dod = (to_strided(x) for x in (q, k, v, do))
    o, lse = spion.attn_fwd(qd, kd, vd, bp, "paper", 0.125)
    dq, dk, dv = spion.attn_bwd(qd, kd, vd, o, dod, lse, bp, "paper", 0.125)
    outs = [x.float().cpu().numpy() for x in (o, lse, dq, dk, dv)]
    _compare(outs, q, k, v, do, fl, B, "paper", 0.125, range(H), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


# ---------------------------------------------------------------- bf16
BF16_CASES = [
    # L, B, d, bh, density, mode   (ragged: nblk not a multiple of the 128-row tile)
    (512, 64, 64, 3, 0.2, "paper"),
    (512, 64, 64, 2, 0.2, "masked"),
    (320, 64, 64, 2, 0.4, "paper"),     # nblk = 5
    (512, 32, 64, 3, 0.15, "paper"),
    (224, 32, 64, 2, 0.3, "masked"),    # nblk = 7
    (256, 32, 64, 1, 1.0, "paper"),     # dense
    (256, 16, 32, 2, 0.25, "paper"),    # CUDA-core bf16 path
    (1024, 64, 64, 2, 0.15, "paper"),   # B=64, stripe columns with many entries (1 CTA/SM kernels)
    (1024, 64, 64, 2, 0.30, "masked"),
    (1088, 64, 64, 1, 0.25, "paper"),   # nblk = 17 (ragged tile)
    (2048, 32, 64, 2, 0.10, "paper"),   # B=32, nblk = 64
    (512, 128, 64, 2, 0.5, "paper"),    # B=128: CUDA-core bf16 path (SURVEY 8(b) envelope)
    (256, 64, 128, 2, 0.5, "masked"),   # d=128: CUDA-core bf16 path
]


@pytest.mark.parametrize("L,B,d,bh,density,mode", BF16_CASES)
def test_bf16_parity(L, B, d, bh, density, mode):
    spion = _spion()
    fl = synth.syn_mask(L // B, density, seed=L + bh)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=L + d, dtype=torch.bfloat16)
    scale = 1 / math.sqrt(d)
    outs = _run(q, k, v, do, bp, mode, scale)
    _compare(outs, q, k, v, do, fl, B, mode, scale, range(bh), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


FUSED_CASES = [c for c in BF16_CASES if c[1] == 64 and c[2] == 64] + [(640, 64, 64, 3, 0.35, "masked")]


@pytest.mark.parametrize("L,B,d,bh,density,mode", FUSED_CASES)
def test_bf16_parity_fused_backward(L, B, d, bh, density, mode):
    """SPION_BWD_FUSED (one pass: dK/dV per column tile, dQ by paired M=128 MMAs and L2 reduce-adds,
    finalised by the last contributor) against the oracle; odd entry counts leave a pair unpaired."""
    spion = _spion()
    fl = synth.syn_mask(L // B, density, seed=L + bh)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=L + d, dtype=torch.bfloat16)
    scale = 1 / math.sqrt(d)
    outs = _run(q, k, v, do, bp, mode, scale, fused=True)
    _compare(outs, q, k, v, do, fl, B, mode, scale, range(bh), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


@pytest.mark.parametrize("cfg", ["listops", "text"])
def test_full_size_all_slices_fused(cfg):
    """SPION_BWD_FUSED at full BASELINE sizes (bench launch configuration), every slice."""
    spion = _spion()
    c = FULL[cfg]
    L, B, bh, d = c["L"], c["B"], c["bh"], 64
    A = synth.lra_scores(L, B, seed=1)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=c["alpha"], sync=True)
    fl, _, _ = oracle.pattern(A.numpy(), B, 31, c["alpha"])
    q, k, v, do = synth.qkvdo(bh, L, d, seed=77, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, "paper", 1 / math.sqrt(d), fused=True)
    _compare(outs, q, k, v, do, fl, B, "paper", 1 / math.sqrt(d), range(bh), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


@pytest.mark.parametrize("L,B,cols", [(1024, 32, (3, 17, 30)), (1088, 64, (0, 9, 16)), (512, 32, (15,))])
def test_bf16_stripe_columns(L, B, cols):
    """Band + full vertical stripes (the LRA-like structure): the dK/dV column tiles take the
    block columns in count order, so stripe columns share tiles and are loaded / stored as
    separate B-row boxes at their own coordinates (ragged tails included)."""
    spion = _spion()
    n = L // B
    fl = np.zeros((n, n), dtype=np.uint8)
    for i in range(n):
        fl[i, max(0, i - 1):i + 2] = 1
    for c in cols:
        fl[:, c] = 1
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(2, L, 64, seed=L + B, dtype=torch.bfloat16)
    for mode in ("paper", "masked"):
        outs = _run(q, k, v, do, bp, mode, 0.125)
        _compare(outs, q, k, v, do, fl, B, mode, 0.125, range(2), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


def test_bf16_empty_rows():
    spion = _spion()
    L, B, d = 512, 64, 64
    fl = synth.syn_mask(8, 0.3, seed=2)
    fl[5] = 0
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(2, L, d, seed=3, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, "paper", 0.125)
    _compare(outs, q, k, v, do, fl, B, "paper", 0.125, range(2), 2e-2, norm_tol=1e-2, lse_tol=1e-3)
    assert (outs[0][:, 320:384] == 0).all()


@pytest.mark.parametrize("B,fused", [(32, False), (64, False), (64, True)])
def test_bf16_empty_block_columns(B, fused):
    """Block columns with no stored block, in the middle of the range: the dK/dV column tiles take
    block columns in count order, so an empty column's tile is a late tile whose rows are NOT
    t*128 + r; its dK/dV rows must still be zero (and the fused backward's dQ must not read them)."""
    spion = _spion()
    L = 1024
    n = L // B
    fl = synth.syn_mask(n, 0.25, seed=12)
    for c in (1, n // 2, n // 2 + 1):
        fl[:, c] = 0
    fl[3] = 0  # and one empty block row (dQ rows zero)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(3, L, 64, seed=31, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, "paper", 0.125, fused=fused)
    _compare(outs, q, k, v, do, fl, B, "paper", 0.125, range(3), 2e-2, norm_tol=1e-2, lse_tol=1e-3)
    for c in (1, n // 2, n // 2 + 1):
        assert (outs[3][:, c * B:(c + 1) * B] == 0).all() and (outs[4][:, c * B:(c + 1) * B] == 0).all()
    assert (outs[2][:, 3 * B:4 * B] == 0).all()


@pytest.mark.parametrize("mode", ["paper", "masked"])
@pytest.mark.parametrize("B", [32, 64])
def test_bf16_all_blocks_empty(mode, B):
    """Degenerate pattern with no stored block (nnzb = 0): O = 0, lse = ln L (PAPER) / -inf
    (MASKED), zero gradients - the tcgen05 kernels' empty-plan path, against the oracle."""
    spion = _spion()
    L, d = 512, 64
    fl = np.zeros((L // B, L // B), dtype=np.uint8)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    assert bp.nnzb == 0
    q, k, v, do = synth.qkvdo(3, L, d, seed=9, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, mode, 0.125)
    _compare(outs, q, k, v, do, fl, B, mode, 0.125, range(3), 0.0, lse_tol=1e-3)
    for x in (outs[0], outs[2], outs[3], outs[4]):
        assert (x == 0).all()


def test_attention_rejects_bad_shapes():
    """bh = 0 and d beyond the supported head widths are refused with SPION_ERR_SHAPE, and
    block = 128 with d = 128 (CUDA-core staging beyond 227 KB) with SPION_ERR_UNSUPPORTED
    (raised by the binding), not silently skipped."""
    spion = _spion()
    from paper_2309_12578_b200 import _native as N
    L, B = 256, 32
    fl = synth.syn_mask(L // B, 0.3, seed=1)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    for bh, d in ((0, 64), (2, 256)):
        q = torch.zeros((bh, L, d), dtype=torch.bfloat16, device=DEV)
        with pytest.raises(Exception):
            spion.attn_fwd(q, q, q, bp, "paper", 0.125)
    bp128 = spion.bsr_from_mask(torch.ones((2, 2), dtype=torch.uint8, device=DEV), 256, 128)
    q = torch.zeros((1, 256, 128), dtype=torch.bfloat16, device=DEV)
    with pytest.raises(N.SpionError) as ei:
        spion.attn_fwd(q, q, q, bp128, "paper", 0.125)
    assert ei.value.status == 7


# ------------------------------------------ full BASELINE sizes, every (batch, head) slice
# the bench's workloads (bench.CONFIGS): alpha per config puts the flood-filled block density near
# the north star's ~10 % on the synthetic LRA scores
FULL = {
    "image": dict(L=1024, B=32, bh=256, alpha=75.0),
    "listops": dict(L=2048, B=64, bh=256, alpha=75.0),
    "text": dict(L=4096, B=64, bh=128, alpha=55.0),
    "retrieval": dict(L=4096, B=64, bh=256, alpha=55.0),  # 2 towers x batch 16 x 8 heads
}


@pytest.mark.parametrize("cfg", ["image", "listops", "text", "retrieval"])
def test_full_size_all_slices(cfg):
    """Bench launch configuration (pattern from synthetic scores, then fwd+bwd over every
    (batch, head)); the oracle recomputes EVERY (batch, head) slice entirely (the dynamic
    scheduler places each slice in a different chunk / heavy-tile position)."""
    spion = _spion()
    c = FULL[cfg]
    L, B, bh, d = c["L"], c["B"], c["bh"], 64
    A = synth.lra_scores(L, B, seed=1)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=c["alpha"], sync=True)
    fl, _, _ = oracle.pattern(A.numpy(), B, 31, c["alpha"])
    n = L // B
    assert (bp.mask.view(n, n).cpu().numpy() == fl).all()
    q, k, v, do = synth.qkvdo(bh, L, d, seed=2024, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, "paper", 1 / math.sqrt(d))
    for x in outs:
        assert np.isfinite(x[np.isfinite(x) | ~np.isinf(x)]).all()
    _compare(outs, q, k, v, do, fl, B, "paper", 1 / math.sqrt(d), range(bh), 2e-2, norm_tol=1e-2,
             lse_tol=1e-3)


def _step_chunks(bh, tensor_bytes):
    """spion_step_host's (batch, head) chunk count (api.cu step_chunks)."""
    cmax = 8 if tensor_bytes > (64 << 20) else 16
    for C in (16, 8, 4, 2):
        if C <= cmax and bh % C == 0 and bh // C >= 8 and tensor_bytes // C >= (4 << 20):
            return C
    return 1


@pytest.mark.parametrize("bh,dtype,mode", [(16, "bf16", "paper"), (256, "bf16", "paper"), (512, "bf16", "masked"),
                                           (48, "f32", "paper")])
def test_step_host_matches_device_calls(bh, dtype, mode):
    """spion_step_host (pipelined over (batch, head) chunks, host buffers) gives the same bytes as
    spion_pattern + spion_attn_fwd + spion_attn_bwd on device buffers (bf16 bh = 16 / 256 / 512 run
    as 1 / 8 / 16 chunks; fp32 on the CUDA-core path)."""
    import ctypes

    spion = _spion()
    from paper_2309_12578_b200 import _native as N

    L, B, d = 1024, 32, 64
    A = synth.lra_scores(L, B, seed=5)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    q, k, v, do = synth.qkvdo(bh, L, d, seed=77, dtype=tdt)
    scale = 1 / math.sqrt(d)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=75.0, sync=True)
    qd, kd, vd, dod = (x.to(DEV) for x in (q, k, v, do))
    o, lse = spion.attn_fwd(qd, kd, vd, bp, mode, scale)
    # the device reference in spion_step_host's (batch, head) chunks: a launch's size decides whether the
    # dK/dV pass splits its heavy tiles (the summation order of those tiles' dK, dV)
    C = _step_chunks(bh, bh * L * d * (2 if dtype == "bf16" else 4))
    bc = bh // C
    grads = [spion.attn_bwd(qd[c * bc:(c + 1) * bc], kd[c * bc:(c + 1) * bc], vd[c * bc:(c + 1) * bc],
                            o[c * bc:(c + 1) * bc], dod[c * bc:(c + 1) * bc], lse[c * bc:(c + 1) * bc], bp, mode, scale)
             for c in range(C)]
    dq, dk, dv = (torch.cat([g[i] for g in grads]) for i in range(3))
    torch.cuda.synchronize()
    lib = N.lib()
    hA = A.pin_memory()
    hq, hk, hv, hdo = (x.pin_memory() for x in (q, k, v, do))
    ho, hdq, hdk, hdv = (torch.empty_like(hq).pin_memory() for _ in range(4))
    hlse = torch.empty((bh, L), dtype=torch.float32).pin_memory()
    ndt = N.BF16 if dtype == "bf16" else N.F32
    nb = lib.spion_step_arena_bytes(bh, L, d, B, ndt)
    arena = torch.empty(nb, dtype=torch.uint8, device=DEV)
    P = lambda t: ctypes.c_void_p(t.data_ptr())
    nnz = ctypes.c_int32(0)
    st = lib.spion_step_host(P(hA), P(hq), P(hk), P(hv), P(hdo), P(ho), P(hlse), P(hdq), P(hdk), P(hdv), bh, L, d, B,
                             31, 75.0, N.THRESH["linear"], ndt, N.SOFTMAX[mode], scale, P(arena), nb,
                             ctypes.byref(nnz), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    N.check(st, "spion_step_host")
    assert nnz.value == bp.nnzb
    for got, want in ((ho, o), (hlse, lse), (hdq, dq), (hdk, dk), (hdv, dv)):
        assert torch.equal(got, want.cpu())


@pytest.mark.parametrize("L,B", [(1024, 32), (2048, 64), (4096, 64)])
def test_plan_matches_host_recomputation(L, B):
    """The attention work plan built by the pattern kernel (slot tiles of S = 128/B block rows /
    columns, union lists with slot masks, descending-work order, heavy-tile counts, and the
    column-tile order: block columns by descending count, stable) equals a plain host recomputation from the block mask."""
    spion = _spion()
    A = synth.lra_scores(L, B, seed=3)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=75.0, sync=True)
    n = L // B
    fl = bp.mask.view(n, n).cpu().numpy().astype(bool)
    plan = bp.plan.view(torch.int32).cpu().numpy()
    S = 128 // B
    nt = (n + S - 1) // S
    fptr = 16
    bptr = fptr + nt + 1
    forder = bptr + nt + 1
    border = forder + nt
    cap = n * nt
    fcol = border + nt
    fmsk, brow = fcol + cap, fcol + 2 * cap
    bmsk = brow + cap
    bperm = bmsk + cap
    assert list(plan[:3]) == [n, S, nt]
    colcnt = fl.sum(0)
    want_perm = sorted(range(n), key=lambda c: (-colcnt[c], c)) + [n] * (nt * S - n)
    assert list(plan[bperm:bperm + nt * S]) == want_perm
    assert plan[7] == sum(1 for c in range(n) if colcnt[c] * n > 2 * fl.sum())
    row_order = list(range(n)) + [n] * (nt * S - n)
    for which, (ptr, order, col, msk, grid, perm) in enumerate(((fptr, forder, fcol, fmsk, fl, row_order),
                                                               (bptr, border, brow, bmsk, fl.T, want_perm))):
        cnts = []
        for t in range(nt):
            slots = perm[t * S:(t + 1) * S]
            rows = np.stack([grid[r] if r < n else np.zeros(n, dtype=bool) for r in slots])
            union = np.nonzero(rows.any(0))[0]
            beg, end = plan[ptr + t], plan[ptr + t + 1]
            assert end - beg == len(union)
            assert (plan[col + beg:col + end] == union).all()
            want_m = [sum(int(rows[s, j]) << s for s in range(S)) for j in union]
            assert list(plan[msk + beg:msk + end]) == want_m
            cnts.append(len(union))
        want_order = sorted(range(nt), key=lambda t: (-cnts[t], t))
        assert list(plan[order:order + nt]) == want_order
        tot = sum(cnts)
        assert plan[5 + which] == sum(1 for c in cnts if c * nt > 2 * tot)


@pytest.mark.parametrize("B", [32, 64])
def test_backward_deterministic(B):
    """SPION_BWD_DETERMINISTIC: every accumulator has one issuing thread and a fixed block order, so
    two backward passes give identical bits; the fused
    (SPION_BWD_FUSED) backward gives an identical dV and dQ, dK within bf16 rounding of the deterministic ones (its
    D = rowsum(dO * O) is summed in another order, and dQ by L2 reduce-adds in scheduling order)."""
    spion = _spion()
    L, bh, d = 2048, 24, 64
    A = synth.lra_scores(L, B, seed=9)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=75.0, sync=True)
    q, k, v, do = (x.to(DEV) for x in synth.qkvdo(bh, L, d, seed=5, dtype=torch.bfloat16))
    o, lse = spion.attn_fwd(q, k, v, bp)
    g1 = spion.attn_bwd(q, k, v, o, do, lse, bp, deterministic=True)
    g1 = [x.clone() for x in g1]
    o2, lse2 = spion.attn_fwd(q, k, v, bp)
    g2 = spion.attn_bwd(q, k, v, o2, do, lse2, bp, deterministic=True)
    assert torch.equal(o, o2) and torch.equal(lse, lse2)
    for a, b in zip(g1, g2):
        assert torch.equal(a, b)
    g0 = spion.attn_bwd(q, k, v, o, do, lse, bp)  # the default is the deterministic path
    for a, b in zip(g0, g1):
        assert torch.equal(a, b)
    g3 = spion.attn_bwd(q, k, v, o, do, lse, bp, fused=True)
    assert torch.equal(g3[2], g1[2])
    for a, b in ((g3[0], g1[0]), (g3[1], g1[1])):
        err = (a.float() - b.float()).abs().max().item()
        assert err <= 1e-2 * b.float().abs().max().item(), err


@pytest.mark.parametrize("B", [32, 64])
def test_backward_repeatable_many_runs(B):
    """Regression for a release-before-read race (round 1): the dQ pass's softmax warps read the O / dO
    tiles from shared memory for D = rowsum(dO * O) and then released the O buffer; the mbarrier arrive
    was issued behind still-outstanding LDS, so the next item's O TMA could overwrite the first rows
    being read (a few rows of D, dQ and dK wrong, ~3 % of runs).  150 backward passes must agree bit for
    bit (D in the workspace included)."""
    spion = _spion()
    L, bh, d = 2048, 32, 64
    A = synth.lra_scores(L, B, seed=4)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=75.0, sync=True)
    q, k, v, do = (x.to(DEV) for x in synth.qkvdo(bh, L, d, seed=2, dtype=torch.bfloat16))
    ws = spion.attn_workspace(bh, L, d, torch.bfloat16, DEV)
    o, lse = spion.attn_fwd(q, k, v, bp)
    ref = [x.clone() for x in spion.attn_bwd(q, k, v, o, do, lse, bp, workspace=ws)]
    D_ref = ws[256:256 + bh * L * 4].clone()
    for rep in range(150):
        g = spion.attn_bwd(q, k, v, o, do, lse, bp, workspace=ws)
        assert torch.equal(ws[256:256 + bh * L * 4], D_ref), rep
        for a, b in zip(g, ref):
            assert torch.equal(a, b), rep


@pytest.mark.parametrize("bh,L", [(6, 256), (16, 1024), (3, 2048), (64, 1024), (40, 512)])  # last two: (batch, head)-split tiles
def test_score_mean_matches_oracle(bh, L):
    """NEXT-1: the dense-phase score matrix A^s (mean over (batch, head) of softmax(scale Q K^T))
    and its squared Frobenius norm against the fp64 oracle; rows of A^s sum to 1."""
    spion = _spion()
    d = 64
    q, k, _, _ = synth.qkvdo(bh, L, d, seed=L + bh, dtype=torch.bfloat16)
    A, ss = spion.score_mean(q.to(DEV), k.to(DEV))
    A = A.cpu().numpy().astype(np.float64)
    ref, ss_ref = oracle.score_mean(q.double().numpy(), k.double().numpy(), 1 / math.sqrt(d))
    err = np.abs(A - ref).max()
    assert err <= 1e-5 * np.abs(ref).max() + 1e-8, err  # measured ~7e-7 relative (fp32 S, ex2.approx)
    assert np.abs(A.sum(1) - 1).max() < 1e-5
    assert abs(ss - ss_ref) <= 1e-5 * ss_ref


@pytest.mark.parametrize("ss,alpha", [((9.0, 6.25, 4.84), 0.25), ((9.0, 6.25, 4.84), 0.15), ((1.0, 1.0, 1.0), 0.0),
                                      ((2.5e3, 2.4e3, 2.31e3), 0.05), ((0.5, 0.75, 0.2), 0.3)])
def test_transition_matches_oracle(ss, alpha):
    """spion_transition (Alg. 2 / Eq. 2 on the device, fp64) equals the oracle's test bit for bit,
    distances included; also chained after score_mean's device sums of squares."""
    spion = _spion()
    sw, dist = spion.transition(torch.tensor(ss, dtype=torch.float64, device=DEV), alpha)
    ok, d1, d2 = oracle.transition(*ss, alpha)
    assert sw == ok
    assert dist.cpu().tolist() == [d1, d2]


def test_transition_after_score_mean():
    spion = _spion()
    L, bh, d = 512, 4, 64
    ss = torch.zeros(3, dtype=torch.float64, device=DEV)
    refs = []
    for i in range(3):
        q, k, _, _ = synth.qkvdo(bh, L, d, seed=100 + i, dtype=torch.bfloat16)
        spion.score_mean(q.to(DEV), k.to(DEV), sumsq=ss[i:i + 1])
        refs.append(oracle.score_mean(q.double().numpy(), k.double().numpy(), 1 / math.sqrt(d))[1])
    for alpha in (1e-6, 1e-3, 1.0):
        sw, dist = spion.transition(ss, alpha)
        ok, d1, d2 = oracle.transition(*refs, alpha)
        got = dist.cpu().numpy()
        assert abs(got[0] - d1) <= 1e-5 * max(1.0, abs(d1)) and abs(got[1] - d2) <= 1e-5 * max(1.0, abs(d2))
        if abs(abs(d1 - d2) - alpha) > 1e-4:  # far from the decision boundary: same decision
            assert sw == ok


def test_concurrent_streams_share_one_pattern():
    """Two fwd+bwd launches sharing ONE pattern on two streams at once (each with its own
    workspace: the scheduler counters live there) equal the sequential results bit for bit."""
    spion = _spion()
    L, B, bh, d = 2048, 64, 32, 64
    A = synth.lra_scores(L, B, seed=4)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=75.0, sync=True)
    sets = [tuple(x.to(DEV) for x in synth.qkvdo(bh, L, d, seed=s, dtype=torch.bfloat16)) for s in (1, 2)]
    ref = []
    for q, k, v, do in sets:
        o, lse = spion.attn_fwd(q, k, v, bp)
        ref.append((o, lse) + spion.attn_bwd(q, k, v, o, do, lse, bp))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in sets]
    wss = [spion.attn_workspace(bh, L, d, torch.bfloat16, DEV) for _ in sets]
    got = [None, None]
    for rep in range(3):
        for i, ((q, k, v, do), st) in enumerate(zip(sets, streams)):
            with torch.cuda.stream(st):
                o, lse = spion.attn_fwd(q, k, v, bp, workspace=wss[i])
                got[i] = (o, lse) + spion.attn_bwd(q, k, v, o, do, lse, bp, workspace=wss[i])
        torch.cuda.synchronize()
        for g, r in zip(got, ref):
            for name, a, b in zip(("o", "lse", "dq", "dk", "dv"), g, r):
                if name == "dq":  # fused backward: fp32 L2 reduce-adds in scheduling order
                    assert (a.float() - b.float()).abs().max() <= 1e-2 * b.float().abs().max(), name
                else:
                    assert torch.equal(a, b), name


def test_autograd_strided_layout():
    """spion.attention() through torch.autograd with the strided [L][heads][d] layout (dO arrives
    contiguous in [heads][L][d] order and is materialised in q's layout) against the oracle."""
    spion = _spion()
    L, B, d, H = 512, 64, 64, 3
    fl = synth.syn_mask(L // B, 0.3, seed=8)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(H, L, d, seed=91, dtype=torch.bfloat16)
    to_strided = lambda x: x.to(DEV).permute(1, 0, 2).contiguous().permute(1, 0, 2)
    qd, kd, vd = (to_strided(x).requires_grad_(True) for x in (q, k, v))
    o = spion.attention(qd, kd, vd, bp, "paper", 0.125)
    o.backward(do.to(DEV))
    _, lse = spion.attn_fwd(qd.detach(), kd.detach(), vd.detach(), bp, "paper", 0.125)
    outs = [x.float().cpu().numpy() for x in (o.detach(), lse, qd.grad, kd.grad, vd.grad)]
    _compare(outs, q, k, v, do, fl, B, "paper", 0.125, range(H), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


@pytest.mark.parametrize("B", [32, 64])
def test_tensor_core_path_is_taken(B):
    """bf16, d = 64, B in {32, 64}: spion_attn_path reports tcgen05 and the tensor-core launch
    counter advances by the kernels of one fwd + bwd."""
    spion = _spion()
    L = 1024
    fl = synth.syn_mask(L // B, 0.2, seed=3)
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q = torch.randn((4, L, 64), device=DEV).to(torch.bfloat16)
    assert spion.attn_path(q, bp) == "tcgen05"
    c0 = spion.tc_launch_count()
    o, lse = spion.attn_fwd(q, q, q, bp)
    c1 = spion.tc_launch_count()
    spion.attn_bwd(q, q, q, o, q, lse, bp)
    c2 = spion.tc_launch_count()
    assert c1 - c0 == 1 and c2 - c1 >= 1


@pytest.mark.parametrize("cfg", ["image", "listops", "text", "retrieval"])
def test_full_size_all_slices_masked(cfg):
    """The MASKED softmax (rows of P sum to 1, reading Q1) at full BASELINE sizes, every slice."""
    spion = _spion()
    c = FULL[cfg]
    L, B, bh, d = c["L"], c["B"], c["bh"], 64
    A = synth.lra_scores(L, B, seed=2)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=c["alpha"], sync=True)
    fl, _, _ = oracle.pattern(A.numpy(), B, 31, c["alpha"])
    q, k, v, do = synth.qkvdo(bh, L, d, seed=4048, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, "masked", 1 / math.sqrt(d))
    _compare(outs, q, k, v, do, fl, B, "masked", 1 / math.sqrt(d), range(bh), 2e-2, norm_tol=1e-2,
             lse_tol=1e-3)


# ---------------------------------------------------------------- small launches (one rank's share)
@pytest.mark.parametrize("cfg,bh", [("text", 16), ("image", 32), ("listops", 8)])
def test_small_launch_all_slices(cfg, bh):
    """One rank's share of a strong-scaled job (few (batch, head) per launch, so the heavy tiles — a
    vertical stripe's ~n entries — are a large part of each CTA's work): every slice against the oracle."""
    spion = _spion()
    c = FULL[cfg]
    L, B, d = c["L"], c["B"], 64
    A = synth.lra_scores(L, B, seed=1)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=c["alpha"], sync=True)
    fl, _, _ = oracle.pattern(A.numpy(), B, 31, c["alpha"])
    q, k, v, do = synth.qkvdo(bh, L, d, seed=77, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, "paper", 1 / math.sqrt(d))
    _compare(outs, q, k, v, do, fl, B, "paper", 1 / math.sqrt(d), range(bh), 2e-2, norm_tol=1e-2, lse_tol=1e-3)


def test_small_launch_matches_large_launch():
    """The same (batch, head) slices in a launch of 16 and inside one of 64: the persistent kernels'
    results do not depend on which CTA takes an item or on the launch's size — bit for bit."""
    spion = _spion()
    L, B, d = 4096, 64, 64
    A = synth.lra_scores(L, B, seed=1001)
    bp = spion.pattern(A.to(DEV), B, filter=31, alpha=55.0, sync=True)
    q, k, v, do = (x.to(DEV) for x in synth.qkvdo(64, L, d, seed=31, dtype=torch.bfloat16))
    o, lse = spion.attn_fwd(q, k, v, bp)
    big = spion.attn_bwd(q, k, v, o, do, lse, bp)
    o16, lse16 = spion.attn_fwd(q[:16], k[:16], v[:16], bp)
    small = spion.attn_bwd(q[:16], k[:16], v[:16], o16, do[:16], lse16, bp)
    assert torch.equal(o16, o[:16]) and torch.equal(lse16, lse[:16])
    for a, b in zip(small, big):
        assert torch.equal(a, b[:16])


@pytest.mark.parametrize("mode", ["paper", "masked"])
def test_single_column_mask(mode):
    """A caller mask whose only blocks are three in one block column (no diagonal): one heavy column
    tile, every other tile and most rows empty."""
    spion = _spion()
    L, B, d, bh = 1024, 64, 64, 4
    n = L // B
    fl = np.zeros((n, n), dtype=np.uint8)
    fl[[0, 5, 9], 3] = 1
    bp = spion.bsr_from_mask(torch.from_numpy(fl).to(DEV), L, B)
    q, k, v, do = synth.qkvdo(bh, L, d, seed=13, dtype=torch.bfloat16)
    outs = _run(q, k, v, do, bp, mode, 1 / math.sqrt(d))
    _compare(outs, q, k, v, do, fl, B, mode, 1 / math.sqrt(d), range(bh), 2e-2, norm_tol=1e-2)
