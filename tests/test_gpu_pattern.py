"""GPU parity of pattern generation (K1 stencil + K2 finalize) against the oracle.

Bar: bit-exact block mask, block-CSR, block-CSC and nnzb (integer work).
Sizes: the tiny config, every LRA shape of BASELINE.json at the paper's alpha
and at alpha=75, plus ragged / degenerate cases.
"""
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


def _check(bp, fl_ref):
    n = fl_ref.shape[0]
    ref = oracle.mask_to_bsr(fl_ref)
    assert (bp.mask.view(n, n).cpu().numpy() == fl_ref).all()
    assert bp.nnzb == ref["nnzb"]
    rp, ci = bp.csr()
    cp, ri = bp.csc()
    assert (rp.cpu().numpy() == ref["brow_ptr"]).all()
    assert (ci.cpu().numpy() == ref["bcol_idx"]).all()
    assert (cp.cpu().numpy() == ref["bcol_ptr"]).all()
    assert (ri.cpu().numpy() == ref["brow_idx"]).all()


CASES = [
    # L, B, F, theta, kind
    (64, 8, 31, 0.1, "absolute"),        # tiny config, fixed threshold
    (64, 8, 31, 75.0, "linear"),
    (1024, 32, 31, 96.0, "linear"),      # LRA Image, paper alpha
    (1024, 32, 31, 75.0, "linear"),
    (2048, 64, 31, 98.0, "linear"),      # ListOps
    (2048, 64, 31, 75.0, "linear"),
    (4096, 64, 31, 99.0, "linear"),      # Text / Retrieval
    (4096, 64, 31, 75.0, "linear"),
    (4096, 32, 31, 90.0, "linear"),      # nblk = 128 (largest supported)
    (1024, 32, 31, 96.0, "nearest"),
    (256, 16, 1, 80.0, "linear"),        # SPION-F (no conv) == F=1
    (256, 16, 3, 50.0, "linear"),
    (192, 64, 31, 50.0, "linear"),       # nblk = 3
    (64, 64, 31, 50.0, "linear"),        # nblk = 1
    (96, 4, 63, 60.0, "linear"),         # h > B (targets span several pool rows)
    (1024, 32, 31, 0.05, "absolute"),
    (1024, 64, 601, 70.0, "linear"),     # wide filter: window > 636 columns (17-float4 lanes)
    (2048, 1024, 31, 50.0, "linear"),    # block wider than the small window
    (1280, 10, 31, 75.0, "linear"),      # B not a multiple of 4 (windows start mid-float4)
]


@pytest.mark.parametrize("L,B,F,theta,kind", CASES)
def test_pattern_bit_exact(L, B, F, theta, kind):
    spion = _spion()
    A = synth.syn_scores(L, B, heads=2, seed=L + B + F)
    bp = spion.pattern(A.to(DEV), B, filter=F, alpha=None if kind == "absolute" else theta,
                       t=theta if kind == "absolute" else None, kind=kind, sync=True)
    fl_ref, _, _ = oracle.pattern(A.numpy(), B, F, theta, kind)
    _check(bp, fl_ref)


@pytest.mark.parametrize("seed", range(6))
def test_pattern_random_scores_with_ties(seed):
    """Quantised values with heavy ties exercise the ==m edges and the order statistics."""
    spion = _spion()
    rng = np.random.default_rng(seed)
    L, B = 256, 16
    A = (rng.integers(0, 4, size=(L, L)) / 3.0).astype(np.float32)
    for alpha in (10.0, 50.0, 90.0, 99.0):
        bp = spion.pattern(torch.from_numpy(A).to(DEV), B, filter=7, alpha=alpha, sync=True)
        fl_ref, _, _ = oracle.pattern(A, B, 7, alpha)
        _check(bp, fl_ref)


def test_pattern_flags_bad_scores():
    spion = _spion()
    from paper_2309_12578_b200 import _native as N
    A = synth.syn_scores(128, 16, heads=1, seed=3)
    A[5, 7] = float("nan")
    with pytest.raises(N.SpionError) as e:
        spion.pattern(A.to(DEV), 16, filter=31, alpha=90.0, sync=True)
    assert e.value.status == 3


@pytest.mark.parametrize("n,density,seed", [(8, 0.3, 0), (32, 0.1, 1), (64, 0.1, 2), (128, 0.05, 3), (5, 0.5, 4)])
def test_bsr_from_mask_matches_oracle(n, density, seed):
    spion = _spion()
    m = synth.syn_mask(n, density, seed)
    rng = np.random.default_rng(seed)
    if n > 4:
        m[rng.integers(0, n)] = 0  # an empty row (user masks only)
    bp = spion.bsr_from_mask(torch.from_numpy(m).to(DEV), n * 32, 32)
    _check(bp, m)


def test_bsr_from_mask_rejects_non_binary():
    spion = _spion()
    from paper_2309_12578_b200 import _native as N
    m = np.eye(8, dtype=np.uint8)
    m[2, 3] = 2
    with pytest.raises(N.SpionError) as e:
        spion.bsr_from_mask(torch.from_numpy(m).to(DEV), 256, 32)
    assert e.value.status == 3


VARIANTS = ["noflood", "prose", "all_seeds", "prose+all_seeds"]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("L,B,F,theta", [(64, 8, 31, 75.0), (1024, 32, 31, 96.0), (1024, 32, 31, 60.0),
                                         (2048, 64, 31, 75.0), (4096, 64, 31, 99.0), (4096, 32, 31, 90.0),
                                         (192, 64, 31, 50.0), (96, 4, 63, 60.0)])
def test_pattern_variants_bit_exact(variant, L, B, F, theta):
    """NEXT-2 variants (SPION-C, prose recursion, all-cells seeding) bit-exact against the oracle,
    including the 64-/128-bit row paths (n <= 64 / n = 128)."""
    spion = _spion()
    A = synth.lra_scores(L, B, seed=L + F) if L >= 1024 else synth.syn_scores(L, B, heads=2, seed=L + F)
    bp = spion.pattern(A.to(DEV), B, filter=F, alpha=theta, sync=True, variant=variant)
    fl_ref, _, _ = oracle.pattern(A.numpy(), B, F, theta, "linear", variant=variant)
    _check(bp, fl_ref)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("variant", VARIANTS)
def test_pattern_variants_ties(seed, variant):
    spion = _spion()
    rng = np.random.default_rng(100 + seed)
    L, B = 256, 16
    A = (rng.integers(0, 4, size=(L, L)) / 3.0).astype(np.float32)
    for alpha in (10.0, 50.0, 90.0):
        bp = spion.pattern(torch.from_numpy(A).to(DEV), B, filter=7, alpha=alpha, sync=True, variant=variant)
        fl_ref, _, _ = oracle.pattern(A, B, 7, alpha, variant=variant)
        _check(bp, fl_ref)


# ---------------------------------------------------------------- multi-device pattern path
SPLIT_CASES = [
    # L, B, F, theta, row cuts (multiples of B; the multi-device bench uses n / world block rows each)
    (64, 8, 31, 75.0, [32]),
    (1024, 32, 31, 75.0, [256, 512, 768]),     # LRA Image over 4 devices
    (2048, 64, 31, 75.0, [1024]),
    (4096, 64, 31, 55.0, [512 * k for k in range(1, 8)]),  # Text over 8 devices
    (96, 4, 63, 60.0, [4, 48, 92]),            # h > B: taps reach pool rows of other slabs
    (1280, 10, 31, 75.0, [0, 640, 1280]),      # empty first and last slab, B not a multiple of 4
]


def _pool_of(bp, n):
    spion = _spion()
    return spion.pool_region(bp)[-n * n:].view(n, n)


@pytest.mark.parametrize("L,B,F,theta,cuts", SPLIT_CASES)
def test_pattern_pool_partition_sum_finalize(L, B, F, theta, cuts):
    """spion_pattern_pool on every slab of a row partition (one workspace each, as one device each),
    the pool regions summed (what an all-reduce does), spion_pattern_finalize: the same pattern as
    spion_pattern, bit for bit; each slab's partial pool equals the oracle pool of the matrix that
    keeps only that slab's rows."""
    spion = _spion()
    A = synth.syn_scores(L, B, heads=2, seed=L + B + F)
    Ad = A.to(DEV)
    n = L // B
    edges = [0] + cuts + [L]
    parts = []
    for r0, r1 in zip(edges[:-1], edges[1:]):
        bp = spion.pattern_pool(Ad[r0:r1], L, B, filter=F, row_begin=r0)
        As = np.zeros_like(A.numpy())
        As[r0:r1] = A.numpy()[r0:r1]
        ref = oracle.pool_sum(oracle.diag_conv(oracle.quantize(As), F), B)
        assert (_pool_of(bp, n).cpu().numpy() == ref).all(), (r0, r1)
        parts.append(bp)
    total = parts[0]
    region = spion.pool_region(total)
    for bp in parts[1:]:
        region += spion.pool_region(bp)
    spion.pattern_finalize(total, alpha=theta, sync=True)
    whole = spion.pattern(Ad, B, filter=F, alpha=theta, sync=True)
    fl_ref, _, _ = oracle.pattern(A.numpy(), B, F, theta)
    _check(total, fl_ref)
    assert torch.equal(total.flat, whole.flat)  # CSR, CSC, mask and the attention plan


def test_pattern_pool_bad_score_in_one_slab():
    spion = _spion()
    from paper_2309_12578_b200 import _native as N
    L, B = 256, 16
    A = synth.syn_scores(L, B, heads=1, seed=5)
    A[200, 3] = 1.5  # outside [0, 1], in the second slab
    Ad = A.to(DEV)
    a = spion.pattern_pool(Ad[:128], L, B, row_begin=0)
    b = spion.pattern_pool(Ad[128:], L, B, row_begin=128)
    spion.pool_region(a).add_(spion.pool_region(b))
    with pytest.raises(N.SpionError) as e:
        spion.pattern_finalize(a, alpha=90.0, sync=True)
    assert e.value.status == 3  # SPION_ERR_DATA


def test_pattern_pool_rejects_bad_ranges():
    spion = _spion()
    from paper_2309_12578_b200 import _native as N
    L, B = 256, 16
    A = synth.syn_scores(L, B, heads=1, seed=6).to(DEV)
    with pytest.raises(N.SpionError) as e:
        spion.pattern_pool(A[8:40], L, B, row_begin=8)  # not at a block boundary
    assert e.value.status == 1  # SPION_ERR_SHAPE
    with pytest.raises(N.SpionError):
        spion.pattern_pool(A[:64], L, B, row_begin=224)  # past L
