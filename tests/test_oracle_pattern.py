"""Pins for the pattern half of the oracle (Alg. 3/4, Eq. 3/4).

Every check here compares the oracle with something other than itself: a
worked example (tests/golden, cited), a library routine (torch conv2d /
avg_pool2d, numpy.quantile), a closed form, brute force on tiny inputs or an
invariant the paper states.
"""
import itertools
import json
import os
import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2309_12578_b200 import accounting
from synth import syn_scores

sys.setrecursionlimit(100000)


def _load(golden_dir, name):
    with open(os.path.join(golden_dir, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ P1
def test_p1_paper_op_counts(golden_dir):
    g = _load(golden_dir, "op_counts_p779.json")
    assert accounting.paper_dense_ops(g["L"], g["D"]) == g["dense_ops"]
    assert accounting.paper_sparse_ops(g["L"], g["D"], g["C"]) == g["sparse_ops"]
    assert g["C"] == int(0.1 * g["L"] ** 2)


# ------------------------------------------------------------- quantise
def test_quantize_exact_values():
    A = np.array([0.0, 1.0, 0.5, 2.0 ** -33, 3 * 2.0 ** -33, 0.25 + 2.0 ** -25], np.float32)
    q = oracle.quantize(A)
    # round half to even: 0.5 -> 0, 1.5 -> 2
    assert list(q) == [0, 2 ** 32, 2 ** 31, 0, 2, 2 ** 30 + 128]


@pytest.mark.parametrize("bad", [-1e-7, 1.0000001, float("nan"), float("inf")])
def test_quantize_rejects_out_of_range(bad):
    with pytest.raises(oracle.OracleError):
        oracle.quantize(np.array([0.5, bad], np.float32))


# ------------------------------------------------------------- P3: conv
def test_p3_diag_conv_worked_example(golden_dir):
    g = _load(golden_dir, "diag_conv_spec.json")
    q = oracle.quantize(np.array(g["A"], np.float32))
    conv = oracle.diag_conv(q, g["F"])
    assert (conv == np.array(g["conv_units"], np.int64) * 2 ** 32).all()


@pytest.mark.parametrize("L,F", [(8, 1), (8, 3), (16, 5), (24, 31), (32, 7), (64, 31)])
def test_diag_conv_matches_torch_conv2d(L, F):
    """Eq. 3 with a diagonal filter of ones == cross-correlation with eye(F), padding h."""
    rng = np.random.default_rng(L * 100 + F)
    q = rng.integers(0, 2 ** 32 + 1, size=(L, L), dtype=np.int64)
    conv = oracle.diag_conv(q, F)
    h = (F - 1) // 2
    ref = torch.nn.functional.conv2d(
        torch.from_numpy(q.astype(np.float64))[None, None],
        torch.eye(F, dtype=torch.float64)[None, None],
        padding=h,
    )[0, 0].numpy()
    assert (conv == ref.astype(np.int64)).all()  # exact: sums < 2^53


@pytest.mark.parametrize("F", [2, 0, -3])
def test_diag_conv_rejects_even_filter(F):
    with pytest.raises(oracle.OracleError):
        oracle.diag_conv(np.zeros((4, 4), np.int64), F)


# ------------------------------------------------------------- P4: pool
def test_avg_pool_worked_example(golden_dir):
    g = _load(golden_dir, "avg_pool_spec.json")
    pool = oracle.pool_sum(np.array(g["conv"], np.int64), g["B"])
    assert (pool == np.array(g["pool_sum"])).all()


@pytest.mark.parametrize("L,B", [(8, 2), (16, 4), (64, 8), (96, 32), (32, 32), (12, 3)])
def test_pool_matches_torch_avg_pool2d(L, B):
    rng = np.random.default_rng(L + B)
    c = rng.integers(0, 2 ** 37, size=(L, L), dtype=np.int64)
    pool = oracle.pool_sum(c, B)
    ref = torch.nn.functional.avg_pool2d(torch.from_numpy(c.astype(np.float64))[None, None], B)[0, 0]
    ref = (ref * (B * B)).numpy()
    # mean * B^2 is exact whenever the block sum is a multiple-free integer < 2^53 and B^2 is a
    # power of two; compare with a 1-ulp-safe integer rounding otherwise
    assert (pool == np.rint(ref).astype(np.int64)).all()


def test_pool_rejects_ragged():
    with pytest.raises(oracle.OracleError):
        oracle.pool_sum(np.zeros((10, 10), np.int64), 4)


def test_p4_F1_is_plain_average_pooling():
    """SPION-F (no conv) == F=1: pool_out is plain avg_pool2d of the quantised scores."""
    A = syn_scores(64, 8, heads=2, seed=5).numpy()
    q = oracle.quantize(A)
    pool = oracle.pool_sum(oracle.diag_conv(q, 1), 8)
    ref = torch.nn.functional.avg_pool2d(torch.from_numpy(q.astype(np.float64))[None, None], 8)[0, 0] * 64
    assert (pool == ref.numpy().astype(np.int64)).all()


def test_conv_pool_closed_form_weights():
    """pool(I,J) = sum_{x,y} q(x,y) w, w = |[max(x-IB-B+1, y-JB-B+1, -h), min(x-IB, y-JB, h)]|
    (a different derivation of Eq. 3 followed by Eq. 4), brute force on small inputs."""
    rng = np.random.default_rng(3)
    for (L, B, F) in [(12, 4, 3), (16, 4, 9), (16, 8, 31), (20, 5, 5)]:
        q = rng.integers(0, 1000, size=(L, L), dtype=np.int64)
        pool = oracle.pool_sum(oracle.diag_conv(q, F), B)
        h = (F - 1) // 2
        n = L // B
        ref = np.zeros((n, n), np.int64)
        for I in range(n):
            for J in range(n):
                s = 0
                for x in range(L):
                    for y in range(L):
                        lo = max(x - I * B - B + 1, y - J * B - B + 1, -h)
                        hi = min(x - I * B, y - J * B, h)
                        if hi >= lo:
                            s += int(q[x, y]) * (hi - lo + 1)
                ref[I, J] = s
        assert (pool == ref).all(), (L, B, F)


# -------------------------------------------------------- P5: threshold
@pytest.mark.parametrize("N,alpha,seed", [(64, 75.0, 1), (1024, 96.0, 2), (4096, 99.0, 3), (1024, 98.0, 4),
                                          (4096, 75.0, 5), (16, 50.0, 6), (100, 33.3, 7)])
def test_p5_linear_threshold_matches_numpy_quantile(N, alpha, seed):
    rng = np.random.default_rng(seed)
    v = rng.integers(0, 2 ** 50, size=N, dtype=np.int64)
    v[: N // 4] = v[N // 2]  # heavy ties
    rng.shuffle(v)
    gt, t = oracle.threshold_gt(v, 8, alpha, "linear")
    ref_t = np.quantile(v.astype(np.float64), alpha / 100.0)
    assert (gt.astype(bool) == (v > ref_t)).all()
    assert abs(t - ref_t) <= 1e-6 * max(1.0, abs(ref_t))


def test_p5_nearest_rank_examples(golden_dir):
    g = _load(golden_dir, "quantile_nearest_spec.json")
    for case in g["cases"]:
        vals = list(range(1, 101)) if case["values"] == "1..100" else case["values"]
        v = np.array(vals, np.int64)
        gt, t = oracle.threshold_gt(v, 1, case["alpha"], "nearest")
        assert t == case["t"]
        assert (gt.astype(bool) == (v > case["t"])).all()


def test_absolute_threshold_units():
    B = 4
    v = np.array([0, 15 * 2 ** 32, 16 * 2 ** 32, 17 * 2 ** 32], np.int64)  # means 0, 15/16, 1, 17/16
    gt, _ = oracle.threshold_gt(v, B, 1.0, "absolute")  # t = mean 1.0 -> sum 16 * 2^32
    assert list(gt) == [0, 0, 0, 1]


# ------------------------------------------------------ P2/P6 flood fill
def _literal_alg4(pool, t, order=(0, 1, 2)):
    """Alg. 4 exactly as printed, no pruning; Alg. 3 seeds and diagonal."""
    n = len(pool)
    fl = [[0] * n for _ in range(n)]
    calls = [0]

    def ff(r, c):
        calls[0] += 1
        if r + 1 == n or c + 1 == n:
            return
        nb = [(r + 1, c), (r, c + 1), (r + 1, c + 1)]  # below, right, diagonal (paper order)
        m = max(pool[a][b] for a, b in nb)
        for k in order:
            a, b = nb[k]
            if pool[a][b] == m and fl[a][b] == 0:
                if pool[a][b] > t:
                    fl[a][b] = 1
                ff(a, b)

    for i in range(n):
        ff(0, i)
    for j in range(n):
        ff(j, 0)
    for k in range(n):
        fl[k][k] = 1
    return np.array(fl, np.uint8), calls[0]


def _oracle_ff(pool, t):
    pool = np.array(pool, np.int64)
    gt = (pool > t).astype(np.uint8)
    return oracle.flood_fill(pool, gt)


def test_p2_flood_fill_worked_examples(golden_dir):
    g = _load(golden_dir, "flood_fill_spec.json")
    for case in g["cases"]:
        fl = _oracle_ff(case["pool"], case["t"])
        assert (fl == np.array(case["fl_out"], np.uint8)).all(), case
        lit, _ = _literal_alg4(case["pool"], case["t"])
        assert (lit == fl).all()


def test_p6_exhaustive_3x3_literal_recursion():
    """All 3^9 grids over {1,5,9} x t in {0,1,5,9}: oracle == literal Alg. 4 (paper visit order),
    and a second visit order gives the same mask (order independence, reading Q14)."""
    vals = (1, 5, 9)
    mismatches = 0
    for cells in itertools.product(vals, repeat=9):
        pool = [list(cells[0:3]), list(cells[3:6]), list(cells[6:9])]
        for t in (0, 1, 5, 9):
            fl = _oracle_ff(pool, t)
            lit, _ = _literal_alg4(pool, t)
            if not (lit == fl).all():
                mismatches += 1
        lit2, _ = _literal_alg4(pool, 5, order=(1, 0, 2))
        if not (lit2 == _oracle_ff(pool, 5)).all():
            mismatches += 1
    assert mismatches == 0


@pytest.mark.parametrize("n", [4, 5, 6])
def test_p6_random_grids_literal_recursion(n):
    rng = np.random.default_rng(n)
    for trial in range(60):
        pool = rng.integers(0, 4, size=(n, n)).tolist()  # many ties
        t = int(rng.integers(0, 4))
        lit, _ = _literal_alg4(pool, t, order=tuple(rng.permutation(3)))
        assert (lit == _oracle_ff(pool, t)).all(), (pool, t)


def test_flood_fill_threshold_above_max_gives_diagonal():
    rng = np.random.default_rng(0)
    pool = rng.integers(0, 100, size=(9, 9))
    fl = _oracle_ff(pool, 1000)
    assert (fl == np.eye(9, dtype=np.uint8)).all()


# ----------------------------------------------------------- BSR / CSC
def test_mask_to_bsr_worked_example(golden_dir):
    g = _load(golden_dir, "mask_to_csr_spec.json")
    bsr = oracle.mask_to_bsr(np.array(g["mask"], np.uint8))
    for k in ("brow_ptr", "bcol_idx", "bcol_ptr", "brow_idx"):
        assert list(bsr[k]) == g[k], k


def test_mask_to_bsr_random_vs_numpy():
    rng = np.random.default_rng(9)
    for n in (1, 3, 8, 33):
        m = (rng.random((n, n)) < 0.3).astype(np.uint8)
        bsr = oracle.mask_to_bsr(m)
        r, c = np.nonzero(m)
        assert list(bsr["bcol_idx"]) == list(c)
        assert list(bsr["brow_ptr"]) == [0] + list(np.cumsum(m.sum(1)))
        cc, rr = np.nonzero(m.T)
        assert list(bsr["brow_idx"]) == list(rr)
        assert list(bsr["bcol_ptr"]) == [0] + list(np.cumsum(m.sum(0)))
        assert bsr["nnzb"] == int(m.sum())


# ------------------------------------------------------- P7 invariants
def test_p7_pattern_invariants():
    L, B = 128, 16
    A = syn_scores(L, B, heads=2, seed=21).numpy()
    prev = None
    for alpha in (50.0, 75.0, 90.0, 96.0, 99.0):
        fl, pool, t = oracle.pattern(A, B, 31, alpha)
        n = L // B
        assert (np.diag(fl) == 1).all()
        if prev is not None:  # monotone non-increasing in alpha (edges do not depend on t)
            assert (fl <= prev).all()
        prev = fl
        # composition equals the unfused steps
        q = oracle.quantize(A)
        pool2 = oracle.pool_sum(oracle.diag_conv(q, 31), B)
        assert (pool2 == pool).all()
        gt, _ = oracle.threshold_gt(pool, B, alpha)
        assert (oracle.flood_fill(pool, gt) == fl).all()


def test_p7_band_gives_diagonal_blocks_and_stripe_gives_stripe():
    L, B = 96, 32
    # identity-dominant band
    A = np.full((L, L), 0.001, np.float32)
    for i in range(L):
        for j in range(max(0, i - 2), min(L, i + 3)):
            A[i, j] = 0.2
    fl, _, _ = oracle.pattern(A, B, 31, 96.0)
    assert (np.diag(fl) == 1).all()
    # dominant column block -> vertical stripe through that block column plus the diagonal
    # (strength decreasing down the column so each step's max-neighbour is the cell below;
    #  a flat column would be entered diagonally from (0,0) and skip (0,1), as Alg. 4 dictates)
    A = np.full((L, L), 0.001, np.float32)
    A[:, 32:64] = (0.05 - 1e-4 * np.arange(L, dtype=np.float32))[:, None]
    fl, _, _ = oracle.pattern(A, B, 3, 50.0)
    assert (fl[:, 1] == 1).all(), fl
    assert (np.diag(fl) == 1).all()


@pytest.mark.parametrize("L,B,F,alpha", [(128, 16, 31, 96.0), (256, 32, 31, 96.0), (256, 64, 31, 98.0),
                                         (256, 32, 3, 99.0)])
def test_p7_uniform_scores_give_block_diagonal(L, B, F, alpha):
    A = np.full((L, L), 1.0 / L, np.float32)
    fl, _, _ = oracle.pattern(A, B, F, alpha)
    assert (fl == np.eye(L // B, dtype=np.uint8)).all()


def test_pattern_rejects_bad_params():
    A = np.zeros((16, 16), np.float32)
    with pytest.raises(oracle.OracleError):
        oracle.pattern(A, 4, 4, 90.0)   # even filter
    with pytest.raises(oracle.OracleError):
        oracle.pattern(A, 4, 3, 100.0)  # alpha out of (0,100)
    A[0, 0] = 2.0
    with pytest.raises(oracle.OracleError):
        oracle.pattern(A, 4, 3, 90.0)   # score outside [0,1]


# ------------------------------------------------------ NEXT-2 pattern variants
def _literal_variant(pool, t, prose=False, all_seeds=False, order=(0, 1, 2)):
    """Alg. 4 written out again with the two readings of SURVEY Q11/Q12, no pruning:
    prose (R2): the recursion continues only from a critical (> t) neighbour;
    all_seeds: every element of pool_out is a seed point."""
    n = len(pool)
    fl = [[0] * n for _ in range(n)]

    def ff(r, c):
        if r + 1 == n or c + 1 == n:
            return
        nb = [(r + 1, c), (r, c + 1), (r + 1, c + 1)]
        m = max(pool[a][b] for a, b in nb)
        for k in order:
            a, b = nb[k]
            if pool[a][b] == m and fl[a][b] == 0:
                if pool[a][b] > t:
                    fl[a][b] = 1
                    ff(a, b)
                elif not prose:
                    ff(a, b)

    seeds = [(r, c) for r in range(n) for c in range(n)] if all_seeds else \
        [(0, i) for i in range(n)] + [(j, 0) for j in range(n)]
    for r, c in seeds:
        ff(r, c)
    for k in range(n):
        fl[k][k] = 1
    return np.array(fl, np.uint8)


def _var(pool, t, variant):
    pool = np.array(pool, np.int64)
    return oracle.flood_fill(pool, (pool > t).astype(np.uint8), variant)


def test_spion_c_is_threshold_plus_diagonal():
    """SPION-C: the top alpha% of pool_out, no flood fill (+ forced diagonal, Q23);
    end to end equals x > numpy.quantile(pool, alpha/100) on the oracle's own pool sums."""
    rng = np.random.default_rng(4)
    A = syn_scores(256, 16, heads=2, seed=8).numpy()
    for alpha in (50.0, 75.0, 96.0):
        fl, pool, _ = oracle.pattern(A, 16, 31, alpha, variant="noflood")
        want = (pool > np.quantile(pool.astype(np.float64), alpha / 100.0)) | np.eye(pool.shape[0], dtype=bool)
        assert (fl.astype(bool) == want).all()
    pool = rng.integers(0, 9, size=(7, 7))
    assert (_var(pool, 4, "noflood").astype(bool) == ((pool > 4) | np.eye(7, dtype=bool))).all()


def test_variants_exhaustive_3x3_literal_recursion():
    """All 3^9 grids over {1,5,9} x t in {1,5}: prose recursion, all-cells seeding and both
    together == the unpruned literal recursions above (two visit orders)."""
    vals = (1, 5, 9)
    for cells in itertools.product(vals, repeat=9):
        pool = [list(cells[0:3]), list(cells[3:6]), list(cells[6:9])]
        for t in (1, 5):
            for prose, seeds, v in ((True, False, "prose"), (False, True, "all_seeds"), (True, True, "prose+all_seeds")):
                want = _literal_variant(pool, t, prose, seeds)
                assert (want == _literal_variant(pool, t, prose, seeds, order=(2, 1, 0))).all()
                assert (_var(pool, t, v) == want).all(), (pool, t, v)


@pytest.mark.parametrize("n", [5, 8, 16])
def test_variant_invariants_random(n):
    """R2 marks a subset of Alg. 4; all-cells seeding a superset; with every
    cell a seed, R1 and R2 coincide and equal the closed form: cells entered by a
    max-neighbour edge from any cell, above t, plus the diagonal."""
    rng = np.random.default_rng(n)
    for trial in range(40):
        pool = rng.integers(0, 5, size=(n, n))
        t = int(rng.integers(0, 5))
        base, prose, alls = _var(pool, t, 0), _var(pool, t, "prose"), _var(pool, t, "all_seeds")
        assert (prose <= base).all() and (base <= alls).all()
        assert (alls == _var(pool, t, "prose+all_seeds")).all()
        entered = np.zeros((n, n), bool)
        for r in range(n - 1):
            for c in range(n - 1):
                nb = [(r + 1, c), (r, c + 1), (r + 1, c + 1)]
                m = max(pool[a, b] for a, b in nb)
                for a, b in nb:
                    entered[a, b] |= pool[a, b] == m
        want = (entered & (pool > t)) | np.eye(n, dtype=bool)
        assert (alls.astype(bool) == want).all()
        if n <= 8:
            assert (prose == _literal_variant(pool.tolist(), t, prose=True)).all()


def test_variants_worked_example(golden_dir):
    """Hand-worked example separating the literal recursion from the prose reading."""
    g = _load(golden_dir, "flood_fill_variants.json")
    for case in g["cases"]:
        for v, want in case["fl"].items():
            assert (_var(case["pool"], case["t"], v) == np.array(want, np.uint8)).all(), v


@pytest.mark.parametrize("L,B,F,cuts", [(64, 8, 31, [24]), (96, 4, 63, [32, 36, 80]), (128, 16, 3, [0, 64, 128]),
                                        (256, 32, 31, [96, 160])])
def test_pool_is_sum_over_row_partition(L, B, F, cuts):
    """Eq. 3-4 are sums over the source rows of A^s: the pool of the whole matrix is the
    sum of the pools of the matrices that keep one slab of rows each (zeros elsewhere) — including
    slabs whose diagonal-filter taps (h > B for F=63, B=4) reach pool rows of a neighbouring slab.
    This is what the multi-device pattern path (spion_pattern_pool + a sum + spion_pattern_finalize)
    relies on; checked here against a direct pool of the unsplit matrix."""
    A = syn_scores(L, B, heads=2, seed=L + F)
    full = oracle.pool_sum(oracle.diag_conv(oracle.quantize(A.numpy()), F), B)
    edges = [0] + [c for c in cuts] + [L]
    acc = np.zeros_like(full)
    for r0, r1 in zip(edges[:-1], edges[1:]):
        As = np.zeros_like(A.numpy())
        As[r0:r1] = A.numpy()[r0:r1]
        acc += oracle.pool_sum(oracle.diag_conv(oracle.quantize(As), F), B)
    assert (acc == full).all()
    # and the pattern from the summed pool is the pattern of the matrix
    gt, _ = oracle.threshold_gt(acc, B, 75.0)
    fl = oracle.flood_fill(acc, gt)
    fl_ref, _, _ = oracle.pattern(A.numpy(), B, F, 75.0)
    assert (fl == fl_ref).all()
