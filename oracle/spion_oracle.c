/*
 * spion_oracle.c — plain, slow, obviously-correct CPU oracle for SPION's
 * layer-wise block-sparse attention hot path (arXiv 2309.12578).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_2309_12578_b200/, libspion.so) never links, loads
 * or calls it, and shares no code, header, table or constant with it.
 *
 * Citations: "P:N" = line N of the paper text.  Readings of
 * ambiguous passages are the Q-numbers listed in DESIGN.md §3.
 *
 * Precision: the paper never states one.  Pattern arithmetic is exact
 * integer arithmetic on the fixed-point encoding q = rint(A * 2^32)
 * (reading Q8); attention arithmetic is IEEE fp64.
 *
 * Every function is single-threaded and re-entrant.
 *
 * Pin status (see tests/test_oracle_*.py and DESIGN.md §4):
 *   spion_oracle_quantize       pinned (exact-value tests)
 *   spion_oracle_diag_conv      pinned (worked example S:232; torch conv2d
 *                               with an identity F×F kernel)
 *   spion_oracle_pool_sum       pinned (torch avg_pool2d × B²)
 *   spion_oracle_threshold_gt   pinned (numpy.quantile, nearest-rank examples)
 *   spion_oracle_flood_fill     pinned (SPEC worked examples; exhaustive
 *                               literal-recursion Alg. 4 on 3x3 grids)
 *   ..._flood_fill_variant      pinned (SPION-C = definition; prose recursion
 *                               and all-cells seeding against unpruned
 *                               recursions written in the test, exhaustive
 *                               3x3 grids; all-seeds closed form; R2 within R1)
 *   spion_oracle_pattern        pinned (composition + invariants P7)
 *   spion_oracle_mask_to_bsr    pinned (S:125 worked example, invariants)
 *   spion_oracle_score_mean     pinned (torch softmax fp64, rows sum to 1, Frobenius
 *                               norm via numpy); _transition: Eq. 2 worked numbers
 *   spion_oracle_attn_fwd/bwd   pinned (SDPA fp64 on all-ones and boolean
 *                               masks, PAPER/MASKED closed form
 *                               worked example, finite differences)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SPION_ORACLE_OK 0
#define SPION_ORACLE_ERR_SHAPE 1
#define SPION_ORACLE_ERR_PARAM 2
#define SPION_ORACLE_ERR_DATA 3

/* threshold kinds (reading Q9) */
#define ORACLE_TH_QUANTILE_LINEAR 0
#define ORACLE_TH_QUANTILE_NEAREST 1
#define ORACLE_TH_ABSOLUTE 2

/* softmax modes (reading Q1) */
#define ORACLE_SOFTMAX_PAPER 0
#define ORACLE_SOFTMAX_MASKED 1

/* ------------------------------------------------------------------ */
/* a2: fixed-point quantisation q = rint(A * 2^32) (reading Q8).       */
/* A must be finite and in [0, 1] (A^s is a softmax probability) */
/* ------------------------------------------------------------------ */
int spion_oracle_quantize(const float *A, int64_t count, int64_t *q)
{
    for (int64_t k = 0; k < count; ++k) {
        double a = (double)A[k];
        if (!(a >= 0.0 && a <= 1.0)) return SPION_ORACLE_ERR_DATA; /* also NaN */
        q[k] = llrint(a * 4294967296.0); /* exact product; round half to even */
    }
    return SPION_ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* a3: Eq. 3 diagonal convolution, centred window and a    */
/* filter of ones on its main diagonal (reading Q5), zero padding so  */
/* the output keeps the L x L shape:                          */
/*     conv_out(i,j) = sum_{f=-h..h} A(i+f, j+f),   h = (F-1)/2        */
/* ------------------------------------------------------------------ */
int spion_oracle_diag_conv(const int64_t *q, int32_t L, int32_t F, int64_t *conv)
{
    if (L <= 0) return SPION_ORACLE_ERR_SHAPE;
    if (F < 1 || (F % 2) == 0) return SPION_ORACLE_ERR_PARAM;
    int32_t h = (F - 1) / 2;
    for (int32_t i = 0; i < L; ++i) {
        for (int32_t j = 0; j < L; ++j) {
            int64_t acc = 0;
            for (int32_t f = -h; f <= h; ++f) {
                int32_t x = i + f, y = j + f;
                if (x < 0 || y < 0 || x >= L || y >= L) continue; /* zero padding */
                acc += q[(int64_t)x * L + y];
            }
            conv[(int64_t)i * L + j] = acc;
        }
    }
    return SPION_ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* a4: Eq. 4 B x B average pooling, non-overlapping blocks */
/* with stride B (reading Q6).  The 1/B^2 factor is dropped: it is a   */
/* positive constant and every later use is a comparison (reading Q7). */
/*     pool(I,J) = sum_{p,q in [0,B)} conv_out(I*B+p, J*B+q)            */
/* ------------------------------------------------------------------ */
int spion_oracle_pool_sum(const int64_t *conv, int32_t L, int32_t B, int64_t *pool)
{
    if (L <= 0 || B <= 0 || (L % B) != 0) return SPION_ORACLE_ERR_SHAPE;
    int32_t n = L / B;
    for (int32_t I = 0; I < n; ++I) {
        for (int32_t J = 0; J < n; ++J) {
            int64_t acc = 0;
            for (int32_t p = 0; p < B; ++p)
                for (int32_t qq = 0; qq < B; ++qq)
                    acc += conv[(int64_t)(I * B + p) * L + (J * B + qq)];
            pool[(int64_t)I * n + J] = acc;
        }
    }
    return SPION_ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* a5: threshold t = alpha% quantile of pool_out, and the      */
/* predicate gt(x) := x > t used by Alg. 4 lines 5/9/13.   */
/*                                                                     */
/* LINEAR (reading Q9, numpy/torch default "linear" method): with v the */
/* ascending values and N = n^2,                                       */
/*     hpos = (N-1) * alpha / 100,  lo = floor(hpos),  frac = hpos - lo */
/*     t    = v[lo] + frac * (v[lo+1] - v[lo])                          */
/* evaluated in long double (v < 2^56 are exact; frac*gap is the only   */
/* rounded term and cannot cross an integer value of x).                */
/* NEAREST: t = v[ceil(alpha/100 * N) - 1].                */
/* ABSOLUTE: t given in pool-mean units, i.e. compared against          */
/*     t * B^2 * 2^32 (pool sums are B^2 * 2^32 times the mean).        */
/* Output: gt[k] = 1 iff pool[k] > t.                                   */
/* ------------------------------------------------------------------ */
static int cmp_i64(const void *a, const void *b)
{
    int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
    return (x > y) - (x < y);
}

int spion_oracle_threshold_gt(const int64_t *pool, int64_t N, int32_t B, double theta,
                              int32_t kind, uint8_t *gt, double *t_out)
{
    if (N <= 0) return SPION_ORACLE_ERR_SHAPE;
    long double t;
    if (kind == ORACLE_TH_ABSOLUTE) {
        t = (long double)((double)theta * (double)((int64_t)B * B) * 4294967296.0);
    } else {
        if (!(theta > 0.0 && theta < 100.0)) return SPION_ORACLE_ERR_PARAM;
        int64_t *v = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
        if (!v) return SPION_ORACLE_ERR_PARAM;
        memcpy(v, pool, sizeof(int64_t) * (size_t)N);
        qsort(v, (size_t)N, sizeof(int64_t), cmp_i64);
        if (kind == ORACLE_TH_QUANTILE_LINEAR) {
            double hpos = (double)(N - 1) * theta / 100.0;
            int64_t lo = (int64_t)floor(hpos);
            double frac = hpos - (double)lo;
            if (lo >= N - 1) { lo = N - 1; frac = 0.0; }
            t = (long double)v[lo];
            if (frac > 0.0) t += (long double)frac * (long double)(v[lo + 1] - v[lo]);
        } else if (kind == ORACLE_TH_QUANTILE_NEAREST) {
            int64_t k = (int64_t)ceil(theta / 100.0 * (double)N) - 1;
            if (k < 0) k = 0;
            if (k > N - 1) k = N - 1;
            t = (long double)v[k];
        } else {
            free(v);
            return SPION_ORACLE_ERR_PARAM;
        }
        free(v);
    }
    for (int64_t k = 0; k < N; ++k) gt[k] = ((long double)pool[k] > t) ? 1 : 0;
    if (t_out) *t_out = (double)t;
    return SPION_ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* a6: Alg. 4 flood_fill, written in the paper's order and  */
/* notation.  `gt` carries the comparison "pool_out[.] > t".            */
/*                                                                     */
/* Literal Alg. 4 re-enters an unmarked (sub-threshold) neighbour every */
/* time it is reached, which is exponential on flat regions (reading    */
/* Q15).  `explored` prunes only such repeated re-entries: the subtree  */
/* below a cell depends on pool_out alone, and a cell skipped by the    */
/* fl_out guard has itself been entered, so the set of marked cells is  */
/* unchanged (tests/test_oracle_pattern.py checks this against the     */
/* unpruned recursion, exhaustively on 3x3 grids).                      */
/* ------------------------------------------------------------------ */
static void flood_fill(const int64_t *pool_out, int32_t n, int32_t r, int32_t c, uint8_t *fl_out,
                       const uint8_t *gt, uint8_t *explored)
{
    /* Alg. 4 l.1-2: stop at the last row / column */
    if (r + 1 == n || c + 1 == n) return;
    int64_t below = pool_out[(int64_t)(r + 1) * n + c];
    int64_t right = pool_out[(int64_t)r * n + (c + 1)];
    int64_t diag = pool_out[(int64_t)(r + 1) * n + (c + 1)];
    /* Alg. 4 l.3 */
    int64_t m = below;
    if (right > m) m = right;
    if (diag > m) m = diag;
    /* Alg. 4 l.4-7: below */
    int64_t k = (int64_t)(r + 1) * n + c;
    if (below == m && fl_out[k] == 0) {
        if (gt[k]) fl_out[k] = 1;
        if (!explored[k]) { explored[k] = 1; flood_fill(pool_out, n, r + 1, c, fl_out, gt, explored); }
    }
    /* Alg. 4 l.8-11: right */
    k = (int64_t)r * n + (c + 1);
    if (right == m && fl_out[k] == 0) {
        if (gt[k]) fl_out[k] = 1;
        if (!explored[k]) { explored[k] = 1; flood_fill(pool_out, n, r, c + 1, fl_out, gt, explored); }
    }
    /* Alg. 4 l.12-15: diagonally below */
    k = (int64_t)(r + 1) * n + (c + 1);
    if (diag == m && fl_out[k] == 0) {
        if (gt[k]) fl_out[k] = 1;
        if (!explored[k]) { explored[k] = 1; flood_fill(pool_out, n, r + 1, c + 1, fl_out, gt, explored); }
    }
}

/* The prose reading of the recursion (reading Q11 R2): "after
 * determining the critical element, the algorithm recursively compares the
 * elements to the right, below and diagonally below the critical element" —
 * recursion continues only from a neighbour that is marked (> t).  Each cell
 * is marked (and entered) at most once, so no pruning is needed. */
static void flood_fill_prose(const int64_t *pool_out, int32_t n, int32_t r, int32_t c, uint8_t *fl_out,
                             const uint8_t *gt)
{
    /* Alg. 4 l.1-2: stop at the last row / column */
    if (r + 1 == n || c + 1 == n) return;
    int64_t below = pool_out[(int64_t)(r + 1) * n + c];
    int64_t right = pool_out[(int64_t)r * n + (c + 1)];
    int64_t diag = pool_out[(int64_t)(r + 1) * n + (c + 1)];
    /* Alg. 4 l.3 */
    int64_t m = below;
    if (right > m) m = right;
    if (diag > m) m = diag;
    /* below, right, diagonally below: a max neighbour above t becomes critical and is recursed from */
    int64_t k = (int64_t)(r + 1) * n + c;
    if (below == m && fl_out[k] == 0 && gt[k]) { fl_out[k] = 1; flood_fill_prose(pool_out, n, r + 1, c, fl_out, gt); }
    k = (int64_t)r * n + (c + 1);
    if (right == m && fl_out[k] == 0 && gt[k]) { fl_out[k] = 1; flood_fill_prose(pool_out, n, r, c + 1, fl_out, gt); }
    k = (int64_t)(r + 1) * n + (c + 1);
    if (diag == m && fl_out[k] == 0 && gt[k]) { fl_out[k] = 1; flood_fill_prose(pool_out, n, r + 1, c + 1, fl_out, gt); }
}

/* Pattern variants (flag bits shared in meaning, not in
 * code, with the product's spion_pattern_variant):
 *   ORACLE_PAT_NOFLOOD   1: SPION-C: no flood fill, the top alpha%
 *                           of pool_out (the gt cells) plus the forced diagonal
 *                           (reading Q23)
 *   ORACLE_PAT_PROSE     2: recursion only from critical (> t) cells (R2)
 *   ORACLE_PAT_ALL_SEEDS 4: every element of pool_out a seed point */
#define ORACLE_PAT_NOFLOOD 1
#define ORACLE_PAT_PROSE 2
#define ORACLE_PAT_ALL_SEEDS 4

/* Alg. 3 lines 4-10: seeds (0,i) for all i, then (j,0) for
 * all j (reading Q12) — or every cell (ORACLE_PAT_ALL_SEEDS) — then the
 * forced diagonal.  Seeds are not marked themselves (reading Q21).
 * fl_out must hold n*n bytes. */
int spion_oracle_flood_fill_variant(const int64_t *pool_out, int32_t n, const uint8_t *gt, int32_t variant,
                                    uint8_t *fl_out)
{
    if (n <= 0) return SPION_ORACLE_ERR_SHAPE;
    if (variant & ~7) return SPION_ORACLE_ERR_PARAM;
    memset(fl_out, 0, (size_t)n * n);
    if (variant & ORACLE_PAT_NOFLOOD) {
        for (int64_t k = 0; k < (int64_t)n * n; ++k) fl_out[k] = gt[k] ? 1 : 0;
    } else if (variant & ORACLE_PAT_PROSE) {
        for (int32_t r = 0; r < n; ++r)
            for (int32_t c = 0; c < n; ++c)
                if ((variant & ORACLE_PAT_ALL_SEEDS) || r == 0 || c == 0) flood_fill_prose(pool_out, n, r, c, fl_out, gt);
    } else {
        uint8_t *explored = (uint8_t *)calloc((size_t)n * n, 1);
        if (!explored) return SPION_ORACLE_ERR_PARAM;
        if (variant & ORACLE_PAT_ALL_SEEDS) {
            for (int32_t r = 0; r < n; ++r)
                for (int32_t c = 0; c < n; ++c) flood_fill(pool_out, n, r, c, fl_out, gt, explored);
        } else {
            for (int32_t i = 0; i < n; ++i) flood_fill(pool_out, n, 0, i, fl_out, gt, explored);
            for (int32_t j = 0; j < n; ++j) flood_fill(pool_out, n, j, 0, fl_out, gt, explored);
        }
        free(explored);
    }
    for (int32_t k = 0; k < n; ++k) fl_out[(int64_t)k * n + k] = 1;
    return SPION_ORACLE_OK;
}

int spion_oracle_flood_fill(const int64_t *pool_out, int32_t n, const uint8_t *gt, uint8_t *fl_out)
{
    return spion_oracle_flood_fill_variant(pool_out, n, gt, 0, fl_out);
}

/* ------------------------------------------------------------------ */
/* a7: block mask -> block-CSR and block-CSC ("row_ptr, col_idx"; */
/* upsampling P:502/P:622 is implicit: block (I,J) stands for the B x B */
/* all-ones square of P).  Indices ascending.  Returns nnzb.            */
/* ------------------------------------------------------------------ */
int64_t spion_oracle_mask_to_bsr(const uint8_t *fl, int32_t n, int32_t *brow_ptr, int32_t *bcol_idx,
                                 int32_t *bcol_ptr, int32_t *brow_idx)
{
    int64_t nnz = 0;
    brow_ptr[0] = 0;
    for (int32_t I = 0; I < n; ++I) {
        for (int32_t J = 0; J < n; ++J)
            if (fl[(int64_t)I * n + J]) bcol_idx[nnz++] = J;
        brow_ptr[I + 1] = (int32_t)nnz;
    }
    int64_t nnz2 = 0;
    bcol_ptr[0] = 0;
    for (int32_t J = 0; J < n; ++J) {
        for (int32_t I = 0; I < n; ++I)
            if (fl[(int64_t)I * n + J]) brow_idx[nnz2++] = I;
        bcol_ptr[J + 1] = (int32_t)nnz2;
    }
    return nnz;
}

/* ------------------------------------------------------------------ */
/* Alg. 3 end to end: quantise, conv, pool, threshold,      */
/* flood fill, forced diagonal.  pool_out (n*n) and fl_out (n*n) are    */
/* outputs; t_out receives the threshold in pool-sum units.             */
/* ------------------------------------------------------------------ */
int spion_oracle_pattern_variant(const float *A, int32_t L, int32_t B, int32_t F, double theta, int32_t kind,
                                 int32_t variant, int64_t *pool_out, uint8_t *fl_out, double *t_out)
{
    if (L <= 0 || B <= 0 || (L % B) != 0) return SPION_ORACLE_ERR_SHAPE;
    if (F < 1 || (F % 2) == 0) return SPION_ORACLE_ERR_PARAM;
    int32_t n = L / B;
    int64_t LL = (int64_t)L * L;
    int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)LL);
    int64_t *conv = (int64_t *)malloc(sizeof(int64_t) * (size_t)LL);
    uint8_t *gt = (uint8_t *)malloc((size_t)n * n);
    int rc = SPION_ORACLE_ERR_PARAM;
    if (!q || !conv || !gt) goto done;
    rc = spion_oracle_quantize(A, LL, q);
    if (rc) goto done;
    rc = spion_oracle_diag_conv(q, L, F, conv);             /* Alg. 3 l.1-2 */
    if (rc) goto done;
    rc = spion_oracle_pool_sum(conv, L, B, pool_out);       /* Alg. 3 l.3 */
    if (rc) goto done;
    rc = spion_oracle_threshold_gt(pool_out, (int64_t)n * n, B, theta, kind, gt, t_out);
    if (rc) goto done;
    rc = spion_oracle_flood_fill_variant(pool_out, n, gt, variant, fl_out);  /* Alg. 3 l.4-10 */
done:
    free(q);
    free(conv);
    free(gt);
    return rc;
}

int spion_oracle_pattern(const float *A, int32_t L, int32_t B, int32_t F, double theta, int32_t kind,
                         int64_t *pool_out, uint8_t *fl_out, double *t_out)
{
    return spion_oracle_pattern_variant(A, L, B, F, theta, kind, 0, pool_out, fl_out, t_out);
}

/* ------------------------------------------------------------------ */
/* a8-a10: sparse attention forward for ONE (batch, head), fp64,        */
/* "dense masked attention with explicit loops":                        */
/*   S^r = (P>0) ⊙ Q K^T  (SDDMM, Eq. 5)                     */
/*   Alg. 6: x <- x*scale; m = max stored; Z = sum_stored    */
/*   exp(x-m) [+ (L - b_cnt) exp(-m) in PAPER mode, l.15]; p = exp(x-m)/Z */
/*   O = S^s V  (SpMM over stored entries only)                   */
/* lse_i = m + ln Z.  A row with no stored entry (only possible for     */
/* user-supplied masks) gives O_i = 0 and lse_i = ln L (PAPER) or -inf  */
/* (MASKED).  Q,K,V,O: [L][d] row-major.  fl: [n][n] block mask.        */
/* P (optional, may be NULL): dense [L][L] probabilities, 0 off-mask.   */
/* ------------------------------------------------------------------ */
int spion_oracle_attn_fwd(const double *Q, const double *K, const double *V, int32_t L, int32_t d,
                          int32_t B, const uint8_t *fl, double scale, int32_t mode, double *O,
                          double *lse, double *P)
{
    if (L <= 0 || d <= 0 || B <= 0 || (L % B) != 0) return SPION_ORACLE_ERR_SHAPE;
    if (mode != ORACLE_SOFTMAX_PAPER && mode != ORACLE_SOFTMAX_MASKED) return SPION_ORACLE_ERR_PARAM;
    int32_t n = L / B;
    double *s = (double *)malloc(sizeof(double) * (size_t)L);
    if (!s) return SPION_ORACLE_ERR_PARAM;
    for (int32_t i = 0; i < L; ++i) {
        int32_t I = i / B;
        int64_t cnt = 0;                       /* b_cnt of Alg. 6 l.3 */
        double m = -INFINITY;
        for (int32_t j = 0; j < L; ++j) {
            if (!fl[(int64_t)I * n + j / B]) continue;
            double dot = 0.0;
            for (int32_t e = 0; e < d; ++e) dot += Q[(int64_t)i * d + e] * K[(int64_t)j * d + e];
            s[j] = dot * scale;                /* Alg. 6 l.8 */
            if (s[j] > m) m = s[j];            /* Alg. 6 l.9-11 */
            ++cnt;
        }
        for (int32_t e = 0; e < d; ++e) O[(int64_t)i * d + e] = 0.0;
        if (P) for (int32_t j = 0; j < L; ++j) P[(int64_t)i * L + j] = 0.0;
        if (cnt == 0) {
            lse[i] = (mode == ORACLE_SOFTMAX_PAPER) ? log((double)L) : -INFINITY;
            continue;
        }
        double Z = 0.0;
        for (int32_t j = 0; j < L; ++j)
            if (fl[(int64_t)I * n + j / B]) Z += exp(s[j] - m);           /* Alg. 6 l.12-14 */
        if (mode == ORACLE_SOFTMAX_PAPER) Z += exp(-m) * (double)(L - cnt); /* Alg. 6 l.15 */
        for (int32_t j = 0; j < L; ++j) {
            if (!fl[(int64_t)I * n + j / B]) continue;
            double p = exp(s[j] - m) / Z;                                  /* Alg. 6 l.16-17 */
            if (P) P[(int64_t)i * L + j] = p;
            for (int32_t e = 0; e < d; ++e) O[(int64_t)i * d + e] += p * V[(int64_t)j * d + e]; /* SpMM */
        }
        lse[i] = m + log(Z);
    }
    free(s);
    return SPION_ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* a11: backward for ONE (batch, head), fp64.  The paper only says a     */
/* custom autograd function is used; these are the derivatives  */
/* of the forward above (reading Q17).  The (L - b_cnt) implicit zeros  */
/* are constants that act only through Z, so with p = exp(s - lse):     */
/*   D_i = sum_e dO_ie O_ie                                             */
/*   for stored (i,j): dp = dO_i . V_j ; ds = p (dp - D_i)              */
/*     dQ_i += scale ds K_j ; dK_j += scale ds Q_i ; dV_j += p dO_i      */
/* O and lse are recomputed by spion_oracle_attn_fwd.                   */
/* ------------------------------------------------------------------ */
int spion_oracle_attn_bwd(const double *Q, const double *K, const double *V, const double *dO,
                          int32_t L, int32_t d, int32_t B, const uint8_t *fl, double scale, int32_t mode,
                          double *dQ, double *dK, double *dV)
{
    if (L <= 0 || d <= 0 || B <= 0 || (L % B) != 0) return SPION_ORACLE_ERR_SHAPE;
    int32_t n = L / B;
    double *O = (double *)malloc(sizeof(double) * (size_t)L * d);
    double *lse = (double *)malloc(sizeof(double) * (size_t)L);
    if (!O || !lse) { free(O); free(lse); return SPION_ORACLE_ERR_PARAM; }
    int rc = spion_oracle_attn_fwd(Q, K, V, L, d, B, fl, scale, mode, O, lse, NULL);
    if (rc) { free(O); free(lse); return rc; }
    memset(dQ, 0, sizeof(double) * (size_t)L * d);
    memset(dK, 0, sizeof(double) * (size_t)L * d);
    memset(dV, 0, sizeof(double) * (size_t)L * d);
    for (int32_t i = 0; i < L; ++i) {
        int32_t I = i / B;
        double Di = 0.0;
        for (int32_t e = 0; e < d; ++e) Di += dO[(int64_t)i * d + e] * O[(int64_t)i * d + e];
        for (int32_t j = 0; j < L; ++j) {
            if (!fl[(int64_t)I * n + j / B]) continue;
            double dot = 0.0, dp = 0.0;
            for (int32_t e = 0; e < d; ++e) {
                dot += Q[(int64_t)i * d + e] * K[(int64_t)j * d + e];
                dp += dO[(int64_t)i * d + e] * V[(int64_t)j * d + e];
            }
            double p = exp(dot * scale - lse[i]);
            double ds = p * (dp - Di);
            for (int32_t e = 0; e < d; ++e) {
                dQ[(int64_t)i * d + e] += scale * ds * K[(int64_t)j * d + e];
                dK[(int64_t)j * d + e] += scale * ds * Q[(int64_t)i * d + e];
                dV[(int64_t)j * d + e] += p * dO[(int64_t)i * d + e];
            }
        }
    }
    free(O);
    free(lse);
    return SPION_ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* the dense-phase score matrix that feeds a1.    */
/* A^s = mean over the `bh` (batch, head) slices of the dense attention */
/* probabilities softmax(scale * Q K^T) (the "attention score matrix"   */
/* averaged across heads; batch mean: SURVEY §8(a) a1), written  */
/* as the definition: every row an explicit max / exp / sum in fp64.    */
/* Q, K: [bh][L][d] fp64 (bf16 inputs widened exactly).  A: [L][L].    */
/* sumsq (may be NULL): sum of A^2, the square of Eq. 2's norm. */
/* ------------------------------------------------------------------ */
int spion_oracle_score_mean(const double *Q, const double *K, int64_t bh, int32_t L, int32_t d, double scale,
                            double *A, double *sumsq)
{
    if (bh <= 0 || L <= 0 || d <= 0) return SPION_ORACLE_ERR_SHAPE;
    double *s = (double *)malloc(sizeof(double) * (size_t)L);
    if (!s) return SPION_ORACLE_ERR_PARAM;
    memset(A, 0, sizeof(double) * (size_t)L * L);
    for (int64_t b = 0; b < bh; ++b) {
        const double *q = Q + b * L * d, *k = K + b * L * d;
        for (int32_t i = 0; i < L; ++i) {
            double m = -INFINITY, Z = 0.0;
            for (int32_t j = 0; j < L; ++j) {
                double dot = 0.0;
                for (int32_t e = 0; e < d; ++e) dot += q[(int64_t)i * d + e] * k[(int64_t)j * d + e];
                s[j] = dot * scale;
                if (s[j] > m) m = s[j];
            }
            for (int32_t j = 0; j < L; ++j) Z += exp(s[j] - m);
            for (int32_t j = 0; j < L; ++j) A[(int64_t)i * L + j] += exp(s[j] - m) / Z / (double)bh;
        }
    }
    if (sumsq) {
        double acc = 0.0;
        for (int64_t k2 = 0; k2 < (int64_t)L * L; ++k2) acc += A[k2] * A[k2];
        *sumsq = acc;
    }
    free(s);
    return SPION_ORACLE_OK;
}

/* Eq. 2: distance_i = | sqrt(sum (A^s_{i-1})^2) - sqrt(sum (A^s_i)^2) |, and Alg. 2's
 * transition test: with three consecutive score matrices (i > 1),
 * transition <=> sqrt((distance_{i-1} - distance_i)^2) < alpha.  Inputs: the three sums of squares. */
int spion_oracle_transition(double sumsq_im2, double sumsq_im1, double sumsq_i, double alpha, double *dist_im1,
                            double *dist_i)
{
    double d1 = fabs(sqrt(sumsq_im2) - sqrt(sumsq_im1));
    double d2 = fabs(sqrt(sumsq_im1) - sqrt(sumsq_i));
    if (dist_im1) *dist_im1 = d1;
    if (dist_i) *dist_i = d2;
    return sqrt((d1 - d2) * (d1 - d2)) < alpha ? 1 : 0;
}

