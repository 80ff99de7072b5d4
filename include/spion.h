/*
 * spion.h — C ABI of libspion.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of SPION (arXiv 2309.12578): layer-wise sparsity
 * pattern generation and block-sparse multi-head attention, forward and
 * backward.
 *
 * Citations "P:N" are lines of the paper text; "Qk" are the
 * readings of ambiguous passages listed in DESIGN.md §3.
 *
 * Conventions (all entry points)
 *  - Pointers named *_dev are DEVICE pointers; *_host are HOST pointers.
 *    The caller owns every buffer, including workspaces; the library never
 *    allocates device memory and keeps no state except a per-process cache
 *    of driver entry points.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    Every call is stream-ordered and asynchronous unless a *_host output
 *    is requested, in which case the call synchronises `stream`.
 *  - Errors never abort and never cross the ABI as exceptions: a call
 *    returns SPION_OK or a status describing the first problem found on the
 *    host (shape, parameter, alignment, workspace size, unsupported
 *    configuration) before anything is launched, or SPION_ERR_CUDA if a
 *    launch failed.  Data errors detectable only on the device (scores
 *    outside [0,1] or NaN) set a flag word in the pattern workspace,
 *    returned by spion_pattern_check().
 *  - Layout of Q, K, V, O, dO, dQ, dK, dV: [bh][L][d], element (b, i, e) at
 *    offset b*stride_bh + i*stride_l + e (elements, d contiguous), with
 *    bh = batch * heads.  lse and D: [bh][L] fp32, contiguous.
 *  - One block pattern per layer, shared by every (batch, head) (P:653,
 *    reading Q16).
 */
#ifndef SPION_H
#define SPION_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SPION_API __attribute__((visibility("default")))
#else
#define SPION_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    SPION_OK = 0,
    SPION_ERR_SHAPE = 1,       /* L % block != 0, L <= 0, bad bh or d          */
    SPION_ERR_PARAM = 2,       /* even filter, alpha outside (0,100), bad enum  */
    SPION_ERR_DATA = 3,        /* scores outside [0,1] / NaN; non-binary mask   */
    SPION_ERR_ALIGN = 4,       /* pointer or stride not 16-byte aligned          */
    SPION_ERR_WORKSPACE = 5,   /* workspace / plan / capacity too small          */
    SPION_ERR_CUDA = 6,        /* a CUDA runtime or driver call failed           */
    SPION_ERR_UNSUPPORTED = 7  /* valid but not implemented (see each call)      */
} spion_status;

typedef enum { SPION_F32 = 0, SPION_BF16 = 1 } spion_dtype;

/* Normaliser of the row softmax (Alg. 6; reading Q1).
 * PAPER : Z = sum_stored exp(s-m) + (L - b_cnt) exp(-m)   (Alg. 6 l.15)
 * MASKED: Z = sum_stored exp(s-m)                           (rows sum to 1) */
typedef enum { SPION_SOFTMAX_PAPER = 0, SPION_SOFTMAX_MASKED = 1 } spion_softmax_mode;

/* Threshold t of the flood fill (reading Q9).
 * QUANTILE_LINEAR : t = alpha% quantile of pool_out, linear interpolation
 *                   between order statistics (numpy/torch default), with
 *                   hpos = ((double)(N-1) * alpha) / 100, N = nblk^2.
 * QUANTILE_NEAREST: t = v[ceil(alpha/100 * N) - 1] (nearest rank).
 * ABSOLUTE        : t given directly in pool-mean units (mean of the B x B
 *                   block of conv_out with a diagonal filter of ones). */
typedef enum {
    SPION_TH_QUANTILE_LINEAR = 0,
    SPION_TH_QUANTILE_NEAREST = 1,
    SPION_TH_ABSOLUTE = 2
} spion_threshold_kind;

/* Pattern variants, bit flags for spion_pattern_variant:
 *   SPION_PAT_NOFLOOD   SPION-C: no flood fill; the top alpha% of
 *                       pool_out (the cells > t) plus the forced diagonal
 *                       (reading Q23).  SPION-F (no convolution) is filter = 1.
 *   SPION_PAT_PROSE     the prose reading of Alg. 4 (reading Q11 R2):
 *                       the fill continues only from critical (> t) cells.
 *   SPION_PAT_ALL_SEEDS every element of pool_out is a seed point (
 *                       reading Q12), instead of row 0 and column 0 (Alg. 3).
 * 0 is Alg. 3/4 as printed (SPION-CF, the paper's model). */
typedef enum {
    SPION_PAT_DEFAULT = 0,
    SPION_PAT_NOFLOOD = 1,
    SPION_PAT_PROSE = 2,
    SPION_PAT_ALL_SEEDS = 4
} spion_pattern_flags;

/* Block pattern in block-CSR + block-CSC form (CSR of P; the nearest
 * neighbour upsampling of Alg. 3 l.11 is implicit: block
 * (I,J) stands for the B x B all-ones square of P).  All pointers are
 * device pointers owned by the caller.  Column (row) indices are strictly
 * ascending within each row (column); brow_ptr[0] = 0, brow_ptr[nblk] =
 * nnzb.  Generated patterns always contain the diagonal.
 * `plan` holds the work lists the attention kernels consume (row tiles of
 * the forward, column tiles of the backward); its contents are private. */
typedef struct {
    int32_t L, block, nblk, nnzb_cap; /* nblk = L / block; nnzb_cap >= nblk*nblk is always safe */
    int32_t *brow_ptr;                /* [nblk+1] */
    int32_t *bcol_idx;                /* [nnzb_cap] */
    int32_t *bcol_ptr;                /* [nblk+1] */
    int32_t *brow_idx;                /* [nnzb_cap] */
    uint8_t *mask;                    /* [nblk*nblk] row-major fl_out, may be NULL */
    int32_t *nnzb;                    /* [1] device scalar */
    void *plan;                       /* >= spion_bsr_plan_bytes(L, block) bytes, 16-byte aligned */
    size_t plan_bytes;
} spion_bsr;

/* Bytes of spion_bsr.plan for a pattern of this shape. */
SPION_API size_t spion_bsr_plan_bytes(int32_t L, int32_t block);

/* Bytes of device workspace spion_pattern needs (pool_out in int64 fixed
 * point, the device flag word and selection scratch). */
SPION_API size_t spion_pattern_workspace_bytes(int32_t L, int32_t block);

/* Pattern generation, Alg. 3 with Alg. 4:
 *   q = rint(A * 2^32) (reading Q8)  ->  Eq. 3 diagonal convolution, centred
 *   window of `filter` taps, zero padding (reading Q5)  ->  Eq. 4
 *   B x B pooling (sums, reading Q7)  ->  threshold t  ->
 *   flood fill seeded at (0,i) and (j,0) (readings Q11-Q15, Q21)
 *   ->  forced diagonal  ->  block-CSR/CSC and plan.
 * scores_dev: [L][L] fp32 row-major, values in [0,1] (head-averaged A^s),
 *   16-byte aligned; L % 4 == 0.
 * block: B >= 1, L % B == 0; nblk = L/B must be <= 128 (else UNSUPPORTED).
 * filter: F odd >= 1, with ceil(((F-1)/2)/B) <= 63.
 * threshold: alpha in (0,100) for QUANTILE_*, t for ABSOLUTE.
 * ws_dev: >= spion_pattern_workspace_bytes(L, block) bytes, 16-byte aligned.
 * out: shape fields are filled in; pointer fields must be set by the caller
 *   (nnzb_cap >= number of blocks produced, nblk*nblk is always enough).
 * nnzb_host: if non-NULL, the call synchronises and stores nnzb there and
 *   returns SPION_ERR_DATA if the device flagged bad scores.
 * Results are bit-identical to the oracle (exact integer arithmetic). */
SPION_API spion_status spion_pattern(const float *scores_dev, int32_t L, int32_t block, int32_t filter,
                           double threshold, spion_threshold_kind kind, void *ws_dev, size_t ws_bytes,
                           spion_bsr *out, int32_t *nnzb_host, void *stream);

/* spion_pattern with a variant: `variant` is a bitwise OR of spion_pattern_flags
 * (any combination; NOFLOOD ignores the other two).  Other bits: SPION_ERR_PARAM.
 * Results are bit-identical to the oracle's spion_oracle_pattern_variant. */
SPION_API spion_status spion_pattern_variant(const float *scores_dev, int32_t L, int32_t block, int32_t filter,
                           double threshold, spion_threshold_kind kind, uint32_t variant, void *ws_dev,
                           size_t ws_bytes, spion_bsr *out, int32_t *nnzb_host, void *stream);

/* Pattern generation split for a multi-device job.  Eq. 3 and
 * Eq. 4 are sums over the source rows of A^s, so the pool of the
 * whole matrix is the SUM of the pools of any partition of its rows: each
 * device pools its own rows, the callers sum the pool regions of their
 * workspaces (e.g. one NCCL all-reduce, 64-bit integer sum: exact and
 * order-independent), and every device finalises the identical pattern.
 *
 * spion_pattern_pool_region: the part of a pattern workspace the callers sum,
 *   as *count_i64 int64 elements starting *offset_bytes into ws (the pool sums
 *   and the bad-score count); returns 0 (count 0) for an invalid shape.
 * spion_pattern_pool: zero-fills the workspace's pool region and adds the
 *   contributions of source rows [row_begin, row_end) (a2-a4).
 *   scores_rows_dev: those rows only, [row_end - row_begin][L] fp32 row-major
 *   (row 0 = source row row_begin), values in [0,1], 16-byte aligned.
 *   row_begin, row_end: multiples of block, 0 <= row_begin <= row_end <= L
 *   (an empty range gives a zero pool).  Other parameters as spion_pattern.
 *   Asynchronous; scores outside [0,1] are counted in the pool region and
 *   reported by spion_pattern_finalize.
 * spion_pattern_finalize: threshold, flood fill, diagonal, CSR/CSC and plan
 *   (a5-a7) from the (summed) pool in ws_dev; threshold, kind, variant, out and
 *   nnzb_host as spion_pattern_variant (SPION_ERR_DATA if any device saw a bad
 *   score).  spion_pattern_pool over [0, L) followed by spion_pattern_finalize
 *   is exactly spion_pattern_variant. */
SPION_API size_t spion_pattern_pool_region(int32_t L, int32_t block, size_t *offset_bytes);
SPION_API spion_status spion_pattern_pool(const float *scores_rows_dev, int32_t L, int32_t block, int32_t filter,
                                          int32_t row_begin, int32_t row_end, void *ws_dev, size_t ws_bytes,
                                          void *stream);
SPION_API spion_status spion_pattern_finalize(int32_t L, int32_t block, double threshold, spion_threshold_kind kind,
                                              uint32_t variant, void *ws_dev, size_t ws_bytes, spion_bsr *out,
                                              int32_t *nnzb_host, void *stream);

/* Synchronises `stream` and reads the device flag word of a pattern
 * workspace: *flags_host = 0 if every score was finite and in [0,1]. */
SPION_API spion_status spion_pattern_check(const void *ws_dev, int32_t *flags_host, void *stream);

/* Block-CSR/CSC and plan from a caller-supplied block mask (e.g. SPION-C or
 * a fixed pattern).  mask_dev: [nblk][nblk] uint8 in {0,1} (device); a
 * non-binary byte sets *nnzb to -1 (and SPION_ERR_DATA if nnzb_host given).
 * Empty rows are allowed (their outputs are zero, see spion_attn_fwd). */
SPION_API spion_status spion_bsr_from_mask(const uint8_t *mask_dev, int32_t L, int32_t block, spion_bsr *out,
                                 int32_t *nnzb_host, void *stream);

/* Attention workspaces (device, caller-owned, 16-byte aligned).  The first 256
 * bytes hold the tensor-core kernels' work-item counters; every call zeroes
 * them (one cudaMemsetAsync on `stream`) before launching, so calls that
 * share one pattern may run concurrently on different streams as long as
 * each has its OWN workspace.  A workspace must not be shared by calls that
 * can run concurrently.
 * spion_attn_fwd_workspace_bytes: the counters only (256 bytes).
 * spion_attn_workspace_bytes: the counters, then D_i = rowsum(dO*O) and
 * -lse_i*log2(e), fp32 [bh][L] each (written by the dQ pass for the dK/dV
 * pass; the backward is atomic-free and deterministic).  Enough for either
 * call. */
SPION_API size_t spion_attn_fwd_workspace_bytes(int64_t bh, int32_t L, int32_t d, spion_dtype dt);
SPION_API size_t spion_attn_workspace_bytes(int64_t bh, int32_t L, int32_t d, spion_dtype dt);

/* Which kernels spion_attn_fwd / spion_attn_bwd run for these arguments
 * (host only, nothing is launched): SPION_PATH_TCGEN05 — the tensor-core
 * kernels (bf16, d == 64, block in {32, 64}, strides multiples of 8, L % 4 ==
 * 0, nblk <= 128, plan present, driver entry point cuTensorMapEncodeTiled
 * available, SPION_DISABLE_TC unset); SPION_PATH_CUDA_CORE — the CUDA-core
 * kernels; a negative value -status if the call would be rejected. */
typedef enum { SPION_PATH_CUDA_CORE = 0, SPION_PATH_TCGEN05 = 1 } spion_attn_path_kind;
SPION_API int32_t spion_attn_path(int64_t bh, int32_t L, int32_t d, int64_t stride_bh, int64_t stride_l,
                                  spion_dtype dt, const spion_bsr *pat);

/* Forward block-sparse attention, per (batch, head) b (Alg. 5 l.4-8,
 * P:662-670; Eq. 5; Alg. 6):
 *   s_ij = scale * Q_i . K_j for (floor(i/B), floor(j/B)) in the pattern (SDDMM)
 *   p_ij = exp(s_ij - lse_i)                        (sparse softmax, mode)
 *   O_i  = sum_stored p_ij V_j                      (SpMM)
 *   lse_i = m_i + ln Z_i  (fp32; log-domain form of Alg. 6 l.15, reading Q2)
 * Rows whose block-row is empty: O_i = 0, lse_i = ln L (PAPER) / -inf (MASKED).
 * dt = SPION_BF16: bf16 Q/K/V/O, fp32 accumulation, P rounded to bf16 before
 *   P.V on the tensor-core path (reading Q18).  Tensor-core (tcgen05) path
 *   for block in {32, 64} and d == 64 (any strides that are multiples of 8
 *   elements: strided TMA tensor maps); other shapes run the CUDA-core path.
 * dt = SPION_F32: fp32 everywhere on CUDA cores (d <= 128, any block | L).
 * scale: normally 1/sqrt(d) (Eq. 1; reading Q4).
 * Pointers 16-byte aligned; strides in elements, multiples of 8 (bf16) or
 * 4 (fp32).  d <= 128.  The CUDA-core path stages one key block in shared
 * memory: shapes whose staging exceeds 227 KB (e.g. block = 128 with
 * d = 128) return SPION_ERR_UNSUPPORTED.
 * ws_dev: >= spion_attn_fwd_workspace_bytes(...) bytes (see above). */
SPION_API spion_status spion_attn_fwd(const void *Q_dev, const void *K_dev, const void *V_dev, void *O_dev,
                            float *lse_dev, int64_t bh, int32_t L, int32_t d, int64_t stride_bh,
                            int64_t stride_l, spion_dtype dt, const spion_bsr *pat, spion_softmax_mode mode,
                            float scale, void *ws_dev, size_t ws_bytes, void *stream);

/* Backward of spion_attn_fwd (the paper's custom autograd; formulas
 * of reading Q17): with p_ij = exp(s_ij - lse_i) and D_i = dO_i . O_i,
 *   dp_ij = dO_i . V_j ; ds_ij = p_ij (dp_ij - D_i)
 *   dQ_i = scale sum_j ds_ij K_j ; dK_j = scale sum_i ds_ij Q_i ; dV_j = sum_i p_ij dO_i
 * The same formulas hold in both modes (the implicit zeros act only
 * through Z).  O and lse are the outputs of spion_attn_fwd.  dQ, dK, dV use
 * the same layout and strides as Q.  ws_dev: >= spion_attn_workspace_bytes
 * (see above).
 * Tensor-core path: a row pass for dQ and a column pass for dK/dV,
 * atomic-free and bitwise reproducible; block 64 can instead run ONE fused
 * pass (spion_attn_bwd_ex, SPION_BWD_FUSED). */
SPION_API spion_status spion_attn_bwd(const void *Q_dev, const void *K_dev, const void *V_dev, const void *O_dev,
                            const void *dO_dev, const float *lse_dev, void *dQ_dev, void *dK_dev,
                            void *dV_dev, int64_t bh, int32_t L, int32_t d, int64_t stride_bh,
                            int64_t stride_l, spion_dtype dt, const spion_bsr *pat, spion_softmax_mode mode,
                            float scale, void *ws_dev, size_t ws_bytes, void *stream);

/* spion_attn_bwd with flags (bitwise OR; other bits, or both bits: SPION_ERR_PARAM):
 * SPION_BWD_DETERMINISTIC — bitwise reproducible results (the two-pass
 *   tensor-core backward; also the default).
 * SPION_BWD_FUSED — block 64 on the tensor-core path: one pass over the
 *   pattern's column tiles computes dK, dV and dQ (dQ = [dS_I0; dS_I1] K per
 *   pair of query blocks, accumulated in fp32 in the workspace by bulk
 *   reduce-adds at L2 and converted by the last contributor), so Q, K, V and
 *   dO are read and S^T, dP^T recomputed once; dQ's summation order depends on
 *   scheduling (results may differ between runs by rounding).  Other shapes
 *   ignore the flag. */
typedef enum { SPION_BWD_DETERMINISTIC = 1, SPION_BWD_FUSED = 2 } spion_bwd_flags;
SPION_API spion_status spion_attn_bwd_ex(const void *Q_dev, const void *K_dev, const void *V_dev, const void *O_dev,
                            const void *dO_dev, const float *lse_dev, void *dQ_dev, void *dK_dev,
                            void *dV_dev, int64_t bh, int32_t L, int32_t d, int64_t stride_bh,
                            int64_t stride_l, spion_dtype dt, const spion_bsr *pat, spion_softmax_mode mode,
                            float scale, uint32_t flags, void *ws_dev, size_t ws_bytes, void *stream);

/* One whole step of the hot path from HOST buffers (the end-to-end call):
 * copies scores, Q, K, V, dO host->device, runs spion_pattern,
 * spion_attn_fwd and spion_attn_bwd, and copies O, lse, dQ, dK, dV back.
 * Tensors are contiguous [bh][L][d] (stride_l = d).  Host buffers should be
 * pinned for asynchronous copies.  dev_arena: caller-owned device memory of
 * >= spion_step_arena_bytes(...) bytes.  Synchronises `stream` and returns
 * nnzb in *nnzb_host (may be NULL).
 * Every parameter is validated before the first copy is enqueued; on an
 * error after that point the call drains its copy streams and `stream`
 * before returning, so no DMA touches the host buffers after it returns.
 * The (batch, head) range is processed in up to 16 contiguous chunks (>= 8 pairs and >= 4 MB per
 * input tensor each), pipelined:
 * the H2D copy of chunk c+1, the attention of chunk c (on `stream`) and the D2H
 * copy of chunk c-1 overlap, on two copy streams the library creates once per
 * device and host thread (with their events: the ABI's only internal state).
 * Results are identical to the unchunked device calls (every (batch, head) is
 * computed independently and deterministically). */
SPION_API size_t spion_step_arena_bytes(int64_t bh, int32_t L, int32_t d, int32_t block, spion_dtype dt);
SPION_API spion_status spion_step_host(const float *scores_host, const void *Q_host, const void *K_host,
                             const void *V_host, const void *dO_host, void *O_host, float *lse_host,
                             void *dQ_host, void *dK_host, void *dV_host, int64_t bh, int32_t L, int32_t d,
                             int32_t block, int32_t filter, double threshold, spion_threshold_kind kind,
                             spion_dtype dt, spion_softmax_mode mode, float scale, void *dev_arena,
                             size_t arena_bytes, int32_t *nnzb_host, void *stream);

/* the dense-phase score matrix that feeds spion_pattern.
 * A_dev[L][L] (fp32, row-major, caller-owned) = mean over the bh (batch, head)
 * slices of softmax(scale Q K^T) — the attention score matrix averaged across
 * heads and batch — and, if sumsq_dev != NULL, *sumsq_dev = sum of A^2
 * (fp64), the square of the norm in Eq. 2 for Alg. 2's transition
 * test (spion_transition below).  Q, K: [bh][L][d] bf16 device, strides as spion_attn_fwd.
 * Needs d = 64, L % 128 == 0, L <= 8192 (else UNSUPPORTED).  ws_dev: >=
 * spion_score_mean_workspace_bytes(bh, L, d) bytes (a dense block pattern,
 * forward scratch and the row normalisers).  Tensor cores: the dense forward
 * gives every row's lse, then one pass forms each 128x128 tile of A over all
 * bh in registers (no atomics on A). */
SPION_API size_t spion_score_mean_workspace_bytes(int64_t bh, int32_t L, int32_t d);
SPION_API spion_status spion_score_mean(const void *Q_dev, const void *K_dev, int64_t bh, int32_t L, int32_t d,
                             int64_t stride_bh, int64_t stride_l, float scale, void *ws_dev, size_t ws_bytes,
                             float *A_dev, double *sumsq_dev, void *stream);

/* Alg. 2's transition test with Eq. 2's distance, on
 * the device in fp64: sumsq_dev[3] = sum (A^s)^2 of the score matrices of
 * three consecutive dense-phase steps i-2, i-1, i (spion_score_mean);
 * distance_k = | sqrt(sumsq[k-1]) - sqrt(sumsq[k]) |; *switch_dev = 1 if
 * sqrt((distance_{i-1} - distance_i)^2) < alpha (switch to the sparse phase),
 * else 0.  dist_dev (nullable): [2] = distance_{i-1}, distance_i.  alpha is
 * the transition tolerance (reading Q10), finite and >= 0.  switch_host
 * (nullable): also copied to the host (synchronises `stream`).  Stream-ordered
 * otherwise, so it can sit inside a captured training step. */
SPION_API spion_status spion_transition(const double *sumsq_dev, double alpha, int32_t *switch_dev,
                                        double *dist_dev, int32_t *switch_host, void *stream);

/* the projections of the sparse-MHA sub-layer (Alg. 5 l.2-3,
 * l.8-9) on the tensor cores, with the head split / concatenation
 * folded into the operand and output addressing:
 *   C[M][N] = alpha * A[M][K] B[N][K]^T, bf16 in, fp32 accumulation, bf16 out.
 * B: [N][K] row-major (a weight in nn.Linear layout, out x in).  A and C are
 * either SPION_GEMM_ROWMAJOR ([M][K], [M][N] contiguous) or SPION_GEMM_HEADS:
 * the attention layout, W tensors [batch*H][L][64] bf16 stacked contiguously
 * (tensor w at element offset w*batch*H*L*64), row m = token (b, l) with
 * M = batch*L, column (A: k, C: n) = w*H*64 + h*64 + e.  So Q|K|V = X W^T with
 * c_layout = HEADS writes the three attention inputs directly (W = 3), and
 * S Wo^T with a_layout = HEADS reads the attention output directly (W = 1).
 * Needs M % 128 == 0, N % 128 == 0, K % 64 == 0 (else UNSUPPORTED); with a
 * HEADS layout also head dim 64, L % 128 == 0 and M == batch*L, K (or N) a
 * multiple of 64*H (else SHAPE).  16-byte aligned pointers.  L, H, batch are
 * ignored for two ROWMAJOR operands.  Persistent tcgen05 kernel: 128 x 128
 * tiles, TMA operand ring, TMEM accumulators, TMA stores. */
typedef enum { SPION_GEMM_ROWMAJOR = 0, SPION_GEMM_HEADS = 1 } spion_gemm_layout;
SPION_API spion_status spion_gemm_bf16(const void *A_dev, const void *B_dev, void *C_dev, int32_t M, int32_t N,
                                       int32_t K, int32_t a_layout, int32_t c_layout, int32_t L, int32_t H,
                                       int32_t batch, float alpha, void *stream);

/* the sparse-MHA sub-layer around the attention (Alg. 5,
 * P:655-674): head split / concatenation and dropout + residual kernels.
 * spion_mha_heads: l.3 split / l.8 concatenate.  packed_dev: [batch][L][W][H][d]
 * bf16 row-major (the projection output, W tensors side by side: W = 3 for
 * Q|K|V, 1 for the concatenated heads); heads_dev: W tensors [batch*H][L][d],
 * tensor w at element offset w*batch*H*L*d (the attention layout).  to_heads =
 * 1: packed -> heads (split); 0: heads -> packed (concatenate, or the split's
 * backward).  d % 8 == 0; 16-byte aligned pointers.
 * spion_dropout_residual: l.9, out = e + dropout(y, p) (e != NULL), or the
 * backward out = dropout(y, p) (e == NULL, y the incoming gradient), bf16, n
 * elements; the keep mask is a counter-based hash of (seed, element index), so
 * the backward with the same seed drops the same elements; kept values are
 * scaled by 1/(1-p); 0 <= p < 1. */
SPION_API spion_status spion_mha_heads(void *packed_dev, void *heads_dev, int64_t batch, int32_t L, int32_t W,
                            int32_t H, int32_t d, int32_t to_heads, void *stream);
SPION_API spion_status spion_dropout_residual(const void *y_dev, const void *e_dev, void *out_dev, int64_t n, float p,
                                   uint64_t seed, void *stream);

/* Number of this library's kernels launched by this thread since process
 * start (host-side counter, for the bench's gpu_launches claim). */
SPION_API int64_t spion_launch_count(void);

/* Number of tensor-core (tcgen05) attention kernels launched by this process
 * (attn_fwd_tc_kernel, attn_bwd_*_tc_kernel): lets tests assert that the
 * tensor-core path, not the CUDA-core path, ran. */
SPION_API int64_t spion_tc_launch_count(void);

/* Human-readable status. */
SPION_API const char *spion_status_str(spion_status s);

#ifdef __cplusplus
}
#endif

#endif /* SPION_H */
