// api.cu — the C ABI of libspion.so (include/spion.h): validation, dispatch,
// workspace carving and the host-buffer step.  No arithmetic of the method
// lives here except the host-side threshold rank (Alg. 3 / P:600), which is a
// scalar computed once per call.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "attn.cuh"

namespace spion {
static std::atomic<long long> g_launches{0}, g_tc_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
void note_tc_launch(int n) { g_tc_launches.fetch_add(n, std::memory_order_relaxed); }
void report_cuda_error(cudaError_t e, const char *what, const char *file, int line) {
    static const bool on = getenv("SPION_DEBUG") != nullptr;
    if (on) fprintf(stderr, "[spion] %s:%d %s -> %s\n", file, line, what, cudaGetErrorString(e));
}
}  // namespace spion

using namespace spion;

extern "C" {

int64_t spion_launch_count(void) { return (int64_t)g_launches.load(); }
int64_t spion_tc_launch_count(void) { return (int64_t)g_tc_launches.load(); }

// debug: copy the event trace of the last traced kernel (SPION_TRACE=1) to host:
// 3 roles (producer, MMA, softmax thread 0) x 1024 (event, globaltimer) pairs
SPION_API int64_t spion_debug_k2_trace(unsigned long long *host) {
    if (!spion::g_k2_trace) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(host, spion::g_k2_trace, 16 * 8, cudaMemcpyDeviceToHost);
    return 8;
}
SPION_API int64_t spion_debug_trace(unsigned long long *host, int64_t cap) {
    if (!spion::g_trace_buf) return 0;
    cudaDeviceSynchronize();
    int64_t n = 8 * 2048 + 4096;  // 8 roles x 2048 events, then [start, end] per CTA
    if (n > cap) n = cap;
    cudaMemcpy(host, spion::g_trace_buf + 16, n * 8, cudaMemcpyDeviceToHost);
    return n;
}

const char *spion_status_str(spion_status s) {
    switch (s) {
        case SPION_OK: return "ok";
        case SPION_ERR_SHAPE: return "shape error (L % block, L, bh or d)";
        case SPION_ERR_PARAM: return "parameter error (filter, threshold, enum)";
        case SPION_ERR_DATA: return "data error (scores outside [0,1]/NaN or non-binary mask)";
        case SPION_ERR_ALIGN: return "alignment error (pointers/strides must be 16-byte aligned)";
        case SPION_ERR_WORKSPACE: return "workspace, plan or capacity too small";
        case SPION_ERR_CUDA: return "CUDA error";
        case SPION_ERR_UNSUPPORTED: return "unsupported configuration";
    }
    return "unknown status";
}

size_t spion_bsr_plan_bytes(int32_t L, int32_t block) {
    if (L <= 0 || block <= 0 || L % block) return 0;
    PlanLayout pl(L / block, block);
    return round_up(pl.words * 4, 256);
}

size_t spion_pattern_workspace_bytes(int32_t L, int32_t block) {
    if (L <= 0 || block <= 0 || L % block) return 0;
    return pattern_ws_bytes(L, block);
}

static spion_status check_bsr_out(const spion_bsr *out, int32_t L, int32_t block) {
    if (!out || !out->brow_ptr || !out->bcol_idx || !out->bcol_ptr || !out->brow_idx || !out->nnzb)
        return SPION_ERR_PARAM;
    if (out->plan && out->plan_bytes < spion_bsr_plan_bytes(L, block)) return SPION_ERR_WORKSPACE;
    if (out->plan && !aligned16(out->plan)) return SPION_ERR_ALIGN;
    if (out->nnzb_cap < L / block) return SPION_ERR_WORKSPACE;  // the diagonal alone needs nblk
    return SPION_OK;
}

spion_status spion_pattern(const float *scores_dev, int32_t L, int32_t block, int32_t filter, double threshold,
                           spion_threshold_kind kind, void *ws_dev, size_t ws_bytes, spion_bsr *out,
                           int32_t *nnzb_host, void *stream) {
    return spion_pattern_variant(scores_dev, L, block, filter, threshold, kind, SPION_PAT_DEFAULT, ws_dev, ws_bytes,
                                 out, nnzb_host, stream);
}

// host-side validation of the pattern parameters and the threshold rank (Alg. 3 / P:600): the
// order-statistic index lo (and whether the LINEAR interpolation fraction is positive) or the
// absolute threshold in fixed point
struct PatternParams {
    long long lo = 0, T_abs = 0;
    int frac_pos = 0;
};
static spion_status pattern_params(int32_t L, int32_t block, int32_t filter, double threshold,
                                   spion_threshold_kind kind, uint32_t variant, PatternParams *pp) {
    if (variant & ~7u) return SPION_ERR_PARAM;
    if (L <= 0 || block <= 0 || L % block) return SPION_ERR_SHAPE;
    if (filter < 1 || filter % 2 == 0) return SPION_ERR_PARAM;
    if (L % 4) return SPION_ERR_ALIGN;
    const int n = L / block;
    if (n > 128) return SPION_ERR_UNSUPPORTED;
    const int h = (filter - 1) / 2;
    if ((h + block - 1) / block > 63) return SPION_ERR_UNSUPPORTED;
    const long long N = (long long)n * n;
    switch (kind) {
        case SPION_TH_QUANTILE_LINEAR: {
            if (!(threshold > 0.0 && threshold < 100.0)) return SPION_ERR_PARAM;
            const double hpos = ((double)(N - 1) * threshold) / 100.0;
            pp->lo = (long long)floor(hpos);
            const double frac = hpos - (double)pp->lo;
            if (pp->lo >= N - 1) { pp->lo = N - 1; pp->frac_pos = 0; }
            else pp->frac_pos = frac > 0.0;
            break;
        }
        case SPION_TH_QUANTILE_NEAREST: {
            if (!(threshold > 0.0 && threshold < 100.0)) return SPION_ERR_PARAM;
            long long k = (long long)ceil(threshold / 100.0 * (double)N) - 1;
            if (k < 0) k = 0;
            if (k > N - 1) k = N - 1;
            pp->lo = k;
            break;
        }
        case SPION_TH_ABSOLUTE: {
            if (!isfinite(threshold)) return SPION_ERR_PARAM;
            // gt(x) <=> x > t * B^2 * 2^32 (pool-mean units); x integral => x > floor(thr)
            const double thr = threshold * (double)((long long)block * block) * 4294967296.0;
            if (thr < 0.0) pp->T_abs = -1;
            else if (thr >= 9.2e18) pp->T_abs = 0x7fffffffffffffffLL;
            else pp->T_abs = (long long)floor(thr);
            break;
        }
        default: return SPION_ERR_PARAM;
    }
    return SPION_OK;
}

spion_status spion_pattern_variant(const float *scores_dev, int32_t L, int32_t block, int32_t filter,
                                   double threshold, spion_threshold_kind kind, uint32_t variant, void *ws_dev,
                                   size_t ws_bytes, spion_bsr *out, int32_t *nnzb_host, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PatternParams pp;
    spion_status st = pattern_params(L, block, filter, threshold, kind, variant, &pp);
    if (st) return st;
    if (!scores_dev || !ws_dev) return SPION_ERR_PARAM;
    if (!aligned16(scores_dev) || !aligned16(ws_dev)) return SPION_ERR_ALIGN;
    if (ws_bytes < pattern_ws_bytes(L, block)) return SPION_ERR_WORKSPACE;
    st = check_bsr_out(out, L, block);
    if (st) return st;
    out->L = L;
    out->block = block;
    out->nblk = L / block;
    st = launch_pattern(scores_dev, L, block, filter, (int)kind, pp.lo, pp.frac_pos, (int)variant, pp.T_abs, ws_dev,
                        out, s);
    if (st) return st;
    if (nnzb_host) {
        int flags = 0;
        SPION_CUDA_TRY(cudaMemcpyAsync(nnzb_host, out->nnzb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SPION_CUDA_TRY(cudaMemcpyAsync(&flags, ws_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPION_CUDA_TRY(cudaStreamSynchronize(s));
        if (flags & FLAG_BAD_SCORE) return SPION_ERR_DATA;
        if (flags & FLAG_CAPACITY) return SPION_ERR_WORKSPACE;
    }
    return SPION_OK;
}

size_t spion_pattern_pool_region(int32_t L, int32_t block, size_t *offset_bytes) {
    if (offset_bytes) *offset_bytes = 0;
    if (L <= 0 || block <= 0 || L % block) return 0;
    const size_t n = (size_t)(L / block);
    if (offset_bytes) *offset_bytes = 8;  // the bad-score count, padding, then the pool (at 256)
    return (256 - 8) / 8 + n * n;
}

spion_status spion_pattern_pool(const float *scores_rows_dev, int32_t L, int32_t block, int32_t filter,
                                int32_t row_begin, int32_t row_end, void *ws_dev, size_t ws_bytes, void *stream) {
    PatternParams pp;
    spion_status st = pattern_params(L, block, filter, 50.0, SPION_TH_QUANTILE_LINEAR, 0, &pp);
    if (st) return st;
    if (row_begin < 0 || row_end < row_begin || row_end > L || row_begin % block || row_end % block)
        return SPION_ERR_SHAPE;
    if (!ws_dev || (!scores_rows_dev && row_end > row_begin)) return SPION_ERR_PARAM;
    if (!aligned16(ws_dev) || (scores_rows_dev && !aligned16(scores_rows_dev))) return SPION_ERR_ALIGN;
    if (ws_bytes < pattern_ws_bytes(L, block)) return SPION_ERR_WORKSPACE;
    return launch_pattern_pool(scores_rows_dev, L, block, filter, row_begin, row_end, ws_dev,
                               static_cast<cudaStream_t>(stream));
}

spion_status spion_pattern_finalize(int32_t L, int32_t block, double threshold, spion_threshold_kind kind,
                                    uint32_t variant, void *ws_dev, size_t ws_bytes, spion_bsr *out,
                                    int32_t *nnzb_host, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    PatternParams pp;
    spion_status st = pattern_params(L, block, 1, threshold, kind, variant, &pp);
    if (st) return st;
    if (!ws_dev) return SPION_ERR_PARAM;
    if (!aligned16(ws_dev)) return SPION_ERR_ALIGN;
    if (ws_bytes < pattern_ws_bytes(L, block)) return SPION_ERR_WORKSPACE;
    st = check_bsr_out(out, L, block);
    if (st) return st;
    out->L = L;
    out->block = block;
    out->nblk = L / block;
    st = launch_pattern_finalize(L, block, (int)kind, pp.lo, pp.frac_pos, (int)variant, pp.T_abs, ws_dev, out, s);
    if (st) return st;
    if (nnzb_host) {
        int flags = 0;
        SPION_CUDA_TRY(cudaMemcpyAsync(nnzb_host, out->nnzb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SPION_CUDA_TRY(cudaMemcpyAsync(&flags, ws_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
        SPION_CUDA_TRY(cudaStreamSynchronize(s));
        if (flags & FLAG_BAD_SCORE) return SPION_ERR_DATA;
        if (flags & FLAG_CAPACITY) return SPION_ERR_WORKSPACE;
    }
    return SPION_OK;
}

spion_status spion_pattern_check(const void *ws_dev, int32_t *flags_host, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!ws_dev || !flags_host) return SPION_ERR_PARAM;
    SPION_CUDA_TRY(cudaMemcpyAsync(flags_host, ws_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SPION_CUDA_TRY(cudaStreamSynchronize(s));
    return SPION_OK;
}

spion_status spion_bsr_from_mask(const uint8_t *mask_dev, int32_t L, int32_t block, spion_bsr *out,
                                 int32_t *nnzb_host, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (L <= 0 || block <= 0 || L % block) return SPION_ERR_SHAPE;
    if (!mask_dev) return SPION_ERR_PARAM;
    const int n = L / block;
    if (n > 128) return SPION_ERR_UNSUPPORTED;
    if (out && out->nnzb_cap < 0) return SPION_ERR_WORKSPACE;
    if (!out || !out->brow_ptr || !out->bcol_idx || !out->bcol_ptr || !out->brow_idx || !out->nnzb)
        return SPION_ERR_PARAM;
    if (out->plan && (out->plan_bytes < spion_bsr_plan_bytes(L, block) || !aligned16(out->plan)))
        return SPION_ERR_WORKSPACE;
    out->L = L;
    out->block = block;
    out->nblk = n;
    spion_status st = launch_bsr_from_mask(mask_dev, L, block, out, nullptr, s);
    if (st) return st;
    if (nnzb_host) {
        SPION_CUDA_TRY(cudaMemcpyAsync(nnzb_host, out->nnzb, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SPION_CUDA_TRY(cudaStreamSynchronize(s));
        if (*nnzb_host < 0) return SPION_ERR_DATA;
        if (*nnzb_host > out->nnzb_cap) return SPION_ERR_WORKSPACE;
    }
    return SPION_OK;
}

// attention workspace: [0, 256) the tensor-core kernels' work-item counters (zeroed by every call,
// so concurrent calls sharing one pattern never share a counter); then, for the backward,
// D_i = rowsum(dO * O) and -lse_i * log2(e), fp32 [bh][L] each
static const size_t ATTN_CTR_BYTES = 256;

size_t spion_attn_fwd_workspace_bytes(int64_t bh, int32_t L, int32_t d, spion_dtype dt) {
    (void)dt;
    if (bh <= 0 || L <= 0 || d <= 0) return 0;
    return ATTN_CTR_BYTES;
}

// bf16 d = 64 (the tensor-core envelope) also reserves the fused backward's fp32 dQ accumulator
// and per-(bh, query block) completion counters (sized for the smallest block, 32)
static size_t attn_ws_base(int64_t bh, int32_t L) { return ATTN_CTR_BYTES + round_up((size_t)bh * L * 4, 256) * 2; }

size_t spion_attn_workspace_bytes(int64_t bh, int32_t L, int32_t d, spion_dtype dt) {
    if (bh <= 0 || L <= 0 || d <= 0) return 0;
    size_t b = attn_ws_base(bh, L);
    if (dt == SPION_BF16 && d == 64) b += fused_bwd_ws_bytes(bh, L, (L + 31) / 32);
    return b;
}

// SPION_FUSED_BWD=1: the fused single-pass backward at B = 64 without the flag (A/B timing)
static bool fused_bwd_forced() {
    static const int v = getenv("SPION_FUSED_BWD") != nullptr;
    return v != 0;
}

static spion_status check_attn_common(const void *Q, const void *K, const void *V, int64_t bh, int32_t L,
                                      int32_t d, int64_t stride_bh, int64_t stride_l, spion_dtype dt,
                                      const spion_bsr *pat, int mode) {
    if (!Q || !K || !V || !pat) return SPION_ERR_PARAM;
    if (bh <= 0 || L <= 0 || d <= 0 || d > 128) return SPION_ERR_SHAPE;
    if (pat->L != L || pat->block <= 0 || L % pat->block || pat->nblk != L / pat->block) return SPION_ERR_SHAPE;
    if (dt != SPION_F32 && dt != SPION_BF16) return SPION_ERR_PARAM;
    if (mode != SPION_SOFTMAX_PAPER && mode != SPION_SOFTMAX_MASKED) return SPION_ERR_PARAM;
    if (stride_l < d || stride_bh < d) return SPION_ERR_SHAPE;
    const int vec = dt == SPION_BF16 ? 8 : 4;
    if (stride_l % vec || stride_bh % vec) return SPION_ERR_ALIGN;
    if (!aligned16(Q) || !aligned16(K) || !aligned16(V)) return SPION_ERR_ALIGN;
    if (!pat->brow_ptr || !pat->bcol_idx || !pat->bcol_ptr || !pat->brow_idx) return SPION_ERR_PARAM;
    return SPION_OK;
}

static AttnArgs make_args(const void *Q, const void *K, const void *V, int64_t bh, int32_t L, int32_t d,
                          int64_t stride_bh, int64_t stride_l, const spion_bsr *pat, int mode, float scale) {
    AttnArgs a;
    memset(&a, 0, sizeof(a));
    a.Q = Q;
    a.K = K;
    a.V = V;
    a.bh = bh;
    a.L = L;
    a.d = d;
    a.stride_bh = stride_bh;
    a.stride_l = stride_l;
    a.B = pat->block;
    a.n = pat->nblk;
    a.mode = mode;
    a.scale = scale;
    a.brow_ptr = pat->brow_ptr;
    a.bcol_idx = pat->bcol_idx;
    a.bcol_ptr = pat->bcol_ptr;
    a.brow_idx = pat->brow_idx;
    a.plan = static_cast<const int *>(pat->plan);
    return a;
}

// which kernels a call with these arguments runs (no launch); see spion_attn_path in spion.h
static int attn_path(const AttnArgs &a, spion_dtype dt) {
    if (dt == SPION_BF16 && tc_supported(a, dt)) return SPION_PATH_TCGEN05;
    if (!simt_supported(a.B, a.d)) return -(int)SPION_ERR_UNSUPPORTED;
    return SPION_PATH_CUDA_CORE;
}

int32_t spion_attn_path(int64_t bh, int32_t L, int32_t d, int64_t stride_bh, int64_t stride_l, spion_dtype dt,
                        const spion_bsr *pat) {
    static const char dummy[16] __attribute__((aligned(16))) = {0};
    spion_status st = check_attn_common(dummy, dummy, dummy, bh, L, d, stride_bh, stride_l, dt, pat, 0);
    if (st) return -(int32_t)st;
    if (bh > 65535) return -(int32_t)SPION_ERR_UNSUPPORTED;
    AttnArgs a = make_args(dummy, dummy, dummy, bh, L, d, stride_bh, stride_l, pat, 0, 1.f);
    return attn_path(a, dt);
}

spion_status spion_attn_fwd(const void *Q_dev, const void *K_dev, const void *V_dev, void *O_dev, float *lse_dev,
                            int64_t bh, int32_t L, int32_t d, int64_t stride_bh, int64_t stride_l, spion_dtype dt,
                            const spion_bsr *pat, spion_softmax_mode mode, float scale, void *ws_dev,
                            size_t ws_bytes, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    spion_status st = check_attn_common(Q_dev, K_dev, V_dev, bh, L, d, stride_bh, stride_l, dt, pat, mode);
    if (st) return st;
    if (!O_dev || !lse_dev || !ws_dev) return SPION_ERR_PARAM;
    if (!aligned16(O_dev) || !aligned16(lse_dev) || !aligned16(ws_dev)) return SPION_ERR_ALIGN;
    if (ws_bytes < spion_attn_fwd_workspace_bytes(bh, L, d, dt)) return SPION_ERR_WORKSPACE;
    if (bh > 65535) return SPION_ERR_UNSUPPORTED;
    AttnArgs a = make_args(Q_dev, K_dev, V_dev, bh, L, d, stride_bh, stride_l, pat, mode, scale);
    a.Oout = O_dev;
    a.lse_out = lse_dev;
    a.sched = static_cast<int *>(ws_dev);
    const int path = attn_path(a, dt);
    if (path < 0) return (spion_status)(-path);
    if (path == SPION_PATH_TCGEN05) {
        SPION_CUDA_TRY(cudaMemsetAsync(ws_dev, 0, ATTN_CTR_BYTES, s));
        return launch_fwd_tc(a, s);
    }
    return launch_fwd_simt(a, dt, s);
}

spion_status spion_attn_bwd(const void *Q_dev, const void *K_dev, const void *V_dev, const void *O_dev,
                            const void *dO_dev, const float *lse_dev, void *dQ_dev, void *dK_dev, void *dV_dev,
                            int64_t bh, int32_t L, int32_t d, int64_t stride_bh, int64_t stride_l, spion_dtype dt,
                            const spion_bsr *pat, spion_softmax_mode mode, float scale, void *ws_dev,
                            size_t ws_bytes, void *stream) {
    return spion_attn_bwd_ex(Q_dev, K_dev, V_dev, O_dev, dO_dev, lse_dev, dQ_dev, dK_dev, dV_dev, bh, L, d, stride_bh,
                             stride_l, dt, pat, mode, scale, 0u, ws_dev, ws_bytes, stream);
}

spion_status spion_attn_bwd_ex(const void *Q_dev, const void *K_dev, const void *V_dev, const void *O_dev,
                               const void *dO_dev, const float *lse_dev, void *dQ_dev, void *dK_dev, void *dV_dev,
                               int64_t bh, int32_t L, int32_t d, int64_t stride_bh, int64_t stride_l, spion_dtype dt,
                               const spion_bsr *pat, spion_softmax_mode mode, float scale, uint32_t flags,
                               void *ws_dev, size_t ws_bytes, void *stream) {
    if (flags & ~(uint32_t)(SPION_BWD_DETERMINISTIC | SPION_BWD_FUSED)) return SPION_ERR_PARAM;
    if ((flags & SPION_BWD_DETERMINISTIC) && (flags & SPION_BWD_FUSED)) return SPION_ERR_PARAM;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    spion_status st = check_attn_common(Q_dev, K_dev, V_dev, bh, L, d, stride_bh, stride_l, dt, pat, mode);
    if (st) return st;
    if (!O_dev || !dO_dev || !lse_dev || !dQ_dev || !dK_dev || !dV_dev || !ws_dev) return SPION_ERR_PARAM;
    if (!aligned16(O_dev) || !aligned16(dO_dev) || !aligned16(dQ_dev) || !aligned16(dK_dev) ||
        !aligned16(dV_dev) || !aligned16(ws_dev) || !aligned16(lse_dev))
        return SPION_ERR_ALIGN;
    if (ws_bytes < spion_attn_workspace_bytes(bh, L, d, dt)) return SPION_ERR_WORKSPACE;
    if (bh > 65535) return SPION_ERR_UNSUPPORTED;
    AttnArgs a = make_args(Q_dev, K_dev, V_dev, bh, L, d, stride_bh, stride_l, pat, mode, scale);
    a.O = O_dev;
    a.dO = dO_dev;
    a.lse = lse_dev;
    a.dQ = dQ_dev;
    a.dK = dK_dev;
    a.dV = dV_dev;
    a.sched = static_cast<int *>(ws_dev);
    float *D = reinterpret_cast<float *>(static_cast<char *>(ws_dev) + ATTN_CTR_BYTES);
    a.D = D;
    a.nlse2 = reinterpret_cast<float *>(static_cast<char *>(ws_dev) + ATTN_CTR_BYTES + round_up((size_t)bh * L * 4, 256));
    const int path = attn_path(a, dt);
    if (path < 0) return (spion_status)(-path);
    if (path == SPION_PATH_TCGEN05) {
        SPION_CUDA_TRY(cudaMemsetAsync(ws_dev, 0, ATTN_CTR_BYTES, s));
        const bool fused = (flags & SPION_BWD_FUSED) || (fused_bwd_forced() && !(flags & SPION_BWD_DETERMINISTIC));
        if (fused && fused_bwd_supported(a))
            return launch_bwd_fused(a, static_cast<char *>(ws_dev) + attn_ws_base(bh, L), s);
        return launch_bwd_tc(a, s);
    }
    st = launch_bwd_preprocess(a, dt, D, s);
    if (st) return st;
    return launch_bwd_simt(a, dt, s);
}

// ------------------------------------------------------------------ host-buffer step
struct Arena {
    size_t scores, Q, K, V, dO, O, lse, dQ, dK, dV, pws, aws, brow_ptr, bcol_idx, bcol_ptr, brow_idx, mask, nnzb,
        plan, total;
};

// spion_step_host pipelines the step over C contiguous (batch, head) chunks: the H2D copy of
// chunk c+1, the attention of chunk c and the D2H copy of chunk c-1 overlap (copy engines in
// both directions and the SMs busy at once).  C (a power of two dividing bh, >= 8 (batch, head)
// pairs per chunk) is the largest of 16/8/4/2 that keeps >= 4 MB per input tensor per chunk, capped
// at 8 above 64 MB per tensor.  Measured on B200 (e2e ms/step, C = 4 / 8 / 16): Image 3.95 / 3.43 /
// 3.79, ListOps 7.58 / 7.55 / 6.62, Text 8.55 / 8.68 / 7.92, Retrieval 15.26 / 14.88 / 15.65; the
// step is bound by ~75 GB/s of combined H2D + D2H PCIe traffic, the chunking sets how much of it
// overlaps.
static int step_chunks(int64_t bh, size_t tensor_bytes) {
    const int cmax = tensor_bytes > ((size_t)64 << 20) ? 8 : 16;
    for (int C : {16, 8, 4, 2})
        if (C <= cmax && bh % C == 0 && bh / C >= 8 && tensor_bytes / C >= ((size_t)4 << 20)) return C;
    return 1;
}

static Arena arena_layout(int64_t bh, int32_t L, int32_t d, int32_t block, spion_dtype dt) {
    Arena A;
    const size_t elt = dt == SPION_BF16 ? 2 : 4;
    const size_t t = (size_t)bh * L * d * elt;
    const int n = L / block;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += round_up(bytes, 256); return r; };
    A.scores = take((size_t)L * L * 4);
    A.Q = take(t);
    A.K = take(t);
    A.V = take(t);
    A.dO = take(t);
    A.O = take(t);
    A.lse = take((size_t)bh * L * 4);
    A.dQ = take(t);
    A.dK = take(t);
    A.dV = take(t);
    A.pws = take(pattern_ws_bytes(L, block));
    const int C = step_chunks(bh, t);
    A.aws = take((size_t)C * spion_attn_workspace_bytes(bh / C, L, d, dt));  // one per bh chunk
    A.brow_ptr = take((size_t)(n + 1) * 4);
    A.bcol_idx = take((size_t)n * n * 4);
    A.bcol_ptr = take((size_t)(n + 1) * 4);
    A.brow_idx = take((size_t)n * n * 4);
    A.mask = take((size_t)n * n);
    A.nnzb = take(16);
    A.plan = take(spion_bsr_plan_bytes(L, block));
    A.total = o;
    return A;
}

size_t spion_step_arena_bytes(int64_t bh, int32_t L, int32_t d, int32_t block, spion_dtype dt) {
    if (bh <= 0 || L <= 0 || d <= 0 || block <= 0 || L % block) return 0;
    return arena_layout(bh, L, d, block, dt).total;
}

spion_status spion_step_host(const float *scores_host, const void *Q_host, const void *K_host, const void *V_host,
                             const void *dO_host, void *O_host, float *lse_host, void *dQ_host, void *dK_host,
                             void *dV_host, int64_t bh, int32_t L, int32_t d, int32_t block, int32_t filter,
                             double threshold, spion_threshold_kind kind, spion_dtype dt, spion_softmax_mode mode,
                             float scale, void *dev_arena, size_t arena_bytes, int32_t *nnzb_host, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (bh <= 0 || L <= 0 || d <= 0 || block <= 0 || L % block) return SPION_ERR_SHAPE;
    if (!scores_host || !Q_host || !K_host || !V_host || !dO_host) return SPION_ERR_PARAM;
    if (!dev_arena || !aligned16(dev_arena)) return SPION_ERR_ALIGN;
    Arena A = arena_layout(bh, L, d, block, dt);
    if (arena_bytes < A.total) return SPION_ERR_WORKSPACE;
    char *base = static_cast<char *>(dev_arena);
    const size_t elt = dt == SPION_BF16 ? 2 : 4;
    const size_t t = (size_t)bh * L * d * elt;
    const int n = L / block;
    const int C = step_chunks(bh, t);
    const int64_t bhc = bh / C;
    const size_t tc = t / C, lc = (size_t)bhc * L * 4, wsc = spion_attn_workspace_bytes(bhc, L, d, dt);
    spion_bsr bsr;
    memset(&bsr, 0, sizeof(bsr));
    bsr.L = L;
    bsr.block = block;
    bsr.nblk = n;
    bsr.nnzb_cap = n * n;
    bsr.brow_ptr = reinterpret_cast<int32_t *>(base + A.brow_ptr);
    bsr.bcol_idx = reinterpret_cast<int32_t *>(base + A.bcol_idx);
    bsr.bcol_ptr = reinterpret_cast<int32_t *>(base + A.bcol_ptr);
    bsr.brow_idx = reinterpret_cast<int32_t *>(base + A.brow_idx);
    bsr.mask = reinterpret_cast<uint8_t *>(base + A.mask);
    bsr.nnzb = reinterpret_cast<int32_t *>(base + A.nnzb);
    bsr.plan = base + A.plan;
    bsr.plan_bytes = spion_bsr_plan_bytes(L, block);
    // every parameter and shape check runs before the first copy is enqueued, so a rejected call
    // never leaves DMA in flight on the caller's host buffers
    {
        PatternParams pp;
        spion_status st = pattern_params(L, block, filter, threshold, kind, 0, &pp);
        if (st) return st;
        if (mode != SPION_SOFTMAX_PAPER && mode != SPION_SOFTMAX_MASKED) return SPION_ERR_PARAM;
        const int32_t path = spion_attn_path(bhc, L, d, (int64_t)L * d, d, dt, &bsr);
        if (path < 0) return (spion_status)(-path);
        if (bhc > 65535) return SPION_ERR_UNSUPPORTED;
    }
    // copy streams and events: created once per device and thread (the ABI's only state)
    constexpr int MAXC = 16;
    struct Pipe {
        int dev = -1;
        cudaStream_t h2d = nullptr, d2h = nullptr;
        cudaEvent_t start, scores, in[MAXC], out[MAXC], done;
    };
    static thread_local Pipe P;
    int dev = 0;
    SPION_CUDA_TRY(cudaGetDevice(&dev));
    if (P.dev != dev) {
        SPION_CUDA_TRY(cudaStreamCreateWithFlags(&P.h2d, cudaStreamNonBlocking));
        SPION_CUDA_TRY(cudaStreamCreateWithFlags(&P.d2h, cudaStreamNonBlocking));
        SPION_CUDA_TRY(cudaEventCreateWithFlags(&P.start, cudaEventDisableTiming));
        SPION_CUDA_TRY(cudaEventCreateWithFlags(&P.scores, cudaEventDisableTiming));
        SPION_CUDA_TRY(cudaEventCreateWithFlags(&P.done, cudaEventDisableTiming));
        for (int c = 0; c < MAXC; ++c) {
            SPION_CUDA_TRY(cudaEventCreateWithFlags(&P.in[c], cudaEventDisableTiming));
            SPION_CUDA_TRY(cudaEventCreateWithFlags(&P.out[c], cudaEventDisableTiming));
        }
        P.dev = dev;
    }
    // once a copy is enqueued, every exit drains both copy streams and the caller's stream
    // first (the header promises a synchronised return; no DMA may outlive the call)
    auto fail = [&](spion_status st) {
        cudaStreamSynchronize(P.h2d);
        cudaStreamSynchronize(P.d2h);
        cudaStreamSynchronize(s);
        return st;
    };
#define STEP_TRY(expr)                                                           \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) {                                                 \
            ::spion::report_cuda_error(_e, #expr, __FILE__, __LINE__);           \
            return fail(SPION_ERR_CUDA);                                         \
        }                                                                        \
    } while (0)
    auto H2D = [&](size_t off, const void *src, size_t bytes) {
        return cudaMemcpyAsync(base + off, src, bytes, cudaMemcpyHostToDevice, P.h2d);
    };
    auto D2H = [&](void *dst, size_t off, size_t bytes) {
        return cudaMemcpyAsync(dst, base + off, bytes, cudaMemcpyDeviceToHost, P.d2h);
    };
    // everything earlier on the caller's stream first
    SPION_CUDA_TRY(cudaEventRecord(P.start, s));
    SPION_CUDA_TRY(cudaStreamWaitEvent(P.h2d, P.start, 0));
    SPION_CUDA_TRY(cudaStreamWaitEvent(P.d2h, P.start, 0));
    STEP_TRY(H2D(A.scores, scores_host, (size_t)L * L * 4));
    STEP_TRY(cudaEventRecord(P.scores, P.h2d));
    for (int c = 0; c < C; ++c) {
        const char *q = static_cast<const char *>(Q_host), *k = static_cast<const char *>(K_host);
        const char *v = static_cast<const char *>(V_host), *g = static_cast<const char *>(dO_host);
        STEP_TRY(H2D(A.Q + c * tc, q + c * tc, tc));
        STEP_TRY(H2D(A.K + c * tc, k + c * tc, tc));
        STEP_TRY(H2D(A.V + c * tc, v + c * tc, tc));
        STEP_TRY(H2D(A.dO + c * tc, g + c * tc, tc));
        STEP_TRY(cudaEventRecord(P.in[c], P.h2d));
    }
    STEP_TRY(cudaStreamWaitEvent(s, P.scores, 0));
    spion_status st = spion_pattern(reinterpret_cast<const float *>(base + A.scores), L, block, filter, threshold,
                                    kind, base + A.pws, pattern_ws_bytes(L, block), &bsr, nullptr, stream);
    if (st) return fail(st);
    for (int c = 0; c < C; ++c) {
        const size_t o = c * tc;
        float *lse = reinterpret_cast<float *>(base + A.lse + c * lc);
        void *ws = base + A.aws + c * wsc;
        STEP_TRY(cudaStreamWaitEvent(s, P.in[c], 0));
        st = spion_attn_fwd(base + A.Q + o, base + A.K + o, base + A.V + o, base + A.O + o, lse, bhc, L, d,
                            (int64_t)L * d, d, dt, &bsr, mode, scale, ws, wsc, stream);
        if (st) return fail(st);
        st = spion_attn_bwd(base + A.Q + o, base + A.K + o, base + A.V + o, base + A.O + o, base + A.dO + o, lse,
                            base + A.dQ + o, base + A.dK + o, base + A.dV + o, bhc, L, d, (int64_t)L * d, d, dt, &bsr,
                            mode, scale, ws, wsc, stream);
        if (st) return fail(st);
        STEP_TRY(cudaEventRecord(P.out[c], s));
        STEP_TRY(cudaStreamWaitEvent(P.d2h, P.out[c], 0));
        if (O_host) STEP_TRY(D2H(static_cast<char *>(O_host) + o, A.O + o, tc));
        if (lse_host) STEP_TRY(D2H(reinterpret_cast<char *>(lse_host) + c * lc, A.lse + c * lc, lc));
        if (dQ_host) STEP_TRY(D2H(static_cast<char *>(dQ_host) + o, A.dQ + o, tc));
        if (dK_host) STEP_TRY(D2H(static_cast<char *>(dK_host) + o, A.dK + o, tc));
        if (dV_host) STEP_TRY(D2H(static_cast<char *>(dV_host) + o, A.dV + o, tc));
    }
#undef STEP_TRY
    SPION_CUDA_TRY(cudaEventRecord(P.done, P.d2h));
    SPION_CUDA_TRY(cudaStreamWaitEvent(s, P.done, 0));
    int32_t nnzb = 0;
    SPION_CUDA_TRY(cudaMemcpyAsync(&nnzb, bsr.nnzb, 4, cudaMemcpyDeviceToHost, s));
    int flags = 0;
    SPION_CUDA_TRY(cudaMemcpyAsync(&flags, base + A.pws, 4, cudaMemcpyDeviceToHost, s));
    SPION_CUDA_TRY(cudaStreamSynchronize(s));
    if (nnzb_host) *nnzb_host = nnzb;
    if (flags & FLAG_BAD_SCORE) return SPION_ERR_DATA;
    return SPION_OK;
}

// ------------------------------------------------------------------ NEXT-1: dense-phase scores
static size_t score_ws_layout(int64_t bh, int32_t L, size_t *o_pat, size_t *o_O, size_t *o_lse) {
    const int n = L / 64;
    size_t o = 0;
    auto take = [&](size_t bytes) { size_t r = o; o += round_up(bytes, 256); return r; };
    *o_pat = take((size_t)(n + 1) * 4 * 2 + (size_t)n * n * 4 * 2 + (size_t)n * n + 16 + 5 * 256 +
                  spion_bsr_plan_bytes(L, 64));
    *o_O = take((size_t)bh * L * 64 * 2);
    *o_lse = take((size_t)bh * L * 4);
    take(ATTN_CTR_BYTES);  // the dense forward's work-item counters (the last 256 bytes)
    return o;
}

size_t spion_score_mean_workspace_bytes(int64_t bh, int32_t L, int32_t d) {
    if (bh <= 0 || L <= 0 || d != 64 || L % 128) return 0;
    size_t a, b, c;
    return score_ws_layout(bh, L, &a, &b, &c);
}

spion_status spion_score_mean(const void *Q_dev, const void *K_dev, int64_t bh, int32_t L, int32_t d,
                              int64_t stride_bh, int64_t stride_l, float scale, void *ws_dev, size_t ws_bytes,
                              float *A_dev, double *sumsq_dev, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!Q_dev || !K_dev || !A_dev || !ws_dev) return SPION_ERR_PARAM;
    if (bh <= 0 || L <= 0 || d <= 0) return SPION_ERR_SHAPE;
    if (d != 64 || L % 128 || L / 64 > 128 || bh > 65535) return SPION_ERR_UNSUPPORTED;
    if (stride_l < d || stride_bh < (int64_t)stride_l * L || stride_l % 8 || stride_bh % 8) return SPION_ERR_ALIGN;
    if (!aligned16(Q_dev) || !aligned16(K_dev) || !aligned16(A_dev) || !aligned16(ws_dev)) return SPION_ERR_ALIGN;
    size_t o_pat, o_O, o_lse;
    if (ws_bytes < score_ws_layout(bh, L, &o_pat, &o_O, &o_lse)) return SPION_ERR_WORKSPACE;
    char *base = static_cast<char *>(ws_dev);
    const int n = L / 64;
    // a dense 64 x 64 block pattern (every block stored): the tensor-core forward in MASKED mode then
    // returns every row's exact normaliser lse_i = ln sum_j exp(scale q_i . k_j)
    spion_bsr bsr;
    memset(&bsr, 0, sizeof(bsr));
    size_t o = o_pat;
    auto take = [&](size_t bytes) { char *r = base + o; o += round_up(bytes, 256); return r; };
    bsr.nnzb_cap = n * n;
    bsr.brow_ptr = reinterpret_cast<int32_t *>(take((size_t)(n + 1) * 4));
    bsr.bcol_idx = reinterpret_cast<int32_t *>(take((size_t)n * n * 4));
    bsr.bcol_ptr = reinterpret_cast<int32_t *>(take((size_t)(n + 1) * 4));
    bsr.brow_idx = reinterpret_cast<int32_t *>(take((size_t)n * n * 4));
    uint8_t *mask = reinterpret_cast<uint8_t *>(take((size_t)n * n));
    bsr.nnzb = reinterpret_cast<int32_t *>(take(16));
    bsr.plan_bytes = spion_bsr_plan_bytes(L, 64);
    bsr.plan = take(bsr.plan_bytes);
    SPION_CUDA_TRY(cudaMemsetAsync(mask, 1, (size_t)n * n, s));
    spion_status st = spion_bsr_from_mask(mask, L, 64, &bsr, nullptr, stream);
    if (st) return st;
    bsr.mask = mask;
    float *lse = reinterpret_cast<float *>(base + o_lse);
    const size_t total = score_ws_layout(bh, L, &o_pat, &o_O, &o_lse);
    st = spion_attn_fwd(Q_dev, K_dev, K_dev, base + o_O, lse, bh, L, d, stride_bh, stride_l, SPION_BF16, &bsr,
                        SPION_SOFTMAX_MASKED, scale, base + total - ATTN_CTR_BYTES, ATTN_CTR_BYTES, stream);
    if (st) return st;
    if (sumsq_dev) SPION_CUDA_TRY(cudaMemsetAsync(sumsq_dev, 0, sizeof(double), s));
    // partial tiles of a (batch, head)-split score pass reuse the forward's (dead) O scratch
    int ks = score_splits(bh, L);
    while (ks > 1 && (size_t)ks * L * L * 4 > (size_t)bh * L * 64 * 2) --ks;
    return launch_score_mean(Q_dev, K_dev, lse, bh, L, stride_bh, stride_l, scale, A_dev, sumsq_dev,
                             reinterpret_cast<float *>(base + o_O), ks, s);
}

spion_status spion_transition(const double *sumsq_dev, double alpha, int32_t *switch_dev, double *dist_dev,
                              int32_t *switch_host, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!sumsq_dev || !switch_dev) return SPION_ERR_PARAM;
    if (!(alpha >= 0.0) || !isfinite(alpha)) return SPION_ERR_PARAM;
    spion_status st = launch_transition(sumsq_dev, alpha, switch_dev, dist_dev, s);
    if (st) return st;
    if (switch_host) {
        SPION_CUDA_TRY(cudaMemcpyAsync(switch_host, switch_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
        SPION_CUDA_TRY(cudaStreamSynchronize(s));
    }
    return SPION_OK;
}

// ------------------------------------------------------------------ NEXT-4: sparse-MHA sub-layer
spion_status spion_gemm_bf16(const void *A_dev, const void *B_dev, void *C_dev, int32_t M, int32_t N, int32_t K,
                             int32_t a_layout, int32_t c_layout, int32_t L, int32_t H, int32_t batch, float alpha,
                             void *stream) {
    if (!A_dev || !B_dev || !C_dev) return SPION_ERR_PARAM;
    if (M <= 0 || N <= 0 || K <= 0) return SPION_ERR_SHAPE;
    if ((a_layout != SPION_GEMM_ROWMAJOR && a_layout != SPION_GEMM_HEADS) ||
        (c_layout != SPION_GEMM_ROWMAJOR && c_layout != SPION_GEMM_HEADS))
        return SPION_ERR_PARAM;
    if (!aligned16(A_dev) || !aligned16(B_dev) || !aligned16(C_dev)) return SPION_ERR_ALIGN;
    if (M % 128 || N % 128 || K % 64) return SPION_ERR_UNSUPPORTED;
    const bool heads = a_layout == SPION_GEMM_HEADS || c_layout == SPION_GEMM_HEADS;
    if (heads) {
        if (L <= 0 || H <= 0 || batch <= 0) return SPION_ERR_SHAPE;
        if (L % 128 || (int64_t)batch * L != M) return SPION_ERR_SHAPE;
        if (a_layout == SPION_GEMM_HEADS && K % (64 * H)) return SPION_ERR_SHAPE;
        if (c_layout == SPION_GEMM_HEADS && N % (64 * H)) return SPION_ERR_SHAPE;
        if ((int64_t)batch * H > 65535 * 4) return SPION_ERR_UNSUPPORTED;
    }
    if (!tc_encode_fn_available()) return SPION_ERR_UNSUPPORTED;
    return launch_gemm_bf16(A_dev, B_dev, C_dev, M, N, K, a_layout == SPION_GEMM_HEADS, c_layout == SPION_GEMM_HEADS,
                            L, H, batch, alpha, static_cast<cudaStream_t>(stream));
}

spion_status spion_mha_heads(void *packed_dev, void *heads_dev, int64_t batch, int32_t L, int32_t W, int32_t H,
                             int32_t d, int32_t to_heads, void *stream) {
    if (!packed_dev || !heads_dev) return SPION_ERR_PARAM;
    if (batch <= 0 || L <= 0 || W <= 0 || H <= 0 || d <= 0) return SPION_ERR_SHAPE;
    if (d % 8) return SPION_ERR_UNSUPPORTED;
    if (!aligned16(packed_dev) || !aligned16(heads_dev)) return SPION_ERR_ALIGN;
    return launch_heads_permute(to_heads ? packed_dev : heads_dev, to_heads ? heads_dev : packed_dev, batch, L, W, H, d,
                                to_heads, static_cast<cudaStream_t>(stream));
}

spion_status spion_dropout_residual(const void *y_dev, const void *e_dev, void *out_dev, int64_t n, float p,
                                    uint64_t seed, void *stream) {
    if (!y_dev || !out_dev) return SPION_ERR_PARAM;
    if (n < 0) return SPION_ERR_SHAPE;
    if (!(p >= 0.f && p < 1.f)) return SPION_ERR_PARAM;
    if (n == 0) return SPION_OK;
    return launch_dropout_residual(y_dev, e_dev, out_dev, n, p, seed, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
