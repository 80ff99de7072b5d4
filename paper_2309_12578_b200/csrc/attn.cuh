// attn.cuh — internal interface between the ABI layer and the attention kernels.
#pragma once
#include "common.cuh"

namespace spion {

struct AttnArgs {
    const void *Q, *K, *V, *O, *dO;
    void *Oout, *dQ, *dK, *dV;
    float *lse_out;
    const float *lse, *D;
    float *nlse2;  // bwd workspace: -lse * log2(e), written by the dQ pass (tensor-core path)
    int64_t bh, stride_bh, stride_l;
    int L, d, B, n;
    int mode;
    float scale;
    const int *brow_ptr, *bcol_idx, *bcol_ptr, *brow_idx;
    const int *plan;
    int *sched;  // tensor-core path: 4 zeroed work-item counters in the caller's workspace
};

extern unsigned long long *g_trace_buf;  // debug event trace (SPION_TRACE=1)
extern unsigned long long *g_k2_trace;   // debug K2 phase stamps (SPION_TRACE=1)

bool simt_supported(int B, int d);
spion_status launch_fwd_simt(const AttnArgs &a, spion_dtype dt, cudaStream_t s);
spion_status launch_bwd_preprocess(const AttnArgs &a, spion_dtype dt, float *D, cudaStream_t s);
spion_status launch_bwd_simt(const AttnArgs &a, spion_dtype dt, cudaStream_t s);

// tensor-core (tcgen05) path; attn_tc.cu
bool tc_supported(const AttnArgs &a, spion_dtype dt);
bool tc_encode_fn_available();  // the driver's cuTensorMapEncodeTiled was found
spion_status launch_fwd_tc(const AttnArgs &a, cudaStream_t s);
spion_status launch_bwd_tc(const AttnArgs &a, cudaStream_t s);

// fused tensor-core backward (B = 64, d = 64; dQ by bulk reduce-add); attn_bwd_fused.cu.
// fws: >= fused_bwd_ws_bytes(bh, L, n) bytes (completion counters + the fp32 dQ accumulator)
bool fused_bwd_supported(const AttnArgs &a);
size_t fused_bwd_ws_bytes(int64_t bh, int L, int n);
spion_status launch_bwd_fused(const AttnArgs &a, void *fws, cudaStream_t s);

// a TMA tensor map (CUtensorMap, 128-byte aligned) over [bh][L][64] bf16, 128B swizzle; attn_tc.cu
bool tc_make_map(void *map, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l, int box_rows);

// NEXT-1 dense-phase score mean; scores.cu
spion_status launch_score_mean(const void *Q, const void *K, const float *lse, int64_t bh, int L, int64_t stride_bh,
                               int64_t stride_l, float scale, float *A, double *sumsq, float *part, int ks,
                               cudaStream_t s);
int score_splits(int64_t bh, int L);
// Alg. 2 / Eq. 2 transition test on three device sums of squares; scores.cu
spion_status launch_transition(const double *sumsq, double alpha, int32_t *flag, double *dist, cudaStream_t s);

// NEXT-4 projection GEMM (tcgen05; head-layout operand gather / output scatter); gemm.cu
spion_status launch_gemm_bf16(const void *A, const void *B, void *C, int M, int N, int K, int a_heads, int c_heads,
                              int L, int H, int batch, float alpha, cudaStream_t s);

// NEXT-4 sub-layer kernels; mha.cu
spion_status launch_heads_permute(const void *src, void *dst, int64_t batch, int L, int W, int H, int d, int to_heads,
                                  cudaStream_t s);
spion_status launch_dropout_residual(const void *y, const void *e, void *out, int64_t n, float p, uint64_t seed,
                                     cudaStream_t s);

// pattern kernels; pattern.cu
size_t pattern_ws_bytes(int L, int block);
spion_status launch_pattern_pool(const float *scores_rows, int L, int B, int F, int row_begin, int row_end, void *ws,
                                 cudaStream_t s);
spion_status launch_pattern_finalize(int L, int B, int kind, long long lo, int frac_pos, int variant, long long T_abs,
                                     void *ws, spion_bsr *out, cudaStream_t s);
spion_status launch_pattern(const float *scores, int L, int B, int F, int kind, long long lo, int frac_pos, int variant,
                            long long T_abs, void *ws, spion_bsr *out, cudaStream_t s);
spion_status launch_bsr_from_mask(const uint8_t *mask, int L, int B, spion_bsr *out, int *flags, cudaStream_t s);

}  // namespace spion
