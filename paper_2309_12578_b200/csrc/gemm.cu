// gemm.cu — tcgen05 GEMM for the sparse-MHA projections (Alg. 5 l.2-3 and
// l.8-9): C[M][N] = alpha * A[M][K] B[N][K]^T, bf16 operands, fp32 accumulation in tensor
// memory, bf16 output.  The head split / concatenation of the sub-layer is folded into the operand
// and output addressing instead of separate permute passes:
//   A: row-major [M][K], or GATHERED from the attention layout [W][batch*H][L][64] — row m = (b, l)
//      token, K-step kk of 64 = head h of tensor w (kk = w*H + h): one TMA box per (tile, K-step);
//   C: row-major [M][N], or SCATTERED into that layout — output column n = (w, h, e), one TMA store
//      box per 64 columns.
// So Q|K|V = X W^{QKV} writes the attention inputs directly, and S W^O reads the attention output
// directly (rows of a 128-token tile never cross a batch item: L % 128 == 0).
//
// Persistent kernel, one CTA per SM, tiles 128 x 128 in N-fastest order (consecutive tiles of a CTA
// share the A rows in L2).  Warps: 0 TMA producer, 1 MMA issuer (TMEM owner), 2..5 epilogue (TMEM
// lane quarter = warp % 4: TMEM -> registers -> bf16 -> SW128 staging -> TMA store).  K-steps of 64
// stream through a 4-stage ring (A 16 KB + B 16 KB per stage); two TMEM accumulators (2 x 128
// columns) let the epilogue of tile i overlap the MMAs of tile i+1; two staging buffers let the TMA
// store of tile i overlap the epilogue of tile i+1.
#include "attn_tc.cuh"

namespace spion {

namespace {
constexpr int GT = 128;            // tile M = N
constexpr int GK = 64;             // K-step (one SW128 row of bf16)
constexpr int G_NST = 4;           // ring stages
constexpr int G_THREADS = 192;
constexpr uint32_t G_TILE = GT * GK * 2;          // 16 KB operand tile
constexpr uint32_t G_STAGE = 2 * G_TILE;          // A + B
constexpr uint32_t G_STG = 2 * G_TILE;            // output staging: two [128][64] bf16 boxes
constexpr size_t G_SMEM = 1024 + G_NST * G_STAGE + 2 * G_STG + 512;
}  // namespace

struct GemmParams {
    int M, N, K;
    int a_heads, c_heads;  // 1: operand A gathered from / output C scattered into [W][BH][L][64]
    int L, H, BH;          // the head layout: L rows per (batch, head), H heads, BH = batch * H
    float alpha;
};

// head-layout coordinates of token row m0 (tile start) and 64-column chunk kk: (l0, plane)
__device__ __forceinline__ void head_coord(const GemmParams &g, int m0, int kk, int &l0, int &plane) {
    const int b = m0 / g.L;
    l0 = m0 - b * g.L;
    const int w = kk / g.H, h = kk - w * g.H;
    plane = w * g.BH + b * g.H + h;
}

__global__ void __launch_bounds__(G_THREADS, 1)
gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC, GemmParams g) {
    constexpr uint32_t IDESC = idesc_bf16(GT, GT, false, false);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sRing = smem;
    uint8_t *sStg = smem + G_NST * G_STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sStg + 2 * G_STG);
    uint64_t *full = bars, *empty = bars + G_NST, *acc_full = bars + 2 * G_NST, *acc_empty = acc_full + 2,
             *stg_free = acc_empty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(stg_free + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < G_NST; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(acc_full + i, 1); mbar_init(acc_empty + i, 128); mbar_init(stg_free + i, 1); }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int mt = g.M / GT, nt = g.N / GT, ntiles = mt * nt, nk = g.K / GK;

    if (warp == 0) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) { prefetch_tmap(&tmA); prefetch_tmap(&tmB); prefetch_tmap(&tmC); }
        int st = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            const int m0 = (t / nt) * GT, n0 = (t % nt) * GT;
            for (int kk = 0; kk < nk; ++kk) {
                mbar_wait(empty + st, ph ^ 1);
                if (elect_one()) {
                    uint8_t *sa = sRing + st * G_STAGE;
                    mbar_arrive_expect_tx(full + st, G_STAGE);
                    if (g.a_heads) {
                        int l0, plane;
                        head_coord(g, m0, kk, l0, plane);
                        tma_load_3d(sa, &tmA, full + st, 0, l0, plane);
                    } else {
                        tma_load_3d(sa, &tmA, full + st, kk * GK, m0, 0);
                    }
                    tma_load_3d(sa + G_TILE, &tmB, full + st, kk * GK, n0, 0);
                }
                __syncwarp();
                if (++st == G_NST) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        int st = 0, it = 0;
        uint32_t ph = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int ab = it & 1;
            if (it >= 2) mbar_wait(acc_empty + ab, ((it >> 1) - 1) & 1);
            tc_fence_after();
            for (int kk = 0; kk < nk; ++kk) {
                mbar_wait(full + st, ph);
                tc_fence_after();
                const uint64_t da = sdesc_sw128(smem_u32(sRing + st * G_STAGE));
                const uint64_t db = sdesc_sw128(smem_u32(sRing + st * G_STAGE + G_TILE));
                if (elect_one()) {
#pragma unroll
                    for (int k = 0; k < GK / 16; ++k) mma_bf16_ss(tmem + ab * GT, da + 2 * k, db + 2 * k, IDESC, (kk | k) != 0);
                    mma_commit(empty + st);
                    if (kk == nk - 1) mma_commit(acc_full + ab);
                }
                __syncwarp();
                if (++st == G_NST) { st = 0; ph ^= 1; }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue (warps 2..5)
        const int q4 = warp & 3;
        const int r = q4 * 32 + lane;  // tile row = TMEM lane
        const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
        const bool leader = warp == 2 && lane == 0;
        int it = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
            const int ab = it & 1, sb = it & 1;
            const int m0 = (t / nt) * GT, n0 = (t % nt) * GT;
            uint8_t *stg = sStg + sb * G_STG;
            mbar_wait(acc_full + ab, (it >> 1) & 1);
            tc_fence_after();
            if (it >= 2) mbar_wait(stg_free + sb, ((it >> 1) - 1) & 1);  // the TMA store two tiles back read it
#pragma unroll
            for (int c = 0; c < 4; ++c) {  // 32-column chunks: box c / 2, half c % 2
                float v[32];
                tmem_ld32(tl + ab * GT + 32 * c, v);
                tmem_ld_wait();
                stage_row_bf16(stg + (c >> 1) * G_TILE, r, v, g.alpha, c & 1);
            }
            tc_fence_before();
            mbar_arrive(acc_empty + ab);
            fence_proxy_async_smem();
            named_bar_sync(1, 128);
            if (leader) {
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    if (g.c_heads) {
                        int l0, plane;
                        head_coord(g, m0, (n0 >> 6) + j, l0, plane);
                        tma_store_3d(&tmC, stg + j * G_TILE, 0, l0, plane);
                    } else {
                        tma_store_3d(&tmC, stg + j * G_TILE, n0 + 64 * j, m0, 0);
                    }
                }
                bulk_commit();
                bulk_wait_read0();
                mbar_arrive(stg_free + sb);
            }
        }
        if (leader) bulk_wait0();
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

// ---------------------------------------------------------------- host
// 3-D bf16 tensor map: dims {inner, rows, planes}, row pitch `pitch` elements, plane pitch `ppitch`
static bool gmap(CUtensorMap *m, const void *base, uint64_t inner, uint64_t rows, uint64_t planes, uint64_t pitch,
                 uint64_t ppitch, uint32_t box_inner, uint32_t box_rows) {
    auto enc = tc_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {inner, rows, planes};
    cuuint64_t strides[2] = {pitch * 2, ppitch * 2};
    cuuint32_t box[3] = {box_inner, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

spion_status launch_gemm_bf16(const void *A, const void *Bm, void *C, int M, int N, int K, int a_heads, int c_heads,
                              int L, int H, int batch, float alpha, cudaStream_t s) {
    static PerDevice attr;
    SPION_CUDA_TRY(smem_attr_once(attr, gemm_bf16_tc_kernel, (int)G_SMEM));
    GemmParams g;
    g.M = M; g.N = N; g.K = K;
    g.a_heads = a_heads; g.c_heads = c_heads;
    g.L = L; g.H = H; g.BH = batch * H;
    g.alpha = alpha;
    CUtensorMap ma, mb, mc;
    const uint64_t BH = (uint64_t)batch * H;
    bool ok = a_heads ? gmap(&ma, A, 64, L, (uint64_t)(K / 64) / H * BH, 64, (uint64_t)L * 64, 64, GT)
                      : gmap(&ma, A, K, M, 1, K, (uint64_t)M * K, 64, GT);
    ok = ok && gmap(&mb, Bm, K, N, 1, K, (uint64_t)N * K, 64, GT);
    ok = ok && (c_heads ? gmap(&mc, C, 64, L, (uint64_t)(N / 64) / H * BH, 64, (uint64_t)L * 64, 64, GT)
                        : gmap(&mc, C, N, M, 1, N, (uint64_t)M * N, 64, GT));
    if (!ok) return SPION_ERR_CUDA;
    const int tiles = (M / GT) * (N / GT);
    const int grid = tiles < tc_num_sms() ? tiles : tc_num_sms();
    gemm_bf16_tc_kernel<<<grid, G_THREADS, G_SMEM, s>>>(ma, mb, mc, g);
    SPION_LAUNCH_CHECK();
    note_tc_launch();
    return SPION_OK;
}

}  // namespace spion
