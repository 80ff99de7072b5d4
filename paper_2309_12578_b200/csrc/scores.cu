// scores.cu — SURVEY §8(f) NEXT-1: the dense-phase score matrix that feeds pattern generation.
//
// A^s = mean over the bh (batch, head) slices of softmax(scale Q K^T) (the attention score
// matrix averaged across heads; batch mean: SURVEY §8(a) a1), as fp32 [L][L], plus
// sum(A^2) for Eq. 2's Frobenius distance.  The row normalisers lse come from the
// tensor-core forward on a dense pattern (spion_score_mean, api.cu); this kernel then forms
// every 128 x 128 output tile once, looping over all bh inside the CTA (no atomics on A):
//   S = Q_tile K_tile^T (tcgen05, N = 128, into one of 4 TMEM buffers) -> p = 2^(s*scale*log2e
//   - lse*log2e) accumulated in registers -> A tile = sum / bh, one coalesced store per row.
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2..(AW+1) accumulators (thread = TMEM
// lane = row; the AW/4 warps of a lane quarter split every S tile's 128 columns).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "attn.cuh"
#include "tc_ptx.cuh"

namespace spion {

using namespace tc;

#ifndef SPION_SCORE_AW  // accumulator warps (8: 64 columns each, 16: 32 columns each)
#define SPION_SCORE_AW 16
#endif
static constexpr int SM_AW = SPION_SCORE_AW, SM_CPW = 512 / SM_AW;  // columns per accumulator thread
static constexpr int SM_NST = 3, SM_NBUF = 4, SM_THREADS = 32 * (2 + SM_AW);
static constexpr uint32_t SM_TILE = 16384;  // 128 rows x 64 bf16, SW128

__global__ void __launch_bounds__(SM_THREADS, 1)
score_mean_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const float *__restrict__ lse, int64_t bh_total, int L, float scale_log2, float *__restrict__ out,
                     double *sumsq, float out_scale) {
    constexpr uint32_t IDESC = idesc_bf16(128, 128, false, false);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t *sQ = smem, *sK = smem + SM_NST * SM_TILE;  // stage s: Q at sQ + s*TILE, K at sK + s*TILE
    uint64_t *bars = reinterpret_cast<uint64_t *>(sK + SM_NST * SM_TILE);
    uint64_t *st_full = bars, *st_empty = bars + SM_NST, *s_full = bars + 2 * SM_NST, *s_free = s_full + SM_NBUF;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(s_free + SM_NBUF);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int i0 = blockIdx.y * 128, j0 = blockIdx.x * 128;
    // (batch, head) range of this CTA: gridDim.z CTAs split the slices of one tile (partial sums)
    const int64_t b_lo = bh_total * blockIdx.z / gridDim.z, bh = bh_total * (blockIdx.z + 1) / gridDim.z - b_lo;
    float *A = out + (int64_t)blockIdx.z * L * L;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SM_NST; ++i) { mbar_init(st_full + i, 1); mbar_init(st_empty + i, 1); }
        for (int i = 0; i < SM_NBUF; ++i) { mbar_init(s_full + i, 1); mbar_init(s_free + i, 32 * SM_AW); }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == 0) {
        // TMA producer: Q rows [i0, i0+128) and K rows [j0, j0+128) of every (batch, head)
        if (lane == 0) { prefetch_tmap(&tmQ); prefetch_tmap(&tmK); }
        for (int64_t b = 0; b < bh; ++b) {
            const int st = (int)(b % SM_NST);
            const uint32_t u = (uint32_t)(b / SM_NST);
            mbar_wait(st_empty + st, (u & 1) ^ 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(st_full + st, 2 * SM_TILE);
                tma_load_3d(sQ + st * SM_TILE, &tmQ, st_full + st, 0, i0, (int)(b_lo + b));
                tma_load_3d(sK + st * SM_TILE, &tmK, st_full + st, 0, j0, (int)(b_lo + b));
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // S = Q K^T into TMEM buffer b % NBUF (128 columns), once the accumulators loaded its last use
        for (int64_t b = 0; b < bh; ++b) {
            const int st = (int)(b % SM_NST), sb = (int)(b % SM_NBUF);
            const uint32_t ub = (uint32_t)(b / SM_NBUF);
            if (ub > 0) mbar_wait(s_free + sb, (ub - 1) & 1);
            mbar_wait(st_full + st, (uint32_t)(b / SM_NST) & 1);
            tc_fence_after();
            const uint64_t dQ = sdesc_sw128(smem_u32(sQ + st * SM_TILE)), dK = sdesc_sw128(smem_u32(sK + st * SM_TILE));
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + sb * 128, dQ + 2 * k, dK + 2 * k, IDESC, k > 0);
                mma_commit(s_full + sb);
                mma_commit(st_empty + st);
            }
            __syncwarp();
        }
    } else {
        // a warp reaches TMEM lanes 32 * (warp % 4) .. + 31: row r = that lane; the AW / 4 warps of
        // a lane quarter split the 128 columns of every S tile (SM_CPW each)
        const int r = (warp & 3) * 32 + lane, cg = (warp - 2) >> 2;
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + cg * SM_CPW;
        const float *lrow = lse + b_lo * L + i0 + r;
        float acc[SM_CPW];
#pragma unroll
        for (int c = 0; c < SM_CPW; ++c) acc[c] = 0.f;
        float nl2 = bh > 0 ? -lrow[0] * 1.4426950408889634f : 0.f;  // -lse * log2(e), one (batch, head) ahead
        for (int64_t b = 0; b < bh; ++b) {
            const int sb = (int)(b % SM_NBUF);
            const float cur = nl2;
            if (b + 1 < bh) nl2 = -lrow[(b + 1) * L] * 1.4426950408889634f;
            mbar_wait(s_full + sb, (uint32_t)(b / SM_NBUF) & 1);
            tc_fence_after();
            float v[SM_CPW];
#pragma unroll
            for (int h = 0; h < SM_CPW / 32; ++h) tmem_ld32(tl + sb * 128 + 32 * h, *reinterpret_cast<float(*)[32]>(v + 32 * h));
            tmem_ld_wait();
            tc_fence_before();
            mbar_arrive(s_free + sb);
#pragma unroll
            for (int c = 0; c < SM_CPW; ++c) acc[c] += ex2(fmaf(v[c], scale_log2, cur));
        }
        const float inv = out_scale;
        float ss = 0.f;
        float4 *dst = reinterpret_cast<float4 *>(A + (int64_t)(i0 + r) * L + j0 + cg * SM_CPW);
#pragma unroll
        for (int c = 0; c < SM_CPW / 4; ++c) {
            const float4 q = make_float4(acc[4 * c] * inv, acc[4 * c + 1] * inv, acc[4 * c + 2] * inv, acc[4 * c + 3] * inv);
            ss = fmaf(q.x, q.x, fmaf(q.y, q.y, fmaf(q.z, q.z, fmaf(q.w, q.w, ss))));
            dst[c] = q;
        }
        if (sumsq) {
            double dss = ss;
            for (int o = 16; o > 0; o >>= 1) dss += __shfl_xor_sync(0xffffffffu, dss, o);
            if (lane == 0) atomicAdd(sumsq, dss);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// sum of the gridDim-split partial tiles in slice order (deterministic), scaled; sum of squares
__global__ void score_reduce_kernel(const float4 *__restrict__ part, int ks, int64_t n4, float inv, float4 *__restrict__ A,
                                    double *sumsq) {
    double ss = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 a = __ldg(part + i);
        for (int z = 1; z < ks; ++z) {
            const float4 b = __ldg(part + z * n4 + i);
            a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
        }
        a.x *= inv; a.y *= inv; a.z *= inv; a.w *= inv;
        A[i] = a;
        ss += (double)(a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w);
    }
    if (sumsq) {
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if ((threadIdx.x & 31) == 0) atomicAdd(sumsq, ss);
    }
}

// (batch, head) split of each output tile: the one with the best wave efficiency over one CTA
// per SM (the kernel holds all 512 TMEM columns), the smallest on ties; 1 when the tiles alone
// fill the GPU (Text: 1024 tiles), e.g. 2 at L = 1024 (64 tiles)
int score_splits(int64_t bh, int L) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t tiles = (int64_t)(L / 128) * (L / 128);
    int best = 1;
    double be = -1.0;
    for (int k = 1; k <= 8 && k <= bh; ++k) {
        const double w = (double)(tiles * k) / sms, e = w / ceil(w);
        if (e > be + 1e-9) { be = e; best = k; }
    }
    return best;
}

spion_status launch_score_mean(const void *Q, const void *K, const float *lse, int64_t bh, int L, int64_t stride_bh,
                               int64_t stride_l, float scale, float *A, double *sumsq, float *part, int ks,
                               cudaStream_t s) {
    alignas(128) CUtensorMap mq, mk;
    if (!tc_make_map(&mq, Q, L, bh, stride_bh, stride_l, 128) || !tc_make_map(&mk, K, L, bh, stride_bh, stride_l, 128))
        return SPION_ERR_CUDA;
    const size_t smem = 1024 + 2 * SM_NST * SM_TILE + 256;
    static PerDevice attr;
    SPION_CUDA_TRY(smem_attr_once(attr, score_mean_tc_kernel, (int)smem));
    if (ks < 1 || !part) ks = 1;
    const float inv = 1.f / (float)bh;
    score_mean_tc_kernel<<<dim3(L / 128, L / 128, ks), SM_THREADS, smem, s>>>(
        mq, mk, lse, bh, L, scale * 1.4426950408889634f, ks == 1 ? A : part, ks == 1 ? sumsq : nullptr,
        ks == 1 ? inv : 1.f);
    SPION_LAUNCH_CHECK();
    if (ks > 1) {
        const int64_t n4 = (int64_t)L * L / 4;
        score_reduce_kernel<<<148 * 8, 256, 0, s>>>(reinterpret_cast<const float4 *>(part), ks, n4, inv,
                                                   reinterpret_cast<float4 *>(A), sumsq);
        SPION_LAUNCH_CHECK();
    }
    return SPION_OK;
}

// Alg. 2 with Eq. 2, one thread in fp64: with s_k = sum (A^s_k)^2 of three
// consecutive dense-phase score matrices, distance_k = | sqrt(s_{k-1}) - sqrt(s_k) |, and the
// training switches to the sparse phase when sqrt((distance_{i-1} - distance_i)^2) < alpha
// (reading Q10: this alpha is the transition tolerance, not the quantile).  Device-side, so the
// test needs no host round trip inside a captured training step.
__global__ void transition_kernel(const double *ss, double alpha, int32_t *flag, double *dist) {
    const double d1 = fabs(sqrt(ss[0]) - sqrt(ss[1]));
    const double d2 = fabs(sqrt(ss[1]) - sqrt(ss[2]));
    const double g = d1 - d2;
    *flag = sqrt(g * g) < alpha ? 1 : 0;
    if (dist) {
        dist[0] = d1;
        dist[1] = d2;
    }
}

spion_status launch_transition(const double *sumsq, double alpha, int32_t *flag, double *dist, cudaStream_t s) {
    transition_kernel<<<1, 1, 0, s>>>(sumsq, alpha, flag, dist);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

}  // namespace spion
