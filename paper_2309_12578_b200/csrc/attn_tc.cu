// attn_tc.cu — tensor-core (tcgen05 + TMA + TMEM) block-sparse attention, sm_100a.
//
// Shapes: bf16, head dim d = 64, block B in {32, 64}.  Every MMA tile has 128
// rows = S = 128/B consecutive block rows (forward) or block columns
// (backward) of one (batch, head) — "slots".  The pattern is shared by all
// (batch, head), so the work list of a slot tile (the union of its
// slots' column / row lists with a per-entry slot bitmask) is built once by
// the pattern kernel (plan).  Entries absent from a slot contribute exact
// zeros (P = 0), so the result per row equals Eq. 5 on that row's blocks.
//
// Forward (row tiles; Alg. 5 l.5-7, Alg. 6), per (bh, tile):
//   for J in tile list:  S = Q K_J^T (tcgen05, TMEM, double buffered)
//                        -> online softmax, thread = row (tcgen05.ld)
//                        -> P (bf16, smem)  -> O += P V_J (tcgen05, TMEM)
//   epilogue: PAPER lse = logaddexp(m + ln l, ln(L - cnt)) (reading Q1/Q2).
// Backward (column tiles; reading Q17), per (bh, tile of key blocks):
//   for I in tile list:  S^T = K Q_I^T, dP^T = V dO_I^T  (TMEM)
//                        -> P^T = exp(s - lse), dS^T = P^T (dP^T - D)  (thread = key)
//                        -> dV += P^T dO_I, dK += dS^T Q_I (TMEM accumulators)
//                        -> dQ_I = dS K  (M=64 MMA) -> fp32 red.add into dQacc
//
// Warp roles (192 threads): warps 0-3 softmax/epilogue (thread = TMEM lane),
// warp 4 TMA producer, warp 5 MMA issuer (one thread) + TMEM allocator.
// Persistent grid: 2 CTAs per SM, work items (bh, tile) strided by gridDim.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "attn.cuh"
#include "tc_ptx.cuh"

namespace spion {

using namespace tc;

static constexpr int TC_THREADS = 192;
static constexpr int FWD_NST = 3;   // K/V ring stages
static constexpr int BWD_NST = 2;   // Q/dO/lse/D ring stages
static constexpr float LOG2E = 1.4426950408889634f;
static constexpr float LN2 = 0.6931471805599453f;

struct TcParams {
    void *O;              // fwd out (bf16)
    float *lse_out;       // fwd out
    const float *lse;     // bwd in
    const float *D;       // bwd in
    float *dQacc;         // bwd out (fp32)
    void *dK, *dV;        // bwd out (bf16)
    const int *plan;
    const int *brow_ptr;
    int64_t bh, stride_bh, stride_l;
    int L, n, ntiles;
    int mode;
    float scale, scale_log2;
    int off_ptr, off_col, off_msk;  // plan word offsets (fwd: fptr/fcol/fmsk, bwd: bptr/brow/bmsk)
    int off_order;                  // tiles in descending work order
    int off_sched;                  // plan words [off_sched] item counter, [off_sched+1] done counter
    int G;                          // (batch, head) chunk of the scheduling order
};

// ---------------------------------------------------------------- dynamic tile scheduler
// Items (bh, tile) are handed out by an atomic counter in the plan, in chunks of G
// (batch, head): within a chunk, tiles in descending order of work (plan order
// list), each for all G bh.  The producer warp fetches an item and broadcasts it
// through a 4-slot shared-memory ring to the MMA thread and the 4 softmax warps.
// The last CTA to finish resets the counters, so every launch starts from zero.
struct Sched {
    int *item;        // [4]
    uint64_t *full;   // [4], count 1
    uint64_t *empty;  // [4], count 5 (MMA thread + 4 softmax warps)
};

__device__ __forceinline__ int sched_produce(const Sched &sc, int k, int *counter, int nitems) {
    const int slot = k & 3;
    const uint32_t ph = (k >> 2) & 1;
    mbar_wait(sc.empty + slot, ph ^ 1);
    int item = atomicAdd(counter, 1);
    if (item >= nitems) item = -1;
    *reinterpret_cast<volatile int *>(sc.item + slot) = item;
    mbar_arrive(sc.full + slot);
    return item;
}

// whole_warp: all 32 lanes call (one arrival by lane 0 after the warp has read the slot);
// otherwise a single thread calls and arrives.
__device__ __forceinline__ int sched_consume(const Sched &sc, int k, bool whole_warp) {
    const int slot = k & 3;
    const uint32_t ph = (k >> 2) & 1;
    mbar_wait(sc.full + slot, ph);
    const int item = *reinterpret_cast<volatile int *>(sc.item + slot);
    if (whole_warp) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(sc.empty + slot);
    } else {
        mbar_arrive(sc.empty + slot);
    }
    return item;
}

__device__ __forceinline__ void decode_item(int item, const TcParams &p, int &bh, int &t) {
    const int per = p.G * p.ntiles;
    const int c = item / per;
    const int rem = item - c * per;
    const int Gc = min(p.G, (int)p.bh - c * p.G);
    const int k = rem / Gc;
    bh = c * p.G + (rem - k * Gc);
    t = p.plan[p.off_order + k];
}

__device__ __forceinline__ void sched_finish(const TcParams &p) {
    if (threadIdx.x == 0) {
        int *ctr = const_cast<int *>(p.plan) + p.off_sched;
        __threadfence();
        if (atomicAdd(ctr + 1, 1) == (int)gridDim.x - 1) {
            atomicExch(ctr, 0);
            atomicExch(ctr + 1, 0);
            __threadfence();
        }
    }
}

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ============================================================================ forward
template <int B>
__global__ void __launch_bounds__(TC_THREADS, 2)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, TcParams p) {
    constexpr int S = 128 / B;
    constexpr uint32_t KV_BYTES = B * 128;
    constexpr uint32_t IDESC_S = idesc_bf16(128, B, false, false);
    constexpr uint32_t IDESC_PV = idesc_bf16(128, 64, false, true);
    constexpr uint32_t COL_S = 0, COL_O = 128;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sQ = smem;
    uint8_t *sP = smem + 16384;
    uint8_t *sKV = smem + 32768;  // stage st: K at st*16384, V at st*16384 + 8192
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem + 32768 + FWD_NST * 16384);
    uint64_t *q_full = bars + 0, *q_empty = bars + 1, *p_full = bars + 2, *pv_done = bars + 3,
             *tmem_free = bars + 4, *s_full = bars + 5 /*[2]*/, *kv_full = bars + 7 /*[NST]*/,
             *kv_empty = bars + 7 + FWD_NST /*[NST]*/;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 7 + 2 * FWD_NST);
    Sched sc{reinterpret_cast<int *>(bars + 7 + 2 * FWD_NST + 1), bars + 7 + 2 * FWD_NST + 3, bars + 7 + 2 * FWD_NST + 7};

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(p_full, 128);
        mbar_init(pv_done, 1);
        mbar_init(tmem_free, 128);
        mbar_init(s_full + 0, 1);
        mbar_init(s_full + 1, 1);
        for (int i = 0; i < FWD_NST; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        for (int i = 0; i < 4; ++i) { mbar_init(sc.full + i, 1); mbar_init(sc.empty + i, 5); }
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t nitems = p.bh * p.ntiles;
    const int *plan = p.plan;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            prefetch_tmap(&tmQ);
            prefetch_tmap(&tmK);
            prefetch_tmap(&tmV);
            int st = 0;
            uint32_t ph = 0;
            int nq = 0;
            int *counter = const_cast<int *>(plan) + p.off_sched;
            for (int ks = 0;; ++ks) {
                const int item = sched_produce(sc, ks, counter, (int)nitems);
                if (item < 0) break;
                int bh, t;
                decode_item(item, p, bh, t);
                const int beg = plan[p.off_ptr + t], end = plan[p.off_ptr + t + 1];
                if (end == beg) continue;
                if (nq > 0) mbar_wait(q_empty, (nq - 1) & 1);
                mbar_arrive_expect_tx(q_full, 16384);
                tma_load_3d(sQ, &tmQ, q_full, 0, t * 128, bh);
                ++nq;
                for (int j = beg; j < end; ++j) {
                    const int J = plan[p.off_col + j];
                    mbar_wait(kv_empty + st, ph ^ 1);
                    mbar_arrive_expect_tx(kv_full + st, 2 * KV_BYTES);
                    tma_load_3d(sKV + st * 16384, &tmK, kv_full + st, 0, J * B, bh);
                    tma_load_3d(sKV + st * 16384 + 8192, &tmV, kv_full + st, 0, J * B, bh);
                    if (++st == FWD_NST) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0, p_ph = 0;
            int nq = 0;
            const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ));
            const uint64_t dP0 = sdesc_sw128(smem_u32(sP));
            for (int ks = 0;; ++ks) {
                const int item = sched_consume(sc, ks, false);
                if (item < 0) break;
                int bh, t;
                decode_item(item, p, bh, t);
                const int beg = plan[p.off_ptr + t], end = plan[p.off_ptr + t + 1];
                const int cnt = end - beg;
                if (cnt == 0) continue;
                if (nq > 0) { mbar_wait(tmem_free, (nq - 1) & 1); tc_fence_after(); }
                mbar_wait(q_full, nq & 1);
                tc_fence_after();
                ++nq;
                int prev_st = 0;
                for (int jj = 0; jj <= cnt; ++jj) {
                    int cur_st = st;
                    if (jj < cnt) {
                        mbar_wait(kv_full + st, ph);
                        tc_fence_after();
                        const uint32_t sb = jj & 1;
                        const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + st * 16384));
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_bf16_ss(tmem + COL_S + sb * 64, dQ0 + 2 * k, dK0 + 2 * k, IDESC_S, k > 0);
                        mma_commit(s_full + sb);
                        if (jj == cnt - 1) mma_commit(q_empty);
                        if (++st == FWD_NST) { st = 0; ph ^= 1; }
                    }
                    if (jj >= 1) {
                        // O += P(jj-1) V(jj-1)
                        mbar_wait(p_full, p_ph);
                        p_ph ^= 1;
                        tc_fence_after();
                        const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + prev_st * 16384 + 8192), 16, 1024);
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            mma_bf16_ss(tmem + COL_O, dP0 + 2 * k, dV0 + 128 * k, IDESC_PV, (jj - 1 > 0) || (k > 0));
                        mma_commit(pv_done);
                        mma_commit(kv_empty + prev_st);
                    }
                    prev_st = cur_st;
                }
            }
        }
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int r = threadIdx.x;  // tile row = TMEM lane
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
        uint32_t sph0 = 0, sph1 = 0, pv_ph = 0;
        const float sl2 = p.scale_log2;
        __nv_bfloat16 *Obase = static_cast<__nv_bfloat16 *>(p.O);
        for (int ks = 0;; ++ks) {
            const int item = sched_consume(sc, ks, true);
            if (item < 0) break;
            int bh, t;
            decode_item(item, p, bh, t);
            const int beg = plan[p.off_ptr + t], end = plan[p.off_ptr + t + 1];
            const int cnt = end - beg;
            const int I = t * S + slot;
            const int row = t * 128 + r;
            const bool valid = row < p.L;
            const int rcnt = (I < p.n) ? (p.brow_ptr[I + 1] - p.brow_ptr[I]) : 0;
            __nv_bfloat16 *orow = Obase + (int64_t)bh * p.stride_bh + (int64_t)row * p.stride_l;
            float *lrow = p.lse_out + (int64_t)bh * p.L + row;
            if (cnt == 0) {
                if (valid) {
                    uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int c = 0; c < 8; ++c) reinterpret_cast<uint4 *>(orow)[c] = z;
                    *lrow = (p.mode == SPION_SOFTMAX_PAPER) ? logf((float)p.L) : -INFINITY;
                }
                continue;
            }
            float m_run = -INFINITY, l_run = 0.f;
            for (int jj = 0; jj < cnt; ++jj) {
                const int msk = plan[p.off_msk + beg + jj];
                const bool active = (msk >> slot) & 1;  // warp-uniform (32 rows per warp, B >= 32)
                const uint32_t sb = jj & 1;
                if (sb == 0) { mbar_wait(s_full + 0, sph0); sph0 ^= 1; }
                else { mbar_wait(s_full + 1, sph1); sph1 ^= 1; }
                tc_fence_after();
                uint32_t packed[B / 2];
                float alpha = 1.f;
                bool rescale = false;
                if (active) {
                    float s[B];
#pragma unroll
                    for (int h = 0; h < B / 32; ++h) {
                        float v[32];
                        tmem_ld32(tl + COL_S + sb * 64 + h * 32, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) s[h * 32 + i] = v[i] * sl2;
                    }
                    float mx = s[0];
#pragma unroll
                    for (int i = 1; i < B; ++i) mx = fmaxf(mx, s[i]);
                    if (m_run == -INFINITY) {
                        m_run = mx;
                    } else if (mx > m_run + 8.f) {  // rescale only on a large max increase
                        alpha = exp2f(m_run - mx);
                        m_run = mx;
                        rescale = true;
                    }
                    float sum = 0.f;
#pragma unroll
                    for (int i = 0; i < B; i += 2) {
                        const float e0 = exp2f(s[i] - m_run), e1 = exp2f(s[i + 1] - m_run);
                        sum += e0 + e1;
                        packed[i / 2] = pack_bf16(e0, e1);
                    }
                    l_run = l_run * alpha + sum;
                } else {
#pragma unroll
                    for (int i = 0; i < B / 2; ++i) packed[i] = 0u;
                }
                // PV(jj-1) must be complete before P is overwritten and O is touched
                if (jj >= 1) {
                    mbar_wait(pv_done, pv_ph);
                    pv_ph ^= 1;
                    tc_fence_after();
                }
                if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float o[32];
                        tmem_ld32(tl + COL_O + h * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= alpha;
                        tmem_st32(tl + COL_O + h * 32, o);
                    }
                    tmem_st_wait();
                }
#pragma unroll
                for (int c = 0; c < B / 8; ++c) {
                    uint4 v = make_uint4(packed[4 * c], packed[4 * c + 1], packed[4 * c + 2], packed[4 * c + 3]);
                    *reinterpret_cast<uint4 *>(sP + sw128_offset(r, c)) = v;
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(p_full);
            }
            mbar_wait(pv_done, pv_ph);
            pv_ph ^= 1;
            tc_fence_after();
            // ---- epilogue: O / Z and lse (log2 domain internally)
            float f = 0.f, lse2;
            const int64_t ecnt = (int64_t)B * rcnt;
            if (rcnt == 0 || l_run == 0.f) {
                lse2 = (p.mode == SPION_SOFTMAX_PAPER) ? log2f((float)p.L) : -INFINITY;
            } else {
                const float lm = m_run + log2f(l_run);
                if (p.mode == SPION_SOFTMAX_PAPER && ecnt < p.L) {
                    const float lz = log2f((float)(p.L - ecnt));  // Alg. 6 l.15 in the log domain
                    const float hi = fmaxf(lm, lz), lo = fminf(lm, lz);
                    lse2 = hi + log2f(1.f + exp2f(lo - hi));
                } else {
                    lse2 = lm;
                }
                f = exp2f(m_run - lse2);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                float o[32];
                tmem_ld32(tl + COL_O + h * 32, o);
                tmem_ld_wait();
                if (valid) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint4 v = make_uint4(pack_bf16(o[8 * c] * f, o[8 * c + 1] * f),
                                             pack_bf16(o[8 * c + 2] * f, o[8 * c + 3] * f),
                                             pack_bf16(o[8 * c + 4] * f, o[8 * c + 5] * f),
                                             pack_bf16(o[8 * c + 6] * f, o[8 * c + 7] * f));
                        reinterpret_cast<uint4 *>(orow)[h * 4 + c] = v;
                    }
                }
            }
            if (valid) *lrow = lse2 * LN2;
            tc_fence_before();
            mbar_arrive(tmem_free);
        }
    }
    __syncthreads();
    sched_finish(p);
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

// ============================================================================ backward
// D_i = dO_i . O_i (fp32 from the bf16 tensors) and dQacc = 0
__global__ void bwd_prep_tc_kernel(const __nv_bfloat16 *O, const __nv_bfloat16 *dO, float *D, float *dQacc,
                                   int64_t bh, int L, int64_t stride_bh, int64_t stride_l) {
    const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= bh * L) return;
    const int64_t b = row / L, i = row % L;
    const __nv_bfloat162 *o = reinterpret_cast<const __nv_bfloat162 *>(O + b * stride_bh + i * stride_l);
    const __nv_bfloat162 *g = reinterpret_cast<const __nv_bfloat162 *>(dO + b * stride_bh + i * stride_l);
    const float2 a = __bfloat1622float2(o[lane]), c = __bfloat1622float2(g[lane]);
    float s = a.x * c.x + a.y * c.y;
    s = warp_sum(s);
    if (lane == 0) D[row] = s;
    reinterpret_cast<float2 *>(dQacc + row * 64)[lane] = make_float2(0.f, 0.f);
}

__global__ void dq_convert_kernel(const float *dQacc, __nv_bfloat16 *dQ, int64_t bh, int L, int64_t stride_bh,
                                  int64_t stride_l, float scale) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one thread per 8 elements
    if (idx >= bh * L * 8) return;
    const int64_t row = idx >> 3;
    const int c = (int)(idx & 7);
    const int64_t b = row / L, i = row % L;
    const float4 a = reinterpret_cast<const float4 *>(dQacc + row * 64)[2 * c];
    const float4 e = reinterpret_cast<const float4 *>(dQacc + row * 64)[2 * c + 1];
    uint4 v = make_uint4(pack_bf16(a.x * scale, a.y * scale), pack_bf16(a.z * scale, a.w * scale),
                         pack_bf16(e.x * scale, e.y * scale), pack_bf16(e.z * scale, e.w * scale));
    reinterpret_cast<uint4 *>(dQ + b * stride_bh + i * stride_l)[c] = v;
}

template <int B>
__global__ void __launch_bounds__(TC_THREADS, 2)
attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO, TcParams p) {
    constexpr int S = 128 / B;
    constexpr uint32_t TILE = B * 128;  // one Q_I or dO_I tile
    constexpr uint32_t IDESC_ST = idesc_bf16(128, B, false, false);   // S^T, dP^T
    constexpr uint32_t IDESC_DKV = idesc_bf16(128, 64, false, true);  // dV, dK
    constexpr uint32_t IDESC_DQ = idesc_bf16(64, 64, true, true);     // dQ
    constexpr uint32_t COL_S = 0, COL_DP = 64, COL_DQ = 0, COL_DV = 128, COL_DK = 192;
    constexpr uint32_t STAGE = 2 * 8192 + 1024;  // Q, dO (<= 8 KB each), lse, D

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sK = smem, *sV = smem + 16384, *sPt = smem + 32768, *sdSt = smem + 49152;
    uint8_t *sStage = smem + 65536;  // [BWD_NST] x STAGE
    uint64_t *bars = reinterpret_cast<uint64_t *>(sStage + BWD_NST * STAGE);
    uint64_t *kv_full = bars + 0, *kv_empty = bars + 1, *s_full = bars + 2, *p_full = bars + 3,
             *dq_full = bars + 4, *dq_free = bars + 5, *q_full = bars + 6 /*[NST]*/,
             *q_empty = bars + 6 + BWD_NST /*[NST]*/;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6 + 2 * BWD_NST);
    Sched sc{reinterpret_cast<int *>(bars + 6 + 2 * BWD_NST + 1), bars + 6 + 2 * BWD_NST + 3, bars + 6 + 2 * BWD_NST + 7};

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(kv_full, 1);
        mbar_init(kv_empty, 1);
        mbar_init(s_full, 1);
        mbar_init(p_full, 128);
        mbar_init(dq_full, 1);
        mbar_init(dq_free, 128);
        for (int i = 0; i < BWD_NST; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 1); }
        for (int i = 0; i < 4; ++i) { mbar_init(sc.full + i, 1); mbar_init(sc.empty + i, 5); }
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int64_t nitems = p.bh * p.ntiles;
    const int *plan = p.plan;

    if (warp == 4) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            prefetch_tmap(&tmK);
            prefetch_tmap(&tmV);
            prefetch_tmap(&tmQ);
            prefetch_tmap(&tmdO);
            int st = 0;
            uint32_t ph = 0;
            int nk = 0;
            int *counter = const_cast<int *>(plan) + p.off_sched;
            for (int ks = 0;; ++ks) {
                const int item = sched_produce(sc, ks, counter, (int)nitems);
                if (item < 0) break;
                int bh, t;
                decode_item(item, p, bh, t);
                const int beg = plan[p.off_ptr + t], end = plan[p.off_ptr + t + 1];
                if (end == beg) continue;
                if (nk > 0) mbar_wait(kv_empty, (nk - 1) & 1);
                mbar_arrive_expect_tx(kv_full, 32768);
                tma_load_3d(sK, &tmK, kv_full, 0, t * 128, bh);
                tma_load_3d(sV, &tmV, kv_full, 0, t * 128, bh);
                ++nk;
                for (int j = beg; j < end; ++j) {
                    const int I = plan[p.off_col + j];
                    mbar_wait(q_empty + st, ph ^ 1);
                    uint8_t *stg = sStage + st * STAGE;
                    mbar_arrive_expect_tx(q_full + st, 2 * TILE + 2 * B * 4);
                    tma_load_3d(stg, &tmQ, q_full + st, 0, I * B, bh);
                    tma_load_3d(stg + 8192, &tmdO, q_full + st, 0, I * B, bh);
                    bulk_load(stg + 16384, p.lse + (int64_t)bh * p.L + (int64_t)I * B, B * 4, q_full + st);
                    bulk_load(stg + 16384 + 512, p.D + (int64_t)bh * p.L + (int64_t)I * B, B * 4, q_full + st);
                    if (++st == BWD_NST) { st = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int st = 0;
            uint32_t ph = 0, p_ph = 0;
            int nk = 0;
            long long steps = 0;  // steps issued by this CTA (dq_free phases)
            const uint64_t dK0 = sdesc_sw128(smem_u32(sK));
            const uint64_t dV0 = sdesc_sw128(smem_u32(sV));
            const uint64_t dPt0 = sdesc_sw128(smem_u32(sPt));
            const uint64_t ddSt0 = sdesc_sw128(smem_u32(sdSt));
            for (int ks = 0;; ++ks) {
                const int item = sched_consume(sc, ks, false);
                if (item < 0) break;
                int bh, t;
                decode_item(item, p, bh, t);
                const int beg = plan[p.off_ptr + t], end = plan[p.off_ptr + t + 1];
                const int cnt = end - beg;
                if (cnt == 0) continue;
                mbar_wait(kv_full, nk & 1);
                tc_fence_after();
                ++nk;
                for (int jj = 0; jj < cnt; ++jj) {
                    mbar_wait(q_full + st, ph);
                    if (steps > 0) mbar_wait(dq_free, (uint32_t)((steps - 1) & 1));  // S region drained
                    tc_fence_after();
                    uint8_t *stg = sStage + st * STAGE;
                    const uint64_t dQ0 = sdesc_sw128(smem_u32(stg));
                    const uint64_t ddO0 = sdesc_sw128(smem_u32(stg + 8192));
                    // S^T = K Q_I^T ; dP^T = V dO_I^T   (M=128 keys, N=B queries, K=d)
#pragma unroll
                    for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + COL_S, dK0 + 2 * k, dQ0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        mma_bf16_ss(tmem + COL_DP, dV0 + 2 * k, ddO0 + 2 * k, IDESC_ST, k > 0);
                    mma_commit(s_full);
                    mbar_wait(p_full, p_ph);
                    p_ph ^= 1;
                    tc_fence_after();
                    // dV += P^T dO_I ; dK += dS^T Q_I   (M=128 keys, N=d, K=B queries; B operand MN-major)
#pragma unroll
                    for (int k = 0; k < B / 16; ++k)
                        mma_bf16_ss(tmem + COL_DV, dPt0 + 2 * k, ddO0 + 128 * k, IDESC_DKV, (jj > 0) || (k > 0));
#pragma unroll
                    for (int k = 0; k < B / 16; ++k)
                        mma_bf16_ss(tmem + COL_DK, ddSt0 + 2 * k, dQ0 + 128 * k, IDESC_DKV, (jj > 0) || (k > 0));
                    // dQ_I = dS K   (M=64 queries, N=d, K=128 keys; both operands MN-major)
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        mma_bf16_ss(tmem + COL_DQ, ddSt0 + 128 * k, dK0 + 128 * k, IDESC_DQ, k > 0);
                    mma_commit(dq_full);
                    mma_commit(q_empty + st);
                    if (jj == cnt - 1) mma_commit(kv_empty);
                    ++steps;
                    if (++st == BWD_NST) { st = 0; ph ^= 1; }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ softmax / gradients
        const int r = threadIdx.x;  // key row of the tile = TMEM lane
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
        uint32_t s_ph = 0, dq_ph = 0;
        int st = 0;
        uint32_t ph = 0;
        const float sl2 = p.scale_log2;
        for (int ks = 0;; ++ks) {
            const int item = sched_consume(sc, ks, true);
            if (item < 0) break;
            int bh, t;
            decode_item(item, p, bh, t);
            const int beg = plan[p.off_ptr + t], end = plan[p.off_ptr + t + 1];
            const int cnt = end - beg;
            const int key = t * 128 + r;
            const bool valid = key < p.L;
            __nv_bfloat16 *dkrow =
                static_cast<__nv_bfloat16 *>(p.dK) + (int64_t)bh * p.stride_bh + (int64_t)key * p.stride_l;
            __nv_bfloat16 *dvrow =
                static_cast<__nv_bfloat16 *>(p.dV) + (int64_t)bh * p.stride_bh + (int64_t)key * p.stride_l;
            if (cnt == 0) {
                if (valid) {
                    uint4 z = make_uint4(0, 0, 0, 0);
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        reinterpret_cast<uint4 *>(dkrow)[c] = z;
                        reinterpret_cast<uint4 *>(dvrow)[c] = z;
                    }
                }
                continue;
            }
            for (int jj = 0; jj < cnt; ++jj) {
                const int I = plan[p.off_col + beg + jj];
                const int msk = plan[p.off_msk + beg + jj];
                const bool active = (msk >> slot) & 1;
                mbar_wait(q_full + st, ph);  // lse_I, D_I in smem (stage also read by the MMA)
                uint8_t *stg = sStage + st * STAGE;
                const float *slse = reinterpret_cast<const float *>(stg + 16384);
                const float *sD = reinterpret_cast<const float *>(stg + 16384 + 512);
                mbar_wait(s_full, s_ph);
                s_ph ^= 1;
                tc_fence_after();
                uint32_t pk[B / 2], dk[B / 2];
                if (active) {
#pragma unroll
                    for (int h = 0; h < B / 32; ++h) {
                        float sv[32], dp[32];
                        tmem_ld32(tl + COL_S + h * 32, sv);
                        tmem_ld32(tl + COL_DP + h * 32, dp);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const int q = h * 32 + i;
                            const float p0 = exp2f(sv[i] * sl2 - slse[q] * LOG2E);
                            const float p1 = exp2f(sv[i + 1] * sl2 - slse[q + 1] * LOG2E);
                            pk[q / 2] = pack_bf16(p0, p1);
                            dk[q / 2] = pack_bf16(p0 * (dp[i] - sD[q]), p1 * (dp[i + 1] - sD[q + 1]));
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < B / 2; ++i) { pk[i] = 0u; dk[i] = 0u; }
                }
#pragma unroll
                for (int c = 0; c < B / 8; ++c) {
                    *reinterpret_cast<uint4 *>(sPt + sw128_offset(r, c)) =
                        make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                    *reinterpret_cast<uint4 *>(sdSt + sw128_offset(r, c)) =
                        make_uint4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(p_full);
                // dQ_I partial (M=64 layout: rows 16w + lane for lane < 16) -> fp32 reduction in L2
                mbar_wait(dq_full, dq_ph);
                dq_ph ^= 1;
                tc_fence_after();
                {
                    float a[32], b2[32];
                    tmem_ld32(tl + COL_DQ, a);
                    tmem_ld32(tl + COL_DQ + 32, b2);
                    tmem_ld_wait();
                    const int qrow = warp * 16 + lane;
                    if (lane < 16 && qrow < B) {
                        float *dst = p.dQacc + ((int64_t)bh * p.L + (int64_t)I * B + qrow) * 64;
#pragma unroll
                        for (int c = 0; c < 8; ++c) red_add_v4(dst + 4 * c, a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            red_add_v4(dst + 32 + 4 * c, b2[4 * c], b2[4 * c + 1], b2[4 * c + 2], b2[4 * c + 3]);
                    }
                }
                if (jj == cnt - 1) {
                    // epilogue: dK (x scale) and dV rows of this key
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        float kv[32], vv[32];
                        tmem_ld32(tl + COL_DK + h * 32, kv);
                        tmem_ld32(tl + COL_DV + h * 32, vv);
                        tmem_ld_wait();
                        if (valid) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) {
                                reinterpret_cast<uint4 *>(dkrow)[h * 4 + c] = make_uint4(
                                    pack_bf16(kv[8 * c] * p.scale, kv[8 * c + 1] * p.scale),
                                    pack_bf16(kv[8 * c + 2] * p.scale, kv[8 * c + 3] * p.scale),
                                    pack_bf16(kv[8 * c + 4] * p.scale, kv[8 * c + 5] * p.scale),
                                    pack_bf16(kv[8 * c + 6] * p.scale, kv[8 * c + 7] * p.scale));
                                reinterpret_cast<uint4 *>(dvrow)[h * 4 + c] =
                                    make_uint4(pack_bf16(vv[8 * c], vv[8 * c + 1]), pack_bf16(vv[8 * c + 2], vv[8 * c + 3]),
                                               pack_bf16(vv[8 * c + 4], vv[8 * c + 5]),
                                               pack_bf16(vv[8 * c + 6], vv[8 * c + 7]));
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(dq_free);
                if (++st == BWD_NST) { st = 0; ph ^= 1; }
            }
        }
    }
    __syncthreads();
    sched_finish(p);
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

// ============================================================================ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

static bool make_map(CUtensorMap *m, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l,
                     int box_rows) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)L, (cuuint64_t)bh};
    cuuint64_t strides[2] = {(cuuint64_t)stride_l * 2, (cuuint64_t)stride_bh * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool tc_supported(const AttnArgs &a, spion_dtype dt) {
    if (dt != SPION_BF16 || a.d != 64 || !(a.B == 32 || a.B == 64) || !a.plan) return false;
    if (a.stride_l % 8 || a.stride_bh % 8) return false;
    if (a.L % 4) return false;
    static int disabled = -1;
    if (disabled < 0) disabled = getenv("SPION_DISABLE_TC") != nullptr;
    return !disabled && get_encode() != nullptr;
}


static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

static TcParams base_params(const AttnArgs &a, bool fwd) {
    TcParams p;
    memset(&p, 0, sizeof(p));
    PlanLayout pl(a.n, a.B);
    p.plan = a.plan;
    p.brow_ptr = a.brow_ptr;
    p.bh = a.bh;
    p.stride_bh = a.stride_bh;
    p.stride_l = a.stride_l;
    p.L = a.L;
    p.n = a.n;
    p.ntiles = pl.ntiles;
    p.mode = a.mode;
    p.scale = a.scale;
    p.scale_log2 = a.scale * LOG2E;
    p.off_ptr = (int)(fwd ? pl.fptr : pl.bptr);
    p.off_col = (int)(fwd ? pl.fcol : pl.brow);
    p.off_msk = (int)(fwd ? pl.fmsk : pl.bmsk);
    p.off_order = (int)(fwd ? pl.forder : pl.border);
    p.off_sched = fwd ? 8 : 10;
    const int grid = 2 * num_sms();
    int G = (2 * grid + pl.ntiles - 1) / pl.ntiles;
    if (G < 1) G = 1;
    if (G > a.bh) G = (int)a.bh;
    p.G = G;
    return p;
}

static const size_t FWD_SMEM = 1024 + 32768 + FWD_NST * 16384 + 256;
static const size_t BWD_SMEM = 1024 + 65536 + BWD_NST * (2 * 8192 + 1024) + 256;

template <int B>
static spion_status fwd_tc_t(const AttnArgs &a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        SPION_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_tc_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FWD_SMEM));
        attr = true;
    }
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mk, a.K, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !make_map(&mv, a.V, a.L, a.bh, a.stride_bh, a.stride_l, B))
        return SPION_ERR_CUDA;
    TcParams p = base_params(a, true);
    p.O = a.Oout;
    p.lse_out = a.lse_out;
    const int64_t items = a.bh * p.ntiles;
    const int grid = (int)((items < 2LL * num_sms()) ? items : 2LL * num_sms());
    attn_fwd_tc_kernel<B><<<grid, TC_THREADS, FWD_SMEM, s>>>(mq, mk, mv, p);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

template <int B>
static spion_status bwd_tc_t(const AttnArgs &a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        SPION_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_tc_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BWD_SMEM));
        attr = true;
    }
    CUtensorMap mk, mv, mq, mdo;
    if (!make_map(&mk, a.K, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mv, a.V, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mq, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !make_map(&mdo, a.dO, a.L, a.bh, a.stride_bh, a.stride_l, B))
        return SPION_ERR_CUDA;
    // D = rowsum(dO * O), dQacc = 0
    const int64_t rows = a.bh * a.L;
    bwd_prep_tc_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(
        static_cast<const __nv_bfloat16 *>(a.O), static_cast<const __nv_bfloat16 *>(a.dO), const_cast<float *>(a.D),
        a.dQacc, a.bh, a.L, a.stride_bh, a.stride_l);
    SPION_LAUNCH_CHECK();
    TcParams p = base_params(a, false);
    p.lse = a.lse;
    p.D = a.D;
    p.dQacc = a.dQacc;
    p.dK = a.dK;
    p.dV = a.dV;
    const int64_t items = a.bh * p.ntiles;
    const int grid = (int)((items < 2LL * num_sms()) ? items : 2LL * num_sms());
    attn_bwd_tc_kernel<B><<<grid, TC_THREADS, BWD_SMEM, s>>>(mk, mv, mq, mdo, p);
    SPION_LAUNCH_CHECK();
    const int64_t n8 = rows * 8;
    dq_convert_kernel<<<(unsigned)((n8 + 255) / 256), 256, 0, s>>>(a.dQacc, static_cast<__nv_bfloat16 *>(a.dQ), a.bh,
                                                                   a.L, a.stride_bh, a.stride_l, a.scale);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

spion_status launch_fwd_tc(const AttnArgs &a, cudaStream_t s) {
    return a.B == 64 ? fwd_tc_t<64>(a, s) : fwd_tc_t<32>(a, s);
}
spion_status launch_bwd_tc(const AttnArgs &a, cudaStream_t s) {
    return a.B == 64 ? bwd_tc_t<64>(a, s) : bwd_tc_t<32>(a, s);
}

}  // namespace spion
