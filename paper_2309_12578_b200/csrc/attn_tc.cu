// attn_tc.cu — tensor-core (tcgen05 + TMA + TMEM) block-sparse attention, sm_100a.
//
// Shapes: bf16, head dim d = 64, block B in {32, 64}.  Every MMA tile has 128
// rows = S = 128/B consecutive block rows (row tiles) or block columns (column
// tiles) of one (batch, head) — "slots".  The pattern is shared by every
// (batch, head), so the work list of a slot tile — the union of its
// slots' column (row) lists, each entry with a slot bitmask — is built once by
// the pattern kernel (the plan).  Entries absent from a slot contribute exact
// zeros (P = 0 / dS = 0), so every row gets exactly Eq. 5 over its own blocks.
// All MMAs are M=128 (full rate on one SM).
//
// attn_fwd_tc   (row tiles; Alg. 5 l.5-7, Alg. 6), per (bh, tile):
//   for J:  S = Q K_J^T (TMEM, double buffered) -> online softmax, thread = row
//           -> P (bf16, smem) -> O += P V_J (TMEM)
//   epilogue: O / Z and lse (PAPER: logaddexp(m + ln l, ln(L - cnt)), readings Q1/Q2)
// attn_bwd_dq_tc (row tiles; reading Q17), per (bh, tile):
//   D = rowsum(dO * O) from the staged tiles (written for the dK/dV kernel);
//   for J:  S = Q K_J^T, dP = dO V_J^T -> dS = exp(S*c - lse)(dP - D) (smem)
//           -> dQ += dS K_J (TMEM);  dQ * scale -> bf16.   No atomics.
// attn_bwd_dkdv_tc (column tiles), per (bh, tile of key blocks):
//   for I:  S^T = K Q_I^T, dP^T = V dO_I^T -> P^T, dS^T (smem)
//           -> dV += P^T dO_I, dK += dS^T Q_I (TMEM);  dK * scale -> bf16.
//
// Warp roles (192 threads): warps 0-3 softmax / epilogue (thread = TMEM lane =
// tile row), warp 4 scheduler + TMA producer, warp 5 MMA issuer (one thread)
// and TMEM allocator.  Persistent grid of 2 CTAs per SM; work items (bh, tile)
// come from an atomic counter in the plan (longest tiles of each bh-chunk first)
// and are broadcast, with their plan entries, through a shared-memory ring.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "attn.cuh"
#include "tc_ptx.cuh"

namespace spion {

using namespace tc;

static constexpr int TC_THREADS = 192;
// ring stages: as many as fit next to the fixed tiles with 2 CTAs per SM (~104 KB each);
// a B=32 stage is half the size of a B=64 one, so it gets twice the depth
template <int B> struct Stages {
    static constexpr int FWD = B == 32 ? 8 : 4;  // K_J + V_J per stage
    static constexpr int DQ = B == 32 ? 6 : 3;   // K_J + V_J per stage
    static constexpr int DKV = B == 32 ? 4 : 2;  // Q_I + dO_I + lse_I + D_I per stage
};
static constexpr int SCHED_CAP = 128;  // max entries of one tile list (nblk <= 128)
static constexpr float LOG2E = 1.4426950408889634f;
static constexpr float LN2 = 0.6931471805599453f;

struct TcParams {
    void *O;              // fwd out / dq in (bf16)
    float *lse_out;       // fwd out
    const float *lse;     // bwd in
    float *D;             // dq out, dkdv in
    void *dQ, *dK, *dV;   // bwd out (bf16)
    const int *plan;
    const int *brow_ptr;
    int64_t bh, stride_bh, stride_l;
    int L, n, ntiles;
    int mode;
    float scale, scale_log2;
    int off_ptr, off_col, off_msk;  // plan word offsets (row tiles: fptr/fcol/fmsk, column tiles: bptr/brow/bmsk)
    int off_order;                  // tiles in descending work order
    int off_sched;                  // plan words [off_sched] item counter, [off_sched+1] done counter
    int G;                          // (batch, head) chunk of the scheduling order
    int S;                          // slots per tile
};

__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    return reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// ---------------------------------------------------------------- dynamic tile scheduler
// Items (bh, tile) are handed out by an atomic counter in the plan, in chunks of G
// (batch, head): within a chunk, tiles in descending order of work, each for all G
// bh.  The producer warp fetches an item, stages its header and tile list in a
// 4-slot shared ring, and signals `full`; the MMA thread and the 4 softmax warps
// release the slot (`empty`, count 5) when they are done with the item.  The last
// CTA to finish resets the counters, so every launch starts from zero.
struct Sched {
    int *hdr;  // [4][8]: item, bh, t, cnt, rc[0..3] (block-row counts of the slots)
    int *col;  // [4][SCHED_CAP]
    int *msk;  // [4][SCHED_CAP]
    uint64_t *full, *empty;  // [4] each
};
static constexpr int SCHED_BYTES = (32 + 2 * 4 * SCHED_CAP) * 4;

__device__ __forceinline__ Sched make_sched(uint8_t *area, uint64_t *bars) {
    Sched s;
    s.hdr = reinterpret_cast<int *>(area);
    s.col = s.hdr + 32;
    s.msk = s.col + 4 * SCHED_CAP;
    s.full = bars;
    s.empty = bars + 4;
    return s;
}

__device__ __forceinline__ void sched_init(const Sched &sc) {
    for (int i = 0; i < 4; ++i) {
        mbar_init(sc.full + i, 1);
        mbar_init(sc.empty + i, 5);
    }
}

// whole producer warp; returns the item (-1 = no more work)
__device__ __forceinline__ int sched_produce(const Sched &sc, int k, const TcParams &p, int nitems, bool want_rc) {
    const int lane = threadIdx.x & 31;
    const int slot = k & 3;
    mbar_wait(sc.empty + slot, ((k >> 2) & 1) ^ 1);
    int item = 0;
    if (lane == 0) item = atomicAdd(const_cast<int *>(p.plan) + p.off_sched, 1);
    item = __shfl_sync(0xffffffffu, item, 0);
    int *h = sc.hdr + slot * 8;
    if (item >= nitems) {
        item = -1;
        if (lane == 0) h[0] = -1;
    } else {
        const int per = p.G * p.ntiles;
        const int c = item / per;
        const int rem = item - c * per;
        const int Gc = min(p.G, (int)p.bh - c * p.G);
        const int kk = rem / Gc;
        const int bh = c * p.G + (rem - kk * Gc);
        const int t = p.plan[p.off_order + kk];
        const int beg = p.plan[p.off_ptr + t], cnt = p.plan[p.off_ptr + t + 1] - beg;
        for (int e = lane; e < cnt; e += 32) {
            sc.col[slot * SCHED_CAP + e] = p.plan[p.off_col + beg + e];
            sc.msk[slot * SCHED_CAP + e] = p.plan[p.off_msk + beg + e];
        }
        if (want_rc && lane < 4) {
            const int I = t * p.S + lane;
            h[4 + lane] = (lane < p.S && I < p.n) ? p.brow_ptr[I + 1] - p.brow_ptr[I] : 0;
        }
        if (lane == 0) { h[0] = item; h[1] = bh; h[2] = t; h[3] = cnt; }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(sc.full + slot);
    return item;
}

__device__ __forceinline__ const int *sched_wait(const Sched &sc, int k) {
    const int slot = k & 3;
    mbar_wait(sc.full + slot, (k >> 2) & 1);
    return sc.hdr + slot * 8;
}

__device__ __forceinline__ void sched_release(const Sched &sc, int k, bool whole_warp) {
    if (whole_warp) {
        __syncwarp();
        if ((threadIdx.x & 31) == 0) mbar_arrive(sc.empty + (k & 3));
    } else {
        mbar_arrive(sc.empty + (k & 3));
    }
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

__device__ __forceinline__ void store_row_bf16(__nv_bfloat16 *dst, const float (&v)[32], float f, int half) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        reinterpret_cast<uint4 *>(dst)[half * 4 + c] =
            make_uint4(pack_bf16(v[8 * c] * f, v[8 * c + 1] * f), pack_bf16(v[8 * c + 2] * f, v[8 * c + 3] * f),
                       pack_bf16(v[8 * c + 4] * f, v[8 * c + 5] * f), pack_bf16(v[8 * c + 6] * f, v[8 * c + 7] * f));
    }
}

__device__ __forceinline__ void zero_row_bf16(__nv_bfloat16 *dst) {
#pragma unroll
    for (int c = 0; c < 8; ++c) reinterpret_cast<uint4 *>(dst)[c] = make_uint4(0, 0, 0, 0);
}

// ============================================================================ forward
template <int B>
__global__ void __launch_bounds__(TC_THREADS, 2)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, TcParams p) {
    constexpr uint32_t KV_BYTES = B * 128;
    constexpr int FWD_NST = Stages<B>::FWD;
    constexpr uint32_t STG = 2 * KV_BYTES;  // K at +0, V at +KV_BYTES
    constexpr uint32_t IDESC_S = idesc_bf16(128, B, false, false);
    constexpr uint32_t IDESC_PV = idesc_bf16(128, 64, false, true);
    constexpr uint32_t COL_S = 0, COL_O = 128;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sQ = smem;
    uint8_t *sP = smem + 16384;
    uint8_t *sKV = smem + 32768;  // stage st: K at st*STG, V at st*STG + KV_BYTES
    uint8_t *sSched = sKV + FWD_NST * STG;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    uint64_t *q_full = bars + 0, *q_empty = bars + 1, *p_full = bars + 2, *pv_done = bars + 3,
             *s_full = bars + 4 /*[2]*/, *kv_full = bars + 6 /*[NST]*/, *kv_empty = bars + 6 + FWD_NST /*[NST]*/;
    Sched sc = make_sched(sSched, bars + 6 + 2 * FWD_NST);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 6 + 2 * FWD_NST + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(p_full, 128);
        mbar_init(pv_done, 1);
        mbar_init(s_full + 0, 1);
        mbar_init(s_full + 1, 1);
        for (int i = 0; i < FWD_NST; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        sched_init(sc);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nitems = (int)(p.bh * p.ntiles);

    if (warp == 4) {
        // ------------------------------------------------------------ scheduler + TMA producer
        if (lane == 0) { prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV); }
        int st = 0, nq = 0;
        uint32_t ph = 0;
        for (int ks = 0;; ++ks) {
            const int item = sched_produce(sc, ks, p, nitems, true);
            if (item < 0) break;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *col = sc.col + (ks & 3) * SCHED_CAP;
            if (lane == 0 && cnt > 0) {
                if (nq > 0) mbar_wait(q_empty, (nq - 1) & 1);
                mbar_arrive_expect_tx(q_full, 16384);
                tma_load_3d(sQ, &tmQ, q_full, 0, t * 128, bh);
                ++nq;
                for (int j = 0; j < cnt; ++j) {
                    mbar_wait(kv_empty + st, ph ^ 1);
                    mbar_arrive_expect_tx(kv_full + st, 2 * KV_BYTES);
                    tma_load_3d(sKV + st * STG, &tmK, kv_full + st, 0, col[j] * B, bh);
                    tma_load_3d(sKV + st * STG + KV_BYTES, &tmV, kv_full + st, 0, col[j] * B, bh);
                    if (++st == FWD_NST) { st = 0; ph ^= 1; }
                }
            }
            __syncwarp();
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            int st = 0, nq = 0;
            uint32_t ph = 0, p_ph = 0;
            const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ));
            const uint64_t dP0 = sdesc_sw128(smem_u32(sP));
            for (int ks = 0;; ++ks) {
                const int *h = sched_wait(sc, ks);
                if (h[0] < 0) break;
                const int cnt = h[3];
                if (cnt > 0) {
                    mbar_wait(q_full, nq & 1);
                    tc_fence_after();
                    ++nq;
                    int prev_st = 0;
                    for (int jj = 0; jj <= cnt; ++jj) {
                        const int cur_st = st;
                        if (jj < cnt) {
                            mbar_wait(kv_full + st, ph);
                            tc_fence_after();
                            const uint32_t sb = jj & 1;
                            const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + st * STG));
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                mma_bf16_ss(tmem + COL_S + sb * 64, dQ0 + 2 * k, dK0 + 2 * k, IDESC_S, k > 0);
                            mma_commit(s_full + sb);
                            if (jj == cnt - 1) mma_commit(q_empty);
                            if (++st == FWD_NST) { st = 0; ph ^= 1; }
                        }
                        if (jj >= 1) {  // O += P(jj-1) V(jj-1)
                            mbar_wait(p_full, p_ph);
                            p_ph ^= 1;
                            tc_fence_after();
                            const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + prev_st * STG + KV_BYTES));
#pragma unroll
                            for (int k = 0; k < B / 16; ++k)
                                mma_bf16_ss(tmem + COL_O, dP0 + 2 * k, dV0 + 128 * k, IDESC_PV, (jj > 1) || (k > 0));
                            mma_commit(pv_done);
                            mma_commit(kv_empty + prev_st);
                        }
                        prev_st = cur_st;
                    }
                }
                sched_release(sc, ks, false);
            }
        }
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int r = threadIdx.x;  // tile row = TMEM lane
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
        uint32_t sph0 = 0, sph1 = 0, pv_ph = 0;
        const float sl2 = p.scale_log2;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], t = h[2], cnt = h[3], rcnt = h[4 + slot];
            const int *msks = sc.msk + (ks & 3) * SCHED_CAP;
            const int row = t * 128 + r;
            const bool valid = row < p.L;
            __nv_bfloat16 *orow =
                static_cast<__nv_bfloat16 *>(p.O) + (int64_t)bh * p.stride_bh + (int64_t)row * p.stride_l;
            float m_run = -INFINITY, l_run = 0.f;
            for (int jj = 0; jj < cnt; ++jj) {
                const bool active = (msks[jj] >> slot) & 1;  // warp-uniform (B >= 32)
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
                    for (int hh = 0; hh < B / 32; ++hh) {
                        float v[32];
                        tmem_ld32(tl + COL_S + sb * 64 + hh * 32, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) s[hh * 32 + i] = v[i] * sl2;
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
                if (jj >= 1) {  // PV(jj-1) complete before P is overwritten and O touched
                    mbar_wait(pv_done, pv_ph);
                    pv_ph ^= 1;
                    tc_fence_after();
                }
                if (__any_sync(0xffffffffu, rescale)) {
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        float o[32];
                        tmem_ld32(tl + COL_O + hh * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= alpha;
                        tmem_st32(tl + COL_O + hh * 32, o);
                    }
                    tmem_st_wait();
                }
#pragma unroll
                for (int c = 0; c < B / 8; ++c)
                    *reinterpret_cast<uint4 *>(sP + sw128_offset(r, c)) =
                        make_uint4(packed[4 * c], packed[4 * c + 1], packed[4 * c + 2], packed[4 * c + 3]);
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(p_full);
            }
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
            if (cnt > 0) {
                mbar_wait(pv_done, pv_ph);
                pv_ph ^= 1;
                tc_fence_after();
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    float o[32];
                    tmem_ld32(tl + COL_O + hh * 32, o);
                    tmem_ld_wait();
                    if (valid) store_row_bf16(orow, o, f, hh);
                }
                tc_fence_before();
            } else if (valid) {
                zero_row_bf16(orow);
            }
            if (valid) p.lse_out[(int64_t)bh * p.L + row] = lse2 * LN2;
            sched_release(sc, ks, true);
        }
    }
    __syncthreads();
    sched_finish(p);
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

// ============================================================================ backward: dQ
template <int B>
__global__ void __launch_bounds__(TC_THREADS, 2)
attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                      const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, TcParams p) {
    constexpr uint32_t KV_BYTES = B * 128;
    constexpr int DQ_NST = Stages<B>::DQ;
    constexpr uint32_t STG = 2 * KV_BYTES;
    constexpr uint32_t IDESC_S = idesc_bf16(128, B, false, false);   // S = Q K^T, dP = dO V^T
    constexpr uint32_t IDESC_DQ = idesc_bf16(128, 64, false, true);  // dQ = dS K
    constexpr uint32_t COL_S = 0, COL_DP = 64, COL_DQ = 128;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    // O is staged in the dS buffer: it is only read (for D) before the first dS is written
    uint8_t *sQ = smem, *sdO = smem + 16384, *sdS = smem + 32768, *sO = sdS;
    uint8_t *sKV = smem + 49152;  // stage st: K at st*STG, V at +KV_BYTES
    uint8_t *sSched = sKV + DQ_NST * STG;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    uint64_t *q_full = bars + 0, *q_empty = bars + 1, *s_full = bars + 2, *ds_full = bars + 3,
             *dq_full = bars + 4, *kv_full = bars + 5 /*[NST]*/, *kv_empty = bars + 5 + DQ_NST /*[NST]*/;
    Sched sc = make_sched(sSched, bars + 5 + 2 * DQ_NST);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 5 + 2 * DQ_NST + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
        mbar_init(s_full, 1);
        mbar_init(ds_full, 128);
        mbar_init(dq_full, 1);
        for (int i = 0; i < DQ_NST; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        sched_init(sc);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nitems = (int)(p.bh * p.ntiles);

    if (warp == 4) {
        if (lane == 0) {
            prefetch_tmap(&tmQ); prefetch_tmap(&tmdO); prefetch_tmap(&tmO);
            prefetch_tmap(&tmK); prefetch_tmap(&tmV);
        }
        int st = 0, nq = 0;
        uint32_t ph = 0;
        for (int ks = 0;; ++ks) {
            const int item = sched_produce(sc, ks, p, nitems, false);
            if (item < 0) break;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *col = sc.col + (ks & 3) * SCHED_CAP;
            if (lane == 0 && cnt > 0) {
                if (nq > 0) mbar_wait(q_empty, (nq - 1) & 1);
                mbar_arrive_expect_tx(q_full, 3 * 16384);
                tma_load_3d(sQ, &tmQ, q_full, 0, t * 128, bh);
                tma_load_3d(sdO, &tmdO, q_full, 0, t * 128, bh);
                tma_load_3d(sO, &tmO, q_full, 0, t * 128, bh);
                ++nq;
                for (int j = 0; j < cnt; ++j) {
                    mbar_wait(kv_empty + st, ph ^ 1);
                    mbar_arrive_expect_tx(kv_full + st, 2 * KV_BYTES);
                    tma_load_3d(sKV + st * STG, &tmK, kv_full + st, 0, col[j] * B, bh);
                    tma_load_3d(sKV + st * STG + KV_BYTES, &tmV, kv_full + st, 0, col[j] * B, bh);
                    if (++st == DQ_NST) { st = 0; ph ^= 1; }
                }
            }
            __syncwarp();
        }
    } else if (warp == 5) {
        if (lane == 0) {
            int st = 0, nq = 0;
            uint32_t ph = 0, ds_ph = 0;
            const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ));
            const uint64_t ddO0 = sdesc_sw128(smem_u32(sdO));
            const uint64_t ddS0 = sdesc_sw128(smem_u32(sdS));
            for (int ks = 0;; ++ks) {
                const int *h = sched_wait(sc, ks);
                if (h[0] < 0) break;
                const int cnt = h[3];
                if (cnt > 0) {
                    mbar_wait(q_full, nq & 1);
                    tc_fence_after();
                    ++nq;
                    for (int jj = 0; jj < cnt; ++jj) {
                        mbar_wait(kv_full + st, ph);
                        tc_fence_after();
                        const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + st * STG));
                        const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + st * STG + KV_BYTES));
#pragma unroll
                        for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + COL_S, dQ0 + 2 * k, dK0 + 2 * k, IDESC_S, k > 0);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_bf16_ss(tmem + COL_DP, ddO0 + 2 * k, dV0 + 2 * k, IDESC_S, k > 0);
                        mma_commit(s_full);
                        mbar_wait(ds_full, ds_ph);
                        ds_ph ^= 1;
                        tc_fence_after();
                        // dQ += dS K_J  (A = dS [rows][keys] K-major, B = K_J as N=d x K=keys, MN-major)
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            mma_bf16_ss(tmem + COL_DQ, ddS0 + 2 * k, dK0 + 128 * k, IDESC_DQ, (jj > 0) || (k > 0));
                        mma_commit(kv_empty + st);
                        if (jj == cnt - 1) { mma_commit(dq_full); mma_commit(q_empty); }
                        if (++st == DQ_NST) { st = 0; ph ^= 1; }
                    }
                }
                sched_release(sc, ks, false);
            }
        }
    } else {
        const int r = threadIdx.x;  // query row of the tile
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
        uint32_t q_ph = 0, s_ph = 0, dq_ph = 0;
        const float sl2 = p.scale_log2;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *msks = sc.msk + (ks & 3) * SCHED_CAP;
            const int row = t * 128 + r;
            const bool valid = row < p.L;
            __nv_bfloat16 *dqrow =
                static_cast<__nv_bfloat16 *>(p.dQ) + (int64_t)bh * p.stride_bh + (int64_t)row * p.stride_l;
            if (cnt == 0) {
                if (valid) zero_row_bf16(dqrow);
                sched_release(sc, ks, true);
                continue;
            }
            const float lse2 = valid ? p.lse[(int64_t)bh * p.L + row] * LOG2E : 0.f;
            mbar_wait(q_full, q_ph);
            q_ph ^= 1;
            // D_i = dO_i . O_i from the staged (swizzled) tiles
            float Dr = 0.f;
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const uint4 a = *reinterpret_cast<const uint4 *>(sO + sw128_offset(r, c));
                const uint4 g = *reinterpret_cast<const uint4 *>(sdO + sw128_offset(r, c));
                const uint32_t av[4] = {a.x, a.y, a.z, a.w}, gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&av[i]));
                    const float2 fg = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&gv[i]));
                    Dr = fmaf(fa.x, fg.x, fmaf(fa.y, fg.y, Dr));
                }
            }
            if (valid) p.D[(int64_t)bh * p.L + row] = Dr;
            for (int jj = 0; jj < cnt; ++jj) {
                const bool active = (msks[jj] >> slot) & 1;
                mbar_wait(s_full, s_ph);  // also implies dQ(jj-1) finished reading sdS
                s_ph ^= 1;
                tc_fence_after();
#pragma unroll
                for (int hh = 0; hh < B / 32; ++hh) {
                    uint32_t pk[16];
                    if (active) {
                        float sv[32], dp[32];
                        tmem_ld32(tl + COL_S + hh * 32, sv);
                        tmem_ld32(tl + COL_DP + hh * 32, dp);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const float p0 = exp2f(fmaf(sv[i], sl2, -lse2));
                            const float p1 = exp2f(fmaf(sv[i + 1], sl2, -lse2));
                            pk[i / 2] = pack_bf16(p0 * (dp[i] - Dr), p1 * (dp[i + 1] - Dr));
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) pk[i] = 0u;
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        *reinterpret_cast<uint4 *>(sdS + sw128_offset(r, hh * 4 + c)) =
                            make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(ds_full);
            }
            mbar_wait(dq_full, dq_ph);
            dq_ph ^= 1;
            tc_fence_after();
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float v[32];
                tmem_ld32(tl + COL_DQ + hh * 32, v);
                tmem_ld_wait();
                if (valid) store_row_bf16(dqrow, v, p.scale, hh);
            }
            tc_fence_before();
            sched_release(sc, ks, true);
        }
    }
    __syncthreads();
    sched_finish(p);
    if (warp == 5) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

// ============================================================================ backward: dK, dV
// K/V tiles are double buffered across items; P^T and dS^T never leave the SM:
// they are written as packed bf16 over the S^T / dP^T columns of TMEM and feed
// the dV / dK MMAs as the A operand straight from tensor memory.
template <int B>
__global__ void __launch_bounds__(TC_THREADS, 2)
attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                        TcParams p) {
    constexpr uint32_t TILE = B * 128;
    constexpr int DKV_NST = Stages<B>::DKV;
    constexpr uint32_t STAGE = 2 * TILE + 1024;  // Q_I, dO_I, lse_I, D_I
    constexpr uint32_t IDESC_ST = idesc_bf16(128, B, false, false);   // S^T = K Q^T, dP^T = V dO^T
    constexpr uint32_t IDESC_DKV = idesc_bf16(128, 64, false, true);  // dV += P^T dO, dK += dS^T Q
    constexpr uint32_t COL_S = 0, COL_DP = 64, COL_DV = 128, COL_DK = 192;  // P^T over S^T, dS^T over dP^T

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sKV = smem;  // buffer kb: K at kb*32768, V at kb*32768 + 16384
    uint8_t *sStage = smem + 65536;
    uint8_t *sSched = sStage + DKV_NST * STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    uint64_t *kv_full = bars + 0 /*[2]*/, *kv_empty = bars + 2 /*[2]*/, *s_full = bars + 4, *p_full = bars + 5,
             *acc_full = bars + 6, *q_full = bars + 7 /*[NST]*/, *q_empty = bars + 7 + DKV_NST /*[NST]*/;
    Sched sc = make_sched(sSched, bars + 7 + 2 * DKV_NST);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 7 + 2 * DKV_NST + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        mbar_init(s_full, 1);
        mbar_init(p_full, 128);
        mbar_init(acc_full, 1);
        for (int i = 0; i < DKV_NST; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 1); }
        sched_init(sc);
        fence_barrier_init();
    }
    if (warp == 5) tmem_alloc<256>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nitems = (int)(p.bh * p.ntiles);

    if (warp == 4) {
        if (lane == 0) { prefetch_tmap(&tmK); prefetch_tmap(&tmV); prefetch_tmap(&tmQ); prefetch_tmap(&tmdO); }
        int st = 0, nk = 0;
        uint32_t ph = 0;
        for (int ks = 0;; ++ks) {
            const int item = sched_produce(sc, ks, p, nitems, false);
            if (item < 0) break;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *rows = sc.col + (ks & 3) * SCHED_CAP;
            if (lane == 0 && cnt > 0) {
                const int kb = nk & 1;
                if (nk >= 2) mbar_wait(kv_empty + kb, ((nk >> 1) - 1) & 1);
                mbar_arrive_expect_tx(kv_full + kb, 32768);
                tma_load_3d(sKV + kb * 32768, &tmK, kv_full + kb, 0, t * 128, bh);
                tma_load_3d(sKV + kb * 32768 + 16384, &tmV, kv_full + kb, 0, t * 128, bh);
                ++nk;
                for (int j = 0; j < cnt; ++j) {
                    const int I = rows[j];
                    mbar_wait(q_empty + st, ph ^ 1);
                    uint8_t *stg = sStage + st * STAGE;
                    mbar_arrive_expect_tx(q_full + st, 2 * TILE + 2 * B * 4);
                    tma_load_3d(stg, &tmQ, q_full + st, 0, I * B, bh);
                    tma_load_3d(stg + TILE, &tmdO, q_full + st, 0, I * B, bh);
                    bulk_load(stg + 2 * TILE, p.lse + (int64_t)bh * p.L + (int64_t)I * B, B * 4, q_full + st);
                    bulk_load(stg + 2 * TILE + 512, p.D + (int64_t)bh * p.L + (int64_t)I * B, B * 4, q_full + st);
                    if (++st == DKV_NST) { st = 0; ph ^= 1; }
                }
            }
            __syncwarp();
        }
    } else if (warp == 5) {
        if (lane == 0) {
            int st = 0, nk = 0;
            uint32_t ph = 0, p_ph = 0;
            for (int ks = 0;; ++ks) {
                const int *h = sched_wait(sc, ks);
                if (h[0] < 0) break;
                const int cnt = h[3];
                if (cnt > 0) {
                    const int kb = nk & 1;
                    mbar_wait(kv_full + kb, (nk >> 1) & 1);
                    tc_fence_after();
                    ++nk;
                    const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + kb * 32768));
                    const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + kb * 32768 + 16384));
                    for (int jj = 0; jj < cnt; ++jj) {
                        mbar_wait(q_full + st, ph);
                        tc_fence_after();
                        uint8_t *stg = sStage + st * STAGE;
                        const uint64_t dQ0 = sdesc_sw128(smem_u32(stg));
                        const uint64_t ddO0 = sdesc_sw128(smem_u32(stg + TILE));
#pragma unroll
                        for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + COL_S, dK0 + 2 * k, dQ0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            mma_bf16_ss(tmem + COL_DP, dV0 + 2 * k, ddO0 + 2 * k, IDESC_ST, k > 0);
                        mma_commit(s_full);
                        if (jj == cnt - 1) mma_commit(kv_empty + kb);  // K/V no longer read by this item
                        mbar_wait(p_full, p_ph);
                        p_ph ^= 1;
                        tc_fence_after();
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            mma_bf16_ts(tmem + COL_DV, tmem + COL_S + 8 * k, ddO0 + 128 * k, IDESC_DKV, (jj > 0) || (k > 0));
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            mma_bf16_ts(tmem + COL_DK, tmem + COL_DP + 8 * k, dQ0 + 128 * k, IDESC_DKV, (jj > 0) || (k > 0));
                        mma_commit(q_empty + st);
                        if (jj == cnt - 1) mma_commit(acc_full);
                        if (++st == DKV_NST) { st = 0; ph ^= 1; }
                    }
                }
                sched_release(sc, ks, false);
            }
        }
    } else {
        const int r = threadIdx.x;  // key row of the tile = TMEM lane
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
        uint32_t s_ph = 0, a_ph = 0, ph = 0;
        int st = 0;
        const float sl2 = p.scale_log2;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *msks = sc.msk + (ks & 3) * SCHED_CAP;
            const int key = t * 128 + r;
            const bool valid = key < p.L;
            __nv_bfloat16 *dkrow =
                static_cast<__nv_bfloat16 *>(p.dK) + (int64_t)bh * p.stride_bh + (int64_t)key * p.stride_l;
            __nv_bfloat16 *dvrow =
                static_cast<__nv_bfloat16 *>(p.dV) + (int64_t)bh * p.stride_bh + (int64_t)key * p.stride_l;
            if (cnt == 0) {
                if (valid) { zero_row_bf16(dkrow); zero_row_bf16(dvrow); }
                sched_release(sc, ks, true);
                continue;
            }
            for (int jj = 0; jj < cnt; ++jj) {
                const bool active = (msks[jj] >> slot) & 1;
                mbar_wait(q_full + st, ph);
                const float *slse = reinterpret_cast<const float *>(sStage + st * STAGE + 2 * TILE);
                const float *sD = slse + 128;
                mbar_wait(s_full, s_ph);
                s_ph ^= 1;
                tc_fence_after();
#pragma unroll
                for (int hh = 0; hh < B / 32; ++hh) {
                    uint32_t pk[16], dk[16];
                    if (active) {
                        float sv[32], dp[32];
                        tmem_ld32(tl + COL_S + hh * 32, sv);
                        tmem_ld32(tl + COL_DP + hh * 32, dp);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            const int q = hh * 32 + i;
                            const float p0 = exp2f(fmaf(sv[i], sl2, -slse[q] * LOG2E));
                            const float p1 = exp2f(fmaf(sv[i + 1], sl2, -slse[q + 1] * LOG2E));
                            pk[i / 2] = pack_bf16(p0, p1);
                            dk[i / 2] = pack_bf16(p0 * (dp[i] - sD[q]), p1 * (dp[i + 1] - sD[q + 1]));
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) { pk[i] = 0u; dk[i] = 0u; }
                    }
                    // packed bf16 P^T / dS^T over the (already read) S^T / dP^T columns
                    tmem_st16(tl + COL_S + hh * 16, pk);
                    tmem_st16(tl + COL_DP + hh * 16, dk);
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full);
                if (++st == DKV_NST) { st = 0; ph ^= 1; }
            }
            mbar_wait(acc_full, a_ph);
            a_ph ^= 1;
            tc_fence_after();
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float kv[32], vv[32];
                tmem_ld32(tl + COL_DK + hh * 32, kv);
                tmem_ld32(tl + COL_DV + hh * 32, vv);
                tmem_ld_wait();
                if (valid) {
                    store_row_bf16(dkrow, kv, p.scale, hh);
                    store_row_bf16(dvrow, vv, 1.f, hh);
                }
            }
            tc_fence_before();
            sched_release(sc, ks, true);
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

// [bh][L][64] bf16 viewed as a 3-D tensor; box = 64 x box_rows x 1, 128-byte swizzle
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
    if (a.L % 4 || a.n > SCHED_CAP) return false;
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

// which: 0 fwd (row tiles), 1 dq (row tiles), 2 dkdv (column tiles)
static TcParams base_params(const AttnArgs &a, int which) {
    TcParams p;
    memset(&p, 0, sizeof(p));
    PlanLayout pl(a.n, a.B);
    const bool rows = which != 2;
    p.plan = a.plan;
    p.brow_ptr = a.brow_ptr;
    p.bh = a.bh;
    p.stride_bh = a.stride_bh;
    p.stride_l = a.stride_l;
    p.L = a.L;
    p.n = a.n;
    p.ntiles = pl.ntiles;
    p.S = pl.S;
    p.mode = a.mode;
    p.scale = a.scale;
    p.scale_log2 = a.scale * LOG2E;
    p.off_ptr = (int)(rows ? pl.fptr : pl.bptr);
    p.off_col = (int)(rows ? pl.fcol : pl.brow);
    p.off_msk = (int)(rows ? pl.fmsk : pl.bmsk);
    p.off_order = (int)(rows ? pl.forder : pl.border);
    p.off_sched = 8 + 2 * which;
    const int grid = 2 * num_sms();
    int G = (2 * grid + pl.ntiles - 1) / pl.ntiles;
    if (G < 1) G = 1;
    if (G > a.bh) G = (int)a.bh;
    p.G = G;
    return p;
}

static const size_t SCHED_AREA = SCHED_BYTES + 256;
template <int B> static size_t fwd_smem() { return 1024 + 32768 + Stages<B>::FWD * 2 * B * 128 + SCHED_AREA; }
template <int B> static size_t dq_smem() { return 1024 + 49152 + Stages<B>::DQ * 2 * B * 128 + SCHED_AREA; }
template <int B> static size_t dkv_smem() { return 1024 + 65536 + Stages<B>::DKV * (2 * B * 128 + 1024) + SCHED_AREA; }

static int grid_for(const TcParams &p) {
    const int64_t items = p.bh * p.ntiles;
    return (int)((items < 2LL * num_sms()) ? items : 2LL * num_sms());
}

template <int B>
static spion_status fwd_tc_t(const AttnArgs &a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        SPION_CUDA_TRY(cudaFuncSetAttribute(attn_fwd_tc_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fwd_smem<B>()));
        attr = true;
    }
    CUtensorMap mq, mk, mv;
    if (!make_map(&mq, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mk, a.K, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !make_map(&mv, a.V, a.L, a.bh, a.stride_bh, a.stride_l, B))
        return SPION_ERR_CUDA;
    TcParams p = base_params(a, 0);
    p.O = a.Oout;
    p.lse_out = a.lse_out;
    attn_fwd_tc_kernel<B><<<grid_for(p), TC_THREADS, fwd_smem<B>(), s>>>(mq, mk, mv, p);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

template <int B>
static spion_status bwd_tc_t(const AttnArgs &a, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        SPION_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dq_tc_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dq_smem<B>()));
        SPION_CUDA_TRY(cudaFuncSetAttribute(attn_bwd_dkdv_tc_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dkv_smem<B>()));
        attr = true;
    }
    CUtensorMap mq128, mdo128, mo128, mkB, mvB, mk128, mv128, mqB, mdoB;
    if (!make_map(&mq128, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mdo128, a.dO, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mo128, a.O, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mkB, a.K, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !make_map(&mvB, a.V, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !make_map(&mk128, a.K, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mv128, a.V, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !make_map(&mqB, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !make_map(&mdoB, a.dO, a.L, a.bh, a.stride_bh, a.stride_l, B))
        return SPION_ERR_CUDA;
    // 1) dQ (row tiles) and D = rowsum(dO * O)
    TcParams p = base_params(a, 1);
    p.O = const_cast<void *>(a.O);
    p.lse = a.lse;
    p.D = const_cast<float *>(a.D);
    p.dQ = a.dQ;
    attn_bwd_dq_tc_kernel<B><<<grid_for(p), TC_THREADS, dq_smem<B>(), s>>>(mq128, mdo128, mo128, mkB, mvB, p);
    SPION_LAUNCH_CHECK();
    // 2) dK, dV (column tiles)
    TcParams q = base_params(a, 2);
    q.lse = a.lse;
    q.D = const_cast<float *>(a.D);
    q.dK = a.dK;
    q.dV = a.dV;
    attn_bwd_dkdv_tc_kernel<B><<<grid_for(q), TC_THREADS, dkv_smem<B>(), s>>>(mk128, mv128, mqB, mdoB, q);
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
