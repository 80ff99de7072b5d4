// attn_tc.cuh — shared pieces of the tensor-core (tcgen05 + TMA + TMEM) attention kernels:
// compile-time knobs, kernel parameters, the persistent work-item scheduler, the softmax
// exponentials and output staging helpers (device), and the tensor-map / launch helpers (host).
// Used by attn_tc.cu (forward, split backward) and attn_bwd_fused.cu (fused backward).
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <math.h>

#include "attn.cuh"
#include "tc_ptx.cuh"

// compile-time knobs (A/B builds: tools/build_variant.py)
#ifndef SPION_PING
#define SPION_PING 1
#endif
// timing-only debug builds (wrong results): skip the MMAs, or the softmax loads and math
#ifndef SPION_DBG_NOMMA
#define SPION_DBG_NOMMA 0
#endif
#ifndef SPION_DBG_NOSOFTMAX
#define SPION_DBG_NOSOFTMAX 0
#endif
#ifndef SPION_G_MULT  // scheduling chunk: ~this many work items per CTA
#define SPION_G_MULT 4
#endif
#ifndef SPION_HEAVY_AHEAD  // heavy tiles are scheduled this many (batch, head) chunks ahead
#define SPION_HEAVY_AHEAD 2
#endif
#ifndef SPION_NSW  // 1: one S-MMA warp per buffer where one CTA owns the SM (0: a single S-MMA warp)
#define SPION_NSW 0
#endif
#ifndef SPION_DQ_TS  // dQ pass: Q / dO of the item in tensor memory (TS score MMAs) where TMEM allows
#define SPION_DQ_TS 1
#endif
#ifndef SPION_TRACE_EVENTS  // 1: per-role event traces of CTA 0 (tools/trace_*.py; costs issue slots)
#define SPION_TRACE_EVENTS 0
#endif
#ifndef SPION_ITEM_FENCE  // the score-MMA issuer starts an item's MMAs only after the previous item's last
#define SPION_ITEM_FENCE 0  // accumulating MMAs were issued (tensor-pipe order: the accumulator finishes first)
#endif
#ifndef SPION_DEFER_DKV  // item epilogues run after the softmax warps' first block of the next item
#define SPION_DEFER_DKV 0
#endif
#ifndef SPION_DEFER_DQ
#define SPION_DEFER_DQ 0
#endif
#ifndef SPION_DEFER_FWD
#define SPION_DEFER_FWD 0
#endif
#ifndef SPION_DKV_EPI  // dK/dV pass: a dedicated epilogue warpgroup (B = 64)
#define SPION_DKV_EPI 0
#endif
#ifndef SPION_L2HINT  // TMA copies carry L2 eviction priorities (read-once tiles first, gathered blocks last)
#define SPION_L2HINT 1
#endif
#ifndef SPION_LANE0  // the MMA-issuing roles run on one thread (lane 0) instead of a converged warp
#define SPION_LANE0 0
#endif
#define ISSUER() (SPION_LANE0 ? true : elect_one())
#define ROLE_SYNC()                   \
    do {                              \
        if (!SPION_LANE0) __syncwarp(); \
    } while (0)
#ifndef SPION_DKV_TS  // dK/dV pass: K / V of the item in tensor memory (TS score MMAs), NBUF 3 -> 2
#define SPION_DKV_TS 0
#endif
#ifndef SPION_DBG_NOLOAD  // per-block operand tiles not loaded
#define SPION_DBG_NOLOAD 0
#endif
#if SPION_DBG_NOMMA
#define MMA_SS(...) ((void)0)
#define MMA_TS(...) ((void)0)
#else
#define MMA_SS(...) mma_bf16_ss(__VA_ARGS__)
#define MMA_TS(...) mma_bf16_ts(__VA_ARGS__)
#endif
#ifndef SPION_POLY  // of every 16 exponentials, how many run as a polynomial on the FMA pipe
#define SPION_POLY 0
#endif

namespace spion {

using namespace tc;

static constexpr int SCHED_CAP = 128;

// 2^x on the FMA pipe (the SFU does 16 ex2/clk/SM, as many as this does on the FP32 pipe):
// Cody-Waite split x = j + f with j = rint(x) taken from the low mantissa bits of x + 1.5*2^23,
// f in [-0.5, 0.5]; 2^f by a degree-3 relative-minimax polynomial (max rel. error 1.0e-4, far
// below the 2^-9 rounding of P / dS to bf16); 2^j added into the exponent field.  x <= -127
// gives +0 (like ex2.approx.ftz underflow).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -127.f);
    const float t = x + 12582912.f;
    const float f = x - (t - 12582912.f);
    const float q = fmaf(fmaf(fmaf(0.05500883f, f, 0.24221103f), f, 0.69328296f), f, 1.f);
    return __int_as_float(__float_as_int(q) + (__float_as_int(t) << 23));
}
// element i of an unrolled row loop: SPION_POLY of every 16 on the FMA pipe, the rest on the SFU
__device__ __forceinline__ float ex2m(float x, int i) { return (i & 15) < SPION_POLY ? ex2_poly(x) : ex2(x); }
// TMA copies with an L2 eviction priority (SPION_L2HINT; plain copies otherwise)
__device__ __forceinline__ void tma_ld(void *dst, const void *tmap, uint64_t *bar, int c0, int c1, int c2, uint64_t pol) {
    if (SPION_L2HINT) tma_load_3d_hint(dst, tmap, bar, c0, c1, c2, pol);
    else tma_load_3d(dst, tmap, bar, c0, c1, c2);
}
__device__ __forceinline__ void tma_st(const void *tmap, const void *src, int c0, int c1, int c2, uint64_t pol) {
    if (SPION_L2HINT) tma_store_3d_hint(tmap, src, c0, c1, c2, pol);
    else tma_store_3d(tmap, src, c0, c1, c2);
}
static constexpr float LOG2E = 1.4426950408889634f;
static constexpr float LN2 = 0.6931471805599453f;

struct TcParams {
    void *O;              // fwd out / dq in (bf16)
    float *lse_out;       // fwd out
    const float *lse;     // bwd in
    float *D;             // dq out, dkdv in
    float *nlse2;         // dq out: -lse * log2(e) (the dK/dV pass stages it instead of lse)
    void *dQ, *dK, *dV;   // bwd out (bf16)
    const int *plan;
    const int *brow_ptr;
    int64_t bh, stride_bh, stride_l;
    int L, n, ntiles;
    int mode;
    float scale, scale_log2;
    int off_ptr, off_col, off_msk;  // plan word offsets (row tiles: fptr/fcol/fmsk, column tiles: bptr/brow/bmsk)
    int off_order;                  // tiles in descending work order
    int *sched;                     // caller workspace: this launch's work-item counter (zeroed per call)
    int off_heavy;                  // plan word: number of heavy tiles (scheduled first)
    int off_perm;                   // column tiles: plan word offset of bperm (slot -> block column)
    int G;                          // (batch, head) chunk of the scheduling order
    int S;                          // slots per tile
    unsigned long long *trace;      // optional event trace of CTA 0 (SPION_TRACE=1), else null
};

// debug event trace of CTA 0 (SPION_TRACE=1): each recording thread owns a region of
// 1024 (event, globaltimer) pairs and a private counter, so recording is a pair of
// fire-and-forget stores (no atomics on the critical path)
struct Tracer {
    unsigned long long *base;
    int n;
    __device__ Tracer(const TcParams &p, int role) : base(nullptr), n(0) {
        if (p.trace && blockIdx.x == 0) base = p.trace + 16 + role * 2048;
    }
    __device__ __forceinline__ void ev(int id) {
        if (SPION_TRACE_EVENTS && base && n < 2048) {  // one 64-bit store: SM clock << 8 | event id
            base[n] = (unsigned long long)id | ((unsigned long long)clock64() << 8);
            ++n;
        }
    }
};

// offset arithmetic on the __shared__ array (not an integer round trip), so the
// compiler keeps the shared address space and emits LDS/STS for the staged tiles
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
}

// ---------------------------------------------------------------- dynamic tile scheduler
// Items (bh, tile) are handed out by an atomic counter in the caller's workspace (zeroed
// by the host before every call, so launches sharing a pattern never share a counter), in chunks of G
// (batch, head): within a chunk, tiles in descending order of work, each for all G
// bh.  The producer warp fetches an item, stages its header and tile list in a
// 4-slot shared ring, and signals `full`; the MMA thread and the 4 softmax warps
// release the slot (`empty`) when they are done with the item.
struct Sched {
    int *hdr;  // [4][8]: item, bh, t, cnt, rc[0..3] (block-row counts of the slots)
    int *col;  // [4][SCHED_CAP]
    int *msk;  // [4][SCHED_CAP]
    // copies of the plan's small arrays, loaded once per CTA (the per-item fetch then needs
    // one global round trip for the tile's list, after the atomic): [0] heavy-tile count,
    // order[ntiles] at TAB_ORDER, ptr[ntiles + 1] at TAB_PTR, block-row counts at TAB_RC
    int *tab;
    uint64_t *full, *empty;  // [4] each
};
static constexpr int TAB_ORDER = 8, TAB_PTR = TAB_ORDER + SCHED_CAP, TAB_RC = TAB_PTR + SCHED_CAP + 8;
static constexpr int TAB_PERM = TAB_RC;  // column-tile kernels (no block-row counts): plan bperm
static constexpr int SCHED_TAB = TAB_RC + SCHED_CAP;
static constexpr int SCHED_BYTES = (32 + 2 * 4 * SCHED_CAP + SCHED_TAB) * 4;

__device__ __forceinline__ Sched make_sched(uint8_t *area, uint64_t *bars) {
    Sched s;
    s.hdr = reinterpret_cast<int *>(area);
    s.col = s.hdr + 32;
    s.msk = s.col + 4 * SCHED_CAP;
    s.tab = s.msk + 4 * SCHED_CAP;
    s.full = bars;
    s.empty = bars + 4;
    return s;
}

// all threads, before the CTA's first __syncthreads: copy the plan's order, pointers and
// (forward) block-row counts into shared memory
__device__ __forceinline__ void sched_load_tables(const Sched &sc, const TcParams &p, bool want_rc) {
    if (threadIdx.x == 0) sc.tab[0] = p.plan[p.off_heavy];
    for (int i = threadIdx.x; i < p.ntiles; i += blockDim.x) sc.tab[TAB_ORDER + i] = p.plan[p.off_order + i];
    for (int i = threadIdx.x; i <= p.ntiles; i += blockDim.x) sc.tab[TAB_PTR + i] = p.plan[p.off_ptr + i];
    if (want_rc)
        for (int i = threadIdx.x; i < p.n; i += blockDim.x) sc.tab[TAB_RC + i] = p.brow_ptr[i + 1] - p.brow_ptr[i];
    else if (p.off_perm)  // column tiles: the slot -> block column table in the same area
        for (int i = threadIdx.x; i < p.ntiles * p.S; i += blockDim.x) sc.tab[TAB_PERM + i] = p.plan[p.off_perm + i];
}

// `consumers` warps release each slot: the MMA warp and every softmax warp
__device__ __forceinline__ void sched_init(const Sched &sc, int consumers = 5) {
    for (int i = 0; i < 4; ++i) {
        mbar_init(sc.full + i, 1);
        mbar_init(sc.empty + i, consumers);
    }
}

// the next item's index from the plan's atomic counter (lane 0; the value is used by a later
// sched_produce, so the atomic's round trip overlaps the current item's TMA issue)
__device__ __forceinline__ int sched_prefetch(const TcParams &p) {
    return (threadIdx.x & 31) == 0 ? atomicAdd(p.sched, 1) : 0;
}

// The producer fetches an item in two halves, so the global-memory round trips (the item
// counter's atomic, prefetched with sched_prefetch, and the tile's entry lists) overlap its TMA
// issue for the current item: sched_fetch_begin claims ring slot k and issues the list loads
// into registers (lane e holds entries e, e+32, e+64, e+96; n <= SCHED_CAP = 128);
// sched_fetch_end stores them to the slot and signals `full`.  Whole producer warp.
struct SchedFetch {
    int item, bh, t, cnt;
    int col[4], msk[4];
};

__device__ __forceinline__ SchedFetch sched_fetch_begin(const Sched &sc, int k, const TcParams &p, int nitems,
                                                        int pre, Tracer *tr = nullptr) {
    const int lane = threadIdx.x & 31;
    const int slot = k & 3;
    SchedFetch f;
    mbar_wait(sc.empty + slot, ((k >> 2) & 1) ^ 1);
    if (tr && lane == 0) tr->ev(5);
    int item = pre != -2 ? pre : sched_prefetch(p);
    item = __shfl_sync(0xffffffffu, item, 0);
    f.item = item < nitems ? item : -1;
    f.bh = f.t = f.cnt = 0;
    if (f.item < 0) return f;
    // chunks of G (batch, head), each chunk's tiles in descending work order (its K/V or
    // Q/dO stay in L2), with the heavy tiles (> 2x the mean work) of chunk c+A handed out
    // before the light tiles of chunk c (A = SPION_HEAVY_AHEAD): long tiles start A chunks
    // early, so none is left for the end of the launch, while the L2 working set stays
    // A + 1 chunks.  Block order (A = 1): H0, H1, L0, H2, L1, ..., H(C-1), L(C-2), L(C-1)
    const int nh = sc.tab[0];
    const int nbh = (int)p.bh, C = (nbh + p.G - 1) / p.G;
    int rem = item, kk = 0, bh = 0;
    auto take = [&](int c, bool heavy) {
        const int Gc = min(p.G, nbh - c * p.G), sz = (heavy ? nh : p.ntiles - nh) * Gc;
        if (rem < sz) {
            const int k2 = rem / Gc;
            bh = c * p.G + (rem - k2 * Gc);
            kk = heavy ? k2 : nh + k2;
            return true;
        }
        rem -= sz;
        return false;
    };
    bool found = false;
    for (int c = 0; c < min(SPION_HEAVY_AHEAD, C) && !found; ++c) found = take(c, true);
    for (int c = 0; c < C && !found; ++c)
        found = (c + SPION_HEAVY_AHEAD < C && take(c + SPION_HEAVY_AHEAD, true)) || take(c, false);
    const int t = sc.tab[TAB_ORDER + kk];
    const int beg = sc.tab[TAB_PTR + t], cnt = sc.tab[TAB_PTR + t + 1] - beg;
    f.bh = bh;
    f.t = t;
    f.cnt = cnt;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int e = lane + 32 * i;
        f.col[i] = e < cnt ? p.plan[p.off_col + beg + e] : 0;
        f.msk[i] = e < cnt ? p.plan[p.off_msk + beg + e] : 0;
    }
    return f;
}

__device__ __forceinline__ void sched_fetch_end(const Sched &sc, int k, const TcParams &p, const SchedFetch &f,
                                                bool want_rc, Tracer *tr = nullptr) {
    const int lane = threadIdx.x & 31;
    const int slot = k & 3;
    int *h = sc.hdr + slot * 8;
    if (f.item < 0) {
        if (lane == 0) h[0] = -1;
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int e = lane + 32 * i;
            if (e < f.cnt) {
                sc.col[slot * SCHED_CAP + e] = f.col[i];
                sc.msk[slot * SCHED_CAP + e] = f.msk[i];
            }
        }
        if (tr && lane == 0) tr->ev(6);
        if (want_rc && lane < 4) {
            const int I = f.t * p.S + lane;
            h[4 + lane] = (lane < p.S && I < p.n) ? sc.tab[TAB_RC + I] : 0;
        }
        if (lane == 0) { h[0] = f.item; h[1] = f.bh; h[2] = f.t; h[3] = f.cnt; }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(sc.full + slot);
}

// both halves at once; returns the item (-1 = no more work).  pre: a prefetched item index
// (sched_prefetch, valid in lane 0), or -2 to fetch one now
__device__ __forceinline__ int sched_produce(const Sched &sc, int k, const TcParams &p, int nitems, bool want_rc,
                                             int pre = -2, Tracer *tr = nullptr) {
    const SchedFetch f = sched_fetch_begin(sc, k, p, nitems, pre, tr);
    sched_fetch_end(sc, k, p, f, want_rc, tr);
    return f.item;
}

// non-blocking warp-uniform test of an mbarrier phase (lane 0's view, broadcast)
__device__ __forceinline__ bool warp_test(uint64_t *bar, uint32_t parity) {
    return __shfl_sync(0xffffffffu, (int)mbar_test(bar, parity), 0) != 0;
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

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// SPION_TRACE: per-CTA [start, end] globaltimer after the role loops (load balance)
__device__ __forceinline__ void sched_finish(const TcParams &p, unsigned long long t_start) {
    if (p.trace && threadIdx.x == 0) {
        p.trace[16 + 8 * 2048 + 2 * blockIdx.x] = t_start;
        p.trace[16 + 8 * 2048 + 2 * blockIdx.x + 1] = gtimer();
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

// row r, columns [32 half, 32 half + 32) of a [128][64] bf16 SW128 K-major tile in shared
// memory (the TMA box layout): 16-byte chunks at their swizzled place, conflict-free
__device__ __forceinline__ void stage_row_bf16(uint8_t *tile, int r, const float (&v)[32], float f, int half) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        *reinterpret_cast<uint4 *>(tile + sw128_offset(r, half * 4 + c)) =
            make_uint4(pack_bf16(v[8 * c] * f, v[8 * c + 1] * f), pack_bf16(v[8 * c + 2] * f, v[8 * c + 3] * f),
                       pack_bf16(v[8 * c + 4] * f, v[8 * c + 5] * f), pack_bf16(v[8 * c + 6] * f, v[8 * c + 7] * f));
    }
}

__device__ __forceinline__ void zero_row_bf16(__nv_bfloat16 *dst) {
#pragma unroll
    for (int c = 0; c < 8; ++c) reinterpret_cast<uint4 *>(dst)[c] = make_uint4(0, 0, 0, 0);
}

// ---------------------------------------------------------------- host helpers (attn_tc.cu)
// 3-D TMA map over [bh][L][64] bf16, box 64 x box_rows x 1, 128-byte swizzle (cached per thread)
bool tc_map(CUtensorMap *m, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l, int box_rows);
int tc_num_sms();
// cuTensorMapEncodeTiled from the driver (null if unavailable)
PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn();
// which: 0 fwd (row tiles), 1 dq (row tiles), 2 dkdv / fused (column tiles); gmult: ~work items per CTA
// in one (batch, head) scheduling chunk
TcParams tc_base_params(const AttnArgs &a, int which, int ctas, int gmult = SPION_G_MULT);
static const size_t SCHED_AREA = SCHED_BYTES + 1024;  // scheduler ring + mbarriers + TMEM slot

}  // namespace spion
