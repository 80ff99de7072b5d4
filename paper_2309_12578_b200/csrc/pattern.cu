// pattern.cu — SPION sparsity-pattern generation on sm_100a (Alg. 3/4).
//
// K1 pattern_pool_kernel  (HBM-bound stencil): q = rint(A*2^32); Eq. 3 diagonal
//    convolution (centred, zero padded, ones on the diagonal; reading Q5) fused
//    with Eq. 4 B x B pooling (sums; reading Q7), exact in 64-bit integers.
//    Identity used: pooling a diagonal box filter is a sum, over the filter
//    taps f, of B x B box sums shifted by (f, f):
//       pool(I,J) = sum_x sum_{f in F_I(x)} Wrow(x, J*B + f),
//       F_I(x) = [max(x-IB-B+1, -h), min(x-IB, h)],  Wrow(x,s) = sum_{q<B} A(x, s+q)
//    and a contiguous range of Wrow is a difference of the second row prefix
//    sum PP.  One warp owns one source row segment at a time; the float4 loads
//    of its next row are in flight while the current row is scanned.
// K2 pattern_finalize_kernel (one CTA): threshold by exact order statistics,
//    max-neighbour edges as 128-bit row bitboards, flood fill as a row sweep
//    (the reach along a row's right-edges is a carry chain: one 128-bit add),
//    forced diagonal, block-CSR/CSC and the attention work plan from popcounts
//    and bit scans.
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"

namespace spion {

#ifndef SPION_GROUP_HEAVY  // plan: column tiles over the block columns sorted by count (0: natural order)
#define SPION_GROUP_HEAVY 1
#endif
#ifndef SPION_HEAVY_FIRST  // plan: tiles with > 2x the mean work scheduled first (attention tail)
#define SPION_HEAVY_FIRST 1
#endif
// ---------------------------------------------------------------- K1
#ifndef SPION_K1_MIN_ROWS  // source rows per warp at least (row split of a block row over CTAs)
#define SPION_K1_MIN_ROWS 4
#endif
#ifndef SPION_K1_PER_SM  // resident K1 CTAs per SM (register cap of the K4 = 4 instantiation)
#define SPION_K1_PER_SM 3
#endif
static constexpr int K1_WARPS = 8;
static constexpr int K1_MAXP = 2;  // (target row, column) pairs per lane

struct K1Geom {
    int L, B, h, A, nI, JC, n_cc, RP;  // RP: source rows per CTA (grid.z splits the B rows)
    int Ioff, nrows;                   // the launch covers source block rows [Ioff, Ioff + nrows)
};

// Window of one CTA: positions [g4, g4 + 128*K4) of a source row (float4-aligned, g4 <= c0);
// lane l owns positions [4*K4*l, 4*K4*(l+1)).
static bool k1_geom(int L, int B, int F, int K4, K1Geom &g, int Ioff = 0, int nrows = -1) {
    g.L = L;
    g.Ioff = Ioff;
    g.nrows = nrows < 0 ? L / B : nrows;
    g.B = B;
    g.h = (F - 1) / 2;
    g.A = (g.h + B - 1) / B;
    g.nI = 2 * g.A + 1;
    const int n = L / B;
    // positions used: [0, W + o] with W = JC*B + 2h, o <= 3
    int jmax = (128 * K4 - 2 * g.h - 4) / B;
    jmax = min(jmax, 32 * K1_MAXP / g.nI);
    if (jmax < 1) return false;
    const int n_cc = (n + jmax - 1) / jmax;
    g.JC = (n + n_cc - 1) / n_cc;
    g.n_cc = (n + g.JC - 1) / g.JC;
    // split the rows of a block row over rs CTAs (>= K1_MIN_ROWS rows per warp each): the rs with the best
    // wave efficiency (waves / ceil(waves)) over the resident CTA slots, the smallest on ties
    static int slots = 0;
    if (!slots) {
        int dev = 0, sms = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        slots = SPION_K1_PER_SM * sms;
    }
    int rs = 1;
    double best = -1.0;
    for (int r = 1; r == 1 || B / r >= SPION_K1_MIN_ROWS * K1_WARPS; r *= 2) {
        const double w = (double)g.n_cc * g.nrows * r / slots, eff = w / ceil(w);
        if (eff > best + 1e-9) { best = eff; rs = r; }
    }
    g.RP = (B + rs - 1) / rs;
    return true;
}

template <int K4>
struct K1Cfg {
    static constexpr int CH = 4 * K4;                    // positions per lane
    static constexpr bool POW2 = (K4 & (K4 - 1)) == 0;
    static constexpr int LOGK4 = K4 == 2 ? 1 : K4 == 4 ? 2 : K4 == 8 ? 3 : 0;
    static constexpr bool HOLD = K4 <= 8;                // lane's q in registers, next row prefetched
    // staging (float4): v at v + v/K4 when K4 is even (an odd lane stride keeps the LDS.128 of a
    // lane's own chunk conflict-free); PP (u64): element-major, lane-minor (conflict-free STS.64)
    static constexpr int STAGE4 = POW2 ? 32 * (K4 + 1) : 32 * K4;
    static constexpr size_t WARP_BYTES = (size_t)STAGE4 * 16 + (size_t)32 * CH * 8;
    static __device__ __forceinline__ int sidx(int v) { return POW2 ? v + (v >> LOGK4) : v; }
    static __device__ __forceinline__ int own4(int lane, int i) { return POW2 ? lane * (K4 + 1) + i : lane * K4 + i; }
    static __device__ __forceinline__ int ppidx(int pos) { return (pos % CH) * 32 + pos / CH; }
};

// K4 = 4 (every LRA shape): registers capped for 3 resident CTAs per SM (78 regs, no spill;
// uncapped it took 96+ and 2 CTAs per SM: -2 us at L = 2048/4096).  The wider windows would spill.
template <int K4>
__global__ void __launch_bounds__(K1_WARPS * 32, K4 == 4 ? SPION_K1_PER_SM : 1)
pattern_pool_kernel(const float *__restrict__ A, K1Geom g, unsigned long long *__restrict__ pool,
                    unsigned long long *__restrict__ bad_count) {
    using C = K1Cfg<K4>;
    constexpr int CH = C::CH;
    extern __shared__ __align__(16) unsigned char k1_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = g.L, B = g.B, h = g.h, n = L / B;
    // A: the rows of the launch's source block rows (row 0 = source row Ioff * B); I0: the block row
    // in the pool's index space
    const int cc = blockIdx.x, I0 = blockIdx.y + g.Ioff;
    const int J0 = cc * g.JC;
    const int ncols = min(g.JC, n - J0);
    const int W = ncols * B + 2 * h;  // window-relative columns k in [0, W], column = c0 + k
    const int c0 = J0 * B - h;
    const int g4 = (c0 >= 0) ? (c0 & ~3) : -((-c0 + 3) & ~3);
    const int o = c0 - g4;            // position = k + o
    const int n4 = (W + o + 1 + 3) >> 2;
    unsigned char *wbase = k1_smem + (size_t)warp * C::WARP_BYTES;
    float4 *stage = reinterpret_cast<float4 *>(wbase);
    unsigned long long *pp = reinterpret_cast<unsigned long long *>(wbase + (size_t)C::STAGE4 * 16);
    unsigned long long *s_acc = reinterpret_cast<unsigned long long *>(k1_smem + (size_t)K1_WARPS * C::WARP_BYTES);
    const int npairs = g.nI * ncols;
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) s_acc[p] = 0ull;

    // loop-invariant (target row offset a, column jj) pairs of this lane
    int pa[K1_MAXP], pj[K1_MAXP];
    unsigned long long acc[K1_MAXP];
#pragma unroll
    for (int t = 0; t < K1_MAXP; ++t) {
        const int p = lane + 32 * t;
        pa[t] = p < npairs ? p / ncols - g.A : (1 << 20);
        pj[t] = p < npairs ? p % ncols : 0;
        acc[t] = 0ull;
    }
    // which of this lane's float4 loads hit [0, L) (the same for every row): zero padding elsewhere
    unsigned vmask = 0;
#pragma unroll
    for (int i = 0; i < K4; ++i) {
        const int v = lane + 32 * i;
        const int gc = g4 + 4 * v;
        if (v < n4 && gc >= 0 && gc < L) vmask |= 1u << i;
    }
    const int colbase = g4 + 4 * lane;
    bool bad = false;
    const int u_begin = blockIdx.z * g.RP, u_end = min(B, u_begin + g.RP);
    __syncthreads();

    auto load_row = [&](int u, float4 (&dst)[K4]) {
        const float *arow = A + (size_t)(blockIdx.y * B + u) * L + colbase;
#pragma unroll
        for (int i = 0; i < K4; ++i)
            dst[i] = ((vmask >> i) & 1u) ? __ldg(reinterpret_cast<const float4 *>(arow + 128 * i))
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    // q = rint(a * 2^32) (reading Q8; a * 2^32 is exact in fp32, round half to even).  For a in
    // [0, 1) q < 2^32 is the u32 conversion; a = 1 saturates it to 2^32 - 1 and is fixed up below.
    auto lo32 = [](float a) -> unsigned { return __float2uint_rn(a * 4294967296.0f); };
    auto elem = [](const float4 &f, int t) -> float { return t == 0 ? f.x : t == 1 ? f.y : t == 2 ? f.z : f.w; };

    float4 cur[K4];
    int u = u_begin + warp;
    if (C::HOLD && u < u_end) load_row(u, cur);
    for (; u < u_end; u += K1_WARPS) {
        if (!C::HOLD) load_row(u, cur);
#pragma unroll
        for (int i = 0; i < K4; ++i) stage[C::sidx(lane + 32 * i)] = cur[i];
        __syncwarp();
        if (C::HOLD && u + K1_WARPS < u_end) load_row(u + K1_WARPS, cur);  // next row in flight

        // pass 1 over the lane chunk: tot = sum q, ppl = sum_e q_e (CH-1-e) (the chunk's P-sum share)
        unsigned lo[C::HOLD ? CH : 1];
        unsigned long long tot = 0, ppl = 0;
        unsigned mxb = 0;  // max of the bit patterns: every element in [0, 1) <=> mxb < bits(1.0f)
#pragma unroll
        for (int i = 0; i < K4; ++i) {
            const float4 f = stage[C::own4(lane, i)];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float a = elem(f, t);
                mxb = max(mxb, __float_as_uint(a));
                const unsigned l = lo32(a);
                if constexpr (C::HOLD) lo[4 * i + t] = l;
                tot += l;
                ppl += (unsigned long long)l * (unsigned)(CH - 1 - (4 * i + t));
            }
        }
        const bool slow = !__all_sync(0xffffffffu, mxb < 0x3f800000u);
        unsigned fix = 0;  // HOLD: bit e set where q_e = 2^32 (a = 1): one more than the saturated u32
        if (slow) {
#pragma unroll
            for (int i = 0; i < K4; ++i) {
                const float4 f = stage[C::own4(lane, i)];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float a = elem(f, t);
                    if (!(a >= 0.f && a <= 1.f)) bad = true;
                    if (a >= 1.f) {
                        const int e = 4 * i + t;
                        if constexpr (C::HOLD) fix |= 1u << e;
                        tot += 1;
                        ppl += (unsigned long long)(CH - 1 - e);
                    }
                }
            }
        }
        // P at the chunk start (off1) and PP at the chunk start (off2); PP of every position
        const unsigned long long off1 = warp_excl_scan_u64(tot, lane);
        const unsigned long long off2 = warp_excl_scan_u64((unsigned long long)CH * off1 + ppl, lane);
        unsigned long long run = off1, run2 = off2;
        if (C::HOLD && !slow) {  // warp-uniform common case: no a = 1 fix-ups
#pragma unroll
            for (int e = 0; e < CH; ++e) {
                pp[e * 32 + lane] = run2;
                run2 += run;
                run += (unsigned long long)lo[C::HOLD ? e : 0];
            }
        } else
#pragma unroll
        for (int i = 0; i < K4; ++i) {
            float4 f;
            if constexpr (!C::HOLD) f = stage[C::own4(lane, i)];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int e = 4 * i + t;
                unsigned long long qv;
                if constexpr (C::HOLD) {
                    qv = (unsigned long long)lo[e] + ((fix >> e) & 1u);
                } else {
                    const float a = elem(f, t);
                    qv = (unsigned long long)lo32(a) + (a >= 1.f ? 1u : 0u);
                }
                pp[e * 32 + lane] = run2;
                run2 += run;
                run += qv;
            }
        }
        __syncwarp();
        // contributions of source row x = I0*B + u to pool rows I0+a, columns J0+jj:
        //   sum_{f in F} Wrow(x, (J0+jj)*B + f) = (PP[s1+1+B] - PP[s0+B]) - (PP[s1+1] - PP[s0])
        auto PP = [&](int k) -> unsigned long long { return pp[C::ppidx(k + o)]; };
#pragma unroll
        for (int t = 0; t < K1_MAXP; ++t) {
            const int a = pa[t];
            const int I = I0 + a;
            if (I < 0 || I >= n) continue;
            const int r = u - a * B;
            const int f0 = max(r - B + 1, -h), f1 = min(r, h);
            if (f0 > f1) continue;
            const int s0 = pj[t] * B + h + f0, s1 = pj[t] * B + h + f1;
            acc[t] += (PP(s1 + 1 + B) - PP(s0 + B)) - (PP(s1 + 1) - PP(s0));
        }
        __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < K1_MAXP; ++t) {
        const int p = lane + 32 * t;
        if (p < npairs && acc[t]) atomicAdd(&s_acc[p], acc[t]);
    }
    // warps that saw a score outside [0, 1] (a sum, so partial pools of several devices add up)
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicAdd(bad_count, 1ull);
    __syncthreads();
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
        const int a = p / ncols - g.A, jj = p % ncols;
        const int I = I0 + a;
        if (I < 0 || I >= n || s_acc[p] == 0ull) continue;
        atomicAdd(&pool[(size_t)I * n + (J0 + jj)], s_acc[p]);
    }
}

template <int K4>
static size_t k1_smem_bytes(const K1Geom &g) {
    return (size_t)K1_WARPS * K1Cfg<K4>::WARP_BYTES + (size_t)g.nI * g.JC * 8;
}

template <int K4>
static spion_status k1_launch(const float *scores, const K1Geom &g, unsigned long long *pool,
                              unsigned long long *bad, cudaStream_t s) {
    static PerDevice attr;
    SPION_CUDA_TRY(smem_attr_once(attr, pattern_pool_kernel<K4>));
    const int rs = (g.B + g.RP - 1) / g.RP;
    pattern_pool_kernel<K4><<<dim3(g.n_cc, g.nrows, rs), K1_WARPS * 32, k1_smem_bytes<K4>(g), s>>>(scores, g, pool, bad);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

// ---------------------------------------------------------------- K2
#ifndef SPION_K2_THREADS
#define SPION_K2_THREADS 1024
#endif
static constexpr int K2_THREADS = SPION_K2_THREADS;
static constexpr int K2_MAXN = 128;  // n = L/B <= 128: one row of the block grid is 4 x 32 bits

// 128-bit row bitboard (bit c = block column c)
struct Bits {
    unsigned long long lo, hi;
};
__device__ __forceinline__ Bits b_and(Bits a, Bits b) { return {a.lo & b.lo, a.hi & b.hi}; }
__device__ __forceinline__ Bits b_or(Bits a, Bits b) { return {a.lo | b.lo, a.hi | b.hi}; }
__device__ __forceinline__ Bits b_xor(Bits a, Bits b) { return {a.lo ^ b.lo, a.hi ^ b.hi}; }
__device__ __forceinline__ Bits b_shl1(Bits a) { return {a.lo << 1, (a.hi << 1) | (a.lo >> 63)}; }
__device__ __forceinline__ Bits b_add(Bits a, Bits b) {
    const unsigned long long lo = a.lo + b.lo;
    return {lo, a.hi + b.hi + (lo < a.lo ? 1ull : 0ull)};
}
__device__ __forceinline__ Bits b_bit(int c) {
    return c < 64 ? Bits{1ull << c, 0ull} : Bits{0ull, 1ull << (c - 64)};
}
__device__ __forceinline__ Bits b_ones(int n) {  // bits [0, n), 1 <= n <= 128
    if (n >= 128) return {~0ull, ~0ull};
    if (n > 64) return {~0ull, ~0ull >> (128 - n)};
    return {~0ull >> (64 - n), 0ull};
}
__device__ __forceinline__ int b_popc(Bits a) { return __popcll(a.lo) + __popcll(a.hi); }
// the row bitboard stored as 4 x 32-bit ballot words in shared memory
__device__ __forceinline__ Bits b_load(const unsigned *w) {
    const uint4 v = *reinterpret_cast<const uint4 *>(w);
    return {(unsigned long long)v.x | ((unsigned long long)v.y << 32),
            (unsigned long long)v.z | ((unsigned long long)v.w << 32)};
}
__device__ __forceinline__ void b_store(unsigned *w, Bits a) {
    *reinterpret_cast<uint4 *>(w) =
        make_uint4((unsigned)a.lo, (unsigned)(a.lo >> 32), (unsigned)a.hi, (unsigned)(a.hi >> 32));
}
__device__ __forceinline__ unsigned b_get(const unsigned *w, int c) { return (w[c >> 5] >> (c & 31)) & 1u; }

// k-th smallest (0-based) of v[0..N) by MSD radix selection, 8-bit digits.  Once the digit
// bucket holding the k-th value has <= 32 members, they are compacted and one warp ranks them
// directly (the remaining low digits would each cost a full histogram pass).
__device__ long long block_select_kth(const long long *v, int N, long long k, unsigned int *hist,
                                      long long *bc, int top_shift) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long prefix = 0;
    for (int shift = top_shift; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        const unsigned long long hmask = (shift >= 56) ? 0ull : (~0ull << (shift + 8));
        for (int i = tid; i < N; i += blockDim.x) {
            unsigned long long x = (unsigned long long)v[i];
            if ((x & hmask) == prefix) atomicAdd(&hist[(x >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            unsigned int c[8];
            unsigned int s = 0;
#pragma unroll
            for (int t = 0; t < 8; ++t) { c[t] = hist[lane * 8 + t]; s += c[t]; }
            int ex = warp_excl_scan_i32((int)s, lane);
            long long below = ex;
#pragma unroll
            for (int t = 0; t < 8; ++t) {
                if (k >= below && k < below + (long long)c[t]) { bc[0] = lane * 8 + t; bc[1] = below; bc[2] = c[t]; }
                below += c[t];
            }
            if (lane == 0) bc[3] = 0;
        }
        __syncthreads();
        prefix |= ((unsigned long long)bc[0]) << shift;
        k -= bc[1];
        const long long cnt = bc[2];
        if (shift > 0 && cnt <= 32) {
            // compact the bucket's members (hist[0..32) reused as the list) and rank them in one warp
            const unsigned long long m = ~0ull << shift;
            unsigned long long *cand = reinterpret_cast<unsigned long long *>(hist);
            __syncthreads();
            for (int i = tid; i < N; i += blockDim.x) {
                const unsigned long long x = (unsigned long long)v[i];
                if ((x & m) == prefix) cand[atomicAdd(reinterpret_cast<unsigned long long *>(&bc[3]), 1ull)] = x;
            }
            __syncthreads();
            if (warp == 0) {
                const unsigned long long x = lane < cnt ? cand[lane] : ~0ull;
                int less = 0, eq_before = 0;
                for (int j = 0; j < (int)cnt; ++j) {
                    const unsigned long long y = __shfl_sync(0xffffffffu, x, j);
                    less += y < x;
                    eq_before += (y == x) && (j < lane);
                }
                if (lane < cnt && less + eq_before == k) bc[0] = (long long)x;
            }
            __syncthreads();
            const long long r = bc[0];
            __syncthreads();
            return r;
        }
        __syncthreads();
    }
    return (long long)prefix;
}

struct K2Args {
    const long long *pool;  // [n][n] fixed-point pool sums
    int n, block;
    int kind;               // spion_threshold_kind
    long long lo;           // LINEAR: floor(hpos); NEAREST: rank k
    int frac_pos;           // LINEAR: frac > 0
    long long T_abs;        // ABSOLUTE: gt <=> x > T_abs
    int variant;            // spion_pattern_flags
    int *flags;
    const unsigned long long *bad;  // K1's count of warps that saw a score outside [0, 1] (nullable)
    int *brow_ptr, *bcol_idx, *bcol_ptr, *brow_idx, *nnzb;
    uint8_t *mask;
    int nnzb_cap;
    int *plan;
    unsigned long long *trace;  // debug (SPION_TRACE=1): phase timestamps
};

__device__ __forceinline__ void k2_stamp(const K2Args &a, int k) {
    if (a.trace && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[k] = t;
    }
}

// shared scratch of the BSR / plan builder
struct K2Scratch {
    unsigned *flw;   // [K2_MAXN][4] row bitboards of the final block mask
    unsigned *colw;  // [K2_MAXN][4] column bitboards (bit r of column c)
    int *cnt;        // [2 * K2_MAXN]
    int *off;        // [2 * (K2_MAXN + 1)]
    int *perm;       // [K2_MAXN + 32] column-tile order (plan bperm)
};

// exclusive scans of cnt[0..m) and cnt[m..2m) into off[0..m] and off[m+1..2m+1]; warp 0 only
__device__ void scan2(const int *cnt, int *off, int m) {
    const int lane = threadIdx.x & 31;
    const int per = (m + 31) / 32;
    for (int which = 0; which < 2; ++which) {
        const int *c = cnt + which * m;
        int *o = off + which * (m + 1);
        int loc = 0;
        for (int t = 0; t < per; ++t) { const int r = lane * per + t; if (r < m) loc += c[r]; }
        int ex = warp_excl_scan_i32(loc, lane);
        for (int t = 0; t < per; ++t) { const int r = lane * per + t; if (r < m) { o[r] = ex; ex += c[r]; } }
        if (lane == 31) o[m] = ex;
    }
    __syncwarp();  // lanes read offsets written by other lanes (racecheck)
}

// Block-CSR / CSC / plan from the row bitboards sc.flw (all threads of the CTA).
__device__ void build_bsr_and_plan(const K2Args &a, const K2Scratch &sc) {
    const int n = a.n, tid = threadIdx.x, nthr = blockDim.x;
    // column bitboards: thread c gathers bit c of every row (warp-uniform broadcast reads)
    for (int c = tid; c < n; c += nthr) {
        unsigned w[4] = {0u, 0u, 0u, 0u};
        const int cw = c >> 5, cb = c & 31;
        for (int r = 0; r < n; ++r) w[r >> 5] |= ((sc.flw[r * 4 + cw] >> cb) & 1u) << (r & 31);
        *reinterpret_cast<uint4 *>(sc.colw + c * 4) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    __syncthreads();
    k2_stamp(a, 7);
    for (int r = tid; r < 2 * n; r += nthr)
        sc.cnt[r] = b_popc(b_load(r < n ? sc.flw + r * 4 : sc.colw + (r - n) * 4));
    __syncthreads();
    if (tid < 32) {
        scan2(sc.cnt, sc.off, n);
    } else if (a.plan) {
        // column-tile order (plan bperm), alongside warp 0's scan: block columns by descending
        // count (stable).  Tiling consecutive columns pairs each stripe column (vertical stripes:
        // long, overlapping row sets) with band columns, so most of the stripe's union entries
        // carry one useful slot of S; sorted by count, stripes share tiles with stripes and the
        // band columns stay mostly consecutive (union entries over the LRA-shaped patterns:
        // -28 % at Text and Image).  Row tiles keep the natural order.  plan[7]: heavy columns
        // (more than twice the mean count), a prefix of the order.
        const PlanLayout pl(n, a.block);
        const int w = (tid >> 5) - 1, nw = (nthr >> 5) - 1, lane = tid & 31;
        for (int c = w; c < n; c += nw) {
            const int cc = SPION_GROUP_HEAVY ? sc.cnt[n + c] : 0;
            int rank = 0;
            for (int v0 = 0; v0 < n; v0 += 32) {
                const int v = v0 + lane;
                const int cv = v < n ? (SPION_GROUP_HEAVY ? sc.cnt[n + v] : 0) : -1;
                rank += __popc(__ballot_sync(0xffffffffu, v < n && (cv > cc || (cv == cc && v < c))));
            }
            if (lane == 0) sc.perm[rank] = c;
        }
        if (w == 0) {
            int tot = 0;
            for (int c = lane; c < n; c += 32) tot += sc.cnt[n + c];
            for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
            int hv = 0;
            for (int c = lane; c < n; c += 32) hv += (long long)sc.cnt[n + c] * n > 2LL * tot;
            for (int o = 16; o > 0; o >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, o);
            if (lane == 0) a.plan[7] = hv;
            for (int i = n + lane; i < pl.ntiles * pl.S; i += 32) sc.perm[i] = n;
        }
    }
    __syncthreads();
    const int nnzb = sc.off[n];
    if (tid == 0) {
        *a.nnzb = nnzb;
        if (nnzb > a.nnzb_cap && a.flags) atomicOr(a.flags, FLAG_CAPACITY);
    }
    k2_stamp(a, 8);
    for (int r = tid; r <= n; r += nthr) { a.brow_ptr[r] = sc.off[r]; a.bcol_ptr[r] = sc.off[n + 1 + r]; }
    // ascending column (row) indices: one warp per row (column), lane l owns bits [4l, 4l + 4)
    const int lane = tid & 31;
    for (int r = tid >> 5; r < 2 * n; r += nthr >> 5) {
        const bool row = r < n;
        const unsigned *w = row ? sc.flw + r * 4 : sc.colw + (r - n) * 4;
        const unsigned nib = (w[lane >> 3] >> ((lane & 7) * 4)) & 15u;
        int o = (row ? sc.off[r] : sc.off[n + 1 + (r - n)]) + warp_excl_scan_i32(__popc(nib), lane);
        int *dst = row ? a.bcol_idx : a.brow_idx;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if ((nib >> k) & 1u) {
                if (o < a.nnzb_cap) dst[o] = 4 * lane + k;
                ++o;
            }
    }
    k2_stamp(a, 9);
    if (a.mask) {
        const int N = n * n;
        for (int i = tid; i < N; i += nthr) a.mask[i] = (uint8_t)b_get(sc.flw + (i / n) * 4, i % n);
    }
    if (!a.plan) return;
    // attention work plan: slot tiles of S consecutive block rows (fwd) / block columns (bwd);
    // one entry per column (row) in the union of the tile's S rows (columns), with a slot mask
    const PlanLayout pl(n, a.block);
    int *plan = a.plan;
    __syncthreads();
    k2_stamp(a, 10);
    for (int i = tid; i < pl.ntiles * pl.S; i += nthr) plan[pl.bperm + i] = sc.perm[i];
    for (int t = tid; t < 2 * pl.ntiles; t += nthr) {
        const bool fwd = t < pl.ntiles;
        const int tt = fwd ? t : t - pl.ntiles;
        const unsigned *src = fwd ? sc.flw : sc.colw;
        Bits u{0ull, 0ull};
        for (int s = 0; s < pl.S; ++s) {
            const int r = fwd ? tt * pl.S + s : sc.perm[tt * pl.S + s];
            if (r < n) u = b_or(u, b_load(src + r * 4));
        }
        sc.cnt[t] = b_popc(u);
    }
    __syncthreads();
    if (tid < 32) {
        scan2(sc.cnt, sc.off, pl.ntiles);
        for (int r = tid; r <= pl.ntiles; r += 32) {
            plan[pl.fptr + r] = sc.off[r];
            plan[pl.bptr + r] = sc.off[pl.ntiles + 1 + r];
        }
        // heavy tiles (more than twice the mean work; e.g. the columns of vertical stripes): the
        // attention kernels schedule these first for every (batch, head), so no long tile is left
        // for the end of the launch (the load-balance tail)
        int heavy[2];
        for (int which = 0; which < 2; ++which) {
            const int *c = sc.cnt + which * pl.ntiles;
            const long long tot = sc.off[which * (pl.ntiles + 1) + pl.ntiles];
            int hv = 0;
            for (int t = tid; t < pl.ntiles; t += 32) hv += SPION_HEAVY_FIRST && (long long)c[t] * pl.ntiles > 2 * tot;
            for (int o = 16; o > 0; o >>= 1) hv += __shfl_xor_sync(0xffffffffu, hv, o);
            heavy[which] = hv;
        }
        if (tid == 0) {
            plan[0] = n; plan[1] = pl.S; plan[2] = pl.ntiles;
            plan[3] = sc.off[pl.ntiles];
            plan[4] = sc.off[2 * pl.ntiles + 1];
            for (int w = 8; w < 16; ++w) plan[w] = 0;  // scheduler counters start at zero
            plan[5] = heavy[0];  // heavy row tiles (a prefix of the descending work order)
            plan[6] = heavy[1];  // heavy column tiles
        }
    }
    __syncthreads();
    k2_stamp(a, 11);
    // one warp per tile: rank in descending work order, then the union list with slot masks
    // (lane l owns union bits [4l, 4l + 4))
    for (int t = tid >> 5; t < 2 * pl.ntiles; t += nthr >> 5) {
        const bool fwd = t < pl.ntiles;
        const int tt = fwd ? t : t - pl.ntiles;
        const unsigned *src = fwd ? sc.flw : sc.colw;
        // tiles in descending order of work (stable): the attention kernels hand out the
        // longest tiles of a bh-chunk first (longest-processing-time-first scheduling)
        const int *cnt = sc.cnt + (fwd ? 0 : pl.ntiles);
        const int c = cnt[tt];
        int rank = 0;
        for (int v0 = 0; v0 < pl.ntiles; v0 += 32) {
            const int v = v0 + lane;
            const bool before = v < pl.ntiles && ((cnt[v] > c) || (cnt[v] == c && v < tt));
            rank += __popc(__ballot_sync(0xffffffffu, before));
        }
        if (lane == 0) plan[(fwd ? pl.forder : pl.border) + rank] = tt;
        const int wsel = lane >> 3, sh = (lane & 7) * 4;
        unsigned nib = 0;
        for (int sl = 0; sl < pl.S; ++sl) {
            const int r = fwd ? tt * pl.S + sl : sc.perm[tt * pl.S + sl];
            if (r < n) nib |= (src[r * 4 + wsel] >> sh) & 15u;
        }
        int o = sc.off[(fwd ? 0 : pl.ntiles + 1) + tt] + warp_excl_scan_i32(__popc(nib), lane);
        int *col = plan + (fwd ? pl.fcol : pl.brow);
        int *msk = plan + (fwd ? pl.fmsk : pl.bmsk);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (!((nib >> k) & 1u)) continue;
            const int j = 4 * lane + k;
            int m = 0;
            for (int sl = 0; sl < pl.S; ++sl) {
                const int r = fwd ? tt * pl.S + sl : sc.perm[tt * pl.S + sl];
                if (r < n) m |= (int)((src[r * 4 + wsel] >> (sh + k)) & 1u) << sl;
            }
            col[o] = j;
            msk[o] = m;
            ++o;
        }
    }
}

static __host__ __device__ constexpr int k2_bits_words() { return 4 * K2_MAXN; }

__global__ void __launch_bounds__(K2_THREADS) pattern_finalize_kernel(K2Args a) {
    extern __shared__ __align__(16) unsigned char k2_smem[];
    const int n = a.n, N = n * n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0 && a.bad && *a.bad && a.flags) atomicOr(a.flags, FLAG_BAD_SCORE);
    long long *s_pool = reinterpret_cast<long long *>(k2_smem);
    unsigned *gtw = reinterpret_cast<unsigned *>(s_pool + ((N + 1) & ~1));  // [n][4] row bitboards: > t
    unsigned *dnw = gtw + k2_bits_words();                      // edge (r,c) -> (r+1,c)
    unsigned *rtw = dnw + k2_bits_words();                      // edge (r,c) -> (r,c+1)
    unsigned *dgw = rtw + k2_bits_words();                      // edge (r,c) -> (r+1,c+1)
    K2Scratch sc;
    sc.flw = dgw + k2_bits_words();
    sc.colw = sc.flw + k2_bits_words();
    sc.cnt = reinterpret_cast<int *>(sc.colw + k2_bits_words());
    sc.off = sc.cnt + 2 * K2_MAXN + 8;
    unsigned int *hist = reinterpret_cast<unsigned int *>(sc.off + 2 * (K2_MAXN + 1) + 8);
    sc.perm = reinterpret_cast<int *>(hist + 256);
    __shared__ long long bc[4];
    __shared__ unsigned long long s_red[2];
    __shared__ unsigned int s_le;

    k2_stamp(a, 0);
    for (int i = tid; i < N; i += blockDim.x) s_pool[i] = a.pool[i];
    if (tid == 0) { s_red[0] = 0ull; s_red[1] = ~0ull; s_le = 0u; }
    __syncthreads();
    k2_stamp(a, 1);

    // ---- threshold as an integer T: gt(x) <=> x > T (reading Q9)
    long long T;
    if (a.kind == SPION_TH_ABSOLUTE) {
        T = a.T_abs;
    } else {
        unsigned long long orv = 0;
        for (int i = tid; i < N; i += blockDim.x) orv |= (unsigned long long)s_pool[i];
        for (int o = 16; o > 0; o >>= 1) orv |= __shfl_xor_sync(0xffffffffu, orv, o);
        if (lane == 0 && orv) atomicOr(&s_red[0], orv);
        __syncthreads();
        const unsigned long long all = s_red[0];
        const int topbit = all ? 63 - __clzll((long long)all) : 0;
        const int top_shift = (topbit / 8) * 8;
        k2_stamp(a, 12);
        const long long v_lo = block_select_kth(s_pool, N, a.lo, hist, bc, top_shift);
        k2_stamp(a, 13);
        if (a.kind == SPION_TH_QUANTILE_LINEAR && a.frac_pos) {
            // t = v[lo] + frac (v[lo+1] - v[lo]) with 0 < frac < 1: x > t <=> x >= v[lo+1] if the
            // gap is positive, else x > v[lo]
            unsigned int le = 0;
            unsigned long long mn = ~0ull;
            for (int i = tid; i < N; i += blockDim.x) {
                long long x = s_pool[i];
                if (x <= v_lo) ++le; else mn = min(mn, (unsigned long long)x);
            }
            for (int o = 16; o > 0; o >>= 1) {
                le += __shfl_xor_sync(0xffffffffu, le, o);
                mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            }
            if (lane == 0) {
                atomicAdd(&s_le, le);
                atomicMin(&s_red[1], mn);
            }
            __syncthreads();
            const bool tie = (long long)s_le >= a.lo + 2;
            T = tie ? v_lo : (long long)s_red[1] - 1;
        } else {
            T = v_lo;
        }
    }
    k2_stamp(a, 2);

    // ---- gt and max-neighbour edges (Alg. 4 l.1-15) as row bitboards: one warp per 32-bit word
    for (int pw = warp; pw < n * 4; pw += K2_THREADS / 32) {
        const int r = pw >> 2, c = (pw & 3) * 32 + lane;
        bool g = false, dn = false, rt = false, dg = false;
        if (c < n) {
            const long long v = s_pool[r * n + c];
            g = v > T;
            if (r + 1 < n && c + 1 < n) {  // Alg. 4 l.1: the last row / column has no out-edges
                const long long below = s_pool[(r + 1) * n + c], right = s_pool[r * n + c + 1],
                                diag = s_pool[(r + 1) * n + c + 1];
                long long m = below > right ? below : right;
                m = m > diag ? m : diag;
                dn = below == m;
                rt = right == m;
                dg = diag == m;
            }
        }
        const unsigned bg = __ballot_sync(0xffffffffu, g), bd = __ballot_sync(0xffffffffu, dn),
                       br = __ballot_sync(0xffffffffu, rt), bq = __ballot_sync(0xffffffffu, dg);
        if (lane == 0) { gtw[pw] = bg; dnw[pw] = bd; rtw[pw] = br; dgw[pw] = bq; }
    }
    __syncthreads();
    k2_stamp(a, 3);

    // ---- flood fill: reach from the seeds (0, i), (j, 0) (Alg. 3 l.5-8) along the edges, row by row.
    //   E_r   = cells of row r entered from row r-1 (down edges, diagonal edges shifted by one)
    //   reach along row r's right edges: R[c] = X[c] | (R[c-1] & rt[c-1]) with X = E_r + seeds.
    //   That recurrence is a carry chain: with g = X & rt, p = rt the carries of g + p are
    //   C[c] = R[c-1] & rt[c-1] (the cells entered by a right edge); R = X | C.
    //   marked = (entered by an edge AND > t) (Alg. 4 l.5-7) OR diagonal (Alg. 3 l.9-10)
    if (a.variant & (SPION_PAT_NOFLOOD | SPION_PAT_ALL_SEEDS)) {
        // no sweep needed.  SPION-C: marked = gt.  Every cell a seed: every cell propagates (so the
        // literal and prose readings coincide), marked = entered by an edge from any cell AND gt,
        // where row r is entered from row r-1 (down / diagonal edges) or from its left neighbour
        const bool nof = a.variant & SPION_PAT_NOFLOOD;
        for (int r = tid; r < n; r += blockDim.x) {
            const Bits gt = b_load(gtw + r * 4);
            Bits fl = gt;
            if (!nof) {
                Bits E = b_shl1(b_load(rtw + r * 4));
                if (r > 0) E = b_or(E, b_or(b_load(dnw + (r - 1) * 4), b_shl1(b_load(dgw + (r - 1) * 4))));
                fl = b_and(E, gt);
            }
            b_store(sc.flw + r * 4, b_and(b_or(fl, b_bit(r)), b_ones(n)));
        }
    } else if (a.variant & SPION_PAT_PROSE) {
        // prose reading: only the seeds and the marked cells propagate.  Along row r the edge
        // c -> c+1 is usable when rt[c] and gt[c+1] (the cell it enters becomes critical), so the
        // propagating set is the same carry chain as below with rt replaced by that link mask
        if (tid == 0) {
            const Bits all = b_ones(n);
            Bits prop{0ull, 0ull}, dn{0ull, 0ull}, dg{0ull, 0ull};
            for (int r = 0; r < n; ++r) {
                const Bits rt = b_load(rtw + r * 4), gt = b_load(gtw + r * 4);
                const Bits E = b_or(b_and(prop, dn), b_shl1(b_and(prop, dg)));  // entered from above
                const Bits seed = r == 0 ? all : Bits{1ull, 0ull};
                const Bits X = b_or(seed, b_and(E, gt));
                const Bits lnk = b_and(rt, Bits{(gt.lo >> 1) | (gt.hi << 63), gt.hi >> 1});
                const Bits gg = b_and(X, lnk);
                const Bits C = b_xor(b_add(gg, lnk), b_xor(gg, lnk));  // entered from the left, critical
                prop = b_or(X, C);
                const Bits entered = b_or(E, b_shl1(b_and(prop, rt)));
                b_store(sc.flw + r * 4, b_and(b_or(b_and(entered, gt), b_bit(r)), all));
                dn = b_load(dnw + r * 4);
                dg = b_load(dgw + r * 4);
            }
        }
    } else if (tid == 0 && n <= 64) {  // the same sweep on 64-bit rows (half the dependent ops)
        const unsigned long long all = ~0ull >> (64 - n);
        unsigned long long vis = 0ull, dn = 0ull, dg = 0ull;
#pragma unroll 4
        for (int r = 0; r < n; ++r) {
            const unsigned long long rt = b_load(rtw + r * 4).lo, gt = b_load(gtw + r * 4).lo;
            const unsigned long long E = (vis & dn) | ((vis & dg) << 1);
            const unsigned long long X = E | (r == 0 ? all : 1ull);
            const unsigned long long gg = X & rt;
            const unsigned long long C = (gg + rt) ^ (gg ^ rt);
            vis = X | C;
            b_store(sc.flw + r * 4, Bits{((E | C) & gt) | (1ull << r), 0ull});
            dn = b_load(dnw + r * 4).lo;
            dg = b_load(dgw + r * 4).lo;
        }
    } else if (tid == 0) {
        const Bits all = b_ones(n);
        Bits vis{0ull, 0ull}, dn{0ull, 0ull}, dg{0ull, 0ull};
#pragma unroll 4
        for (int r = 0; r < n; ++r) {
            const Bits rt = b_load(rtw + r * 4), gt = b_load(gtw + r * 4);
            const Bits E = b_or(b_and(vis, dn), b_shl1(b_and(vis, dg)));
            const Bits X = b_or(E, r == 0 ? all : Bits{1ull, 0ull});
            const Bits gg = b_and(X, rt);
            const Bits C = b_xor(b_add(gg, rt), b_xor(gg, rt));
            vis = b_or(X, C);
            const Bits fl = b_or(b_and(b_or(E, C), gt), b_bit(r));
            b_store(sc.flw + r * 4, fl);
            dn = b_load(dnw + r * 4);
            dg = b_load(dgw + r * 4);
        }
    }
    __syncthreads();
    k2_stamp(a, 4);
    k2_stamp(a, 5);
    build_bsr_and_plan(a, sc);
    __syncthreads();
    k2_stamp(a, 6);
}

__global__ void __launch_bounds__(K2_THREADS) bsr_from_mask_kernel(const uint8_t *mask_in, K2Args a) {
    extern __shared__ __align__(16) unsigned char k2_smem[];
    const int n = a.n, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    K2Scratch sc;
    sc.flw = reinterpret_cast<unsigned *>(k2_smem);
    sc.colw = sc.flw + k2_bits_words();
    sc.cnt = reinterpret_cast<int *>(sc.colw + k2_bits_words());
    sc.off = sc.cnt + 2 * K2_MAXN + 8;
    sc.perm = sc.off + 2 * (K2_MAXN + 1) + 8 + 256;
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int pw = warp; pw < n * 4; pw += K2_THREADS / 32) {
        const int r = pw >> 2, c = (pw & 3) * 32 + lane;
        const uint8_t v = c < n ? mask_in[r * n + c] : 0;
        if (v > 1) s_bad = 1;
        const unsigned b = __ballot_sync(0xffffffffu, v != 0);
        if (lane == 0) sc.flw[pw] = b;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) { *a.nnzb = -1; if (a.flags) atomicOr(a.flags, FLAG_BAD_MASK); }
        return;
    }
    build_bsr_and_plan(a, sc);
}

// ---------------------------------------------------------------- host side
unsigned long long *g_k2_trace = nullptr;
size_t pattern_ws_bytes(int L, int block) {
    const int n = L / block;
    return 256 + round_up((size_t)n * n * 8, 256);
}

static size_t k2_smem_bytes(int n, bool with_pool) {
    size_t b = with_pool ? (((size_t)n * n + 1) & ~(size_t)1) * 8 + 4 * (size_t)k2_bits_words() * 4 : 0;  // pool, gt/dn/rt/dg
    b += 2 * (size_t)k2_bits_words() * 4;                                             // fl, columns
    b += (2 * K2_MAXN + 8) * 4 + (2 * (K2_MAXN + 1) + 8) * 4 + 256 * 4 + (K2_MAXN + 32) * 4 + 64;
    return b;
}

// pattern workspace: [0, 4) flags (K2; reported by the ABI), [8, 16) K1's bad-score count (u64),
// [256, 256 + 8 n^2) the pool sums (i64).  [8, 256 + 8 n^2) is the part a multi-device caller sums.
static constexpr size_t PWS_BAD = 8, PWS_POOL = 256;

spion_status launch_pattern_pool(const float *scores_rows, int L, int B, int F, int row_begin, int row_end, void *ws,
                                 cudaStream_t s) {
    const int n = L / B;
    if (n > K2_MAXN) return SPION_ERR_UNSUPPORTED;
    char *w = static_cast<char *>(ws);
    unsigned long long *bad = reinterpret_cast<unsigned long long *>(w + PWS_BAD);
    unsigned long long *pool = reinterpret_cast<unsigned long long *>(w + PWS_POOL);
    SPION_CUDA_TRY(cudaMemsetAsync(ws, 0, PWS_POOL + (size_t)n * n * 8, s));
    const int I0 = row_begin / B, nr = (row_end - row_begin) / B;
    if (nr == 0) return SPION_OK;
    K1Geom g4, g8, g;
    spion_status st;
    const bool ok4 = k1_geom(L, B, F, 4, g4, I0, nr), ok8 = k1_geom(L, B, F, 8, g8, I0, nr);
    // fewest window positions per source row (ties: the 16-position lanes, more CTAs)
    if (ok4 && (!ok8 || g4.n_cc * 4 <= g8.n_cc * 8)) st = k1_launch<4>(scores_rows, g4, pool, bad, s);
    else if (ok8) st = k1_launch<8>(scores_rows, g8, pool, bad, s);
    else if (k1_geom(L, B, F, 17, g, I0, nr)) st = k1_launch<17>(scores_rows, g, pool, bad, s);
    else return SPION_ERR_UNSUPPORTED;  // B + F > ~2170 columns per window
    return st;
}

spion_status launch_pattern_finalize(int L, int B, int kind, long long lo, int frac_pos, int variant, long long T_abs,
                                     void *ws, spion_bsr *out, cudaStream_t s) {
    const int n = L / B;
    if (n > K2_MAXN) return SPION_ERR_UNSUPPORTED;
    char *w = static_cast<char *>(ws);
    K2Args a;
    memset(&a, 0, sizeof(a));
    a.pool = reinterpret_cast<const long long *>(w + PWS_POOL);
    a.bad = reinterpret_cast<const unsigned long long *>(w + PWS_BAD);
    a.n = n;
    a.block = B;
    a.kind = kind;
    a.lo = lo;
    a.frac_pos = frac_pos;
    a.T_abs = T_abs;
    a.variant = variant;
    a.flags = reinterpret_cast<int *>(ws);
    a.brow_ptr = out->brow_ptr;
    a.bcol_idx = out->bcol_idx;
    a.bcol_ptr = out->bcol_ptr;
    a.brow_idx = out->brow_idx;
    a.nnzb = out->nnzb;
    a.mask = out->mask;
    a.nnzb_cap = out->nnzb_cap;
    a.plan = reinterpret_cast<int *>(out->plan);
    if (getenv("SPION_TRACE")) {
        static unsigned long long *tb = nullptr;
        if (!tb) SPION_CUDA_TRY(cudaMalloc(&tb, 64 * 8));
        a.trace = tb;
        g_k2_trace = tb;
    }
    const size_t smem2 = k2_smem_bytes(n, true);
    if (smem2 > 227 * 1024) return SPION_ERR_UNSUPPORTED;
    static PerDevice attr2;
    SPION_CUDA_TRY(smem_attr_once(attr2, pattern_finalize_kernel));
    pattern_finalize_kernel<<<1, K2_THREADS, smem2, s>>>(a);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

spion_status launch_pattern(const float *scores, int L, int B, int F, int kind, long long lo, int frac_pos, int variant,
                            long long T_abs, void *ws, spion_bsr *out, cudaStream_t s) {
    spion_status st = launch_pattern_pool(scores, L, B, F, 0, L, ws, s);
    if (st) return st;
    return launch_pattern_finalize(L, B, kind, lo, frac_pos, variant, T_abs, ws, out, s);
}

spion_status launch_bsr_from_mask(const uint8_t *mask, int L, int B, spion_bsr *out, int *flags, cudaStream_t s) {
    const int n = L / B;
    if (n > K2_MAXN) return SPION_ERR_UNSUPPORTED;
    K2Args a;
    memset(&a, 0, sizeof(a));
    a.n = n;
    a.block = B;
    a.flags = flags;
    a.brow_ptr = out->brow_ptr;
    a.bcol_idx = out->bcol_idx;
    a.bcol_ptr = out->bcol_ptr;
    a.brow_idx = out->brow_idx;
    a.nnzb = out->nnzb;
    a.mask = out->mask;
    a.nnzb_cap = out->nnzb_cap;
    a.plan = reinterpret_cast<int *>(out->plan);
    const size_t smem = k2_smem_bytes(n, false);
    static PerDevice attr;
    SPION_CUDA_TRY(smem_attr_once(attr, bsr_from_mask_kernel));
    bsr_from_mask_kernel<<<1, K2_THREADS, smem, s>>>(mask, a);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

}  // namespace spion
