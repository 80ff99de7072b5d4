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
//    sum PP.  One warp owns one source row segment at a time.
// K2 pattern_finalize_kernel (one CTA): threshold by exact order statistics,
//    max-neighbour edges, flood fill as an anti-diagonal wavefront, forced
//    diagonal, block-CSR/CSC and the attention work plan.
#include <stdio.h>

#include "common.cuh"

namespace spion {

// ---------------------------------------------------------------- K1
static constexpr int K1_WARPS = 8;
static constexpr int K1_MAXP = 4;  // (target row, column) pairs per lane

struct K1Geom {
    int L, B, h, A, nI, JC, n_cc, W, CH;
};

static K1Geom k1_geom(int L, int B, int F) {
    K1Geom g;
    g.L = L;
    g.B = B;
    g.h = (F - 1) / 2;
    g.A = (g.h + B - 1) / B;
    g.nI = 2 * g.A + 1;
    int n = L / B;
    int jc = 8;
    while (jc > 1 && g.nI * jc > 32 * K1_MAXP) --jc;
    if (jc > n) jc = n;
    g.JC = jc;
    g.n_cc = (n + jc - 1) / jc;
    g.W = jc * B + 2 * g.h;
    int ch = (g.W + 2 + 31) / 32;
    if ((ch & 1) == 0) ++ch;  // odd chunk -> conflict-free strided smem access
    g.CH = ch;
    return g;
}

__global__ void __launch_bounds__(K1_WARPS * 32)
pattern_pool_kernel(const float *__restrict__ A, K1Geom g, unsigned long long *__restrict__ pool,
                    int *__restrict__ flags) {
    extern __shared__ __align__(16) unsigned char k1_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int L = g.L, B = g.B, h = g.h, n = L / B;
    const int cc = blockIdx.x, I0 = blockIdx.y;
    const int J0 = cc * g.JC;
    const int ncols = min(g.JC, n - J0);
    const int W = ncols * B + 2 * h;  // columns [c0, c0 + W)
    const int c0 = J0 * B - h;
    const int CH = g.CH;
    const int ROW = 32 * CH;
    unsigned long long *rowq = reinterpret_cast<unsigned long long *>(k1_smem) + (size_t)warp * ROW;
    unsigned long long *s_acc = reinterpret_cast<unsigned long long *>(k1_smem) + (size_t)K1_WARPS * ROW;
    const int npairs = g.nI * ncols;
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) s_acc[p] = 0ull;

    unsigned long long acc[K1_MAXP];
#pragma unroll
    for (int t = 0; t < K1_MAXP; ++t) acc[t] = 0ull;
    bool bad = false;

    // float4 window covering [c0, c0+W)
    const int g4 = (c0 >= 0) ? (c0 & ~3) : -((-c0 + 3) & ~3);
    const int n4 = (c0 + W - g4 + 3) >> 2;
    __syncthreads();

    for (int u = warp; u < B; u += K1_WARPS) {
        const int x = I0 * B + u;
        const float *arow = A + (size_t)x * L;
        // stage: coalesced float4 loads -> q (int64 fixed point) in smem, zero outside [0,L)
        for (int k = lane; k < ROW; k += 32) rowq[k] = 0ull;
        __syncwarp();
        for (int v = lane; v < n4; v += 32) {
            const int gc = g4 + 4 * v;
            if (gc < 0 || gc >= L) continue;
            float4 a4 = __ldg(reinterpret_cast<const float4 *>(arow + gc));
            float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const int k = gc + t - c0;
                if (k < 0 || k >= W) continue;
                const float a = av[t];
                if (!(a >= 0.f && a <= 1.f)) bad = true;
                // a * 2^32 is exact in fp32; round half to even (reading Q8)
                rowq[k] = (unsigned long long)__float2ll_rn(a * 4294967296.0f);
            }
        }
        __syncwarp();
        // pass A: chunk totals of q
        const int k0 = lane * CH;
        unsigned long long tot = 0;
        for (int t = 0; t < CH; ++t) tot += rowq[k0 + t];
        unsigned long long off = warp_excl_scan_u64(tot, lane);
        // pass B: P[k] = sum_{c<k} q[c], in place; totals of P
        unsigned long long run = off, tot2 = 0;
        for (int t = 0; t < CH; ++t) {
            unsigned long long qv = rowq[k0 + t];
            rowq[k0 + t] = run;
            tot2 += run;
            run += qv;
        }
        unsigned long long off2 = warp_excl_scan_u64(tot2, lane);
        // pass C: PP[k] = sum_{k'<k} P[k'], in place
        unsigned long long run2 = off2;
        for (int t = 0; t < CH; ++t) {
            unsigned long long pv = rowq[k0 + t];
            rowq[k0 + t] = run2;
            run2 += pv;
        }
        __syncwarp();
        // contributions of row x to pool rows I0+a, columns J0+jj
#pragma unroll
        for (int t = 0; t < K1_MAXP; ++t) {
            const int p = lane + 32 * t;
            if (p >= npairs) break;
            const int a = p / ncols - g.A, jj = p % ncols;
            const int I = I0 + a;
            if (I < 0 || I >= n) continue;
            const int r = u - a * B;
            const int f0 = max(r - B + 1, -h), f1 = min(r, h);
            if (f0 > f1) continue;
            const int s0 = jj * B + h + f0, s1 = jj * B + h + f1;
            acc[t] += (rowq[s1 + 1 + B] - rowq[s0 + B]) - (rowq[s1 + 1] - rowq[s0]);
        }
        __syncwarp();
    }
#pragma unroll
    for (int t = 0; t < K1_MAXP; ++t) {
        const int p = lane + 32 * t;
        if (p < npairs && acc[t]) atomicAdd(&s_acc[p], acc[t]);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flags, FLAG_BAD_SCORE);
    __syncthreads();
    for (int p = threadIdx.x; p < npairs; p += blockDim.x) {
        const int a = p / ncols - g.A, jj = p % ncols;
        const int I = I0 + a;
        if (I < 0 || I >= n || s_acc[p] == 0ull) continue;
        atomicAdd(&pool[(size_t)I * n + (J0 + jj)], s_acc[p]);
    }
}

// ---------------------------------------------------------------- K2
static constexpr int K2_THREADS = 1024;

// k-th smallest (0-based) of v[0..N) by MSD radix selection, 8-bit digits.
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
                if (k >= below && k < below + (long long)c[t]) { bc[0] = lane * 8 + t; bc[1] = below; }
                below += c[t];
            }
        }
        __syncthreads();
        prefix |= ((unsigned long long)bc[0]) << shift;
        k -= bc[1];
        __syncthreads();
    }
    return (long long)prefix;
}

// BSR / CSC / plan from the block mask in shared memory (fl: n*n bytes).
__device__ void build_bsr_and_plan(const uint8_t *fl, int n, int block, int *brow_ptr, int *bcol_idx,
                                   int *bcol_ptr, int *brow_idx, uint8_t *mask_out, int *nnzb_out,
                                   int nnzb_cap, int *plan, int *flags, int *s_cnt, int *s_off) {
    const int tid = threadIdx.x;
    for (int i = tid; mask_out && i < n * n; i += blockDim.x) mask_out[i] = fl[i];
    // row and column counts
    for (int r = tid; r < 2 * n; r += blockDim.x) {
        int c = 0;
        if (r < n) { for (int j = 0; j < n; ++j) c += fl[r * n + j]; }
        else { int col = r - n; for (int i = 0; i < n; ++i) c += fl[i * n + col]; }
        s_cnt[r] = c;
    }
    __syncthreads();
    if (tid < 32) {  // exclusive scans of the two count arrays (n <= 128 -> <= 4 per lane)
        for (int which = 0; which < 2; ++which) {
            const int *cnt = s_cnt + which * n;
            int *off = s_off + which * (n + 1);
            int per = (n + 31) / 32;
            int loc = 0;
            for (int t = 0; t < per; ++t) { int r = tid * per + t; if (r < n) loc += cnt[r]; }
            int ex = warp_excl_scan_i32(loc, tid);
            for (int t = 0; t < per; ++t) { int r = tid * per + t; if (r < n) { off[r] = ex; ex += cnt[r]; } }
            if (tid == 31) off[n] = ex;
        }
    }
    __syncthreads();
    const int nnzb = s_off[n];
    if (tid == 0) {
        *nnzb_out = nnzb;
        if (nnzb > nnzb_cap && flags) atomicOr(flags, FLAG_CAPACITY);
    }
    for (int r = tid; r <= n; r += blockDim.x) { brow_ptr[r] = s_off[r]; bcol_ptr[r] = s_off[n + 1 + r]; }
    for (int r = tid; r < 2 * n; r += blockDim.x) {
        if (r < n) {
            int o = s_off[r];
            for (int j = 0; j < n; ++j)
                if (fl[r * n + j]) { if (o < nnzb_cap) bcol_idx[o] = j; ++o; }
        } else {
            int col = r - n;
            int o = s_off[n + 1 + col];
            for (int i = 0; i < n; ++i)
                if (fl[i * n + col]) { if (o < nnzb_cap) brow_idx[o] = i; ++o; }
        }
    }
    // attention work plan: slot tiles of S consecutive block rows (fwd) / columns (bwd)
    if (plan) {
        PlanLayout pl(n, block);
        __syncthreads();
        for (int t = tid; t < 2 * pl.ntiles; t += blockDim.x) {
            const bool fwd = t < pl.ntiles;
            const int tt = fwd ? t : t - pl.ntiles;
            int c = 0;
            for (int j = 0; j < n; ++j) {
                int m = 0;
                for (int s = 0; s < pl.S; ++s) {
                    int r = tt * pl.S + s;
                    if (r < n && (fwd ? fl[r * n + j] : fl[j * n + r])) m |= 1 << s;
                }
                c += (m != 0);
            }
            s_cnt[t] = c;
        }
        __syncthreads();
        if (tid < 32) {
            for (int which = 0; which < 2; ++which) {
                const int *cnt = s_cnt + which * pl.ntiles;
                int *ptr = plan + (which ? pl.bptr : pl.fptr);
                int per = (pl.ntiles + 31) / 32;
                int loc = 0;
                for (int q = 0; q < per; ++q) { int r = tid * per + q; if (r < pl.ntiles) loc += cnt[r]; }
                int ex = warp_excl_scan_i32(loc, tid);
                for (int q = 0; q < per; ++q) { int r = tid * per + q; if (r < pl.ntiles) { ptr[r] = ex; s_off[which * (pl.ntiles + 1) + r] = ex; ex += cnt[r]; } }
                if (tid == 31) { ptr[pl.ntiles] = ex; plan[3 + which] = ex; }
            }
            if (tid == 0) {
                plan[0] = n; plan[1] = pl.S; plan[2] = pl.ntiles;
                for (int w = 5; w < 16; ++w) plan[w] = 0;  // scheduler counters start at zero
            }
        }
        __syncthreads();
        // tiles in descending order of work (stable): the attention kernels hand out the
        // longest tiles of a bh-chunk first (longest-processing-time-first scheduling)
        for (int t = tid; t < 2 * pl.ntiles; t += blockDim.x) {
            const bool fwd = t < pl.ntiles;
            const int tt = fwd ? t : t - pl.ntiles;
            const int *cnt = s_cnt + (fwd ? 0 : pl.ntiles);
            const int c = cnt[tt];
            int rank = 0;
            for (int u = 0; u < pl.ntiles; ++u) rank += (cnt[u] > c) || (cnt[u] == c && u < tt);
            plan[(fwd ? pl.forder : pl.border) + rank] = tt;
        }
        for (int t = tid; t < 2 * pl.ntiles; t += blockDim.x) {
            const bool fwd = t < pl.ntiles;
            const int tt = fwd ? t : t - pl.ntiles;
            int o = s_off[(fwd ? 0 : 1) * (pl.ntiles + 1) + tt];
            int *col = plan + (fwd ? pl.fcol : pl.brow);
            int *msk = plan + (fwd ? pl.fmsk : pl.bmsk);
            for (int j = 0; j < n; ++j) {
                int m = 0;
                for (int s = 0; s < pl.S; ++s) {
                    int r = tt * pl.S + s;
                    if (r < n && (fwd ? fl[r * n + j] : fl[j * n + r])) m |= 1 << s;
                }
                if (m) { col[o] = j; msk[o] = m; ++o; }
            }
        }
    }
}

struct K2Args {
    const long long *pool;  // [n][n] fixed-point pool sums
    int n, block;
    int kind;               // spion_threshold_kind
    long long lo;           // LINEAR: floor(hpos); NEAREST: rank k
    int frac_pos;           // LINEAR: frac > 0
    long long T_abs;        // ABSOLUTE: gt <=> x > T_abs
    int *flags;
    int *brow_ptr, *bcol_idx, *bcol_ptr, *brow_idx, *nnzb;
    uint8_t *mask;
    int nnzb_cap;
    int *plan;
};

__global__ void __launch_bounds__(K2_THREADS) pattern_finalize_kernel(K2Args a) {
    extern __shared__ __align__(16) unsigned char k2_smem[];
    const int n = a.n, N = n * n, tid = threadIdx.x;
    long long *s_pool = reinterpret_cast<long long *>(k2_smem);
    const int N16 = (N + 15) & ~15;
    uint8_t *s_cell = reinterpret_cast<uint8_t *>(s_pool + N);
    uint8_t *s_fl = s_cell + N16;
    int *s_cnt = reinterpret_cast<int *>(s_fl + N16);
    int *s_off = s_cnt + 2 * n + 8;
    unsigned int *hist = reinterpret_cast<unsigned int *>(s_off + 2 * (n + 1) + 8);
    __shared__ long long bc[4];
    __shared__ unsigned long long s_red[2];

    for (int i = tid; i < N; i += blockDim.x) s_pool[i] = a.pool[i];
    if (tid == 0) { s_red[0] = 0ull; s_red[1] = ~0ull; }
    __syncthreads();

    // ---- threshold as an integer T: gt(x) <=> x > T (reading Q9)
    long long T;
    if (a.kind == SPION_TH_ABSOLUTE) {
        T = a.T_abs;
    } else {
        unsigned long long orv = 0;
        for (int i = tid; i < N; i += blockDim.x) orv |= (unsigned long long)s_pool[i];
        for (int o = 16; o > 0; o >>= 1) orv |= __shfl_xor_sync(0xffffffffu, orv, o);
        if ((tid & 31) == 0 && orv) atomicOr(&s_red[0], orv);
        __syncthreads();
        const unsigned long long all = s_red[0];
        const int topbit = all ? 63 - __clzll((long long)all) : 0;
        const int top_shift = (topbit / 8) * 8;
        const long long v_lo = block_select_kth(s_pool, N, a.lo, hist, bc, top_shift);
        if (a.kind == SPION_TH_QUANTILE_LINEAR && a.frac_pos) {
            // t = v[lo] + frac (v[lo+1] - v[lo]) with 0 < frac < 1: x > t <=> x >= v[lo+1] if the
            // gap is positive, else x > v[lo]
            unsigned int le = 0;
            unsigned long long mn = ~0ull;
            for (int i = tid; i < N; i += blockDim.x) {
                long long x = s_pool[i];
                if (x <= v_lo) ++le; else mn = min(mn, (unsigned long long)x);
            }
            __shared__ unsigned int s_le;
            if (tid == 0) s_le = 0;
            __syncthreads();
            atomicAdd(&s_le, le);
            atomicMin(&s_red[1], mn);
            __syncthreads();
            const bool tie = (long long)s_le >= a.lo + 2;
            T = tie ? v_lo : (long long)s_red[1] - 1;
        } else {
            T = v_lo;
        }
    }

    // ---- gt and max-neighbour edges (Alg. 4 l.3-15)
    for (int i = tid; i < N; i += blockDim.x) {
        const int r = i / n, c = i % n;
        uint8_t f = (s_pool[i] > T) ? 1 : 0;
        if (r + 1 < n && c + 1 < n) {  // Alg. 4 l.1: last row / column has no out-edges
            const long long below = s_pool[i + n], right = s_pool[i + 1], diag = s_pool[i + n + 1];
            long long m = below > right ? below : right;
            m = m > diag ? m : diag;
            if (below == m) f |= 2;
            if (right == m) f |= 4;
            if (diag == m) f |= 8;
        }
        s_cell[i] = f;
    }
    __syncthreads();

    // ---- flood fill: reach from the seeds row 0 / column 0 (Alg. 3 l.5-8) along the edges,
    //      anti-diagonal by anti-diagonal (every edge goes from r+c to r+c+1 or r+c+2)
    const int nw = ((n + 31) / 32) * 32;
    if (tid < nw) {
        for (int d = 0; d <= 2 * n - 2; ++d) {
            const int r = tid, c = d - tid;
            if (r < n && c >= 0 && c < n) {
                bool inr = false;
                if (r > 0 && (s_cell[(r - 1) * n + c] & (16 | 2)) == (16 | 2)) inr = true;
                if (c > 0 && (s_cell[r * n + c - 1] & (16 | 4)) == (16 | 4)) inr = true;
                if (r > 0 && c > 0 && (s_cell[(r - 1) * n + c - 1] & (16 | 8)) == (16 | 8)) inr = true;
                uint8_t f = s_cell[r * n + c];
                if (inr) f |= 32;
                if (inr || r == 0 || c == 0) f |= 16;  // visited
                s_cell[r * n + c] = f;
            }
            asm volatile("bar.sync 1, %0;" ::"r"(nw) : "memory");
        }
    }
    __syncthreads();
    // marked = reached by an edge and > t (Alg. 4 l.5-7), plus the forced diagonal (Alg. 3 l.9-10)
    for (int i = tid; i < N; i += blockDim.x) {
        const int r = i / n, c = i % n;
        const uint8_t f = s_cell[i];
        s_fl[i] = (((f & 32) && (f & 1)) || r == c) ? 1 : 0;
    }
    __syncthreads();
    build_bsr_and_plan(s_fl, n, a.block, a.brow_ptr, a.bcol_idx, a.bcol_ptr, a.brow_idx, a.mask, a.nnzb,
                       a.nnzb_cap, a.plan, a.flags, s_cnt, s_off);
}

__global__ void __launch_bounds__(K2_THREADS) bsr_from_mask_kernel(const uint8_t *mask_in, K2Args a) {
    extern __shared__ __align__(16) unsigned char k2_smem[];
    const int n = a.n, N = n * n, tid = threadIdx.x;
    uint8_t *s_fl = k2_smem;
    int *s_cnt = reinterpret_cast<int *>(s_fl + ((N + 15) & ~15));
    int *s_off = s_cnt + 2 * n + 8;
    __shared__ int s_bad;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    for (int i = tid; i < N; i += blockDim.x) {
        uint8_t v = mask_in[i];
        if (v > 1) s_bad = 1;
        s_fl[i] = v ? 1 : 0;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) { *a.nnzb = -1; if (a.flags) atomicOr(a.flags, FLAG_BAD_MASK); }
        return;
    }
    build_bsr_and_plan(s_fl, n, a.block, a.brow_ptr, a.bcol_idx, a.bcol_ptr, a.brow_idx, a.mask, a.nnzb,
                       a.nnzb_cap, a.plan, a.flags, s_cnt, s_off);
}

// ---------------------------------------------------------------- host side
size_t pattern_ws_bytes(int L, int block) {
    const int n = L / block;
    return 256 + round_up((size_t)n * n * 8, 256);
}

static size_t k2_smem_bytes(int n, bool with_pool) {
    const size_t N = (size_t)n * n;
    const size_t N16 = round_up(N, 16);
    size_t b = with_pool ? N * 8 + 2 * N16 : N16;
    b += (2 * n + 8) * 4 + (2 * (n + 1) + 8) * 4 + 256 * 4 + 64;
    return b;
}

spion_status launch_pattern(const float *scores, int L, int B, int F, int kind, long long lo, int frac_pos,
                            long long T_abs, void *ws, spion_bsr *out, cudaStream_t s) {
    const int n = L / B;
    int *flags = reinterpret_cast<int *>(ws);
    unsigned long long *pool = reinterpret_cast<unsigned long long *>(static_cast<char *>(ws) + 256);
    SPION_CUDA_TRY(cudaMemsetAsync(ws, 0, 256 + (size_t)n * n * 8, s));
    K1Geom g = k1_geom(L, B, F);
    const size_t smem1 = ((size_t)K1_WARPS * 32 * g.CH + (size_t)g.nI * g.JC) * 8;
    if (smem1 > 200 * 1024) return SPION_ERR_UNSUPPORTED;
    static bool attr1 = false;
    if (!attr1) {
        SPION_CUDA_TRY(allow_max_dyn_smem(pattern_pool_kernel));
        attr1 = true;
    }
    pattern_pool_kernel<<<dim3(g.n_cc, n), K1_WARPS * 32, smem1, s>>>(scores, g, pool, flags);
    SPION_LAUNCH_CHECK();

    K2Args a;
    a.pool = reinterpret_cast<const long long *>(pool);
    a.n = n;
    a.block = B;
    a.kind = kind;
    a.lo = lo;
    a.frac_pos = frac_pos;
    a.T_abs = T_abs;
    a.flags = flags;
    a.brow_ptr = out->brow_ptr;
    a.bcol_idx = out->bcol_idx;
    a.bcol_ptr = out->bcol_ptr;
    a.brow_idx = out->brow_idx;
    a.nnzb = out->nnzb;
    a.mask = out->mask;
    a.nnzb_cap = out->nnzb_cap;
    a.plan = reinterpret_cast<int *>(out->plan);
    const size_t smem2 = k2_smem_bytes(n, true);
    static bool attr2 = false;
    if (!attr2) {
        SPION_CUDA_TRY(allow_max_dyn_smem(pattern_finalize_kernel));
        attr2 = true;
    }
    if (smem2 > 227 * 1024) return SPION_ERR_UNSUPPORTED;
    pattern_finalize_kernel<<<1, K2_THREADS, smem2, s>>>(a);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

spion_status launch_bsr_from_mask(const uint8_t *mask, int L, int B, spion_bsr *out, int *flags, cudaStream_t s) {
    const int n = L / B;
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
    static bool attr = false;
    if (!attr) {
        SPION_CUDA_TRY(allow_max_dyn_smem(bsr_from_mask_kernel));
        attr = true;
    }
    bsr_from_mask_kernel<<<1, K2_THREADS, smem, s>>>(mask, a);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

}  // namespace spion
