// attn_bwd_fused.cu — fused tensor-core backward of block-sparse attention (bf16, d = 64,
// block B = 64): ONE pass over column tiles computes dK, dV and dQ (reading Q17, SURVEY 8(a)
// a11), so Q, K, V and dO are read once and S^T / dP^T are recomputed and exponentiated once.
//
// Per work item (bh, column tile t = S = 2 key blocks, 128 keys; plan column tiles, block
// columns in count order), for every query block I of the tile's union list ("entry"):
//   S^T = K Q_I^T, dP^T = V dO_I^T                 tcgen05 SS MMAs -> TMEM (2 buffer pairs)
//   P^T = exp2(S^T c - lse_I log2e), dS^T = P^T (dP^T - D_I)  (thread = key row = TMEM lane)
//   dV += P^T dO_I, dK += dS^T Q_I                 TS MMAs, P^T / dS^T packed bf16 in TMEM
//   dS^T also goes to shared memory (bf16, SW128, row = key), and for every PAIR of entries
//   (I0, I1): [dQ_I0; dQ_I1] = [dS_I0; dS_I1] K     one M = 128 SS MMA (A = dS, MN-major:
//   the two entries' tiles are the two 64-query chunks of A; B = the tile's K, MN-major)
//   -> TMEM -> fp32 rows staged in the pair's (now consumed) dS buffer -> one 1-D bulk
//   reduce-add (cp.reduce.async.bulk .add.f32, performed at L2) per entry into the fp32
//   accumulator dQacc[bh][I*64 .. +64][64] of the workspace.
// A per-(bh, I) counter of completed contributions (the plan says how many column tiles hold
// I) elects the LAST contributor, which converts dQacc rows to bf16 (x scale) into dQ and
// discards the fp32 lines from L2 (no write-back).  dK, dV: epilogue as in the split kernel.
// attn_bwd_prep_kernel (before): D = rowsum(dO * O), -lse * log2(e), zeroed dQacc and
// counters, and dQ = 0 for query rows whose block row holds no block.
//
// Warp roles (512 threads, one CTA per SM, all 512 TMEM columns):
//   0..7   softmax: warpgroup 0 takes the even entries of an item, warpgroup 1 the odd ones
//          (so warpgroup w always fills half w of a pair's dS buffer); dK/dV epilogue
//   8..11  dQ warpgroup: TMEM -> staged fp32 rows -> bulk reduce-adds, completion counting,
//          finalisation (dQacc -> bf16 dQ) of the query blocks it completes
//   12 scheduler + TMA producer   13 S^T/dP^T MMA issuer (TMEM owner)
//   14 dV/dK/dQ MMA issuer        15 dK/dV TMA storer
// TMEM: S^T|dP^T buffer pairs at [0,128) [128,256), dK [256,320), dV [320,384), dQ pair
// accumulators [384,448) [448,512).
#include "attn_tc.cuh"

// timing-only debug builds (wrong dQ): no completion counting / finalisation; no dQ staging or
// reduce-adds; no dQ MMA
#ifndef SPION_FDBG_NOFIN
#define SPION_FDBG_NOFIN 0
#endif
#ifndef SPION_FDBG_NODQ
#define SPION_FDBG_NODQ 0
#endif
#ifndef SPION_FDBG_NODQMMA
#define SPION_FDBG_NODQMMA 0
#endif
#ifndef SPION_FDBG_NODISCARD  // keep finalised fp32 lines in L2 (A/B of discard.global.L2)
#define SPION_FDBG_NODISCARD 0
#endif
#ifndef SPION_FDBG_NOFINLOAD  // count completions but skip the finalisation loads / stores (timing)
#define SPION_FDBG_NOFINLOAD 0
#endif

namespace spion {

namespace {
constexpr int FB = 64;                 // block size of the fused path
constexpr int F_NBUF = 2;              // S^T/dP^T buffer pairs
constexpr int F_NST = 5;               // Q_I / dO_I / lse_I / D_I stages
constexpr int F_THREADS = 512;
constexpr int W_DQ0 = 8, W_PROD = 12, W_MMA = 13, W_MMA2 = 14, W_STORE = 15;
constexpr uint32_t F_TILE = FB * 128;               // one B-row operand tile (8 KB)
constexpr uint32_t F_STAGE = 2 * F_TILE + 1024;     // Q_I, dO_I, -lse_I log2e, D_I
constexpr uint32_t F_KV = 32768;                    // K (16 KB) + V (16 KB) of a 128-key tile
constexpr uint32_t F_DSP = 32768;                   // a pair's dS (2 x 16 KB) / staged fp32 dQ
constexpr uint32_t COL_DK = 256, COL_DV = 320, COL_DQ = 384;
constexpr int F_SCHED_CONSUMERS = 15;  // 8 softmax + 4 dQ warps + S-MMA, MMA2, storer
constexpr int BAR_DQ = 1;              // named barrier of the dQ warpgroup
constexpr size_t F_SMEM = 1024 + 2 * F_KV + F_NST * F_STAGE + 2 * F_DSP + SCHED_AREA + 1024;
}  // namespace

struct FusedParams {
    float *dQacc;   // [bh][L][64] fp32 (zeroed by the prep kernel)
    int *done;      // [bh][n] completed contributions per query block (zeroed by the prep kernel)
    void *dQ;       // bf16 output
};

// ---------------------------------------------------------------- prep: D, -lse log2e, zeroing
// 8 threads per query row (16-byte chunks of O / dO, one 32-byte chunk of the row's dQacc)
__global__ void __launch_bounds__(256) attn_bwd_prep_kernel(const __nv_bfloat16 *O, const __nv_bfloat16 *dO,
                                                             const float *lse, float *D, float *nlse2, float *dQacc,
                                                             int *done, __nv_bfloat16 *dQ, const int *brow_ptr,
                                                             int64_t bh, int L, int B, int n, int64_t stride_bh,
                                                             int64_t stride_l) {
    const int64_t gt = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t row = gt >> 3;
    const int c = (int)(gt & 7);
    if (gt < bh * n) done[gt] = 0;
    if (row >= bh * L) return;
    const int64_t b = row / L;
    const int i = (int)(row - b * L);
    const int64_t off = b * stride_bh + (int64_t)i * stride_l + c * 8;
    const uint4 o = *reinterpret_cast<const uint4 *>(O + off);
    const uint4 g = *reinterpret_cast<const uint4 *>(dO + off);
    const uint32_t ov[4] = {o.x, o.y, o.z, o.w}, gv[4] = {g.x, g.y, g.z, g.w};
    float acc = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&ov[k]));
        const float2 e = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&gv[k]));
        acc = fmaf(a.x, e.x, fmaf(a.y, e.y, acc));
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    float4 *z = reinterpret_cast<float4 *>(dQacc + row * 64 + c * 8);
    z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
    const int I = i / B;
    if (brow_ptr[I + 1] == brow_ptr[I])  // no stored block in this query block row: no contribution
        *reinterpret_cast<uint4 *>(dQ + off) = make_uint4(0, 0, 0, 0);
    if (c == 0) {
        D[row] = acc;
        nlse2[row] = -lse[row] * LOG2E;
    }
}

// ---------------------------------------------------------------- the fused kernel
__global__ void __launch_bounds__(F_THREADS, 1)
attn_bwd_fused_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                         const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                         const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV,
                         const __grid_constant__ CUtensorMap tmAcc, TcParams p, FusedParams f) {
    constexpr int NST = F_NST, NBUF = F_NBUF;
    constexpr uint32_t BUFW = 2 * FB;  // S^T at b*BUFW, dP^T at b*BUFW + FB
    constexpr uint32_t IDESC_ST = idesc_bf16(128, FB, false, false);  // S^T = K Q^T, dP^T = V dO^T
    constexpr uint32_t IDESC_DKV = idesc_bf16(128, 64, false, true);  // dV += P^T dO, dK += dS^T Q
    constexpr uint32_t IDESC_DQ = idesc_bf16(128, 64, true, true);    // [dQ0; dQ1] = [dS0; dS1] K

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sKV = smem;                     // [2] K at +0, V at +16384
    uint8_t *sStage = smem + 2 * F_KV;       // [NST]
    uint8_t *sDS = sStage + NST * F_STAGE;   // [2] pair buffers
    uint8_t *sSched = sDS + 2 * F_DSP;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    uint64_t *kv_full = bars + 0, *kv_empty = bars + 2, *acc_full = bars + 4, *acc_empty = bars + 5,
             *s_full = bars + 6, *p_full = s_full + 2 * NBUF, *freeb = p_full + NBUF, *q_full = freeb + NBUF,
             *q_empty = q_full + NST, *dq_full = q_empty + NST, *dq_empty = dq_full + 2, *ds_empty = dq_empty + 2,
             *staged = ds_empty + 2, *sched_bars = staged + 2;
    Sched sc = make_sched(sSched, sched_bars);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sched_bars + 8);
    int *expc = reinterpret_cast<int *>(tmem_slot + 4);  // [n] contributions expected per query block
    int *fin = expc + SCHED_CAP;                         // dQ warpgroup: finalisation queue (2 + 2 * 64 ints)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        mbar_init(acc_full, 1);
        mbar_init(acc_empty, 256);
        for (int i = 0; i < 2 * NBUF; ++i) mbar_init(s_full + i, 1);
        for (int i = 0; i < NBUF; ++i) { mbar_init(p_full + i, 128); mbar_init(freeb + i, 1); }
        for (int i = 0; i < NST; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 1); }
        for (int i = 0; i < 2; ++i) {
            mbar_init(dq_full + i, 1);
            mbar_init(dq_empty + i, 128);
            mbar_init(ds_empty + i, 1);
            mbar_init(staged + i, 256);
        }
        sched_init(sc, F_SCHED_CONSUMERS);
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < p.n; i += blockDim.x) expc[i] = 0;
    if (warp == W_MMA) tmem_alloc<512>(tmem_slot);
    sched_load_tables(sc, p, false);
    __syncthreads();
    // contributions expected per query block I: the column tiles whose union row list holds I
    for (int e = threadIdx.x; e < sc.tab[TAB_PTR + p.ntiles]; e += blockDim.x) atomicAdd(expc + p.plan[p.off_col + e], 1);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int nitems = (int)(p.bh * p.ntiles);
    // register budgets per warpgroup (each warpgroup executes one setmaxnreg at the top of its branch):
    // softmax 2 x 128 x 168 + dQ 128 x 120 + single-lane roles 128 x 56 = 65536
    if (warp >= W_PROD) {
    regs_dec<56>();
    if (warp == W_PROD) {
        // ------------------------------------------------------------ scheduler + TMA producer
        if (lane == 0) {
            prefetch_tmap(&tmK); prefetch_tmap(&tmV); prefetch_tmap(&tmQ); prefetch_tmap(&tmdO);
            prefetch_tmap(&tmdK); prefetch_tmap(&tmdV); prefetch_tmap(&tmAcc);
        }
        int st = 0, nk = 0, pre = -2;
        uint32_t ph = 0;
        for (int ks = 0;; ++ks) {
            const int item = sched_produce(sc, ks, p, nitems, false, pre);
            pre = -2;
            if (item < 0) break;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *rows = sc.col + (ks & 3) * SCHED_CAP;
            if (cnt > 0) {
                const int kb = nk & 1;
                if (nk >= 2) mbar_wait(kv_empty + kb, ((nk >> 1) - 1) & 1);
                if (elect_one()) {
                    // the tile's S block columns (plan bperm), one B-row box each; an empty slot loads
                    // block column 0 instead (finite values: its dS rows are zero, and 0 * K must be 0
                    // in the dQ contraction over the tile's keys; never stored)
                    const int *pm = sc.tab + TAB_PERM + t * p.S;
                    mbar_arrive_expect_tx(kv_full + kb, (uint32_t)p.S * 2 * F_TILE);
                    for (int sl = 0; sl < p.S; ++sl) {
                        const int c = pm[sl] < p.n ? pm[sl] : 0;
                        tma_load_3d(sKV + kb * F_KV + sl * F_TILE, &tmK, kv_full + kb, 0, c * FB, bh);
                        tma_load_3d(sKV + kb * F_KV + 16384 + sl * F_TILE, &tmV, kv_full + kb, 0, c * FB, bh);
                    }
                }
                __syncwarp();
                ++nk;
                for (int j = 0; j < cnt; ++j) {
                    const int I = rows[j];
                    if (j == (cnt > 2 ? cnt - 2 : 0)) pre = sched_prefetch(p);
                    mbar_wait(q_empty + st, ph ^ 1);
                    uint8_t *stg = sStage + st * F_STAGE;
                    if (elect_one()) {
                        mbar_arrive_expect_tx(q_full + st, 2 * F_TILE + 2 * FB * 4);
                        tma_load_3d(stg, &tmQ, q_full + st, 0, I * FB, bh);
                        tma_load_3d(stg + F_TILE, &tmdO, q_full + st, 0, I * FB, bh);
                        bulk_load(stg + 2 * F_TILE, p.lse + (int64_t)bh * p.L + (int64_t)I * FB, FB * 4, q_full + st);
                        bulk_load(stg + 2 * F_TILE + 512, p.D + (int64_t)bh * p.L + (int64_t)I * FB, FB * 4, q_full + st);
                    }
                    __syncwarp();
                    if (++st == NST) { st = 0; ph ^= 1; }
                }
            }
            __syncwarp();
        }
    } else if (warp == W_MMA) {
        // ------------------------------------------------------------ S^T / dP^T issuer
        int sst = 0, nk = 0;
        uint32_t sph = 0, g = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int cnt = h[3];
            if (cnt > 0) {
                const int kb = nk & 1;
                mbar_wait(kv_full + kb, (nk >> 1) & 1);
                tc_fence_after();
                ++nk;
                const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + kb * F_KV));
                const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + kb * F_KV + 16384));
                for (int sj = 0; sj < cnt; ++sj) {
                    const uint32_t gs = g + sj, b = gs % NBUF, u = gs / NBUF;
                    if (u > 0) mbar_wait(freeb + b, (u - 1) & 1);
                    mbar_wait(q_full + sst, sph);
                    tc_fence_after();
                    uint8_t *stg = sStage + sst * F_STAGE;
                    const uint32_t cs = b * BUFW;
                    const uint64_t dQ0 = sdesc_sw128(smem_u32(stg));
                    const uint64_t ddO0 = sdesc_sw128(smem_u32(stg + F_TILE));
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) MMA_SS(tmem + cs, dK0 + 2 * k, dQ0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                        for (int k = 0; k < 4; ++k) MMA_SS(tmem + cs + FB, dV0 + 2 * k, ddO0 + 2 * k, IDESC_ST, k > 0);
                        mma_commit(s_full + 2 * b + (sj & 1));
                    }
                    __syncwarp();
                    if (++sst == NST) { sst = 0; sph ^= 1; }
                }
                g += cnt;
            }
            sched_release(sc, ks, true);
        }
    } else if (warp == W_MMA2) {
        // ------------------------------------------------------------ dV / dK / dQ issuer
        int pst = 0, na = 0;
        uint32_t g = 0, gp = 0;  // gp: global pair counter (dQ accumulator gp % 2, dS buffer gp % 2)
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int cnt = h[3];
            if (cnt > 0) {
                const int kb = (na & 1);  // K/V buffer of this item (the producer's nk order)
                if (na > 0) mbar_wait(acc_empty, (na - 1) & 1);  // the last item's dK/dV were read
                ++na;
                const uint64_t dKmn = sdesc_sw128(smem_u32(sKV + kb * F_KV));  // K as the MN-major B of dQ
                for (int pj = 0; pj < cnt; ++pj) {
                    const uint32_t gq = g + pj, b = gq % NBUF, u = gq / NBUF;
                    mbar_wait(p_full + b, u & 1);
                    tc_fence_after();
                    uint8_t *stg = sStage + pst * F_STAGE;
                    const uint64_t dQ0 = sdesc_sw128(smem_u32(stg));
                    const uint64_t ddO0 = sdesc_sw128(smem_u32(stg + F_TILE));
                    const uint32_t cs = b * BUFW;
                    const bool pair_end = (pj & 1) || pj == cnt - 1;
                    if (pair_end && gp >= 2) mbar_wait(dq_empty + (gp & 1), ((gp >> 1) - 1) & 1);
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int k = 0; k < FB / 16; ++k)
                            MMA_TS(tmem + COL_DV, tmem + cs + 32 * (k / 2) + 8 * (k % 2), ddO0 + 128 * k, IDESC_DKV,
                                   (pj > 0) || (k > 0));
#pragma unroll
                        for (int k = 0; k < FB / 16; ++k)
                            MMA_TS(tmem + COL_DK, tmem + cs + FB + 32 * (k / 2) + 8 * (k % 2), dQ0 + 128 * k,
                                   IDESC_DKV, (pj > 0) || (k > 0));
                        mma_commit(freeb + b);
                        mma_commit(q_empty + pst);
                        if (pair_end) {
                            // [dQ_I0; dQ_I1] = [dS_I0; dS_I1] K over the tile's 128 keys (8 K-steps of 16)
                            const uint64_t dS0 = sdesc_sw128(smem_u32(sDS + (gp & 1) * F_DSP), F_DSP / 2, 1024);
#pragma unroll
                            for (int k = 0; k < 8; ++k)
                                if (!SPION_FDBG_NODQMMA)
                                    MMA_SS(tmem + COL_DQ + (gp & 1) * 64, dS0 + 128 * k, dKmn + 128 * k, IDESC_DQ, k > 0);
                            mma_commit(dq_full + (gp & 1));
                        }
                        if (pj == cnt - 1) mma_commit(acc_full);
                    }
                    __syncwarp();
                    if (pair_end) ++gp;
                    if (++pst == NST) pst = 0;
                }
                g += cnt;
            }
            sched_release(sc, ks, true);
        }
    } else if (warp == W_STORE) {
        // ------------------------------------------------------------ dK / dV TMA storer
        int ns = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], t = h[2], cnt = h[3];
            if (cnt > 0) {
                const int sb = ns & 1;
                mbar_wait(staged + sb, (ns >> 1) & 1);
                ++ns;
                if (lane == 0) {
                    const int *pm = sc.tab + TAB_PERM + t * p.S;
                    for (int sl = 0; sl < p.S; ++sl) {
                        const int c = pm[sl];
                        if (c >= p.n) continue;
                        tma_store_3d(&tmdK, sKV + sb * F_KV + sl * F_TILE, 0, c * FB, bh);
                        tma_store_3d(&tmdV, sKV + sb * F_KV + 16384 + sl * F_TILE, 0, c * FB, bh);
                    }
                    bulk_commit();
                    bulk_wait_read0();
                    mbar_arrive(kv_empty + sb);
                }
                __syncwarp();
            }
            sched_release(sc, ks, true);
        }
        if (lane == 0) bulk_wait0();
    }
    } else if (warp >= W_DQ0) {
        // ------------------------------------------------------------ dQ warpgroup
        // Per pair: TMEM -> staged fp32 rows -> TMA reduce-adds (leader).  Completion bookkeeping is
        // lagged so no global round trip blocks the pair loop: at pair p the leader waits for pair
        // p-1's reductions (issued a pair ago), issues its two completion-counter atomics, and consumes
        // the atomics issued at pair p-1 (for pair p-2): a query block whose count reached the plan's
        // contribution count joins a shared-memory queue.  Finalising one queued block takes two
        // pairs: its fp32 rows are loaded into registers at the end of one pair and converted /
        // stored (and their L2 lines discarded) at the end of the next.
        regs_dec<120>();
        const int q4 = warp & 3;
        const int row = q4 * 32 + lane;   // accumulator row = TMEM lane: pair half row / 64, query row % 64
        const int half = row >> 6, qr = row & 63;
        const int tq = threadIdx.x - W_DQ0 * 32;  // 0..127: finalise row tq/2, 32-column half tq&1
        const uint32_t tl = tmem + ((uint32_t)(q4 * 32) << 16);
        const bool leader = warp == W_DQ0 && lane == 0;
        int *fq = fin;              // [0] head (leader only), [1] tail, [2..] ring of FQ (bh, I)
        constexpr int FQ = 64;
        if (leader) { fq[0] = 0; fq[1] = 0; }
        // leader state: the previous pair, awaiting completion (A); completed entries not yet counted
        // (pending, shared memory); counter atomics issued, results not yet consumed (R, registers).
        // The counting is batched: one release fence per batch of up to 8 entries.
        int a_n = 0, a_bh = 0, a_I0 = 0, a_I1 = 0;
        int *pend = fq + 2 + 2 * FQ;  // [8][2] (bh, I)
        int np = 0, nr = 0;
        int rr[8], rbh[8], rI[8];
        auto push = [&](int bh, int I) {
            const int t = fq[1];
            fq[2 + 2 * (t % FQ)] = bh;
            fq[3 + 2 * (t % FQ)] = I;
            fq[1] = t + 1;
        };
        auto consume_r = [&]() {  // leader: the batch of atomics issued before has returned
            bool any = false;
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < nr && rr[i] == expc[rI[i]] - 1) {
                    push(rbh[i], rI[i]);
                    any = true;
                }
            if (any) __threadfence();  // acquire: the other contributors' reductions happen-before the loads
            nr = 0;
        };
        auto flush = [&]() {  // leader: count every pending (completed) entry
            consume_r();
            if (np == 0) return;
            fence_proxy_async_global();
            __threadfence();  // release: this CTA's completed reductions before its counter increments
#pragma unroll
            for (int i = 0; i < 8; ++i)
                if (i < np) {
                    rbh[i] = pend[2 * i];
                    rI[i] = pend[2 * i + 1];
                    rr[i] = atomicAdd(f.done + (int64_t)rbh[i] * p.n + rI[i], 1);
                }
            nr = np;
            np = 0;
        };
        auto complete_a = [&]() {  // leader: pair A's reductions are complete -> pending
            for (int e = 0; e < a_n; ++e) {
                pend[2 * np] = a_bh;
                pend[2 * np + 1] = e == 0 ? a_I0 : a_I1;
                ++np;
            }
            a_n = 0;
            if (np >= 6) flush();
        };
        // finaliser state (every thread): one block loaded in registers, waiting to be stored
        int f_bh = -1, f_I = 0, f_head = 0;
        float fv[32];
        auto fin_store = [&]() {
            if (f_bh < 0) return;
            __nv_bfloat16 *dst = static_cast<__nv_bfloat16 *>(f.dQ) + (int64_t)f_bh * p.stride_bh +
                                 (int64_t)(f_I * FB + (tq >> 1)) * p.stride_l;
            store_row_bf16(dst, fv, p.scale, tq & 1);
            // the 16 KB of fp32 rows are dead: drop them from L2 without a write-back
            if (!SPION_FDBG_NODISCARD) discard_l2_line(f.dQacc + ((int64_t)f_bh * p.L + (int64_t)f_I * FB) * 64 + tq * 32);
            f_bh = -1;
        };
        auto fin_load = [&](int tail) {  // after a barrier: start the next queued block, if any
            if (f_head >= tail) return;
            if (SPION_FDBG_NOFINLOAD) { f_head = tail; return; }
            f_bh = fq[2 + 2 * (f_head % FQ)];
            f_I = fq[3 + 2 * (f_head % FQ)];
            ++f_head;
            const float4 *src = reinterpret_cast<const float4 *>(
                f.dQacc + ((int64_t)f_bh * p.L + (int64_t)f_I * FB + (tq >> 1)) * 64 + (tq & 1) * 32);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float4 x = __ldcg(src + c);
                fv[4 * c] = x.x; fv[4 * c + 1] = x.y; fv[4 * c + 2] = x.z; fv[4 * c + 3] = x.w;
            }
        };
        uint32_t gp = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], cnt = h[3];
            const int *rows = sc.col + (ks & 3) * SCHED_CAP;
            for (int pj = 0; pj < cnt; pj += 2) {
                const bool paired = pj + 1 < cnt;
                const int acc = gp & 1;
                uint8_t *slot = sDS + acc * F_DSP;
                mbar_wait(dq_full + acc, (gp >> 1) & 1);
                tc_fence_after();
                float v0[32], v1[32];
                tmem_ld32(tl + COL_DQ + acc * 64, v0);
                tmem_ld32(tl + COL_DQ + acc * 64 + 32, v1);
                tmem_ld_wait();
                tc_fence_before();
                mbar_arrive(dq_empty + acc);
                // the dQ MMA has completed, so the pair's dS buffer is free: stage the fp32 rows there
                if ((half == 0 || paired) && !SPION_FDBG_NODQ) {
                    // two [64 rows][32 fp32] TMA boxes per entry, 128-byte swizzled (the reduce's tensor
                    // map unswizzles): 16-byte chunk c of row qr at (c ^ (qr & 7)) -> conflict-free STS
                    uint8_t *dst = slot + half * (F_DSP / 2) + qr * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const uint32_t sw = (uint32_t)((c ^ (qr & 7)) << 4);
                        *reinterpret_cast<float4 *>(dst + sw) = make_float4(v0[4 * c], v0[4 * c + 1], v0[4 * c + 2], v0[4 * c + 3]);
                        *reinterpret_cast<float4 *>(dst + 8192 + sw) =
                            make_float4(v1[4 * c], v1[4 * c + 1], v1[4 * c + 2], v1[4 * c + 3]);
                    }
                }
                fence_proxy_async_smem();
                named_bar_sync(BAR_DQ, 128);
                fin_store();  // the block loaded at the previous pair
                if (leader) {
                    if (SPION_FDBG_NODQ) {
                        mbar_arrive(ds_empty + acc);
                    } else {
                        const int I0 = rows[pj], I1 = paired ? rows[pj + 1] : 0;
                        tma_reduce_add_3d(&tmAcc, slot, 0, I0 * FB, bh);
                        tma_reduce_add_3d(&tmAcc, slot + 8192, 32, I0 * FB, bh);
                        if (paired) {
                            tma_reduce_add_3d(&tmAcc, slot + F_DSP / 2, 0, I1 * FB, bh);
                            tma_reduce_add_3d(&tmAcc, slot + F_DSP / 2 + 8192, 32, I1 * FB, bh);
                        }
                        bulk_commit();
                        bulk_wait_read<0>();  // staged rows consumed: the softmax may refill the buffer
                        mbar_arrive(ds_empty + acc);
                        bulk_wait<1>();       // the previous pair's reductions are complete
                        if (!SPION_FDBG_NOFIN) complete_a();
                        a_n = paired ? 2 : 1; a_bh = bh; a_I0 = I0; a_I1 = I1;
                    }
                }
                named_bar_sync(BAR_DQ, 128);
                if (!SPION_FDBG_NOFIN) {
                    const int tail = fq[1];
                    while (tail - f_head > FQ / 2) {     // backlog (bursts of completions): catch up now
                        fin_load(tail);
                        fin_store();
                    }
                    fin_load(tail);
                }
                ++gp;
            }
            sched_release(sc, ks, true);
        }
        // drain: the last pair's reductions, every pending count, every queued block
        if (leader && !SPION_FDBG_NODQ && !SPION_FDBG_NOFIN) {
            bulk_wait<0>();
            complete_a();
            flush();      // the last batch of atomics ...
            consume_r();  // ... and its results
        }
        named_bar_sync(BAR_DQ, 128);
        if (!SPION_FDBG_NOFIN) {
            const int tail = fq[1];
            fin_store();
            while (f_head < tail) {
                fin_load(tail);
                fin_store();
            }
        }
    } else {
        // ------------------------------------------------------------ softmax / dK-dV epilogue
        regs_inc<168>();
        const int r = (warp & 3) * 32 + lane;  // key row of the tile = TMEM lane
        const int wg = warp >> 2;              // warpgroup: even (0) / odd (1) entries of an item
        const int slot = r / FB;
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t a_ph = 0, ph = 0, g = 0, sph = 0, gp = 0;
        int st = 0, nk = 0;
        const float sl2 = p.scale_log2;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *msks = sc.msk + (ks & 3) * SCHED_CAP;
            const int pcol = sc.tab[TAB_PERM + t * p.S + slot];  // this row's block column (n: empty slot)
            const int key = pcol * FB + (r % FB);
            if (cnt == 0) {
                if (pcol < p.n) {
                    __nv_bfloat16 *dkrow = static_cast<__nv_bfloat16 *>(p.dK) + (int64_t)bh * p.stride_bh +
                                           (int64_t)key * p.stride_l;
                    __nv_bfloat16 *dvrow = static_cast<__nv_bfloat16 *>(p.dV) + (int64_t)bh * p.stride_bh +
                                           (int64_t)key * p.stride_l;
                    zero_row_bf16(wg == 0 ? dkrow : dvrow);
                }
                sched_release(sc, ks, true);
                continue;
            }
            for (int jj = 0; jj < cnt; ++jj) {
                if ((jj & 1) != wg) {
                    if (++st == NST) { st = 0; ph ^= 1; }
                    if (jj & 1 || jj == cnt - 1) ++gp;
                    continue;
                }
                const bool active = (msks[jj] >> slot) & 1;
                const uint32_t gs = g + jj, sb = gs % NBUF;
                mbar_wait(s_full + 2 * sb + wg, (sph >> sb) & 1);
                sph ^= 1u << sb;
                mbar_wait(q_full + st, ph);
                const float *snl2 = reinterpret_cast<const float *>(sStage + st * F_STAGE + 2 * F_TILE);
                const float *sD = snl2 + 128;
                // this entry's half of the pair's dS buffer must have been drained (pair gp - 2)
                if (gp >= 2) mbar_wait(ds_empty + (gp & 1), ((gp >> 1) - 1) & 1);
                uint8_t *dsrow = sDS + (gp & 1) * F_DSP + wg * (F_DSP / 2);
                tc_fence_after();
                const uint32_t cs = sb * BUFW;
#pragma unroll
                for (int hh = 0; hh < FB / 32; ++hh) {
                    const uint32_t c32 = hh * 32;
                    uint32_t pk[16], dk[16];
                    if (active && !SPION_DBG_NOSOFTMAX) {
                        float sv[32], dp[32];
                        tmem_ld32(tl + cs + c32, sv);
                        tmem_ld32(tl + cs + FB + c32, dp);
                        tmem_ld_wait();
                        const uint64_t sl22 = f2pack(sl2, sl2);
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            // the query block's -lse log2e and D, 4 columns per broadcast LDS.128
                            const float4 a = reinterpret_cast<const float4 *>(snl2 + c32)[i / 4];
                            const float4 b = reinterpret_cast<const float4 *>(sD + c32)[i / 4];
                            const float nl[4] = {a.x, a.y, a.z, a.w}, dd[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                            for (int j = 0; j < 4; j += 2) {
                                float a0, a1, d0, d1;
                                f2unpack(ffma2(f2pack(sv[i + j], sv[i + j + 1]), sl22, f2pack(nl[j], nl[j + 1])), a0,
                                         a1);
                                const float p0 = ex2m(a0, i + j), p1 = ex2m(a1, i + j + 1);
                                pk[(i + j) / 2] = pack_bf16(p0, p1);
                                f2unpack(fmul2(f2pack(p0, p1),
                                               fsub2(f2pack(dp[i + j], dp[i + j + 1]), f2pack(dd[j], dd[j + 1]))),
                                         d0, d1);
                                dk[(i + j) / 2] = pack_bf16(d0, d1);
                            }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) { pk[i] = 0u; dk[i] = 0u; }
                    }
                    tmem_st16(tl + cs + c32, pk);
                    tmem_st16(tl + cs + FB + c32, dk);
                    // dS^T row r (queries c32 .. c32+31) into the pair buffer: SW128, row = key
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        *reinterpret_cast<uint4 *>(dsrow + sw128_offset(r, hh * 4 + c)) =
                            make_uint4(dk[4 * c], dk[4 * c + 1], dk[4 * c + 2], dk[4 * c + 3]);
                }
                fence_proxy_async_smem();  // dS^T (generic proxy) -> the dQ MMA (async proxy)
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full + sb);
                if (++st == NST) { st = 0; ph ^= 1; }
                if (jj & 1 || jj == cnt - 1) ++gp;
            }
            mbar_wait(acc_full, a_ph);
            a_ph ^= 1;
            tc_fence_after();
            // dK (warpgroup 0, x scale) / dV (warpgroup 1) -> bf16 staged in this item's K/V buffer
            const int kb = nk & 1;
            ++nk;
            uint8_t *dst = sKV + kb * F_KV + (wg == 0 ? 0 : 16384);
            const uint32_t col = wg == 0 ? COL_DK : COL_DV;
            const float fsc = wg == 0 ? p.scale : 1.f;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float w[32];
                tmem_ld32(tl + col + hh * 32, w);
                tmem_ld_wait();
                stage_row_bf16(dst, r, w, fsc, hh);
            }
            tc_fence_before();
            mbar_arrive(acc_empty);
            fence_proxy_async_smem();
            mbar_arrive(staged + kb);
            g += cnt;
            sched_release(sc, ks, true);
        }
    }
    __syncthreads();
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
}

// ---------------------------------------------------------------- host
bool fused_bwd_supported(const AttnArgs &a) { return a.B == FB && a.d == 64; }

size_t fused_bwd_ws_bytes(int64_t bh, int L, int n) {
    return round_up((size_t)bh * n * 4, 256) + round_up((size_t)bh * L * 64 * 4, 256);
}

// dQacc [bh][L][64] fp32 as a 3-D tensor; box 32 x 64 x 1 (128-byte rows), 128-byte swizzle
static bool acc_map(CUtensorMap *m, float *base, int L, int64_t bh) {
    auto enc = tc_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)L, (cuuint64_t)bh};
    cuuint64_t strides[2] = {64 * 4, (cuuint64_t)L * 64 * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)FB, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

spion_status launch_bwd_fused(const AttnArgs &a, void *fws, cudaStream_t s) {
    static PerDevice attr;
    SPION_CUDA_TRY(smem_attr_once(attr, attn_bwd_fused_tc_kernel, (int)F_SMEM));
    FusedParams f;
    f.done = static_cast<int *>(fws);
    f.dQacc = reinterpret_cast<float *>(static_cast<char *>(fws) + round_up((size_t)a.bh * a.n * 4, 256));
    f.dQ = a.dQ;
    {
        const int64_t rows = a.bh * a.L;
        const int64_t thr = rows * 8 > a.bh * a.n ? rows * 8 : a.bh * a.n;
        attn_bwd_prep_kernel<<<(unsigned)((thr + 255) / 256), 256, 0, s>>>(
            static_cast<const __nv_bfloat16 *>(a.O), static_cast<const __nv_bfloat16 *>(a.dO), a.lse,
            const_cast<float *>(a.D), a.nlse2, f.dQacc, f.done, static_cast<__nv_bfloat16 *>(a.dQ), a.brow_ptr, a.bh,
            a.L, a.B, a.n, a.stride_bh, a.stride_l);
        SPION_LAUNCH_CHECK();
    }
    CUtensorMap mk, mv, mq, mdo, mdk, mdv, macc;
    if (!acc_map(&macc, f.dQacc, a.L, a.bh)) return SPION_ERR_CUDA;
    if (!tc_map(&mk, a.K, a.L, a.bh, a.stride_bh, a.stride_l, FB) ||
        !tc_map(&mv, a.V, a.L, a.bh, a.stride_bh, a.stride_l, FB) ||
        !tc_map(&mq, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, FB) ||
        !tc_map(&mdo, a.dO, a.L, a.bh, a.stride_bh, a.stride_l, FB) ||
        !tc_map(&mdk, a.dK, a.L, a.bh, a.stride_bh, a.stride_l, FB) ||
        !tc_map(&mdv, a.dV, a.L, a.bh, a.stride_bh, a.stride_l, FB))
        return SPION_ERR_CUDA;
    TcParams p = tc_base_params(a, 2, 1);
    p.lse = a.nlse2;  // staged per query block: -lse * log2(e)
    p.D = const_cast<float *>(a.D);
    p.dK = a.dK;
    p.dV = a.dV;
    const int64_t items = p.bh * p.ntiles;
    const int grid = (int)(items < tc_num_sms() ? items : tc_num_sms());
    attn_bwd_fused_tc_kernel<<<grid, F_THREADS, F_SMEM, s>>>(mk, mv, mq, mdo, mdk, mdv, macc, p, f);
    SPION_LAUNCH_CHECK();
    note_tc_launch();
    return SPION_OK;
}

}  // namespace spion
