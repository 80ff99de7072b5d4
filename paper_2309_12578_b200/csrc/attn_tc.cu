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
//           -> P (bf16, TMEM) -> O += P V_J (TMEM)
//   epilogue: O / Z and lse (PAPER: logaddexp(m + ln l, ln(L - cnt)), readings Q1/Q2)
// attn_bwd_dq_tc (row tiles; reading Q17), per (bh, tile):
//   D = rowsum(dO * O) from the staged tiles (written for the dK/dV kernel);
//   for J:  S = Q K_J^T, dP = dO V_J^T -> dS = exp(S*c - lse)(dP - D) (TMEM)
//           -> dQ += dS K_J (TMEM);  dQ * scale -> bf16.   No atomics.
// attn_bwd_dkdv_tc (column tiles), per (bh, tile of key blocks):
//   for I:  S^T = K Q_I^T, dP^T = V dO_I^T -> P^T, dS^T (TMEM)
//           -> dV += P^T dO_I, dK += dS^T Q_I (TMEM);  dK * scale -> bf16.
//
// Warp roles: warps 0..MW-1 softmax / epilogue (thread = TMEM lane = tile row;
// with MW = 8 the two warpgroups take alternate blocks, so the TMEM loads and
// exponentials of one overlap the other's),
// warp MW scheduler + TMA producer, warp MW+1 MMA issuer (one elected lane of a
// converged warp) and TMEM allocator.  The forward has MW = 4; the backward
// kernels MW = 8 where one CTA owns the SM.  A softmax thread writes its packed bf16
// P / dS over the first half of each 32-column chunk it has read itself.  One CTA per SM owns all 512 TMEM
// columns: S (and dP) rotate through NBUF buffers so the MMA warp runs up to NBUF
// blocks ahead of the softmax warps; P / dS are written back
// into TMEM as packed bf16 and consumed as the A operand of the next MMA
// (tcgen05 TS form), so they never touch shared memory.  Per-item tiles (Q, or
// K/V) are double buffered across work items.  Persistent grid; work items
// (bh, tile) come from an atomic counter in the plan (longest tiles of each
// bh-chunk first) and are broadcast, with their plan entries, through a
// shared-memory ring.
#include "attn_tc.cuh"

namespace spion {

static constexpr int TC_THREADS = 256;  // forward: 4 softmax warps + producer + S-MMA + storer + PV-MMA
// backward: MW softmax warps, then the producer, S-MMA, storer, second MMA and NSW - 1 more S-MMA warps
__host__ __device__ constexpr int bwd_threads(int mw, int nsw) { return 32 * (mw + 3 + nsw); }  // W_MMA3.. = MW + 4..
// Per-kernel, per-B configuration.  CTAS CTAs per SM share the 512 TMEM columns
// (COLS each) and ~227 KB of shared memory; NBUF score buffers let the MMA warp run
// up to NBUF blocks ahead of the softmax warps; TMA rings have NST >= NBUF stages
// (which keeps the look-ahead deadlock free).  Two CTAs per SM where they fit (more
// softmax warps per SM), one CTA with deeper buffering for the B=64 backward.
#ifndef SPION_DKV_CTAS32
#define SPION_DKV_CTAS32 2
#endif
#ifndef SPION_DKV_NST32
#define SPION_DKV_NST32 4
#endif
#ifndef SPION_FWD_NST32
#define SPION_FWD_NST32 8
#endif
#ifndef SPION_DKV_ACCB  // dK/dV accumulator pairs where one CTA owns the SM (1: epilogue not deferred)
#define SPION_DKV_ACCB 1
#endif
template <int B> struct Cfg {
    static constexpr int FWD_CTAS = 2, FWD_COLS = 256;
    static constexpr int FWD_NBUF = (256 - 64) / B;      // S/P buffers of B columns + O
    static constexpr int FWD_NST = B == 32 ? SPION_FWD_NST32 : 4;  // K_J + V_J per stage
    static constexpr int DQ_CTAS = B == 32 ? 2 : 1, DQ_COLS = 512 / DQ_CTAS;
    static constexpr int DQ_NBUF = (DQ_COLS - 64) / (2 * B);   // S+dP buffers + dQ
    static constexpr int DQ_NST = B == 32 ? 3 : 8;             // K_J + V_J per stage
    static constexpr int DKV_CTAS = B == 32 ? SPION_DKV_CTAS32 : 1, DKV_COLS = 512 / DKV_CTAS;
    // dK/dV accumulator pairs: two where one CTA owns the SM, so an item's epilogue (deferred by the
    // softmax warps until after their first block of the next item) never waits on, nor stalls, the
    // tensor pipe; S^T+dP^T buffers take the rest of the columns
    static constexpr int DKV_ACCB = DKV_CTAS == 1 ? SPION_DKV_ACCB : 1;
    // K and V of the item copied into TMEM (tcgen05.cp) where one CTA owns the SM: S^T = K Q_I^T and
    // dP^T = V dO_I^T then run as TS MMAs (A from tensor memory), at the cost of 64 columns
    static constexpr bool DKV_TS = SPION_DKV_TS && DKV_CTAS == 1;
    static constexpr int DKV_NBUF = (DKV_COLS - 128 * DKV_ACCB - (DKV_TS ? 64 : 0)) / (2 * B);
    static constexpr int DKV_NST = B == 32 ? SPION_DKV_NST32 : 7;  // Q_I + dO_I + lse_I + D_I per stage
    // K/V (and dK/dV staging) buffers across items: three where one CTA owns the SM, so the next
    // item's K/V can load while the previous item's dK/dV store still holds its buffer
    static constexpr int DKV_KVB = DKV_CTAS == 1 ? 3 : 2;
    // softmax warps of the backward kernels: two warpgroups (each takes half of a block's
    // columns) where one CTA owns the SM, one warpgroup where two CTAs share it
    static constexpr int DQ_MW = DQ_CTAS == 1 ? 8 : 4, DKV_MW = DKV_CTAS == 1 ? 8 : 4;
    // with two softmax warpgroups: alternate blocks (ping-pong) or split every block's columns
    static constexpr bool PING = SPION_PING;
    // S-MMA issuing warps: where one CTA owns the SM, one per TMEM score buffer (warp w issues
    // the blocks whose buffer is w), so one warp's per-block issue overhead (waits, descriptors,
    // commits, reconvergence) is not the limit, and every buffer's uses (and every ring stage's,
    // NST % NBUF == 0) stay in order within one warp, as mbarrier parity waits require
    static constexpr int DQ_NSW = DQ_CTAS == 1 && SPION_NSW ? DQ_NBUF : 1;
    static constexpr int DKV_NSW = 1;
    // a dedicated epilogue warpgroup (dK/dV accumulators -> bf16 staging) where one CTA with two softmax
    // warpgroups owns the SM, so the softmax warps run into the next item while an item's last dV/dK
    // MMAs drain and its accumulators are read (512 threads, setmaxnreg budgets)
    static constexpr bool DKV_EPI = SPION_DKV_EPI && DKV_CTAS == 1 && DKV_MW == 8 && DKV_NSW == 1;
    static constexpr int DKV_THREADS = bwd_threads(DKV_MW, DKV_NSW) + (DKV_EPI ? 128 : 0);
    static_assert(FWD_NST >= FWD_NBUF && DQ_NST >= DQ_NBUF && DKV_NST >= DKV_NBUF, "ring shallower than look-ahead");
};
// ============================================================================ forward
// Per (bh, row tile): Q tile double buffered across items; K_J/V_J stream through a
// TMA ring; S_J lands in one of NBUF TMEM buffers so the MMA warp can run up to NBUF
// blocks ahead of the softmax warps; P_J (bf16) is written back over S_J in TMEM and
// feeds O += P_J V_J as the A operand from tensor memory.  Buffers rotate by a
// global block counter g: buffer g % NBUF, use g / NBUF (mbarrier phase parity).
template <int B>
__global__ void __launch_bounds__(TC_THREADS, Cfg<B>::FWD_CTAS)
attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, TcParams p) {
    constexpr int NST = Cfg<B>::FWD_NST, NBUF = Cfg<B>::FWD_NBUF;
    constexpr uint32_t KV_BYTES = B * 128, STG = 2 * KV_BYTES;  // stage: K at +0, V at +KV_BYTES
    constexpr uint32_t IDESC_S = idesc_bf16(128, B, false, false);
    constexpr uint32_t IDESC_PV = idesc_bf16(128, 64, false, true);
    constexpr uint32_t COL_O = NBUF * B;  // S / P buffer b at columns [B b, B b + B)
    constexpr int W_PROD = 4, W_MMA = 5, W_STORE = 6, W_MMA2 = 7;

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sQ = smem;           // [2] x 16 KB
    uint8_t *sKV = smem + 32768;  // [NST] x STG
    uint8_t *sSched = sKV + NST * STG;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    // s_full[b]: S in buffer b is ready; p_full[b]: packed P in buffer b is written;
    // freeb[b]: the P.V that read buffer b completed (guards the next S into b, O rescales
    // and the epilogue).  Per buffer, so no parity waiter can fall two phases behind.
    uint64_t *q_full = bars + 0, *q_empty = bars + 2, *s_full = bars + 4, *p_full = s_full + NBUF,
             *freeb = p_full + NBUF, *kv_full = freeb + NBUF, *kv_empty = kv_full + NST;
    Sched sc = make_sched(sSched, kv_empty + NST);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(kv_empty + NST + 8);
    uint64_t *staged = kv_empty + NST + 9;  // [2]: O of the item using Q buffer qb staged
    // li: the P.V issuer has issued an item's last MMA (the S issuer starts the next item's MMAs
    // behind it, so the item's accumulator completes without queueing behind look-ahead MMAs)
    uint64_t *li = staged + 2;
    uint64_t *o_empty = staged + 3;  // the (deferred) epilogue has read the O accumulator

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        // q_empty: the last S of the item, and the epilogue's TMA store of O (staged in the
        // same buffer) having read shared memory
        for (int i = 0; i < 2; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 2); }
        for (int i = 0; i < NBUF; ++i) { mbar_init(s_full + i, 1); mbar_init(p_full + i, 128); mbar_init(freeb + i, 1); }
        for (int i = 0; i < NST; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        for (int i = 0; i < 2; ++i) mbar_init(staged + i, 128);
        mbar_init(li, 1);
        mbar_init(o_empty, 128);
        sched_init(sc, 7);
        fence_barrier_init();
    }
    if (warp == W_MMA) tmem_alloc<Cfg<B>::FWD_COLS>(tmem_slot);
    sched_load_tables(sc, p, true);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const unsigned long long t_start = p.trace ? gtimer() : 0ull;
    const int nitems = (int)(p.bh * p.ntiles);

    if (warp == W_PROD) {
        // ------------------------------------------------------------ scheduler + TMA producer
        Tracer tr(p, 0);
        if (lane == 0) { prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmV); prefetch_tmap(&tmO); }
        // The next item is fetched from the scheduler when the current one starts, and its Q tile
        // is issued as soon as a Q buffer frees up (tested between the current item's K/V stages),
        // so the S-MMA warp finds it resident when it moves on.
        int st = 0, nq = 0;
        uint32_t ph = 0;
        int pre = sched_prefetch(p);
        int item = sched_produce(sc, 0, p, nitems, true, pre);
        pre = sched_prefetch(p);
        bool issued = false;
        auto item_tile = [&](int ks, bool block) -> bool {  // Q of ring item ks (false: buffer busy)
            const int *h = sc.hdr + (ks & 3) * 8;
            if (h[3] == 0) return true;
            const int qb = nq & 1;
            if (nq >= 2) {
                const uint32_t par = ((nq >> 1) - 1) & 1;
                if (block) mbar_wait(q_empty + qb, par);
                else if (!warp_test(q_empty + qb, par)) return false;
            }
            if (elect_one()) {
                mbar_arrive_expect_tx(q_full + qb, 16384);
                tma_ld(sQ + qb * 16384, &tmQ, q_full + qb, 0, h[2] * 128, h[1], l2_evict_first());
            }
            __syncwarp();
            ++nq;
            return true;
        };
        for (int ks = 0; item >= 0; ++ks) {
            if (!issued) item_tile(ks, true);
            // the next item: list loads issued now, stored after two of this item's stages
            const SchedFetch nf = sched_fetch_begin(sc, ks + 1, p, nitems, pre);
            pre = sched_prefetch(p);
            const int nitem = nf.item;
            bool ended = false, nissued = nitem < 0;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], cnt = h[3];
            const int *col = sc.col + (ks & 3) * SCHED_CAP;
            if (lane == 0) tr.ev(1);
            for (int j = 0; j < cnt; ++j) {  // whole warp runs the loop; one elected lane issues the TMA
                if (!ended && j == 2) { sched_fetch_end(sc, ks + 1, p, nf, true); ended = true; }
                if (ended && !nissued) nissued = item_tile(ks + 1, false);
                mbar_wait(kv_empty + st, ph ^ 1);
                if (lane == 0) tr.ev(3);
                if (elect_one()) {
                    if (SPION_DBG_NOLOAD) {
                        mbar_arrive(kv_full + st);
                    } else {
                        mbar_arrive_expect_tx(kv_full + st, STG);
                        const uint64_t keep = l2_evict_last();  // K_J, V_J: read by every tile listing J
                        tma_ld(sKV + st * STG, &tmK, kv_full + st, 0, col[j] * B, bh, keep);
                        tma_ld(sKV + st * STG + KV_BYTES, &tmV, kv_full + st, 0, col[j] * B, bh, keep);
                    }
                }
                __syncwarp();
                if (++st == NST) { st = 0; ph ^= 1; }
            }
            if (!ended) sched_fetch_end(sc, ks + 1, p, nf, true);
            issued = nissued;
            item = nitem;
        }
    } else if (warp == W_MMA) {
        if (!SPION_LANE0 || lane == 0) {  // SPION_LANE0: the issuing role runs on one thread
        // ------------------------------------------------------------ S issuer (converged warp,
        // one elected lane issues): S = Q K_J^T up to NBUF blocks ahead of the softmax
        Tracer tr(p, 1);
        int sst = 0, nq = 0;
        uint32_t sph = 0, g = 0;  // global block counter (buffer = g % NBUF)
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            if (lane == 0) tr.ev(10);
            const int cnt = h[3];
            if (cnt > 0) {
                const int qb = nq & 1;
                mbar_wait(q_full + qb, (nq >> 1) & 1);
                if (lane == 0) tr.ev(11);
                if (SPION_ITEM_FENCE && nq > 0) mbar_wait(li, (nq - 1) & 1);
                tc_fence_after();
                ++nq;
                const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ + qb * 16384));
                for (int sj = 0; sj < cnt; ++sj) {
                    const uint32_t gs = g + sj, b = gs % NBUF, u = gs / NBUF;
                    mbar_wait(kv_full + sst, sph);
                    if (lane == 0) tr.ev(44);
                    if (u > 0) mbar_wait(freeb + b, (u - 1) & 1);
                    if (lane == 0) tr.ev(42);
                    tc_fence_after();
                    const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + sst * STG));
                    if (ISSUER()) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) MMA_SS(tmem + b * B, dQ0 + 2 * k, dK0 + 2 * k, IDESC_S, k > 0);
                        tr.ev(43);
                        mma_commit(s_full + b);
                        if (sj == cnt - 1) mma_commit(q_empty + qb);
                        tr.ev(41);
                    }
                    ROLE_SYNC();
                    if (++sst == NST) { sst = 0; sph ^= 1; }
                }
                g += cnt;
            }
            sched_release(sc, ks, !SPION_LANE0);
        }
        }
    } else if (warp == W_MMA2) {
        if (!SPION_LANE0 || lane == 0) {  // SPION_LANE0: the issuing role runs on one thread
        // ------------------------------------------------------------ P.V issuer: O += P_J V_J
        // (P from TMEM) as each P arrives.  A second issuing warp, so the tensor pipe is fed by
        // whichever stream is ready while the other waits (a commit stalls its issuing thread).
        Tracer tr(p, 4);
        int pst = 0, no = 0;
        uint32_t g = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int cnt = h[3];
            if (SPION_DEFER_FWD && cnt > 0) {  // the previous item's (deferred) epilogue has read O
                if (no > 0) mbar_wait(o_empty, (no - 1) & 1);
                ++no;
            }
            for (int pj = 0; pj < cnt; ++pj) {
                const uint32_t gp = g + pj, b = gp % NBUF, u = gp / NBUF;
                mbar_wait(p_full + b, u & 1);
                if (lane == 0) tr.ev(13);
                tc_fence_after();
                const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + pst * STG + KV_BYTES));
                if (ISSUER()) {
#pragma unroll
                    for (int k = 0; k < B / 16; ++k)
                        MMA_TS(tmem + COL_O, tmem + b * B + 8 * k, dV0 + 128 * k, IDESC_PV, (pj > 0) || (k > 0));
                    tr.ev(32);
                    if (SPION_ITEM_FENCE && pj == cnt - 1) mbar_arrive(li);
                    mma_commit(freeb + b);
                    mma_commit(kv_empty + pst);  // S(pj) (K) completed before P(pj) existed
                    tr.ev(33);
                }
                ROLE_SYNC();
                if (++pst == NST) pst = 0;
            }
            g += cnt;
            sched_release(sc, ks, !SPION_LANE0);
        }
        }
    } else if (warp == W_STORE) {
        // storer: once the softmax warps have staged an item's output tile(s) in shared
        // memory, one TMA store per tile; the buffer is released when the store has read it
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
                    tma_st(&tmO, sQ + sb * 16384, 0, t * 128, bh, l2_evict_first());
                    bulk_commit();
                    bulk_wait_read0();
                    mbar_arrive(q_empty + sb);
                }
                __syncwarp();
            }
            sched_release(sc, ks, true);
        }
        if (lane == 0) bulk_wait0();
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int r = threadIdx.x;  // tile row = TMEM lane
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)(warp * 32) << 16);
        uint32_t g = 0;
        int nq = 0;
        const float sl2 = p.scale_log2;
        Tracer tr(p, threadIdx.x == 0 ? 2 : 3);
        const bool trc = threadIdx.x == 0 || threadIdx.x == 64;
        // pending epilogue (SPION_DEFER_FWD): O / Z of an item whose blocks are done, staged after the
        // first block of the next item, so the softmax warps do not idle while its last P.V drains (the
        // next item's first P.V waits for it through o_empty)
        int dfr_qb = -1, dfr_cnt = 0;
        uint32_t dfr_g = 0;
        float dfr_f = 0.f;
        auto epilogue = [&]() {
            if (dfr_qb < 0) return;
            // every P.V of the item that is not yet known complete (the last NBUF at most)
            for (int pj = (dfr_cnt > NBUF ? dfr_cnt - NBUF : 0); pj < dfr_cnt; ++pj) {
                const uint32_t gp = dfr_g + pj;
                mbar_wait(freeb + gp % NBUF, (gp / NBUF) & 1);
            }
            if (trc) tr.ev(23);
            tc_fence_after();
            // O / Z -> bf16 staged in the item's Q buffer (its last S is done), one TMA store
            uint8_t *sO = sQ + dfr_qb * 16384;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                float o[32];
                tmem_ld32(tl + COL_O + hh * 32, o);
                tmem_ld_wait();
                stage_row_bf16(sO, r, o, dfr_f, hh);
            }
            tc_fence_before();
            if (SPION_DEFER_FWD) mbar_arrive(o_empty);
            fence_proxy_async_smem();  // generic-proxy writes -> the TMA store (async proxy)
            mbar_arrive(staged + dfr_qb);
            tc_fence_before();
            if (trc) tr.ev(24);
            dfr_qb = -1;
        };
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            if (trc) tr.ev(20);
            const int bh = h[1], t = h[2], cnt = h[3], rcnt = h[4 + slot];
            const int *msks = sc.msk + (ks & 3) * SCHED_CAP;
            const int row = t * 128 + r;
            const bool valid = row < p.L;
            __nv_bfloat16 *orow =
                static_cast<__nv_bfloat16 *>(p.O) + (int64_t)bh * p.stride_bh + (int64_t)row * p.stride_l;
            float m_run = -INFINITY, l_run = 0.f;
            for (int jj = 0; jj < cnt; ++jj) {
                const bool active = (msks[jj] >> slot) & 1;  // warp-uniform (B >= 32)
                const uint32_t gs = g + jj, sb = gs % NBUF;
                mbar_wait(s_full + sb, (gs / NBUF) & 1);
                if (trc) tr.ev(21);
                tc_fence_after();
                uint32_t packed[B / 2];
                float alpha = 1.f;
                bool rescale = false;
                if (active && !SPION_DBG_NOSOFTMAX) {
                    float s[B];  // raw scores; the softmax scale is folded into the exponent
#pragma unroll
                    for (int hh = 0; hh < B / 32; ++hh) {
                        float v[32];
                        tmem_ld32(tl + sb * B + hh * 32, v);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) s[hh * 32 + i] = v[i];
                    }
                    float m4[4] = {s[0], s[1], s[2], s[3]};  // 4 independent chains (latency)
#pragma unroll
                    for (int i = 4; i < B; ++i) m4[i & 3] = fmaxf(m4[i & 3], s[i]);
                    float mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                    if (trc) tr.ev(52);
                    mx *= sl2;  // scale > 0: max commutes with the scaling (log2 domain)
                    if (m_run == -INFINITY) {
                        m_run = mx;
                    } else if (mx > m_run + 8.f) {  // rescale only on a large max increase
                        alpha = ex2(m_run - mx);
                        m_run = mx;
                        rescale = true;
                    }
                    // packed fp32x2: s * scale*log2(e) - m for two columns per FFMA2; two running sums
                    const uint64_t sl22 = f2pack(sl2, sl2), nm2 = f2pack(-m_run, -m_run);
                    uint64_t sum2[2] = {0ull, 0ull};  // two independent FADD2 chains
#pragma unroll
                    for (int i = 0; i < B; i += 2) {
                        float a0, a1;
                        f2unpack(ffma2(f2pack(s[i], s[i + 1]), sl22, nm2), a0, a1);
                        const float e0 = ex2m(a0, i), e1 = ex2m(a1, i + 1);
                        sum2[(i >> 1) & 1] = fadd2(sum2[(i >> 1) & 1], f2pack(e0, e1));
                        packed[i / 2] = pack_bf16(e0, e1);
                    }
                    float s0, s1;
                    f2unpack(fadd2(sum2[0], sum2[1]), s0, s1);
                    l_run = l_run * alpha + (s0 + s1);
                    if (trc) tr.ev(53);
                } else {
#pragma unroll
                    for (int i = 0; i < B / 2; ++i) packed[i] = 0u;
                }
                if (__any_sync(0xffffffffu, rescale)) {  // O *= alpha once every earlier P.V is complete
                    for (int pj = (jj > NBUF ? jj - NBUF : 0); pj < jj; ++pj) {
                        const uint32_t gp = g + pj;
                        mbar_wait(freeb + gp % NBUF, (gp / NBUF) & 1);
                    }
                    tc_fence_after();
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        float o[32];
                        tmem_ld32(tl + COL_O + hh * 32, o);
                        tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] *= alpha;
                        tmem_st32(tl + COL_O + hh * 32, o);
                    }
                }
#pragma unroll
                for (int hh = 0; hh < B / 32; ++hh) {
                    uint32_t v[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) v[i] = packed[hh * 16 + i];
                    tmem_st16(tl + sb * B + hh * 16, v);
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full + sb);
                if (trc) tr.ev(22);
                if (jj == 0) epilogue();  // the previous item's (deferred), after this item's first block
            }
            epilogue();  // (an item without blocks)
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
                dfr_qb = nq & 1;
                ++nq;
                dfr_cnt = cnt;
                dfr_g = g;
                dfr_f = f;
                if (!SPION_DEFER_FWD) epilogue();
            } else if (valid) {
                zero_row_bf16(orow);
            }
            if (valid) p.lse_out[(int64_t)bh * p.L + row] = lse2 * LN2;
            g += cnt;
            sched_release(sc, ks, true);
        }
        epilogue();  // the last item's
    }
    __syncthreads();
    sched_finish(p, t_start);
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc<Cfg<B>::FWD_COLS>(tmem);
    }
}

// ============================================================================ backward: dQ
// Per (bh, row tile): D = rowsum(dO * O) (written for the dK/dV kernel); for each
// block J: S, dP into one of NBUF TMEM buffer pairs -> dS = exp(S c - lse)(dP - D),
// packed bf16 over S -> dQ += dS K_J (A from TMEM).  No atomics, no fp32 round trip.
template <int B>
__global__ void __launch_bounds__(bwd_threads(Cfg<B>::DQ_MW, Cfg<B>::DQ_NSW), Cfg<B>::DQ_CTAS)
attn_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                      const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdQ, TcParams p) {
    constexpr int NST = Cfg<B>::DQ_NST, NBUF = Cfg<B>::DQ_NBUF, MW = Cfg<B>::DQ_MW, NSW = Cfg<B>::DQ_NSW;
    constexpr bool PP = MW == 8 && Cfg<B>::PING;   // warpgroups take alternate blocks
    constexpr int CPT = PP || MW == 4 ? B : B / 2;  // columns of a block per softmax thread
    constexpr int W_PROD = MW, W_MMA = MW + 1, W_STORE = MW + 2, W_MMA2 = MW + 3, W_MMA3 = MW + 4;
    constexpr uint32_t BUFW = 2 * B;  // S at b*BUFW, dP at b*BUFW + B
    constexpr uint32_t COL_DQ = NBUF * BUFW;
    // Q and dO of the item copied into TMEM (tcgen05.cp) where the columns allow: S = Q K_J^T and
    // dP = dO V_J^T then run as TS MMAs (A from tensor memory), reading only K_J / V_J from shared
    // memory (SS MMAs at N = 64 are shared-memory bound: 48 vs 32 cycles per K = 16 step)
    constexpr bool TSQ = SPION_DQ_TS && (NBUF * BUFW + 64 + 64 <= Cfg<B>::DQ_COLS);
    constexpr uint32_t COL_QA = COL_DQ + 64, COL_DOA = COL_QA + 32;
    constexpr uint32_t KV_BYTES = B * 128, STG = 2 * KV_BYTES;
    constexpr uint32_t IDESC_S = idesc_bf16(128, B, false, false);   // S = Q K^T, dP = dO V^T
    constexpr uint32_t IDESC_DQ = idesc_bf16(128, 64, false, true);  // dQ += dS K

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sQ = smem, *sdO = smem + 32768, *sO = smem + 65536;  // sQ, sdO: [2] x 16 KB
    uint8_t *sKV = smem + 81920;                                    // [NST] x STG
    uint8_t *sSched = sKV + NST * STG;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    uint64_t *q_full = bars + 0, *q_empty = bars + 2, *o_full = bars + 4, *o_empty = bars + 5, *dq_full = bars + 6,
             *s_full = bars + 7, *ds_full = s_full + 2 * NBUF, *freeb = ds_full + NBUF, *kv_full = freeb + NBUF,
             *kv_empty = kv_full + NST;
    Sched sc = make_sched(sSched, kv_empty + NST);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(kv_empty + NST + 8);
    uint64_t *staged = kv_empty + NST + 9;  // [2]: dQ of the item using Q buffer qb staged
    uint64_t *acc_empty = staged + 2;       // the epilogue has read the dQ accumulator
    uint64_t *li = acc_empty + 1;           // the dQ issuer has issued an item's last MMA (as forward)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        // q_empty: the last MMA of the item, and the epilogue's TMA store of dQ (staged in the
        // same buffer) having read shared memory
        for (int i = 0; i < 2; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, NSW + 1); }
        // s_full[2b + w]: S, dP of buffer b ready for softmax warpgroup w (PP) — one barrier per
        // (buffer, consumer) so every barrier has one in-order producer and one in-order consumer
        for (int i = 0; i < 2 * NBUF; ++i) mbar_init(s_full + i, 1);
        for (int i = 0; i < NBUF; ++i) { mbar_init(ds_full + i, PP ? 128 : 32 * MW); mbar_init(freeb + i, 1); }
        mbar_init(o_full, 1);
        mbar_init(o_empty, 32 * MW);
        mbar_init(dq_full, 1);
        for (int i = 0; i < NST; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, 1); }
        for (int i = 0; i < 2; ++i) mbar_init(staged + i, 32 * MW);
        mbar_init(acc_empty, 32 * MW);
        mbar_init(li, 1);
        sched_init(sc, 2 + NSW + MW);
        fence_barrier_init();
    }
    if (warp == W_MMA) tmem_alloc<Cfg<B>::DQ_COLS>(tmem_slot);
    sched_load_tables(sc, p, false);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const unsigned long long t_start = p.trace ? gtimer() : 0ull;
    const int nitems = (int)(p.bh * p.ntiles);

    if (warp == W_PROD) {
        if (lane == 0) {
            prefetch_tmap(&tmQ); prefetch_tmap(&tmdO); prefetch_tmap(&tmO);
            prefetch_tmap(&tmK); prefetch_tmap(&tmV); prefetch_tmap(&tmdQ);
        }
        // next item fetched at the start of the current one; its Q/dO and O tiles issued as soon as
        // their buffers free up (tested between the current item's K/V stages)
        int st = 0, nq = 0;
        uint32_t ph = 0;
        int pre = sched_prefetch(p);
        int item = sched_produce(sc, 0, p, nitems, false, pre);
        pre = sched_prefetch(p);
        int tstate = 0;  // per-item tiles of the item being prepared: 1 = Q/dO issued, 2 = O too
        auto item_tile = [&](int ks, bool block) -> bool {
            const int *h = sc.hdr + (ks & 3) * 8;
            if (h[3] == 0) return true;
            const int bh = h[1], t = h[2], qb = nq & 1;
            if (tstate == 0) {
                if (nq >= 2) {
                    const uint32_t par = ((nq >> 1) - 1) & 1;
                    if (block) mbar_wait(q_empty + qb, par);
                    else if (!warp_test(q_empty + qb, par)) return false;
                }
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full + qb, 32768);
                    const uint64_t once = l2_evict_first();  // the item's own rows
                    tma_ld(sQ + qb * 16384, &tmQ, q_full + qb, 0, t * 128, bh, once);
                    tma_ld(sdO + qb * 16384, &tmdO, q_full + qb, 0, t * 128, bh, once);
                }
                __syncwarp();
                tstate = 1;
            }
            if (nq >= 1) {
                if (block) mbar_wait(o_empty, (nq - 1) & 1);
                else if (!warp_test(o_empty, (nq - 1) & 1)) return false;
            }
            if (elect_one()) {
                mbar_arrive_expect_tx(o_full, 16384);
                tma_ld(sO, &tmO, o_full, 0, t * 128, bh, l2_evict_first());
            }
            __syncwarp();
            tstate = 0;
            ++nq;
            return true;
        };
        bool issued = false;
        for (int ks = 0; item >= 0; ++ks) {
            if (!issued) item_tile(ks, true);
            // the next item: list loads issued now, stored after two of this item's stages
            const SchedFetch nf = sched_fetch_begin(sc, ks + 1, p, nitems, pre);
            pre = sched_prefetch(p);
            const int nitem = nf.item;
            bool ended = false, nissued = nitem < 0;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], cnt = h[3];
            const int *col = sc.col + (ks & 3) * SCHED_CAP;
            for (int j = 0; j < cnt; ++j) {  // whole warp runs the loop; one elected lane issues the TMA
                if (!ended && j == 2) { sched_fetch_end(sc, ks + 1, p, nf, false); ended = true; }
                if (ended && !nissued) nissued = item_tile(ks + 1, false);
                mbar_wait(kv_empty + st, ph ^ 1);
                if (elect_one()) {
                    if (SPION_DBG_NOLOAD) {
                        mbar_arrive(kv_full + st);
                    } else {
                        mbar_arrive_expect_tx(kv_full + st, STG);
                        const uint64_t keep = l2_evict_last();  // K_J, V_J: read by every tile listing J
                        tma_ld(sKV + st * STG, &tmK, kv_full + st, 0, col[j] * B, bh, keep);
                        tma_ld(sKV + st * STG + KV_BYTES, &tmV, kv_full + st, 0, col[j] * B, bh, keep);
                    }
                }
                __syncwarp();
                if (++st == NST) { st = 0; ph ^= 1; }
            }
            if (!ended) sched_fetch_end(sc, ks + 1, p, nf, false);
            issued = nissued;
            item = nitem;
        }
    } else if (warp == W_MMA || warp >= W_MMA3) {
        if (!SPION_LANE0 || lane == 0) {  // SPION_LANE0: the issuing role runs on one thread
        // S / dP issuers (converged warps, one elected lane issues), up to NBUF blocks ahead;
        // with NSW = NBUF, warp sw issues the blocks whose score buffer is sw
        const int sw = warp == W_MMA ? 0 : warp - W_MMA3 + 1;
        int sst = 0, nq = 0;
        uint32_t sph = 0, g = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int cnt = h[3];
            if (cnt > 0) {
                const int qb = nq & 1;
                mbar_wait(q_full + qb, (nq >> 1) & 1);
                if (SPION_ITEM_FENCE && NSW == 1 && nq > 0) mbar_wait(li, (nq - 1) & 1);
                tc_fence_after();
                ++nq;
                const uint64_t dQ0 = sdesc_sw128(smem_u32(sQ + qb * 16384));
                const uint64_t ddO0 = sdesc_sw128(smem_u32(sdO + qb * 16384));
                if (TSQ && ISSUER()) {  // in issue order with the MMAs below (and the last item's)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        tmem_cp_128x256b(tmem + COL_QA + 8 * k, dQ0 + 2 * k);
                        tmem_cp_128x256b(tmem + COL_DOA + 8 * k, ddO0 + 2 * k);
                    }
                }
                ROLE_SYNC();
                for (int sj = 0; sj < cnt; ++sj) {
                    const uint32_t gs = g + sj, b = gs % NBUF, u = gs / NBUF;
                    if (NSW > 1 && (int)b != sw) {
                        if (++sst == NST) { sst = 0; sph ^= 1; }
                        continue;
                    }
                    // buffer first: its release implies every earlier block's stage arrived, so
                    // the stage wait below can never see a phase from two uses back
                    if (u > 0) mbar_wait(freeb + b, (u - 1) & 1);
                    mbar_wait(kv_full + sst, sph);
                    tc_fence_after();
                    const uint32_t cs = b * BUFW;
                    const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + sst * STG));
                    const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + sst * STG + KV_BYTES));
                    if (ISSUER()) {
                        if (TSQ) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) MMA_TS(tmem + cs, tmem + COL_QA + 8 * k, dK0 + 2 * k, IDESC_S, k > 0);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                MMA_TS(tmem + cs + B, tmem + COL_DOA + 8 * k, dV0 + 2 * k, IDESC_S, k > 0);
                        } else {
#pragma unroll
                            for (int k = 0; k < 4; ++k) MMA_SS(tmem + cs, dQ0 + 2 * k, dK0 + 2 * k, IDESC_S, k > 0);
#pragma unroll
                            for (int k = 0; k < 4; ++k) MMA_SS(tmem + cs + B, ddO0 + 2 * k, dV0 + 2 * k, IDESC_S, k > 0);
                        }
                        mma_commit(s_full + 2 * b + (PP ? (sj & 1) : 0));
                    }
                    ROLE_SYNC();
                    if (++sst == NST) { sst = 0; sph ^= 1; }
                }
                if (ISSUER()) mma_commit(q_empty + qb);  // Q, dO no longer read by this warp's MMAs
                ROLE_SYNC();
                g += cnt;
            }
            sched_release(sc, ks, !SPION_LANE0);
        }
        }
    } else if (warp == W_MMA2) {
        if (!SPION_LANE0 || lane == 0) {  // SPION_LANE0: the issuing role runs on one thread
        // dQ issuer: dQ += dS_J K_J (dS from TMEM) as each dS arrives; a second issuing warp so
        // the tensor pipe is fed while the other waits (a commit stalls its issuing thread)
        int pst = 0, na = 0;
        uint32_t g = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int cnt = h[3];
            if (cnt > 0) {
                if (na > 0) mbar_wait(acc_empty, (na - 1) & 1);  // the last item's dQ was read
                ++na;
                for (int pj = 0; pj < cnt; ++pj) {
                    const uint32_t gp = g + pj, b = gp % NBUF, u = gp / NBUF;
                    mbar_wait(ds_full + b, u & 1);
                    tc_fence_after();
                    const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + pst * STG));
                    if (ISSUER()) {
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            MMA_TS(tmem + COL_DQ, tmem + b * BUFW + 32 * (k / 2) + 8 * (k % 2), dK0 + 128 * k, IDESC_DQ,
                                        (pj > 0) || (k > 0));
                        if (SPION_ITEM_FENCE && NSW == 1 && pj == cnt - 1) mbar_arrive(li);
                        mma_commit(freeb + b);
                        mma_commit(kv_empty + pst);
                        if (pj == cnt - 1) mma_commit(dq_full);
                    }
                    ROLE_SYNC();
                    if (++pst == NST) pst = 0;
                }
                g += cnt;
            }
            sched_release(sc, ks, !SPION_LANE0);
        }
        }
    } else if (warp == W_STORE) {
        // storer: once the softmax warps have staged an item's output tile(s) in shared
        // memory, one TMA store per tile; the buffer is released when the store has read it
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
                    tma_st(&tmdQ, sQ + sb * 16384, 0, t * 128, bh, l2_evict_first());
                    bulk_commit();
                    bulk_wait_read0();
                    mbar_arrive(q_empty + sb);
                }
                __syncwarp();
            }
            sched_release(sc, ks, true);
        }
        if (lane == 0) bulk_wait0();
    } else {
        const int r = (warp & 3) * 32 + lane;  // query row of the tile = TMEM lane
        const int wg = warp >> 2;              // warpgroup: alternate blocks (MW = 8); epilogue halves
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t dq_ph = 0, g = 0, sph = 0;  // sph: phase bit per score buffer (this warpgroup's uses)
        int nq = 0;
        const float sl2 = p.scale_log2;
        // pending epilogue (SPION_DEFER_DQ): the Q buffer of an item whose blocks are done; run after this
        // warpgroup's first block of the next item, so the softmax warps do not idle while the item's last
        // dQ MMAs drain (the next item's first dQ MMA waits for it through acc_empty)
        int dfr_qb = -1;
        auto epilogue = [&]() {
            if (dfr_qb < 0) return;
            mbar_wait(dq_full, dq_ph);
            dq_ph ^= 1;
            tc_fence_after();
            // dQ -> bf16 staged in the item's Q buffer (every MMA of the item is done), one TMA store
            uint8_t *sdQ = sQ + dfr_qb * 16384;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                if (MW == 8 && hh != wg) continue;  // two warpgroups: one 32-column half each
                float v[32];
                tmem_ld32(tl + COL_DQ + hh * 32, v);
                tmem_ld_wait();
                stage_row_bf16(sdQ, r, v, p.scale, hh);
            }
            tc_fence_before();
            mbar_arrive(acc_empty);  // the next item's first dQ MMA may overwrite the accumulator
            fence_proxy_async_smem();  // generic-proxy writes -> the TMA store (async proxy)
            mbar_arrive(staged + dfr_qb);
            tc_fence_before();
            dfr_qb = -1;
        };
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
                if (valid && wg == 0) zero_row_bf16(dqrow);
                sched_release(sc, ks, true);
                continue;
            }
            const int qb = nq & 1;
            const float nl2 = valid ? -__ldcg(p.lse + (int64_t)bh * p.L + row) * LOG2E : 0.f;
            // D_i = dO_i . O_i from the staged (swizzled) tiles
            mbar_wait(q_full + qb, (nq >> 1) & 1);
            mbar_wait(o_full, nq & 1);
            ++nq;
            float Dr = 0.f;
            {
                const uint8_t *rdO = sdO + qb * 16384;
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    const uint4 a = *reinterpret_cast<const uint4 *>(sO + sw128_offset(r, c));
                    const uint4 gg = *reinterpret_cast<const uint4 *>(rdO + sw128_offset(r, c));
                    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, gv[4] = {gg.x, gg.y, gg.z, gg.w};
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&av[i]));
                        const float2 fg = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162 *>(&gv[i]));
                        Dr = fmaf(fa.x, fg.x, fmaf(fa.y, fg.y, Dr));
                    }
                }
            }
            // the release must follow the LAST shared-memory load of O / dO: an mbarrier arrive does not
            // wait for outstanding LDS (ptxas issued it right behind them), so the producer could see it,
            // TMA the next item's O over the tile and corrupt rows still being read.  The proxy fence
            // (generic reads before the async-proxy TMA writes that follow the release) waits for them.
            fence_proxy_async_smem();
            mbar_arrive(o_empty);
            if (valid && wg == 0) {
                p.D[(int64_t)bh * p.L + row] = Dr;
                p.nlse2[(int64_t)bh * p.L + row] = nl2;
            }
            // two warpgroups (MW = 8) take alternate blocks, so one's TMEM loads and exponentials
            // overlap the other's; a thread handles every column of its row of the block
            for (int jj = (PP ? wg : 0); jj < cnt; jj += (PP ? 2 : 1)) {
                const bool active = (msks[jj] >> slot) & 1;
                const uint32_t gs = g + jj, sb = gs % NBUF;
                // also implies the dQ MMA that read sb before
                mbar_wait(s_full + 2 * sb + (PP ? wg : 0), PP ? (sph >> sb) & 1 : (gs / NBUF) & 1);
                sph ^= 1u << sb;
                tc_fence_after();
                const uint32_t cs = sb * BUFW;
#pragma unroll
                for (int hh = 0; hh < CPT / 32; ++hh) {
                    const uint32_t c32 = (PP ? 0 : wg * CPT) + hh * 32;  // 32-column chunk
                    uint32_t pk[16];
                    if (active && !SPION_DBG_NOSOFTMAX) {
                        float sv[32], dp[32];
                        tmem_ld32(tl + cs + c32, sv);
                        tmem_ld32(tl + cs + B + c32, dp);
                        tmem_ld_wait();
                        const uint64_t sl22 = f2pack(sl2, sl2), nl22 = f2pack(nl2, nl2), D2 = f2pack(Dr, Dr);
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {  // packed fp32x2 (FFMA2 / FADD2 / FMUL2)
                            float a0, a1, d0, d1;
                            f2unpack(ffma2(f2pack(sv[i], sv[i + 1]), sl22, nl22), a0, a1);
                            const float p0 = ex2m(a0, i), p1 = ex2m(a1, i + 1);
                            f2unpack(fmul2(f2pack(p0, p1), fsub2(f2pack(dp[i], dp[i + 1]), D2)), d0, d1);
                            pk[i / 2] = pack_bf16(d0, d1);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) pk[i] = 0u;
                    }
                    tmem_st16(tl + cs + c32, pk);  // packed dS over this warp's own consumed S columns
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(ds_full + sb);
                epilogue();  // the previous item's (deferred), after this item's first block
            }
            epilogue();  // (no block of this warpgroup in this item)
            dfr_qb = qb;
            if (!SPION_DEFER_DQ) epilogue();
            g += cnt;
            sched_release(sc, ks, true);
        }
        epilogue();  // the last item's
    }
    __syncthreads();
    sched_finish(p, t_start);
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc<Cfg<B>::DQ_COLS>(tmem);
    }
}

// ============================================================================ backward: dK, dV
// Per (bh, column tile): K/V tiles double buffered across items; for each query
// block I: S^T, dP^T into one of NBUF TMEM buffer pairs (the MMA warp runs up to NBUF
// blocks ahead of the softmax warps); P^T, dS^T packed over them feed dV += P^T dO_I,
// dK += dS^T Q_I as A operands from tensor memory.
template <int B>
__global__ void __launch_bounds__(Cfg<B>::DKV_THREADS, Cfg<B>::DKV_CTAS)
attn_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmdO,
                        const __grid_constant__ CUtensorMap tmdK, const __grid_constant__ CUtensorMap tmdV, TcParams p) {
    constexpr int NST = Cfg<B>::DKV_NST, NBUF = Cfg<B>::DKV_NBUF, MW = Cfg<B>::DKV_MW, NSW = Cfg<B>::DKV_NSW;
    constexpr int KVB = Cfg<B>::DKV_KVB, ACCB = Cfg<B>::DKV_ACCB;
    constexpr bool PP = MW == 8 && Cfg<B>::PING;   // warpgroups take alternate blocks
    constexpr int CPT = PP || MW == 4 ? B : B / 2;  // columns of a block per softmax thread
    constexpr int W_PROD = MW, W_MMA = MW + 1, W_STORE = MW + 2, W_MMA2 = MW + 3, W_MMA3 = MW + 4;
    constexpr bool EPI = Cfg<B>::DKV_EPI;
    constexpr int W_EPI = MW + 3 + NSW;  // EPI: warps W_EPI .. W_EPI + 3 (TMEM lane quarters 0..3)
    constexpr int NEPI = EPI ? 128 : 32 * MW;  // threads that read the accumulators and stage dK/dV
    constexpr uint32_t BUFW = 2 * B;  // S^T at b*BUFW, dP^T at b*BUFW + B
    constexpr uint32_t COL_DK = NBUF * BUFW, COL_DV = NBUF * BUFW + 64;  // + 128 * accumulator pair
    constexpr bool TSKV = Cfg<B>::DKV_TS;
    constexpr uint32_t COL_KA = NBUF * BUFW + 128 * ACCB, COL_VA = COL_KA + 32;  // TSKV: K, V as A operands
    constexpr uint32_t TILE = B * 128;
    constexpr uint32_t STAGE = 2 * TILE + 1024;  // Q_I, dO_I, lse_I, D_I
    constexpr uint32_t IDESC_ST = idesc_bf16(128, B, false, false);   // S^T = K Q^T, dP^T = V dO^T
    constexpr uint32_t IDESC_DKV = idesc_bf16(128, 64, false, true);  // dV += P^T dO, dK += dS^T Q

    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sKV = smem;  // buffer kb: K at kb*32768, V at kb*32768 + 16384
    uint8_t *sStage = smem + KVB * 32768;
    uint8_t *sSched = sStage + NST * STAGE;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sSched + SCHED_BYTES);
    uint64_t *kv_full = bars + 0, *kv_empty = bars + 3, *acc_full = bars + 6, *s_full = bars + 8,
             *p_full = s_full + 2 * NBUF, *freeb = p_full + NBUF, *q_full = freeb + NBUF, *q_empty = q_full + NST;
    Sched sc = make_sched(sSched, q_empty + NST);
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(q_empty + NST + 8);
    uint64_t *staged = q_empty + NST + 9;  // [KVB]: dK/dV of the item using K/V buffer kb staged there
    uint64_t *acc_empty = staged + 3;      // [ACCB]: the epilogue has read accumulator pair a
    uint64_t *li = acc_empty + 2;          // the dV/dK issuer has issued an item's last MMAs (as forward)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        // kv_empty: the last S^T/dP^T MMA of the item, and the epilogue's TMA store of dK/dV
        // (staged in the same buffer) having read shared memory
        for (int i = 0; i < KVB; ++i) { mbar_init(kv_full + i, 1); mbar_init(kv_empty + i, NSW + 1); }
        // s_full[2b + w]: S^T, dP^T of buffer b ready for softmax warpgroup w (PP) — one barrier
        // per (buffer, consumer), so each has one in-order producer and one in-order consumer
        for (int i = 0; i < 2 * NBUF; ++i) mbar_init(s_full + i, 1);
        for (int i = 0; i < NBUF; ++i) { mbar_init(p_full + i, PP ? 128 : 32 * MW); mbar_init(freeb + i, 1); }
        for (int i = 0; i < ACCB; ++i) { mbar_init(acc_full + i, 1); mbar_init(acc_empty + i, NEPI); }
        for (int i = 0; i < NST; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 1); }
        for (int i = 0; i < KVB; ++i) mbar_init(staged + i, NEPI);
        mbar_init(li, 1);
        sched_init(sc, 2 + NSW + MW + (EPI ? 4 : 0));
        fence_barrier_init();
    }
    if (warp == W_MMA) tmem_alloc<Cfg<B>::DKV_COLS>(tmem_slot);
    sched_load_tables(sc, p, false);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const unsigned long long t_start = p.trace ? gtimer() : 0ull;
    const int nitems = (int)(p.bh * p.ntiles);
    // EPI: register budgets per warpgroup (one setmaxnreg at the top of each warpgroup's branch):
    // softmax 2 x 128 x 168 + single-lane roles 128 x 64 + epilogue 128 x 96 <= 65536
    if (warp >= W_PROD && (!EPI || warp < W_EPI)) {
    if (EPI) regs_dec<64>();
    if (warp == W_PROD) {
        Tracer tr(p, 0);
        if (lane == 0) {
            prefetch_tmap(&tmK); prefetch_tmap(&tmV); prefetch_tmap(&tmQ); prefetch_tmap(&tmdO);
            prefetch_tmap(&tmdK); prefetch_tmap(&tmdV);
        }
        // next item fetched at the start of the current one; its K/V tiles issued as soon as their
        // buffer frees up (tested between the current item's Q/dO stages)
        int st = 0, nk = 0;
        uint32_t ph = 0;
        int pre = sched_prefetch(p);
        int item = sched_produce(sc, 0, p, nitems, false, pre, &tr);
        pre = sched_prefetch(p);
        auto item_tile = [&](int ks, bool block) -> bool {  // K/V of ring item ks (false: buffer busy)
            const int *h = sc.hdr + (ks & 3) * 8;
            if (h[3] == 0) return true;
            const int bh = h[1], t = h[2], kb = nk % KVB;
            if (nk >= KVB) {
                const uint32_t par = ((nk / KVB) - 1) & 1;
                if (block) mbar_wait(kv_empty + kb, par);
                else if (!warp_test(kv_empty + kb, par)) return false;
            }
            if (lane == 0) tr.ev(2);
            if (elect_one()) {
                // the tile's S block columns (plan bperm: heavy columns grouped), one B-row box
                // each at slot offset s*B rows (same SW128 layout as one 128-row box); empty
                // slots are not loaded (their rows are masked in every entry, never stored)
                const int *pm = sc.tab + TAB_PERM + t * p.S;
                int nval = 0;
                for (int sl = 0; sl < p.S; ++sl) nval += pm[sl] < p.n;
                mbar_arrive_expect_tx(kv_full + kb, (uint32_t)nval * 2 * B * 128);
                for (int sl = 0; sl < p.S; ++sl) {
                    const int c = pm[sl];
                    if (c >= p.n) continue;
                    const uint64_t once = l2_evict_first();  // the item's own key rows
                    tma_ld(sKV + kb * 32768 + sl * B * 128, &tmK, kv_full + kb, 0, c * B, bh, once);
                    tma_ld(sKV + kb * 32768 + 16384 + sl * B * 128, &tmV, kv_full + kb, 0, c * B, bh, once);
                }
            }
            __syncwarp();
            ++nk;
            return true;
        };
        bool issued = false;
        for (int ks = 0; item >= 0; ++ks) {
            if (lane == 0) tr.ev(1);
            if (!issued) item_tile(ks, true);
            // the next item: list loads issued now, stored after two of this item's stages
            const SchedFetch nf = sched_fetch_begin(sc, ks + 1, p, nitems, pre, &tr);
            pre = sched_prefetch(p);
            const int nitem = nf.item;
            bool ended = false, nissued = nitem < 0;
            const int *h = sc.hdr + (ks & 3) * 8;
            const int bh = h[1], cnt = h[3];
            const int *rows = sc.col + (ks & 3) * SCHED_CAP;
            for (int j = 0; j < cnt; ++j) {  // whole warp runs the loop; one elected lane issues the copies
                if (!ended && j == 2) { sched_fetch_end(sc, ks + 1, p, nf, false, &tr); ended = true; }
                if (ended && !nissued) nissued = item_tile(ks + 1, false);
                const int I = rows[j];
                mbar_wait(q_empty + st, ph ^ 1);
                if (lane == 0) tr.ev(3);
                uint8_t *stg = sStage + st * STAGE;
                if (elect_one()) {
                    if (SPION_DBG_NOLOAD) {
                        mbar_arrive(q_full + st);
                    } else {
                        mbar_arrive_expect_tx(q_full + st, 2 * TILE + 2 * B * 4);
                        const uint64_t keep = l2_evict_last();  // Q_I, dO_I: read by every tile listing I
                        tma_ld(stg, &tmQ, q_full + st, 0, I * B, bh, keep);
                        tma_ld(stg + TILE, &tmdO, q_full + st, 0, I * B, bh, keep);
                        bulk_load(stg + 2 * TILE, p.lse + (int64_t)bh * p.L + (int64_t)I * B, B * 4, q_full + st);
                        bulk_load(stg + 2 * TILE + 512, p.D + (int64_t)bh * p.L + (int64_t)I * B, B * 4, q_full + st);
                    }
                }
                __syncwarp();
                if (++st == NST) { st = 0; ph ^= 1; }
            }
            if (!ended) sched_fetch_end(sc, ks + 1, p, nf, false, &tr);
            issued = nissued;
            item = nitem;
        }
    } else if (warp == W_MMA || (warp >= W_MMA3 && warp < W_EPI)) {
        if (!SPION_LANE0 || lane == 0) {  // SPION_LANE0: the issuing role runs on one thread
        // S^T / dP^T issuers (converged warps, one elected lane issues), up to NBUF blocks ahead;
        // with NSW = NBUF, warp sw issues the blocks whose score buffer is sw
        const int sw = warp == W_MMA ? 0 : warp - W_MMA3 + 1;
        Tracer tr(p, sw == 0 ? 1 : 4 + sw);
        int sst = 0, nk = 0;
        uint32_t sph = 0, g = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            if (lane == 0) tr.ev(10);
            const int cnt = h[3];
            if (cnt > 0) {
                const int kb = nk % KVB;
                mbar_wait(kv_full + kb, (nk / KVB) & 1);
                if (lane == 0) tr.ev(11);
                if (SPION_ITEM_FENCE && NSW == 1 && nk > 0) mbar_wait(li, (nk - 1) & 1);
                tc_fence_after();
                ++nk;
                const uint64_t dK0 = sdesc_sw128(smem_u32(sKV + kb * 32768));
                const uint64_t dV0 = sdesc_sw128(smem_u32(sKV + kb * 32768 + 16384));
                if (TSKV && ISSUER()) {  // in issue order with the MMAs below (and the last item's)
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        tmem_cp_128x256b(tmem + COL_KA + 8 * k, dK0 + 2 * k);
                        tmem_cp_128x256b(tmem + COL_VA + 8 * k, dV0 + 2 * k);
                    }
                }
                ROLE_SYNC();
                for (int sj = 0; sj < cnt; ++sj) {
                    const uint32_t gs = g + sj, b = gs % NBUF, u = gs / NBUF;
                    if (NSW > 1 && (int)b != sw) {
                        if (++sst == NST) { sst = 0; sph ^= 1; }
                        continue;
                    }
                    if (lane == 0) tr.ev(40);
                    // buffer first: its release implies every earlier block's stage arrived, so
                    // the stage wait below can never see a phase from two uses back
                    if (u > 0) mbar_wait(freeb + b, (u - 1) & 1);
                    if (lane == 0) tr.ev(42);
                    mbar_wait(q_full + sst, sph);
                    if (lane == 0) tr.ev(12);
                    tc_fence_after();
                    uint8_t *stg = sStage + sst * STAGE;
                    const uint32_t cs = b * BUFW;
                    const uint64_t dQ0 = sdesc_sw128(smem_u32(stg));
                    const uint64_t ddO0 = sdesc_sw128(smem_u32(stg + TILE));
                    if (ISSUER()) {
                        if (TSKV) {
#pragma unroll
                            for (int k = 0; k < 4; ++k) MMA_TS(tmem + cs, tmem + COL_KA + 8 * k, dQ0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                            for (int k = 0; k < 4; ++k)
                                MMA_TS(tmem + cs + B, tmem + COL_VA + 8 * k, ddO0 + 2 * k, IDESC_ST, k > 0);
                        } else {
#pragma unroll
                            for (int k = 0; k < 4; ++k) MMA_SS(tmem + cs, dK0 + 2 * k, dQ0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                            for (int k = 0; k < 4; ++k) MMA_SS(tmem + cs + B, dV0 + 2 * k, ddO0 + 2 * k, IDESC_ST, k > 0);
                        }
                        tr.ev(43);
                        mma_commit(s_full + 2 * b + (PP ? (sj & 1) : 0));
                        tr.ev(41);
                    }
                    ROLE_SYNC();
                    if (lane == 0) tr.ev(14);
                    if (++sst == NST) { sst = 0; sph ^= 1; }
                }
                // K/V no longer read by this warp's MMAs of the item (the same lane issued them)
                if (ISSUER()) mma_commit(kv_empty + kb);
                ROLE_SYNC();
                g += cnt;
            }
            sched_release(sc, ks, !SPION_LANE0);
        }
        }
    } else if (warp == W_MMA2) {
        if (!SPION_LANE0 || lane == 0) {  // SPION_LANE0: the issuing role runs on one thread
        // dV / dK issuer: dV += P^T dO_I, dK += dS^T Q_I (A from TMEM) as each block's P^T / dS^T
        // arrives; a second issuing warp so the tensor pipe is fed while the other waits
        Tracer tr(p, 4);
        int pst = 0, na = 0;
        uint32_t g = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int cnt = h[3];
            if (cnt > 0) {
                const int ab = na % ACCB;  // accumulator pair of this item
                if (na >= ACCB) mbar_wait(acc_empty + ab, ((na / ACCB) - 1) & 1);  // its last user was read
                ++na;
                const uint32_t cdk = COL_DK + 128 * ab, cdv = COL_DV + 128 * ab;
                for (int pj = 0; pj < cnt; ++pj) {
                    const uint32_t gp = g + pj, b = gp % NBUF, u = gp / NBUF;
                    if (lane == 0) tr.ev(30);
                    mbar_wait(p_full + b, u & 1);
                    if (lane == 0) tr.ev(13);
                    tc_fence_after();
                    uint8_t *stg = sStage + pst * STAGE;
                    const uint64_t dQ0 = sdesc_sw128(smem_u32(stg));
                    const uint64_t ddO0 = sdesc_sw128(smem_u32(stg + TILE));
                    const uint32_t cs = b * BUFW;
                    if (ISSUER()) {
                        tr.ev(31);
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            MMA_TS(tmem + cdv, tmem + cs + 32 * (k / 2) + 8 * (k % 2), ddO0 + 128 * k, IDESC_DKV,
                                        (pj > 0) || (k > 0));
#pragma unroll
                        for (int k = 0; k < B / 16; ++k)
                            MMA_TS(tmem + cdk, tmem + cs + B + 32 * (k / 2) + 8 * (k % 2), dQ0 + 128 * k, IDESC_DKV,
                                        (pj > 0) || (k > 0));
                        tr.ev(32);
                        if (SPION_ITEM_FENCE && NSW == 1 && pj == cnt - 1) mbar_arrive(li);
                        mma_commit(freeb + b);
                        mma_commit(q_empty + pst);
                        if (pj == cnt - 1) mma_commit(acc_full + ab);
                        tr.ev(33);
                    }
                    ROLE_SYNC();
                    if (lane == 0) tr.ev(15);
                    if (++pst == NST) pst = 0;
                }
                g += cnt;
            }
            sched_release(sc, ks, !SPION_LANE0);
        }
        }
    } else if (warp == W_STORE) {
        // storer: once the softmax warps have staged an item's output tile(s) in shared
        // memory, one TMA store per tile; the buffer is released when the store has read it
        int ns = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            const int bh = h[1], t = h[2], cnt = h[3];
            if (cnt > 0) {
                const int sb = ns % KVB;
                mbar_wait(staged + sb, (ns / KVB) & 1);
                ++ns;
                if (lane == 0) {
                    const int *pm = sc.tab + TAB_PERM + t * p.S;
                    for (int sl = 0; sl < p.S; ++sl) {
                        const int c = pm[sl];
                        if (c >= p.n) continue;
                        tma_st(&tmdK, sKV + sb * 32768 + sl * B * 128, 0, c * B, bh, l2_evict_first());
                        tma_st(&tmdV, sKV + sb * 32768 + 16384 + sl * B * 128, 0, c * B, bh, l2_evict_first());
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
    } else if (EPI && warp >= W_EPI) {
        regs_dec<96>();
        // ------------------------------------------------------------ epilogue warpgroup: per item,
        // once its last dV/dK MMAs are done, dK * scale and dV -> bf16 staged in the item's K/V buffer
        const int r = (warp & 3) * 32 + lane;  // key row of the tile = TMEM lane
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        int nk = 0, na = 0;
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            if (h[3] > 0) {
                const int kb = nk % KVB, ab = na % ACCB;
                mbar_wait(acc_full + ab, (uint32_t)(na / ACCB) & 1);
                tc_fence_after();
                uint8_t *sdK = sKV + kb * 32768, *sdV = sdK + 16384;
                const uint32_t cdk = COL_DK + 128 * ab, cdv = COL_DV + 128 * ab;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    float kv[32], vv[32];
                    tmem_ld32(tl + cdk + hh * 32, kv);
                    tmem_ld32(tl + cdv + hh * 32, vv);
                    tmem_ld_wait();
                    stage_row_bf16(sdK, r, kv, p.scale, hh);
                    stage_row_bf16(sdV, r, vv, 1.f, hh);
                }
                tc_fence_before();
                mbar_arrive(acc_empty + ab);  // a later item's first dV/dK MMAs may overwrite the pair
                fence_proxy_async_smem();     // generic-proxy writes -> the TMA store (async proxy)
                mbar_arrive(staged + kb);
                ++nk;
                ++na;
            }
            sched_release(sc, ks, true);
        }
    } else {
        if (EPI) regs_inc<168>();
        const int r = (warp & 3) * 32 + lane;  // key row of the tile = TMEM lane
        const int wg = warp >> 2;              // warpgroup: alternate blocks (MW = 8); epilogue halves
        const int slot = r / B;
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        uint32_t ph = 0, g = 0, sph = 0;  // sph: phase bit per score buffer (this warpgroup's uses)
        int st = 0, nk = 0, na = 0;
        const float sl2 = p.scale_log2;
        Tracer tr(p, 2 + (threadIdx.x == 128));
        const bool trc = threadIdx.x == 0 || threadIdx.x == 128;
        // pending epilogue: K/V buffer (staging) and accumulator pair of an item whose blocks are done
        int dfr_kb = -1, dfr_ab = 0;
        uint32_t dfr_par = 0;
        auto epilogue = [&]() {
            if (EPI || dfr_kb < 0) return;
            mbar_wait(acc_full + dfr_ab, dfr_par);
            if (trc) tr.ev(23);
            tc_fence_after();
            // dK, dV -> bf16 staged in the item's K/V buffer (free: every S^T/dP^T MMA is done),
            // then one TMA store per tile (coalesced; rows past L clipped)
            uint8_t *sdK = sKV + dfr_kb * 32768, *sdV = sdK + 16384;
            const uint32_t cdk = COL_DK + 128 * dfr_ab, cdv = COL_DV + 128 * dfr_ab;
            if (MW == 8) {  // warpgroup 0 stages dK, warpgroup 1 stages dV
                const uint32_t col = wg == 0 ? cdk : cdv;
                uint8_t *dst = wg == 0 ? sdK : sdV;
                const float f = wg == 0 ? p.scale : 1.f;
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    float w[32];
                    tmem_ld32(tl + col + hh * 32, w);
                    tmem_ld_wait();
                    stage_row_bf16(dst, r, w, f, hh);
                }
            } else {
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    float kv[32], vv[32];
                    tmem_ld32(tl + cdk + hh * 32, kv);
                    tmem_ld32(tl + cdv + hh * 32, vv);
                    tmem_ld_wait();
                    stage_row_bf16(sdK, r, kv, p.scale, hh);
                    stage_row_bf16(sdV, r, vv, 1.f, hh);
                }
            }
            tc_fence_before();
            mbar_arrive(acc_empty + dfr_ab);  // a later item's first dV/dK MMAs may overwrite the pair
            fence_proxy_async_smem();         // generic-proxy writes -> the TMA store (async proxy)
            mbar_arrive(staged + dfr_kb);
            tc_fence_before();
            if (trc) tr.ev(24);
            dfr_kb = -1;
        };
        for (int ks = 0;; ++ks) {
            const int *h = sched_wait(sc, ks);
            if (h[0] < 0) break;
            if (trc) tr.ev(20);
            const int bh = h[1], t = h[2], cnt = h[3];
            const int *msks = sc.msk + (ks & 3) * SCHED_CAP;
            // tile row r is key row r % B of block column bperm[t * S + r / B] (n: an empty slot)
            const int pcol = sc.tab[TAB_PERM + t * p.S + slot];
            const int key = pcol * B + (r % B);
            const bool valid = pcol < p.n;
            __nv_bfloat16 *dkrow =
                static_cast<__nv_bfloat16 *>(p.dK) + (int64_t)bh * p.stride_bh + (int64_t)key * p.stride_l;
            __nv_bfloat16 *dvrow =
                static_cast<__nv_bfloat16 *>(p.dV) + (int64_t)bh * p.stride_bh + (int64_t)key * p.stride_l;
            if (cnt == 0) {
                if (valid && (MW == 4 || wg == 0)) zero_row_bf16(dkrow);
                if (valid && (MW == 4 || wg == 1)) zero_row_bf16(dvrow);
                sched_release(sc, ks, true);
                continue;
            }
            // two warpgroups (MW = 8) take alternate blocks, so one's TMEM loads and exponentials
            // overlap the other's; a thread handles every column of its row of the block
            for (int jj = 0; jj < cnt; ++jj) {
                if (PP && (jj & 1) != wg) {
                    if (++st == NST) { st = 0; ph ^= 1; }
                    continue;
                }
                const bool active = (msks[jj] >> slot) & 1;
                const uint32_t gs = g + jj, sb = gs % NBUF;
                // also implies the dV/dK MMAs that read sb before
                mbar_wait(s_full + 2 * sb + (PP ? wg : 0), PP ? (sph >> sb) & 1 : (gs / NBUF) & 1);
                sph ^= 1u << sb;
                // lse_I, D_I: after the S wait, whose MMA already waited this stage's load (so
                // this parity wait can never see the stage's previous use)
                mbar_wait(q_full + st, ph);
                const float *snl2 = reinterpret_cast<const float *>(sStage + st * STAGE + 2 * TILE);
                const float *sD = snl2 + 128;
                if (trc) tr.ev(21);
                tc_fence_after();
                const uint32_t cs = sb * BUFW;
#pragma unroll
                for (int hh = 0; hh < CPT / 32; ++hh) {
                    const uint32_t c32 = (PP ? 0 : wg * CPT) + hh * 32;  // 32-column chunk
                    uint32_t pk[16], dk[16];
                    if (active && !SPION_DBG_NOSOFTMAX) {
                        float sv[32], dp[32], nl[32], dd[32];
                        tmem_ld32(tl + cs + c32, sv);
                        tmem_ld32(tl + cs + B + c32, dp);
#pragma unroll
                        for (int i = 0; i < 8; ++i) {  // broadcast LDS.128 of the query block's offsets
                            const float4 a = reinterpret_cast<const float4 *>(snl2 + c32)[i];
                            const float4 b = reinterpret_cast<const float4 *>(sD + c32)[i];
                            nl[4 * i] = a.x; nl[4 * i + 1] = a.y; nl[4 * i + 2] = a.z; nl[4 * i + 3] = a.w;
                            dd[4 * i] = b.x; dd[4 * i + 1] = b.y; dd[4 * i + 2] = b.z; dd[4 * i + 3] = b.w;
                        }
                        tmem_ld_wait();
                        const uint64_t sl22 = f2pack(sl2, sl2);
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {  // packed fp32x2 (FFMA2 / FADD2 / FMUL2)
                            float a0, a1, d0, d1;
                            f2unpack(ffma2(f2pack(sv[i], sv[i + 1]), sl22, f2pack(nl[i], nl[i + 1])), a0, a1);
                            const float p0 = ex2m(a0, i), p1 = ex2m(a1, i + 1);
                            pk[i / 2] = pack_bf16(p0, p1);
                            f2unpack(fmul2(f2pack(p0, p1), fsub2(f2pack(dp[i], dp[i + 1]), f2pack(dd[i], dd[i + 1]))), d0, d1);
                            dk[i / 2] = pack_bf16(d0, d1);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 16; ++i) { pk[i] = 0u; dk[i] = 0u; }
                    }
                    // packed bf16 P^T / dS^T over this warp's own (already read) S^T / dP^T columns
                    tmem_st16(tl + cs + c32, pk);
                    tmem_st16(tl + cs + B + c32, dk);
                }
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(p_full + sb);
                if (trc) tr.ev(22);
                if (++st == NST) { st = 0; ph ^= 1; }
                epilogue();  // the previous item's (deferred), after this item's first block
            }
            epilogue();  // (no block of this warpgroup in this item)
            // this item's epilogue: now (one accumulator pair), or deferred until after this warpgroup's
            // first block of the next item (two pairs: the tensor pipe is busy with the next item's
            // score MMAs, so waiting here for the last dV/dK MMAs would idle the softmax warps)
            dfr_kb = nk % KVB;
            dfr_ab = na % ACCB;
            dfr_par = (uint32_t)(na / ACCB) & 1;
            ++nk;
            ++na;
            if (ACCB == 1 && !SPION_DEFER_DKV) epilogue();
            g += cnt;
            sched_release(sc, ks, true);
        }
        epilogue();  // the last item's
    }
    __syncthreads();
    sched_finish(p, t_start);
    if (warp == W_MMA) {
        tc_fence_after();
        tmem_dealloc<Cfg<B>::DKV_COLS>(tmem);
    }
}

// ============================================================================ host side
PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
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
bool tc_make_map(void *map, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l, int box_rows);
static bool encode_map(CUtensorMap *m, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l,
                       int box_rows) {
    auto enc = tc_encode_fn();
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
// Tensor maps are pure functions of (address, shape, strides, box), so encoded maps are cached per
// host thread (a small round-robin table): a step that re-launches on the same buffers encodes
// nothing (the backward needs ten maps per call).
bool tc_map(CUtensorMap *m, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l,
                     int box_rows) {
    struct Entry {
        const void *base;
        int64_t bh, stride_bh, stride_l;
        int L, box_rows;
        alignas(64) CUtensorMap map;
    };
    constexpr int CAP = 48;
    static thread_local Entry cache[CAP];
    static thread_local int used = 0, next = 0;
    for (int i = 0; i < used; ++i) {
        const Entry &e = cache[i];
        if (e.base == base && e.L == L && e.bh == bh && e.stride_bh == stride_bh && e.stride_l == stride_l &&
            e.box_rows == box_rows) {
            *m = e.map;
            return true;
        }
    }
    if (!encode_map(m, base, L, bh, stride_bh, stride_l, box_rows)) return false;
    Entry &e = cache[next];
    e.base = base; e.bh = bh; e.stride_bh = stride_bh; e.stride_l = stride_l; e.L = L; e.box_rows = box_rows;
    e.map = *m;
    next = (next + 1) % CAP;
    if (used < CAP) ++used;
    return true;
}

bool tc_make_map(void *map, const void *base, int L, int64_t bh, int64_t stride_bh, int64_t stride_l, int box_rows) {
    return tc_map(static_cast<CUtensorMap *>(map), base, L, bh, stride_bh, stride_l, box_rows);
}

bool tc_encode_fn_available() { return tc_encode_fn() != nullptr; }

bool tc_supported(const AttnArgs &a, spion_dtype dt) {
    if (dt != SPION_BF16 || a.d != 64 || !(a.B == 32 || a.B == 64) || !a.plan) return false;
    if (a.stride_l % 8 || a.stride_bh % 8) return false;
    if (a.L % 4 || a.n > SCHED_CAP) return false;
    static int disabled = -1;
    if (disabled < 0) disabled = getenv("SPION_DISABLE_TC") != nullptr;
    return !disabled && tc_encode_fn() != nullptr;
}

unsigned long long *g_trace_buf = nullptr;
int tc_num_sms() {
    static int n[64] = {0};
    const int dev = current_device() & 63;
    if (!n[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    }
    return n[dev];
}

// which: 0 fwd (row tiles), 1 dq (row tiles), 2 dkdv (column tiles)
TcParams tc_base_params(const AttnArgs &a, int which, int ctas, int gmult) {
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
    p.sched = a.sched + which;
    p.off_heavy = rows ? 5 : 6;
    p.off_perm = rows ? 0 : (int)pl.bperm;
    const int grid = ctas * tc_num_sms();
    int G = (gmult * grid + pl.ntiles - 1) / pl.ntiles;  // (batch, head) per chunk: ~G_MULT items per CTA
    if (G < 1) G = 1;
    if (G > a.bh) G = (int)a.bh;
    p.G = G;
    static unsigned long long *trace_buf = nullptr;
    static int want = -1;
    if (want < 0) want = getenv("SPION_TRACE") != nullptr;
    if (want) {
        if (!trace_buf) cudaMalloc(&trace_buf, (16 + 8 * 2048 + 4096) * 8);
        cudaMemset(trace_buf, 0, (16 + 8 * 2048 + 4096) * 8);
        p.trace = trace_buf;
        g_trace_buf = trace_buf;
    }
    return p;
}

template <int B> static size_t fwd_smem() { return 1024 + 32768 + Cfg<B>::FWD_NST * 2 * B * 128 + SCHED_AREA; }
template <int B> static size_t dq_smem() { return 1024 + 81920 + Cfg<B>::DQ_NST * 2 * B * 128 + SCHED_AREA; }
template <int B> static size_t dkv_smem() {
    return 1024 + Cfg<B>::DKV_KVB * 32768 + Cfg<B>::DKV_NST * (2 * B * 128 + 1024) + SCHED_AREA;
}

static int grid_for(const TcParams &p, int ctas) {
    const int64_t items = p.bh * p.ntiles;
    return (int)((items < (int64_t)ctas * tc_num_sms()) ? items : (int64_t)ctas * tc_num_sms());
}

template <int B>
static spion_status fwd_tc_t(const AttnArgs &a, cudaStream_t s) {
    static PerDevice attr;
    SPION_CUDA_TRY(smem_attr_once(attr, attn_fwd_tc_kernel<B>, (int)fwd_smem<B>()));
    CUtensorMap mq, mk, mv, mo;
    if (!tc_map(&mq, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !tc_map(&mk, a.K, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mv, a.V, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mo, a.Oout, a.L, a.bh, a.stride_bh, a.stride_l, 128))
        return SPION_ERR_CUDA;
    TcParams p = tc_base_params(a, 0, Cfg<B>::FWD_CTAS);
    p.O = a.Oout;
    p.lse_out = a.lse_out;
    attn_fwd_tc_kernel<B><<<grid_for(p, Cfg<B>::FWD_CTAS), TC_THREADS, fwd_smem<B>(), s>>>(mq, mk, mv, mo, p);
    SPION_LAUNCH_CHECK();
    note_tc_launch();
    return SPION_OK;
}

template <int B>
static spion_status bwd_tc_t(const AttnArgs &a, cudaStream_t s) {
    static PerDevice attr_dq, attr_dkv;
    SPION_CUDA_TRY(smem_attr_once(attr_dq, attn_bwd_dq_tc_kernel<B>, (int)dq_smem<B>()));
    SPION_CUDA_TRY(smem_attr_once(attr_dkv, attn_bwd_dkdv_tc_kernel<B>, (int)dkv_smem<B>()));
    CUtensorMap mq128, mdo128, mo128, mkB, mvB, mqB, mdoB, mdq128, mdkB, mdvB;
    if (!tc_map(&mq128, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !tc_map(&mdo128, a.dO, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !tc_map(&mo128, a.O, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !tc_map(&mkB, a.K, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mvB, a.V, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mqB, a.Q, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mdoB, a.dO, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mdq128, a.dQ, a.L, a.bh, a.stride_bh, a.stride_l, 128) ||
        !tc_map(&mdkB, a.dK, a.L, a.bh, a.stride_bh, a.stride_l, B) ||
        !tc_map(&mdvB, a.dV, a.L, a.bh, a.stride_bh, a.stride_l, B))
        return SPION_ERR_CUDA;
    // 1) dQ (row tiles) and D = rowsum(dO * O)
    TcParams p = tc_base_params(a, 1, Cfg<B>::DQ_CTAS);
    p.O = const_cast<void *>(a.O);
    p.lse = a.lse;
    p.D = const_cast<float *>(a.D);
    p.nlse2 = a.nlse2;
    p.dQ = a.dQ;
    attn_bwd_dq_tc_kernel<B><<<grid_for(p, Cfg<B>::DQ_CTAS), bwd_threads(Cfg<B>::DQ_MW, Cfg<B>::DQ_NSW), dq_smem<B>(), s>>>(mq128, mdo128, mo128, mkB, mvB, mdq128, p);
    SPION_LAUNCH_CHECK();
    // 2) dK, dV (column tiles)
    TcParams q = tc_base_params(a, 2, Cfg<B>::DKV_CTAS);
    q.lse = a.nlse2;  // staged per query block: -lse * log2(e)
    q.D = const_cast<float *>(a.D);
    q.dK = a.dK;
    q.dV = a.dV;
    attn_bwd_dkdv_tc_kernel<B><<<grid_for(q, Cfg<B>::DKV_CTAS), Cfg<B>::DKV_THREADS, dkv_smem<B>(), s>>>(
        mkB, mvB, mqB, mdoB, mdkB, mdvB, q);
    SPION_LAUNCH_CHECK();
    note_tc_launch(2);
    return SPION_OK;
}

spion_status launch_fwd_tc(const AttnArgs &a, cudaStream_t s) {
    return a.B == 64 ? fwd_tc_t<64>(a, s) : fwd_tc_t<32>(a, s);
}
spion_status launch_bwd_tc(const AttnArgs &a, cudaStream_t s) {
    return a.B == 64 ? bwd_tc_t<64>(a, s) : bwd_tc_t<32>(a, s);
}

}  // namespace spion
