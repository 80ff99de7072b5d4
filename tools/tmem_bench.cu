// tmem_bench.cu — microbenchmark: tcgen05.ld (32x32b.x32) and tcgen05.st throughput per SM vs warp
// count, and MUFU.EX2 throughput.  Timing only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2309_12578_b200/csrc \
//        tools/tmem_bench.cu -o tools/tmem_bench
#include <cuda_runtime.h>
#include <stdio.h>
#include <cuda_bf16.h>
#include "tc_ptx.cuh"
using namespace spion::tc;

template <int MODE>  // 0 ld, 1 st, 2 ex2
__global__ void kern(int reps, long long *out, float *sink) {
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int warp = threadIdx.x >> 5;
    const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)((warp >> 2) * 64);
    float acc = 0.f, x = threadIdx.x * 1e-3f;
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (MODE == 0) {
            float v[32], w[32];
            tmem_ld32(tl, v);
            tmem_ld32(tl + 32, w);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) acc += v[i] + w[i];
        } else if (MODE == 1) {
            uint32_t v[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = r + i;
            tmem_st16(tl, v);
            tmem_st16(tl + 16, v);
            tmem_st_wait();
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) { x = ex2(x) * 0.5f; }
            acc += x;
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

// MMA throughput (warp 0 issues SS or TS N=64 MMAs into columns [0,128)) while `lw` other
// warps stream tcgen05.ld from columns [256, 320) and optionally write packed bf16 back
template <bool TS, bool ST>
__global__ void contend(int reps, long long *out, float *sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    __shared__ volatile int done;
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int warp = threadIdx.x >> 5;
    constexpr uint32_t IDESC = idesc_bf16(128, 64, false, false);
    float acc = 0.f;
    if (warp == 0) {
        const uint64_t dA = sdesc_sw128(smem_u32(smem)), dB = sdesc_sw128(smem_u32(smem + 16384));
        long long t0 = clock64();
        if (elect_one()) {
            for (int r = 0; r < reps; ++r) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (TS) mma_bf16_ts(tmem + 64 * (r & 1), tmem + 384 + 8 * k, dB + 2 * k, IDESC, k > 0);
                    else mma_bf16_ss(tmem + 64 * (r & 1), dA + 2 * k, dB + 2 * k, IDESC, k > 0);
                }
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; done = 1; }
    } else {
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 256;
        while (!done) {
            float v[32];
            tmem_ld32(tl, v);
            tmem_ld_wait();
            for (int i = 0; i < 32; ++i) acc += v[i];
            if (ST) {
                uint32_t u[16];
                for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i]);
                tmem_st16(tl + 64, u);
                tmem_st_wait();
            }
        }
    }
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <bool TS, bool ST>
void run_contend(int lw) {
    long long *d, h;
    float *s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4096 * 4);
    const int reps = 1000;
    auto k = contend<TS, ST>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
    k<<<1, 32 * (1 + lw), 49152>>>(reps, d, s);
    k<<<1, 32 * (1 + lw), 49152>>>(reps, d, s);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("MMA %s N=64 with %2d tcgen05.ld%s warps: %6.1f cyc/MMA %s\n", TS ? "TS" : "SS", lw, ST ? "+st" : "", (double)h / (reps * 4),
           cudaGetErrorString(e));
}

// the dK/dV kernel's per-block MMA sequence (S^T, dP^T: SS N=64 K=64; dV, dK: TS N=64 K=64,
// B MN-major) issued back to back by warp 0, with `lw` warps doing OTHER traffic:
// OTHER = 0 none, 1 tcgen05.ld, 2 LDS.128 streaming, 3 ld + st
template <int OTHER>
__global__ void seq(int reps, long long *out, float *sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    __shared__ volatile int done;
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const int warp = threadIdx.x >> 5;
    constexpr uint32_t IDESC_ST = idesc_bf16(128, 64, false, false);
    constexpr uint32_t IDESC_DKV = idesc_bf16(128, 64, false, true);
    float acc = 0.f;
    if (warp == 0) {
        const uint64_t dK0 = sdesc_sw128(smem_u32(smem)), dV0 = sdesc_sw128(smem_u32(smem + 16384));
        const uint64_t dQ0 = sdesc_sw128(smem_u32(smem + 32768)), ddO0 = sdesc_sw128(smem_u32(smem + 40960));
        long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem, dK0 + 2 * k, dQ0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + 64, dV0 + 2 * k, ddO0 + 2 * k, IDESC_ST, k > 0);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    mma_bf16_ts(tmem + 256, tmem + 32 * (k / 2) + 8 * (k % 2), ddO0 + 128 * k, IDESC_DKV, 1);
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    mma_bf16_ts(tmem + 320, tmem + 64 + 32 * (k / 2) + 8 * (k % 2), dQ0 + 128 * k, IDESC_DKV, 1);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) { out[0] = t1 - t0; done = 1; }
    } else {
        const uint32_t tl = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384;
        const float4 *src = reinterpret_cast<const float4 *>(smem + 65536);
        int i0 = threadIdx.x;
        while (!done) {
            if (OTHER == 1 || OTHER == 3) {
                float v[32];
                tmem_ld32(tl, v);
                tmem_ld_wait();
                for (int i = 0; i < 32; ++i) acc += v[i];
                if (OTHER == 3) {
                    uint32_t u[16];
                    for (int i = 0; i < 16; ++i) u[i] = __float_as_uint(v[i]);
                    tmem_st16(tl + 64, u);
                    tmem_st_wait();
                }
            } else if (OTHER == 2) {
#pragma unroll
                for (int i = 0; i < 8; ++i) { float4 a = src[(i0 + 64 * i) & 2047]; acc += a.x + a.w; }
                i0 += 7;
            }
        }
    }
    if (acc == 12345.f) sink[threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int OTHER>
void run_seq(int lw) {
    long long *d, h;
    float *s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4096 * 4);
    const int reps = 500;
    auto k = seq<OTHER>;
    const int sm = 65536 + 32768;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    k<<<1, 32 * (1 + lw), sm>>>(reps, d, s);
    k<<<1, 32 * (1 + lw), sm>>>(reps, d, s);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("dKdV MMA sequence (8 SS + 8 TS), other=%d with %2d warps: %6.1f cyc/block (ideal 8*48+8*32=640) %s\n", OTHER, lw,
           (double)h / reps, cudaGetErrorString(e));
}

// issue cost: clock before/after issuing NM SS N=64 MMAs (with or without a commit) into an empty pipe
template <int NM, bool COMMIT>
__global__ void issue_cost(long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t IDESC = idesc_bf16(128, 64, false, false);
    const uint64_t dA = sdesc_sw128(smem_u32(smem)), dB = sdesc_sw128(smem_u32(smem + 16384));
    long long tot = 0, tot2 = 0;
    for (int r = 0; r < 20; ++r) {
        long long t0 = clock64(), t1 = 0;
        if (elect_one()) {
#pragma unroll
            for (int k = 0; k < NM; ++k) mma_bf16_ss(tmem + 64 * (k / 4 % 4), dA + 2 * (k % 4), dB + 2 * (k % 4), IDESC, k % 4 > 0);
            t1 = clock64();
            if (COMMIT) mma_commit(&bar);
        }
        __syncwarp();
        long long t2 = clock64();
        if (!COMMIT && elect_one()) mma_commit(&bar);
        __syncwarp();
        mbar_wait(&bar, r & 1);
        long long t3 = clock64();
        if (r >= 4) { tot += t1 - t0; tot2 += t2 - t0; }
        (void)t3;
    }
    if (threadIdx.x == 0) { out[0] = tot / 16; out[1] = tot2 / 16; }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}
template <int NM, bool COMMIT>
void run_issue() {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    auto k = issue_cost<NM, COMMIT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 49152);
    k<<<1, 32, 49152>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("issue %2d SS MMAs%s: %5lld cyc to issue, %5lld cyc incl. commit/syncwarp (exec %d) %s\n", NM, COMMIT ? " + commit" : "", h[0], h[1],
           NM * 48, cudaGetErrorString(e));
}

template <int MODE>
void run(int warps) {
    long long *d, h;
    float *s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4096);
    const int reps = 2000;
    kern<MODE><<<1, warps * 32>>>(reps, d, s);
    kern<MODE><<<1, warps * 32>>>(reps, d, s);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = (double)h / reps;
    if (MODE == 0)
        printf("tcgen05.ld 2x(32x32b.x32) warps=%2d: %7.1f cyc/iter  -> %6.1f B/cyc/SM %s\n", warps, cyc, warps * 32 * 64 * 4 / cyc, cudaGetErrorString(e));
    else if (MODE == 1)
        printf("tcgen05.st 2x(32x32b.x16) warps=%2d: %7.1f cyc/iter  -> %6.1f B/cyc/SM %s\n", warps, cyc, warps * 32 * 32 * 4 / cyc, cudaGetErrorString(e));
    else
        printf("ex2 (dependent chains)  warps=%2d: %7.1f cyc/iter  -> %6.2f ex2/cyc/SM %s\n", warps, cyc, warps * 32 * 32 / cyc, cudaGetErrorString(e));
}

int main() {
    run_issue<4, false>();
    run_issue<8, false>();
    run_issue<16, false>();
    run_issue<32, false>();
    run_issue<4, true>();
    run_issue<8, true>();
    run_issue<16, true>();
    run_seq<0>(0);
    run_seq<1>(8);
    run_seq<2>(8);
    run_seq<3>(8);
    run_seq<2>(16);
    for (int lw : {0, 4, 8, 16}) run_contend<false, false>(lw);
    for (int lw : {0, 4, 8, 16}) run_contend<true, false>(lw);
    for (int lw : {8, 16}) run_contend<false, true>(lw);
    for (int w : {4, 8, 16}) run<0>(w);
    for (int w : {4, 8, 16}) run<1>(w);
    for (int w : {4, 8, 16, 32}) run<2>(w);
    return 0;
}
