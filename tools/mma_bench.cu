// mma_bench.cu — microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) for the
// SS form (A, B from shared memory) and the TS form (A from tensor memory), several N,
// one or all SMs.  Operand contents are irrelevant (timing only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2309_12578_b200/csrc \
//        tools/mma_bench.cu -o tools/mma_bench -lcuda
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include "tc_ptx.cuh"

using namespace spion::tc;

template <int N, bool TS, int NACC>
__global__ void __launch_bounds__(128, 1) bench(int reps, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *sA = smem, *sB = smem + 16384;  // A 128x64, B N x 64 (SW128 K-major)
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t IDESC = idesc_bf16(128, N, false, false);
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        const uint64_t dA = sdesc_sw128(smem_u32(sA)), dB = sdesc_sw128(smem_u32(sB));
        // warm-up
        for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem, dA + 2 * k, dB + 2 * k, IDESC, k > 0);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            const uint32_t d = tmem + (uint32_t)((r % NACC) * N) % 256;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (TS) mma_bf16_ts(d, tmem + 256 + 8 * k, dB + 2 * k, IDESC, k > 0);
                else mma_bf16_ss(d, dA + 2 * k, dB + 2 * k, IDESC, k > 0);
            }
        }
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

// latency: one K=64 group (4 MMAs, or 8 = two groups as in S+dP) + commit, waited serially
template <int N, bool TS, int G>
__global__ void __launch_bounds__(128, 1) lat(int reps, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *sA = smem, *sB = smem + 16384;
    if (threadIdx.x < 32) tmem_alloc<512>(&slot);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t IDESC = idesc_bf16(128, N, false, false);
    if (threadIdx.x == 0) {
        const uint64_t dA = sdesc_sw128(smem_u32(sA)), dB = sdesc_sw128(smem_u32(sB));
        long long t0 = 0, tiss = 0;
        for (int r = 0; r < reps + 1; ++r) {
            if (r == 1) t0 = clock64();
            const long long ti = clock64();
            for (int g = 0; g < G; ++g)
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (TS) mma_bf16_ts(tmem + g * N, tmem + 256 + 8 * k, dB + 2 * k, IDESC, k > 0);
                    else mma_bf16_ss(tmem + g * N, dA + 2 * k, dB + 2 * k, IDESC, k > 0);
                }
            mma_commit(&bar);
            if (r > 0) tiss += clock64() - ti;
            mbar_wait(&bar, r & 1);
            tc_fence_after();
        }
        out[blockIdx.x] = clock64() - t0;
        out[1] = tiss;
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<512>(tmem);
}

template <int N, bool TS, int G>
static void run_lat() {
    const int reps = 1000;
    long long *d, h, hi[2];
    cudaMalloc(&d, 2 * sizeof(long long));
    auto k = lat<N, TS, G>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768 + 1024);
    k<<<1, 128, 16384 + 32768 + 1024>>>(reps, d);
    cudaDeviceSynchronize();
    cudaMemcpy(hi, d, sizeof(hi), cudaMemcpyDeviceToHost);
    h = hi[0];
    printf("latency %s N=%3d groups=%d (K=64 each) issue->mbarrier: %6.1f cycles (ideal %5.1f), issue alone %6.1f\n", TS ? "TS" : "SS", N, G,
           (double)h / reps, G * 4 * 128.0 * N / 256.0, (double)hi[1] / reps);
    cudaFree(d);
}

template <int N, bool TS, int NACC>
static void run(int grid) {
    const int reps = 2000;
    long long *d;
    cudaMalloc(&d, grid * sizeof(long long));
    auto k = bench<N, TS, NACC>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768 + 1024);
    k<<<grid, 128, 16384 + 32768 + 1024>>>(reps, d);
    k<<<grid, 128, 16384 + 32768 + 1024>>>(reps, d);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const double per = mx / (reps * 4.0);
    const double ideal = 128.0 * N / 256.0;
    printf("%s N=%3d acc=%d grid=%3d: %6.1f cycles/MMA (ideal %5.1f, %4.0f%%)  %s\n", TS ? "TS" : "SS", N, NACC, grid, per,
           ideal, 100 * ideal / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run_lat<64, false, 1>();
    run_lat<64, false, 2>();
    run_lat<64, true, 1>();
    run_lat<64, true, 2>();
    run_lat<32, false, 2>();
    run_lat<32, true, 2>();
    run_lat<128, false, 1>();
    for (int grid : {1, 148}) {
        run<64, false, 1>(grid);
        run<64, true, 1>(grid);
        run<64, false, 4>(grid);
        run<64, true, 4>(grid);
        run<128, false, 1>(grid);
        run<128, true, 1>(grid);
        run<256, false, 1>(grid);
        run<256, true, 1>(grid);
        run<32, false, 1>(grid);
        run<32, true, 1>(grid);
    }
    return 0;
}
