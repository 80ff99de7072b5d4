// hop_bench.cu — latency of the synchronisation hops the attention kernels chain per block:
// mbarrier arrive -> try_wait / test_wait wake-up between two warps (ping-pong), and
// tcgen05.commit (no MMA in flight) -> mbarrier -> waiting warp.  Timing only.
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdio.h>
#include <stdint.h>
#include "tc_ptx.cuh"
using namespace spion::tc;

__device__ __forceinline__ void wait_spin(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n\t.reg .pred P;\n\tmbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\tselp.b32 %0, 1, 0, P;\n\t}"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}

template <int MODE>  // 0: arrive/try_wait ping-pong, 1: test_wait spin ping-pong, 2: commit hop (A commits, B waits, B arrives back)
__global__ void hop(int reps, long long *out) {
    __shared__ uint64_t ba, bb;
    __shared__ uint32_t slot;
    if (threadIdx.x < 32) tmem_alloc<32>(&slot);
    if (threadIdx.x == 0) { mbar_init(&ba, 1); mbar_init(&bb, 1); fence_barrier_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (warp == 0) {
            if (MODE == 2) {
                if (elect_one()) mma_commit(&ba);
                __syncwarp();
            } else if (lane == 0) {
                mbar_arrive(&ba);
            }
            if (MODE == 1) wait_spin(&bb, r & 1); else mbar_wait(&bb, r & 1);
        } else {
            if (MODE == 1) wait_spin(&ba, r & 1); else mbar_wait(&ba, r & 1);
            if (lane == 0) mbar_arrive(&bb);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) out[0] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x < 32) tmem_dealloc<32>(slot);
}
template <int MODE>
void run(const char *name) {
    long long *d, h;
    cudaMalloc(&d, 8);
    hop<MODE><<<1, 64>>>(1000, d);
    hop<MODE><<<1, 64>>>(1000, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s round trip %6.1f cycles (2 hops) %s\n", name, (double)h / 1000, cudaGetErrorString(e));
}
int main() {
    run<0>("arrive -> try_wait, both ways");
    run<1>("arrive -> test_wait spin, both ways");
    run<2>("tcgen05.commit -> try_wait, arrive back");
    return 0;
}
