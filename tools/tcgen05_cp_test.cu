// tcgen05_cp_test.cu — does tcgen05.cp (shared -> tensor memory, 128x256b) place a SW128
// K-major bf16 tile [128][64] in TMEM in the A-operand layout of a TS MMA (row = lane, two
// bf16 per 32-bit column, K = 16 per 8 columns)?  Checks (1) the copied bits via tcgen05.ld,
// (2) D_ts = A(TMEM) B^T equals D_ss = A(smem) B^T, and times (3) SS vs TS with a cp'd A.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2309_12578_b200/csrc \
//        tools/tcgen05_cp_test.cu -o tools/tcgen05_cp_test
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "tc_ptx.cuh"

using namespace spion::tc;

__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ uint16_t val(int r, int c) { return (uint16_t)(0x3c00 + ((r * 7 + c * 3) & 0x1ff)); }

__global__ void __launch_bounds__(128, 1) cp_test(int *err, float *dss, float *dts, long long *cyc) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t *sA = smem, *sB = smem + 16384;  // A [128][64], B [64][64], SW128 K-major
    const int t = threadIdx.x;
    // fill A and B (bf16 bit patterns of moderate values)
    for (int r = t; r < 128; r += 128)
        for (int ch = 0; ch < 8; ++ch) {
            uint16_t v[8];
            for (int e = 0; e < 8; ++e) v[e] = val(r, ch * 8 + e);
            *reinterpret_cast<uint4 *>(sA + sw128_offset(r, ch)) = *reinterpret_cast<uint4 *>(v);
        }
    for (int r = t; r < 64; r += 128)
        for (int ch = 0; ch < 8; ++ch) {
            uint16_t v[8];
            for (int e = 0; e < 8; ++e) v[e] = (uint16_t)(0x3c00 + ((r * 5 + (ch * 8 + e) * 11) & 0xff));
            *reinterpret_cast<uint4 *>(sB + sw128_offset(r, ch)) = *reinterpret_cast<uint4 *>(v);
        }
    fence_proxy_async_smem();
    if (t < 32) tmem_alloc<512>(&slot);
    if (t == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    constexpr uint32_t IDESC = idesc_bf16(128, 64, false, false);
    const uint32_t COL_A = 256, COL_SS = 0, COL_TS = 64;
    if (t == 0) {
        const uint64_t dA = sdesc_sw128(smem_u32(sA)), dB = sdesc_sw128(smem_u32(sB));
        for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + COL_A + 8 * k, dA + 2 * k);
        for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + COL_SS, dA + 2 * k, dB + 2 * k, IDESC, k > 0);
        for (int k = 0; k < 4; ++k) mma_bf16_ts(tmem + COL_TS, tmem + COL_A + 8 * k, dB + 2 * k, IDESC, k > 0);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        // timing: 256 TS MMAs re-reading the copied A vs 256 SS
        long long t0 = clock64();
        for (int r = 0; r < 64; ++r)
            for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + 128, dA + 2 * k, dB + 2 * k, IDESC, k > 0);
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        long long t1 = clock64();
        for (int r = 0; r < 64; ++r)
            for (int k = 0; k < 4; ++k) mma_bf16_ts(tmem + 128, tmem + COL_A + 8 * k, dB + 2 * k, IDESC, k > 0);
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t2 = clock64();
        // cp + dependent TS MMA latency (the item-start cost)
        for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + COL_A + 8 * k, dA + 2 * k);
        for (int k = 0; k < 4; ++k) mma_bf16_ts(tmem + 128, tmem + COL_A + 8 * k, dB + 2 * k, IDESC, k > 0);
        mma_commit(&bar);
        mbar_wait(&bar, 1);
        long long t3 = clock64();
        cyc[0] = (t1 - t0) / 256;
        cyc[1] = (t2 - t1) / 256;
        cyc[2] = t3 - t2;
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // (1) copied bits
    const int w = t >> 5, row = t;  // thread = lane = row
    const uint32_t tl = tmem + ((uint32_t)(w * 32) << 16);
    float v[32];
    tmem_ld32(tl + COL_A, v);
    tmem_ld_wait();
    int bad = 0;
    for (int c = 0; c < 32; ++c) {
        const uint32_t u = __float_as_uint(v[c]);
        const uint32_t want = (uint32_t)val(row, 2 * c) | ((uint32_t)val(row, 2 * c + 1) << 16);
        if (u != want) ++bad;
    }
    // (2) D_ts == D_ss
    float a[32], b[32];
    for (int h = 0; h < 2; ++h) {
        tmem_ld32(tl + COL_SS + 32 * h, a);
        tmem_ld32(tl + COL_TS + 32 * h, b);
        tmem_ld_wait();
        for (int c = 0; c < 32; ++c) {
            dss[row * 64 + 32 * h + c] = a[c];
            dts[row * 64 + 32 * h + c] = b[c];
            if (a[c] != b[c]) bad += 1000;
        }
    }
    atomicAdd(err, bad);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (t < 32) tmem_dealloc<512>(tmem);
}

int main() {
    int *err;
    float *dss, *dts;
    long long *cyc;
    cudaMallocManaged(&err, 4);
    cudaMallocManaged(&dss, 128 * 64 * 4);
    cudaMallocManaged(&dts, 128 * 64 * 4);
    cudaMallocManaged(&cyc, 3 * 8);
    *err = 0;
    cudaFuncSetAttribute(cp_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    cp_test<<<1, 128, 40000>>>(err, dss, dts, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("tcgen05.cp test: %s, mismatches %d (bits: units, D_ts vs D_ss: thousands)\n", cudaGetErrorString(e), *err);
    printf("D_ss[0][0..3] = %g %g %g %g ; D_ts = %g %g %g %g\n", dss[0], dss[1], dss[2], dss[3], dts[0], dts[1],
           dts[2], dts[3]);
    printf("SS N=64 K=16: %lld cyc/MMA, TS (A copied by tcgen05.cp): %lld cyc/MMA, cp(4x128x256b)+4 TS+commit: %lld cyc\n",
           cyc[0], cyc[1], cyc[2]);
    return (e == cudaSuccess && *err == 0) ? 0 : 1;
}
