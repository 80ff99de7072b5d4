// common.cuh — shared helpers of libspion.so (product path; no oracle code).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "spion.h"

namespace spion {

// host-side launch counter (spion_launch_count)
void note_launch(int n = 1);
// host-side counter of tensor-core (tcgen05) attention kernel launches (spion_tc_launch_count)
void note_tc_launch(int n = 1);

// SPION_DEBUG=1 in the environment prints the failing CUDA call
void report_cuda_error(cudaError_t e, const char *what, const char *file, int line);

#define SPION_CUDA_TRY(expr)                                                      \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) {                                                  \
            ::spion::report_cuda_error(_e, #expr, __FILE__, __LINE__);            \
            return SPION_ERR_CUDA;                                                \
        }                                                                         \
    } while (0)

#define SPION_LAUNCH_CHECK()                                                      \
    do {                                                                          \
        ::spion::note_launch();                                                   \
        cudaError_t _e = cudaGetLastError();                                      \
        if (_e != cudaSuccess) {                                                  \
            ::spion::report_cuda_error(_e, "kernel launch", __FILE__, __LINE__);  \
            return SPION_ERR_CUDA;                                                \
        }                                                                         \
    } while (0)

// opt a kernel into the largest dynamic shared memory the device allows
template <typename F>
static inline cudaError_t allow_max_dyn_smem(F *func) {
    int dev = 0, optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    cudaFuncAttributes fa;
    e = cudaFuncGetAttributes(&fa, func);
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes);
}

// "done once per device" flags: kernel attributes (e.g. the dynamic shared memory limit) belong
// to the current device's context, so a process driving several GPUs sets them once per device
struct PerDevice {
    std::atomic<unsigned long long> bits{0};
};
static inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev;
}
// raise func's dynamic shared memory limit to `bytes` (or the device maximum, bytes < 0) once per device
template <typename F>
static inline cudaError_t smem_attr_once(PerDevice &flag, F *func, int bytes = -1) {
    const unsigned long long bit = 1ull << (current_device() & 63);
    if (flag.bits.load(std::memory_order_acquire) & bit) return cudaSuccess;
    cudaError_t e = bytes < 0 ? allow_max_dyn_smem(func)
                              : cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) flag.bits.fetch_or(bit, std::memory_order_release);
    return e;
}

static inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
static inline size_t round_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// ---- element load/store for the two I/O dtypes
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
template <typename T> __device__ __forceinline__ T from_f32(float x);
template <> __device__ __forceinline__ float from_f32<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
// exclusive prefix sum over the warp (64-bit)
__device__ __forceinline__ unsigned long long warp_excl_scan_u64(unsigned long long v, int lane) {
    unsigned long long incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    return incl - v;
}
__device__ __forceinline__ int warp_excl_scan_i32(int v, int lane) {
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    return incl - v;
}

// ---- plan layout (int32 words; see pattern.cu)
struct PlanLayout {
    int n, S, ntiles;
    // header words: [0] n [1] S [2] ntiles [3] fwd entries [4] bwd entries
    //               [5] heavy row tiles [6] heavy column tiles (prefixes of the work orders)
    //               [7] heavy block columns (> 2x the mean count; a prefix of bperm)
    //               [8..15] reserved (the attention kernels' work-item counters live in the
    //               caller's attention workspace, not in the shared pattern)
    size_t fptr, bptr, forder, border, fcol, fmsk, brow, bmsk, bperm, words;
    __host__ __device__ PlanLayout(int n_, int block) {
        n = n_;
        S = block >= 128 ? 1 : 128 / block;
        if (S > 32) S = 32;
        if (S < 1) S = 1;
        ntiles = (n + S - 1) / S;
        fptr = 16;
        bptr = fptr + ntiles + 1;
        forder = bptr + ntiles + 1;
        border = forder + ntiles;
        size_t cap = (size_t)n * ntiles;
        fcol = border + ntiles;
        fmsk = fcol + cap;
        brow = fmsk + cap;
        bmsk = brow + cap;
        bperm = bmsk + cap;  // column tile t, slot s -> block column bperm[t*S + s] (n: empty slot)
        words = bperm + (size_t)ntiles * S;
    }
};

// device flag word bits (pattern workspace)
enum : int { FLAG_BAD_SCORE = 1, FLAG_CAPACITY = 2, FLAG_BAD_MASK = 4 };

}  // namespace spion
