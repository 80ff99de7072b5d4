// mha.cu — SURVEY §8(f) NEXT-4: the sparse-MHA sub-layer around the attention (Alg. 5 l.2-3
// and l.8-9): split of the QKV projection into per-head [bh][L][d] tensors, the
// concatenation of the heads for W^O, and the dropout + residual of l.9 — HBM-bound layout /
// elementwise kernels, 16-byte vectors, one pass each.  The projections themselves are plain
// GEMMs (cuBLAS, through the caller).
#include "attn.cuh"

namespace spion {

// [batch][L][W][H][d] (row-major projection output, W tensors side by side) <-> W tensors
// [batch*H][L][d].  One thread moves one 16-byte chunk (8 bf16); consecutive threads walk a
// row of the projection output, so the wide side is read / written fully coalesced.
__global__ void heads_permute_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int64_t chunks,
                                     int L, int W, int H, int dch, int64_t tstride, int to_heads) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
        // i indexes the [batch][L][W][H][dch] chunk grid
        int64_t r = i;
        const int c = (int)(r % dch); r /= dch;
        const int h = (int)(r % H); r /= H;
        const int w = (int)(r % W); r /= W;
        const int l = (int)(r % L);
        const int64_t b = r / L;
        const int64_t hidx = w * tstride + ((b * H + h) * (int64_t)L + l) * dch + c;  // [w][bh][L][dch]
        if (to_heads) dst[hidx] = src[i];
        else dst[i] = src[hidx];
    }
}

// counter-based keep mask: a 32-bit finalizer of (seed, element index); deterministic, so the
// backward regenerates the forward's mask without storing it
__device__ __forceinline__ uint32_t mix32(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return (uint32_t)x;
}

// forward: out = e + keep(y) / (1 - p);  backward (e == nullptr): out = keep(y) / (1 - p)
__global__ void dropout_residual_kernel(const __nv_bfloat16 *__restrict__ y, const __nv_bfloat16 *__restrict__ e,
                                        __nv_bfloat16 *__restrict__ out, int64_t n, uint32_t thresh, float scale,
                                        uint64_t seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const bool keep = mix32(seed * 0x9e3779b97f4a7c15ull + (uint64_t)i) >= thresh;
        float v = keep ? __bfloat162float(y[i]) * scale : 0.f;
        if (e) v += __bfloat162float(e[i]);
        out[i] = __float2bfloat16_rn(v);
    }
}

static int grid_for_elems(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

spion_status launch_heads_permute(const void *src, void *dst, int64_t batch, int L, int W, int H, int d, int to_heads,
                                  cudaStream_t s) {
    const int dch = d / 8;
    const int64_t chunks = batch * L * W * H * (int64_t)dch;
    const int64_t tstride = batch * H * (int64_t)L * dch;  // chunks per [bh][L][d] tensor
    heads_permute_kernel<<<grid_for_elems(chunks), 256, 0, s>>>(static_cast<const uint4 *>(src), static_cast<uint4 *>(dst),
                                                                 chunks, L, W, H, dch, tstride, to_heads);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

spion_status launch_dropout_residual(const void *y, const void *e, void *out, int64_t n, float p, uint64_t seed,
                                     cudaStream_t s) {
    const double t = (double)p * 4294967296.0;
    const uint32_t thresh = p <= 0.f ? 0u : (t >= 4294967295.0 ? 0xffffffffu : (uint32_t)t);
    const float scale = p < 1.f ? 1.f / (1.f - p) : 0.f;
    dropout_residual_kernel<<<grid_for_elems(n), 256, 0, s>>>(static_cast<const __nv_bfloat16 *>(y),
                                                              static_cast<const __nv_bfloat16 *>(e),
                                                              static_cast<__nv_bfloat16 *>(out), n, thresh, scale, seed);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

}  // namespace spion
