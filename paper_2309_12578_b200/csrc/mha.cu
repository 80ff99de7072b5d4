// mha.cu — SURVEY §8(f) NEXT-4: the sparse-MHA sub-layer around the attention (Alg. 5 l.2-3
// and l.8-9): split of the QKV projection into per-head [bh][L][d] tensors, the
// concatenation of the heads for W^O, and the dropout + residual of l.9 — HBM-bound layout /
// elementwise kernels, 16-byte vectors, one pass each.  The projections themselves are plain
// GEMMs (cuBLAS, through the caller).
#include "attn.cuh"

namespace spion {

// [batch][L][W][H][d] (row-major projection output, W tensors side by side) <-> W tensors
// [batch*H][L][d], in 16-byte chunks (8 bf16).  Block (x, b) owns rows [x*RPB, x*RPB + RPB) of
// batch item b; thread k owns chunk k of every such row (k -> (w, h, c) decomposed once, no
// per-element index division), so the packed side is read / written fully coalesced and the
// head side in 128-byte runs (one head row = d/8 chunks).
constexpr int PERM_RPB = 16;
__global__ void __launch_bounds__(256)
heads_permute_kernel(const uint4 *__restrict__ src, uint4 *__restrict__ dst, int L, int W, int H, int dch,
                     int64_t tstride, int to_heads) {
    const int RC = W * H * dch;  // chunks per packed row
    const int64_t b = blockIdx.y;
    const int l0 = blockIdx.x * PERM_RPB, l1 = min(L, l0 + PERM_RPB);
    for (int k = threadIdx.x; k < RC; k += blockDim.x) {
        const int c = k % dch, h = (k / dch) % H, w = k / (dch * H);
        const int64_t pbase = b * L * (int64_t)RC + k;                                      // packed
        const int64_t hbase = w * tstride + (b * H + h) * (int64_t)L * dch + c;            // heads
        if (to_heads) {
#pragma unroll 4
            for (int l = l0; l < l1; ++l) dst[hbase + (int64_t)l * dch] = __ldg(src + pbase + (int64_t)l * RC);
        } else {
#pragma unroll 4
            for (int l = l0; l < l1; ++l) dst[pbase + (int64_t)l * RC] = __ldg(src + hbase + (int64_t)l * dch);
        }
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

// forward: out = e + keep(y) / (1 - p);  backward (e == nullptr): out = keep(y) / (1 - p).
// 8 elements (one 16-byte vector of each operand) per thread and step; `vec` = every pointer
// 16-byte aligned, else one element per step
__device__ __forceinline__ float dr_one(float y, uint64_t i, uint32_t thresh, float scale, uint64_t seed) {
    return mix32(seed * 0x9e3779b97f4a7c15ull + i) >= thresh ? y * scale : 0.f;
}
__global__ void dropout_residual_kernel(const __nv_bfloat16 *__restrict__ y, const __nv_bfloat16 *__restrict__ e,
                                        __nv_bfloat16 *__restrict__ out, int64_t n, uint32_t thresh, float scale,
                                        uint64_t seed, int vec) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t done = 0;
    if (vec) {
        const int64_t n8 = n / 8;
        for (int64_t v = i0; v < n8; v += stride) {
            const uint4 yv = __ldg(reinterpret_cast<const uint4 *>(y) + v);
            uint4 ev = make_uint4(0u, 0u, 0u, 0u);
            if (e) ev = __ldg(reinterpret_cast<const uint4 *>(e) + v);
            const __nv_bfloat16 *yb = reinterpret_cast<const __nv_bfloat16 *>(&yv);
            const __nv_bfloat16 *eb = reinterpret_cast<const __nv_bfloat16 *>(&ev);
            uint4 ov;
            __nv_bfloat16 *ob = reinterpret_cast<__nv_bfloat16 *>(&ov);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float r = dr_one(__bfloat162float(yb[j]), (uint64_t)(8 * v + j), thresh, scale, seed);
                if (e) r += __bfloat162float(eb[j]);
                ob[j] = __float2bfloat16_rn(r);
            }
            reinterpret_cast<uint4 *>(out)[v] = ov;
        }
        done = n8 * 8;
    }
    for (int64_t i = done + i0; i < n; i += stride) {
        float r = dr_one(__bfloat162float(y[i]), (uint64_t)i, thresh, scale, seed);
        if (e) r += __bfloat162float(e[i]);
        out[i] = __float2bfloat16_rn(r);
    }
}

static int grid_for_elems(int64_t n) {
    int64_t g = (n + 255) / 256;
    return (int)(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

spion_status launch_heads_permute(const void *src, void *dst, int64_t batch, int L, int W, int H, int d, int to_heads,
                                  cudaStream_t s) {
    const int dch = d / 8;
    const int64_t tstride = batch * H * (int64_t)L * dch;  // chunks per [bh][L][d] tensor
    if (batch > 65535) return SPION_ERR_SHAPE;
    const dim3 grid((L + PERM_RPB - 1) / PERM_RPB, (unsigned)batch);
    const int rc = W * H * dch;
    heads_permute_kernel<<<grid, rc >= 256 ? 256 : ((rc + 31) / 32) * 32, 0, s>>>(
        static_cast<const uint4 *>(src), static_cast<uint4 *>(dst), L, W, H, dch, tstride, to_heads);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

spion_status launch_dropout_residual(const void *y, const void *e, void *out, int64_t n, float p, uint64_t seed,
                                     cudaStream_t s) {
    const double t = (double)p * 4294967296.0;
    const uint32_t thresh = p <= 0.f ? 0u : (t >= 4294967295.0 ? 0xffffffffu : (uint32_t)t);
    const float scale = p < 1.f ? 1.f / (1.f - p) : 0.f;
    dropout_residual_kernel<<<grid_for_elems((n + 7) / 8), 256, 0, s>>>(static_cast<const __nv_bfloat16 *>(y),
                                                              static_cast<const __nv_bfloat16 *>(e),
                                                              static_cast<__nv_bfloat16 *>(out), n, thresh, scale, seed,
                                                              aligned16(y) && (!e || aligned16(e)) && aligned16(out));
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

}  // namespace spion
