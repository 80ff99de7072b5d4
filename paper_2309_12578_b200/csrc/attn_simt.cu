// attn_simt.cu — block-sparse attention on CUDA cores (fp32 arithmetic).
//
// The fp32 mode of the ABI (tolerance 1e-4; tf32 tensor cores are too coarse)
// and the bf16 shapes the tensor-core path does not cover (block not in
// {32,64}, d != 64).  Same mathematics as attn_tc.cu:
//   fwd (Eq. 5, Alg. 5 l.4-8, Alg. 6): online softmax over the stored blocks
//       of a block row; PAPER mode adds ln(L - cnt) in the log domain
//       (reading Q2): lse = logaddexp(m + ln l, ln(L - cnt)).
//   bwd (reading Q17): D_i = dO_i . O_i; p = exp(s - lse); ds = p (dO_i.V_j - D_i);
//       dK/dV column-stationary (CSC), dQ row-stationary (CSR) — deterministic.
#include <math.h>

#include "attn.cuh"

namespace spion {

static constexpr int SIMT_WARPS = 4;



template <typename T>
__device__ __forceinline__ void load_tile(float *dst, int ld, const T *src, int64_t stride_l, int rows, int d) {
    for (int idx = threadIdx.x; idx < rows * d; idx += blockDim.x) {
        const int r = idx / d, e = idx % d;
        dst[r * ld + e] = to_f32(src[(int64_t)r * stride_l + e]);
    }
}

// ------------------------------------------------------------------ forward
template <typename T>
__global__ void __launch_bounds__(SIMT_WARPS * 32) attn_fwd_simt_kernel(AttnArgs a) {
    extern __shared__ float sm[];
    const int B = a.B, d = a.d, dp = d + 1;
    const int I = blockIdx.x;
    const int64_t b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *Qs = sm;                 // [B][d+1]
    float *Ks = Qs + B * dp;        // [B][d+1]
    float *Vs = Ks + B * dp;        // [B][d]
    float *Os = Vs + B * d;         // [B][d]
    float *ms = Os + B * d;         // [B]
    float *ls = ms + B;             // [B]
    float *Ps = ls + B;             // [SIMT_WARPS][B]
    const T *Qg = static_cast<const T *>(a.Q) + b * a.stride_bh + (int64_t)I * B * a.stride_l;
    load_tile(Qs, dp, Qg, a.stride_l, B, d);
    for (int idx = threadIdx.x; idx < B * d; idx += blockDim.x) Os[idx] = 0.f;
    for (int r = threadIdx.x; r < B; r += blockDim.x) { ms[r] = -INFINITY; ls[r] = 0.f; }
    const int beg = a.brow_ptr[I], end = a.brow_ptr[I + 1];
    for (int idx = beg; idx < end; ++idx) {
        const int J = a.bcol_idx[idx];
        __syncthreads();
        const int64_t off = b * a.stride_bh + (int64_t)J * B * a.stride_l;
        load_tile(Ks, dp, static_cast<const T *>(a.K) + off, a.stride_l, B, d);
        load_tile(Vs, d, static_cast<const T *>(a.V) + off, a.stride_l, B, d);
        __syncthreads();
        for (int ii = warp; ii < B; ii += SIMT_WARPS) {
            float mloc = -INFINITY;
            for (int jj = lane; jj < B; jj += 32) {
                float s = 0.f;
                for (int e = 0; e < d; ++e) s = fmaf(Qs[ii * dp + e], Ks[jj * dp + e], s);
                s *= a.scale;  // Alg. 6 l.8
                Ps[warp * B + jj] = s;
                mloc = fmaxf(mloc, s);
            }
            mloc = warp_max(mloc);
            const float m_old = ms[ii];
            const float m_new = fmaxf(m_old, mloc);
            const float alpha = (m_old == -INFINITY) ? 0.f : expf(m_old - m_new);
            float lsum = 0.f;
            for (int jj = lane; jj < B; jj += 32) {
                const float p = expf(Ps[warp * B + jj] - m_new);
                Ps[warp * B + jj] = p;
                lsum += p;
            }
            lsum = warp_sum(lsum);
            __syncwarp();
            for (int e = lane; e < d; e += 32) {
                float acc = Os[ii * d + e] * alpha;
                for (int jj = 0; jj < B; ++jj) acc = fmaf(Ps[warp * B + jj], Vs[jj * d + e], acc);
                Os[ii * d + e] = acc;
            }
            __syncwarp();
            if (lane == 0) { ms[ii] = m_new; ls[ii] = ls[ii] * alpha + lsum; }
            __syncwarp();
        }
    }
    __syncthreads();
    const int64_t cnt = (int64_t)B * (end - beg);
    T *Og = static_cast<T *>(a.Oout) + b * a.stride_bh + (int64_t)I * B * a.stride_l;
    for (int ii = warp; ii < B; ii += SIMT_WARPS) {
        float lse, f;
        if (cnt == 0) {
            lse = (a.mode == SPION_SOFTMAX_PAPER) ? logf((float)a.L) : -INFINITY;
            f = 0.f;
        } else {
            const float m = ms[ii], l = ls[ii];
            const float lse_m = m + logf(l);
            if (a.mode == SPION_SOFTMAX_PAPER && cnt < a.L) {
                const float lz = logf((float)(a.L - cnt));  // Alg. 6 l.15 in the log domain
                const float hi = fmaxf(lse_m, lz), lo = fminf(lse_m, lz);
                lse = hi + log1pf(expf(lo - hi));
            } else {
                lse = lse_m;
            }
            f = expf(m - lse);
        }
        for (int e = lane; e < d; e += 32) Og[(int64_t)ii * a.stride_l + e] = from_f32<T>(Os[ii * d + e] * f);
        if (lane == 0) a.lse_out[b * a.L + (int64_t)I * B + ii] = lse;
    }
}

// ----------------------------------------------------- D_i = rowsum(dO * O)
template <typename T>
__global__ void bwd_preprocess_kernel(AttnArgs a, float *D) {
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (row >= a.bh * a.L) return;
    const int64_t b = row / a.L, i = row % a.L;
    const T *o = static_cast<const T *>(a.O) + b * a.stride_bh + i * a.stride_l;
    const T *g = static_cast<const T *>(a.dO) + b * a.stride_bh + i * a.stride_l;
    float s = 0.f;
    for (int e = lane; e < a.d; e += 32) s = fmaf(to_f32(o[e]), to_f32(g[e]), s);
    s = warp_sum(s);
    if (lane == 0) D[row] = s;
}

// ------------------------------------------------- dQ (row-stationary, CSR)
template <typename T>
__global__ void __launch_bounds__(SIMT_WARPS * 32) attn_dq_simt_kernel(AttnArgs a) {
    extern __shared__ float sm[];
    const int B = a.B, d = a.d, dp = d + 1;
    const int I = blockIdx.x;
    const int64_t b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *Qs = sm;              // [B][d+1]
    float *dOs = Qs + B * dp;    // [B][d+1]
    float *Ks = dOs + B * dp;    // [B][d+1]
    float *Vs = Ks + B * dp;     // [B][d+1]
    float *dQs = Vs + B * dp;    // [B][d]
    float *Ps = dQs + B * d;     // [SIMT_WARPS][B]
    const int64_t qoff = b * a.stride_bh + (int64_t)I * B * a.stride_l;
    load_tile(Qs, dp, static_cast<const T *>(a.Q) + qoff, a.stride_l, B, d);
    load_tile(dOs, dp, static_cast<const T *>(a.dO) + qoff, a.stride_l, B, d);
    for (int idx = threadIdx.x; idx < B * d; idx += blockDim.x) dQs[idx] = 0.f;
    const float *lse = a.lse + b * a.L + (int64_t)I * B;
    const float *D = a.D + b * a.L + (int64_t)I * B;
    const int beg = a.brow_ptr[I], end = a.brow_ptr[I + 1];
    for (int idx = beg; idx < end; ++idx) {
        const int J = a.bcol_idx[idx];
        __syncthreads();
        const int64_t off = b * a.stride_bh + (int64_t)J * B * a.stride_l;
        load_tile(Ks, dp, static_cast<const T *>(a.K) + off, a.stride_l, B, d);
        load_tile(Vs, dp, static_cast<const T *>(a.V) + off, a.stride_l, B, d);
        __syncthreads();
        for (int ii = warp; ii < B; ii += SIMT_WARPS) {
            const float li = lse[ii], Di = D[ii];
            for (int jj = lane; jj < B; jj += 32) {
                float s = 0.f, dpv = 0.f;
                for (int e = 0; e < d; ++e) {
                    s = fmaf(Qs[ii * dp + e], Ks[jj * dp + e], s);
                    dpv = fmaf(dOs[ii * dp + e], Vs[jj * dp + e], dpv);
                }
                const float p = expf(s * a.scale - li);
                Ps[warp * B + jj] = p * (dpv - Di);
            }
            __syncwarp();
            for (int e = lane; e < d; e += 32) {
                float acc = dQs[ii * d + e];
                for (int jj = 0; jj < B; ++jj) acc = fmaf(Ps[warp * B + jj], Ks[jj * dp + e], acc);
                dQs[ii * d + e] = acc;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    T *dQg = static_cast<T *>(a.dQ) + qoff;
    for (int idx = threadIdx.x; idx < B * d; idx += blockDim.x) {
        const int r = idx / d, e = idx % d;
        dQg[(int64_t)r * a.stride_l + e] = from_f32<T>(dQs[idx] * a.scale);
    }
}

// --------------------------------------------- dK, dV (column-stationary, CSC)
template <typename T>
__global__ void __launch_bounds__(SIMT_WARPS * 32) attn_dkdv_simt_kernel(AttnArgs a) {
    extern __shared__ float sm[];
    const int B = a.B, d = a.d, dp = d + 1;
    const int J = blockIdx.x;
    const int64_t b = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *Ks = sm;               // [B][d+1]
    float *Vs = Ks + B * dp;      // [B][d+1]
    float *Qs = Vs + B * dp;      // [B][d+1]
    float *dOs = Qs + B * dp;     // [B][d+1]
    float *dKs = dOs + B * dp;    // [B][d]
    float *dVs = dKs + B * d;     // [B][d]
    float *ls = dVs + B * d;      // [B]
    float *Ds = ls + B;           // [B]
    float *Ps = Ds + B;           // [SIMT_WARPS][B]
    float *Ss = Ps + SIMT_WARPS * B;  // [SIMT_WARPS][B]
    const int64_t koff = b * a.stride_bh + (int64_t)J * B * a.stride_l;
    load_tile(Ks, dp, static_cast<const T *>(a.K) + koff, a.stride_l, B, d);
    load_tile(Vs, dp, static_cast<const T *>(a.V) + koff, a.stride_l, B, d);
    for (int idx = threadIdx.x; idx < B * d; idx += blockDim.x) { dKs[idx] = 0.f; dVs[idx] = 0.f; }
    const int beg = a.bcol_ptr[J], end = a.bcol_ptr[J + 1];
    for (int idx = beg; idx < end; ++idx) {
        const int I = a.brow_idx[idx];
        __syncthreads();
        const int64_t qoff = b * a.stride_bh + (int64_t)I * B * a.stride_l;
        load_tile(Qs, dp, static_cast<const T *>(a.Q) + qoff, a.stride_l, B, d);
        load_tile(dOs, dp, static_cast<const T *>(a.dO) + qoff, a.stride_l, B, d);
        for (int r = threadIdx.x; r < B; r += blockDim.x) {
            ls[r] = a.lse[b * a.L + (int64_t)I * B + r];
            Ds[r] = a.D[b * a.L + (int64_t)I * B + r];
        }
        __syncthreads();
        for (int jj = warp; jj < B; jj += SIMT_WARPS) {
            for (int ii = lane; ii < B; ii += 32) {
                float s = 0.f, dpv = 0.f;
                for (int e = 0; e < d; ++e) {
                    s = fmaf(Qs[ii * dp + e], Ks[jj * dp + e], s);
                    dpv = fmaf(dOs[ii * dp + e], Vs[jj * dp + e], dpv);
                }
                const float p = expf(s * a.scale - ls[ii]);
                Ps[warp * B + ii] = p;
                Ss[warp * B + ii] = p * (dpv - Ds[ii]);
            }
            __syncwarp();
            for (int e = lane; e < d; e += 32) {
                float av = dVs[jj * d + e], ak = dKs[jj * d + e];
                for (int ii = 0; ii < B; ++ii) {
                    av = fmaf(Ps[warp * B + ii], dOs[ii * dp + e], av);
                    ak = fmaf(Ss[warp * B + ii], Qs[ii * dp + e], ak);
                }
                dVs[jj * d + e] = av;
                dKs[jj * d + e] = ak;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    T *dKg = static_cast<T *>(a.dK) + koff;
    T *dVg = static_cast<T *>(a.dV) + koff;
    for (int idx = threadIdx.x; idx < B * d; idx += blockDim.x) {
        const int r = idx / d, e = idx % d;
        dKg[(int64_t)r * a.stride_l + e] = from_f32<T>(dKs[idx] * a.scale);
        dVg[(int64_t)r * a.stride_l + e] = from_f32<T>(dVs[idx]);
    }
}

// ------------------------------------------------------------------ host side
static size_t fwd_smem(int B, int d) { return sizeof(float) * ((size_t)B * (d + 1) * 2 + (size_t)B * d * 2 + 2 * B + SIMT_WARPS * B); }
static size_t dq_smem(int B, int d) { return sizeof(float) * ((size_t)B * (d + 1) * 4 + (size_t)B * d + SIMT_WARPS * B); }
static size_t dkdv_smem(int B, int d) { return sizeof(float) * ((size_t)B * (d + 1) * 4 + (size_t)B * d * 2 + 2 * B + 2 * SIMT_WARPS * B); }

bool simt_supported(int B, int d) { return B >= 1 && d >= 1 && d <= 128 && dkdv_smem(B, d) <= 227 * 1024; }

template <typename T>
static spion_status set_attrs() {
    static PerDevice f0, f1, f2;
    SPION_CUDA_TRY(smem_attr_once(f0, attn_fwd_simt_kernel<T>));
    SPION_CUDA_TRY(smem_attr_once(f1, attn_dq_simt_kernel<T>));
    SPION_CUDA_TRY(smem_attr_once(f2, attn_dkdv_simt_kernel<T>));
    return SPION_OK;
}

template <typename T>
static spion_status fwd_simt_t(const AttnArgs &a, cudaStream_t s) {
    spion_status st = set_attrs<T>();
    if (st) return st;
    attn_fwd_simt_kernel<T><<<dim3(a.n, (unsigned)a.bh), SIMT_WARPS * 32, fwd_smem(a.B, a.d), s>>>(a);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

template <typename T>
static spion_status bwd_preprocess_t(const AttnArgs &a, float *D, cudaStream_t s) {
    const int64_t rows = a.bh * a.L;
    bwd_preprocess_kernel<T><<<(unsigned)((rows + 7) / 8), 256, 0, s>>>(a, D);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

template <typename T>
static spion_status bwd_simt_t(const AttnArgs &a, cudaStream_t s) {
    spion_status st = set_attrs<T>();
    if (st) return st;
    attn_dq_simt_kernel<T><<<dim3(a.n, (unsigned)a.bh), SIMT_WARPS * 32, dq_smem(a.B, a.d), s>>>(a);
    SPION_LAUNCH_CHECK();
    attn_dkdv_simt_kernel<T><<<dim3(a.n, (unsigned)a.bh), SIMT_WARPS * 32, dkdv_smem(a.B, a.d), s>>>(a);
    SPION_LAUNCH_CHECK();
    return SPION_OK;
}

spion_status launch_fwd_simt(const AttnArgs &a, spion_dtype dt, cudaStream_t s) {
    return dt == SPION_F32 ? fwd_simt_t<float>(a, s) : fwd_simt_t<__nv_bfloat16>(a, s);
}
spion_status launch_bwd_preprocess(const AttnArgs &a, spion_dtype dt, float *D, cudaStream_t s) {
    return dt == SPION_F32 ? bwd_preprocess_t<float>(a, D, s) : bwd_preprocess_t<__nv_bfloat16>(a, D, s);
}
spion_status launch_bwd_simt(const AttnArgs &a, spion_dtype dt, cudaStream_t s) {
    return dt == SPION_F32 ? bwd_simt_t<float>(a, s) : bwd_simt_t<__nv_bfloat16>(a, s);
}

}  // namespace spion
