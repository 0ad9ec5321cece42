// Emulated-bfloat16 operator path: the reference's BF16 kernel contract
// (_kernels_numba.py:113-126, 166-211, 230-238; precision.py:65-85) on B200.
//
// Semantics restated exactly: storage is FP32; every term rounds the scaled
// matrix entry s_e * K[i,j] (an FP32 product) to bfloat16 with round-to-
// nearest-even (NaN payloads quieted, infinities kept), multiplies it by the
// (pre-quantized) FP32 input and accumulates in FP32, in j order, with no FMA
// contraction -- numba's arithmetic.  The fused kernels optionally quantize
// the gathered input themselves (the operator's _masked_input,
// operator.py:83-88, fused into the gather).
//
// This path is NOT the production path: the north star keeps BF16 only as the
// documented negative result (PAPER.md:1522-1552 -- BF16 conditioning products
// of 2.4e3-9.1e3, iterative-refinement stagnation), which bench/test code
// reproduces on B200.  It runs on CUDA cores; per-term rounding of s_e*K does
// not factor into a tensor-core GEMM (the rounded matrix differs per element).

#include <cstring>

#include "tf_common.cuh"

namespace tf {

// bf16_rne: tf_common.cuh

constexpr int BF_BLOCK = 128;

// f_i = sum_j bf16(s * K_ij) * u_j  (FP32, j order, no FMA)
__device__ __forceinline__ float bf16_row(const float* __restrict__ ke, int i, float s, const float (&u)[NLOC])
{
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < NLOC; ++j) acc = __fadd_rn(acc, __fmul_rn(bf16_rne(__fmul_rn(s, ke[i * NLOC + j])), u[j]));
    return acc;
}

template <bool ATOMIC>
__global__ void __launch_bounds__(BF_BLOCK)
k_edof_bf16(const int32_t* __restrict__ edof, const float* __restrict__ scale, const float* __restrict__ v,
            float* __restrict__ w, long long n, const int32_t* __restrict__ order, int quantize,
            const __grid_constant__ KeMat<float> ke)
{
    const long long t = (long long)blockIdx.x * BF_BLOCK + threadIdx.x;
    if (t >= n) return;
    const long long e = order ? (long long)order[t] : t;
    int idx[NLOC];
    float u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) {
        idx[q] = edof[e * NLOC + q];
        const float x = idx[q] >= 0 ? v[idx[q]] : 0.0f;
        u[q] = quantize ? bf16_rne(x) : x;
    }
    const float s = scale[e];
    for (int i = 0; i < NLOC; ++i) {
        const float acc = bf16_row(ke.a, i, s, u);
        if (idx[i] >= 0) {
            if (ATOMIC)
                atomicAdd(w + idx[i], acc);
            else
                w[idx[i]] = __fadd_rn(w[idx[i]], acc);
        }
    }
}

// FP64 evaluation of the quantized system (operator.py:143-152 apply_fp64 for
// bf16): sum_j f64(bf16(s K_ij)) * f64(bf16(x_j)) accumulated in FP64
__global__ void __launch_bounds__(BF_BLOCK)
k_edof_bf16_f64(const int32_t* __restrict__ edof, const float* __restrict__ scale, const double* __restrict__ v,
                double* __restrict__ w, long long n, const __grid_constant__ KeMat<float> ke)
{
    const long long e = (long long)blockIdx.x * BF_BLOCK + threadIdx.x;
    if (e >= n) return;
    int idx[NLOC];
    double u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) {
        idx[q] = edof[e * NLOC + q];
        u[q] = idx[q] >= 0 ? (double)bf16_rne((float)v[idx[q]]) : 0.0;
    }
    const float s = scale[e];
    for (int i = 0; i < NLOC; ++i) {
        double acc = 0.0;
        for (int j = 0; j < NLOC; ++j)
            acc = __dadd_rn(acc, __dmul_rn((double)bf16_rne(__fmul_rn(s, ke.a[i * NLOC + j])), u[j]));
        if (idx[i] >= 0) atomicAdd(w + idx[i], acc);
    }
}

__global__ void k_gemm_bf16(const float* __restrict__ u_elem, const float* __restrict__ scale,
                            float* __restrict__ f_elem, long long n, const __grid_constant__ KeMat<float> ke)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    float u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) u[q] = u_elem[e * NLOC + q];
    const float s = scale[e];
    for (int i = 0; i < NLOC; ++i) f_elem[e * NLOC + i] = bf16_row(ke.a, i, s, u);
}

// out[edof[e,l]] += bf16(s_e * ke_diag[l])  (FP32 accumulation)
__global__ void k_jacobi_bf16(const int32_t* __restrict__ edof, const float* __restrict__ scale,
                              float* __restrict__ out, long long n, const __grid_constant__ KeMat<float> kd)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n * NLOC) {
        const int d = edof[t];
        if (d >= 0) atomicAdd(out + d, bf16_rne(__fmul_rn(scale[t / NLOC], kd.a[t % NLOC])));
    }
}

__global__ void k_round_bf16(long long n, const float* __restrict__ x, float* __restrict__ y)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) y[t] = bf16_rne(x[t]);
}

}  // namespace tf

using namespace tf;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int tf_matvec_edof_bf16(const int32_t* edof, const float* ke, const float* scale, const float* v, float* w,
                        int64_t n_elem, int mode, const int32_t* color_elems, const int64_t* color_offsets,
                        int n_colors, int quantize_input, void* stream)
{
    if (n_elem <= 0) return TF_OK;
    TF_REQUIRE(edof && ke && scale && v && w, "null pointer");
    KeMat<float> k;
    memcpy(k.a, ke, sizeof(k.a));
    if (mode == TF_SCATTER_ATOMIC) {
        k_edof_bf16<true><<<(unsigned)((n_elem + BF_BLOCK - 1) / BF_BLOCK), BF_BLOCK, 0, S(stream)>>>(
            edof, scale, v, w, n_elem, nullptr, quantize_input, k);
        TF_CHECK_LAUNCH();
    } else if (mode == TF_SCATTER_COLORED) {
        TF_REQUIRE(color_elems && color_offsets && n_colors > 0, "coloured scatter needs a colouring");
        for (int c = 0; c < n_colors; ++c) {
            const long long a = color_offsets[c], b = color_offsets[c + 1];
            if (b <= a) continue;
            k_edof_bf16<false><<<(unsigned)((b - a + BF_BLOCK - 1) / BF_BLOCK), BF_BLOCK, 0, S(stream)>>>(
                edof, scale, v, w, b - a, color_elems + a, quantize_input, k);
            TF_CHECK_LAUNCH();
        }
    } else {
        set_error("unknown scatter mode %d", mode);
        return TF_ERR_ARG;
    }
    return TF_OK;
}

int tf_matvec_edof_bf16_f64(const int32_t* edof, const float* ke, const float* scale, const double* v, double* w,
                            int64_t n_elem, void* stream)
{
    if (n_elem <= 0) return TF_OK;
    TF_REQUIRE(edof && ke && scale && v && w, "null pointer");
    KeMat<float> k;
    memcpy(k.a, ke, sizeof(k.a));
    k_edof_bf16_f64<<<(unsigned)((n_elem + BF_BLOCK - 1) / BF_BLOCK), BF_BLOCK, 0, S(stream)>>>(edof, scale, v, w,
                                                                                               n_elem, k);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_gemm_bf16(const float* u_elem, const float* ke, const float* scale, float* f_elem, int64_t n_elem,
                 void* stream)
{
    if (n_elem <= 0) return TF_OK;
    KeMat<float> k;
    memcpy(k.a, ke, sizeof(k.a));
    k_gemm_bf16<<<(unsigned)((n_elem + 127) / 128), 128, 0, S(stream)>>>(u_elem, scale, f_elem, n_elem, k);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_jacobi_edof_bf16(const int32_t* edof, const float* ke_diag, const float* scale, float* out, int64_t n_elem,
                        void* stream)
{
    if (n_elem <= 0) return TF_OK;
    KeMat<float> k;
    memset(&k, 0, sizeof(k));
    memcpy(k.a, ke_diag, NLOC * sizeof(float));
    const long long n = n_elem * NLOC;
    k_jacobi_bf16<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(edof, scale, out, n_elem, k);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_round_bf16(int64_t n, const float* x, float* y, void* stream)
{
    if (n <= 0) return TF_OK;
    k_round_bf16<<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(n, x, y);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

}  // extern "C"
