// General connectivity, deterministic scatter, bitwise the reference's
// fused_serial (_kernels_numba.py:146-162): every DOF receives its elements'
// row sums in ascending element order, each row summed exactly as numba
// does (FP64: (s_e*K[i][j])*u_j in j order, no FMA; FP32: float32 products,
// float64 row sum, out = f32(f64(out) + row)).
//
//   pass 1  k_edof_rows  one thread per element: the 24 row sums (FP64) into
//                        a (n_elem, 24) workspace -- coalesced edof row loads
//                        via shared memory, as the atomic kernel
//   pass 2  k_dof_pull   one thread per DOF: walks its (element, row) list in
//                        ascending element order (a CSR built once per mesh)
//                        and accumulates into w
// The CSR (DOF -> flat element-row indices, ascending) is built on the device
// with a stable CUB radix sort (tf_edof_csr_build).  Replaces the colour-
// ordered passes of the serial mode (deterministic but not the reference's
// summation order) with the reference's exact order.

#include <cub/cub.cuh>

#include <cstring>

#include "tf_common.cuh"

namespace tf {

constexpr int PULL_ROWS_BLOCK = 128;

template <typename T>
__global__ void __launch_bounds__(PULL_ROWS_BLOCK)
k_edof_rows(const int32_t* __restrict__ edof, const T* __restrict__ scale, const T* __restrict__ v,
            double* __restrict__ rows, long long n, const __grid_constant__ KeMat<T> ke)
{
    const long long e = (long long)blockIdx.x * PULL_ROWS_BLOCK + threadIdx.x;
    if (e >= n) return;
    T u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) {
        const int d = __ldg(edof + e * NLOC + q);
        u[q] = d >= 0 ? ld_nc(v + d) : T(0);
    }
    const T se = ld_nc(scale + e);
    for (int i = 0; i < NLOC; ++i) {
        double t = 0.0;
        if (sizeof(T) == 8) {
#pragma unroll
            for (int j = 0; j < NLOC; ++j)
                t = __dadd_rn(t, __dmul_rn(__dmul_rn((double)se, (double)ke.a[i * NLOC + j]), (double)u[j]));
        } else {
#pragma unroll
            for (int j = 0; j < NLOC; ++j) {
                const float kk = __fmul_rn((float)se, (float)ke.a[i * NLOC + j]);
                t = __dadd_rn(t, (double)__fmul_rn(kk, (float)u[j]));
            }
        }
        rows[e * NLOC + i] = t;
    }
}

template <typename T>
__global__ void k_dof_pull(const int64_t* __restrict__ off, const int32_t* __restrict__ ent,
                           const double* __restrict__ rows, T* __restrict__ w, long long n_dof, int accumulate)
{
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_dof) return;
    const long long a = off[d], b = off[d + 1];
    double acc64 = accumulate ? (double)w[d] : 0.0;
    float acc32 = accumulate ? (float)w[d] : 0.0f;
    // chunks of 8 (a hex-mesh node has <= 8 elements): all loads of a chunk
    // in flight before the in-order accumulation
    for (long long k0 = a; k0 < b; k0 += 8) {
        int e[8];
        double r[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) e[q] = k0 + q < b ? __ldg(ent + k0 + q) : -1;
#pragma unroll
        for (int q = 0; q < 8; ++q) r[q] = e[q] >= 0 ? __ldg(rows + e[q]) : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (e[q] < 0) break;
            if (sizeof(T) == 8)
                acc64 = __dadd_rn(acc64, r[q]);
            else
                acc32 = (float)__dadd_rn((double)acc32, r[q]);
        }
    }
    w[d] = sizeof(T) == 8 ? (T)acc64 : (T)acc32;
}

// Jacobi diagonal in the reference's order (_kernels_numba.py:217-226):
// acc[d] += f64(s_e * Ke[l][l]) over d's (element, corner-row) entries in
// ascending element order -- the product in the working dtype, the sum in
// FP64, no FMA.  One thread per DOF through the same CSR as k_dof_pull.
template <typename T>
__global__ void k_jacobi_pull(const int64_t* __restrict__ off, const int32_t* __restrict__ ent,
                              const T* __restrict__ scale, double* __restrict__ acc, long long n_dof,
                              const __grid_constant__ KeMat<T> kd)
{
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_dof) return;
    double a = acc[d];
    for (long long k = off[d]; k < off[d + 1]; ++k) {
        const int t = __ldg(ent + k);
        const int e = t / NLOC, l = t - e * NLOC;
        const T prod = sizeof(T) == 8 ? (T)__dmul_rn((double)ld_nc(scale + e), (double)kd.a[l])
                                      : (T)__fmul_rn((float)ld_nc(scale + e), (float)kd.a[l]);
        a = __dadd_rn(a, (double)prod);
    }
    acc[d] = a;
}

// three-stage scatter_serial in the reference's order (_kernels_numba.py:
// 129-132): acc[d] (FP64) += f_elem[e][i] over d's entries in ascending
// element order
template <typename T>
__global__ void k_scatter_pull(const int64_t* __restrict__ off, const int32_t* __restrict__ ent,
                               const T* __restrict__ f_elem, double* __restrict__ acc, long long n_dof)
{
    const long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_dof) return;
    double a = acc[d];
    for (long long k = off[d]; k < off[d + 1]; ++k) a = __dadd_rn(a, (double)ld_nc(f_elem + __ldg(ent + k)));
    acc[d] = a;
}

// emulated-bf16 fused_serial rows (_kernels_numba.py:166-177): FP32 row sums
// of bf16(s_e*K[i][j]) * u_j in j order without FMA, stored exactly in the
// FP64 row workspace; k_dof_pull<float> then adds them in ascending element
// order with FP32 rounding (f32(f64(a) + f64(b)) == a + b in binary32)
__global__ void __launch_bounds__(PULL_ROWS_BLOCK)
k_edof_rows_bf16(const int32_t* __restrict__ edof, const float* __restrict__ scale, const float* __restrict__ v,
                 double* __restrict__ rows, long long n, const __grid_constant__ KeMat<float> ke)
{
    const long long e = (long long)blockIdx.x * PULL_ROWS_BLOCK + threadIdx.x;
    if (e >= n) return;
    float u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) {
        const int d = __ldg(edof + e * NLOC + q);
        u[q] = d >= 0 ? ld_nc(v + d) : 0.0f;
    }
    const float se = ld_nc(scale + e);
    for (int i = 0; i < NLOC; ++i) {
        float t = 0.0f;
#pragma unroll
        for (int j = 0; j < NLOC; ++j) t = __fadd_rn(t, __fmul_rn(bf16_rne(__fmul_rn(se, ke.a[i * NLOC + j])), u[j]));
        rows[e * NLOC + i] = (double)t;
    }
}

__global__ void k_iota_flat(int32_t* __restrict__ x, long long n)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) x[t] = (int32_t)t;
}

__global__ void k_count_dofs(const int32_t* __restrict__ keys, long long n, int64_t* __restrict__ cnt)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) atomicAdd(reinterpret_cast<unsigned long long*>(cnt + keys[t] + 1), 1ull);
}

}  // namespace tf

using namespace tf;

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int tf_edof_csr_build(const int32_t* edof, int64_t n_elem, int64_t n_dof, int64_t* offsets, int32_t* entries,
                      void* stream)
{
    TF_REQUIRE(edof && offsets && entries && n_elem > 0 && n_dof > 0, "bad arguments");
    const long long n = n_elem * NLOC;
    TF_REQUIRE(n < (1LL << 31), "too many element rows for int32 CSR entries");
    cudaStream_t st = S(stream);
    int32_t *keys_out = nullptr, *vals_in = nullptr;
    void* temp = nullptr;
    size_t temp_bytes = 0, scan_bytes = 0;
    TF_CUDA_TRY(cudaMallocAsync(&keys_out, sizeof(int32_t) * n, st));
    TF_CUDA_TRY(cudaMallocAsync(&vals_in, sizeof(int32_t) * n, st));
    k_iota_flat<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(vals_in, n);
    TF_CHECK_LAUNCH();
    int end_bit = 1;
    while ((1LL << end_bit) < n_dof + 1 && end_bit < 32) ++end_bit;
    // stable LSD radix sort of (dof, flat index): ascending element order within a DOF
    TF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, edof, keys_out, vals_in, entries, (int)n, 0,
                                                end_bit, st));
    TF_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, offsets + 1, offsets + 1, (int)n_dof, st));
    TF_CUDA_TRY(cudaMallocAsync(&temp, std::max(temp_bytes, scan_bytes), st));
    TF_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, temp_bytes, edof, keys_out, vals_in, entries, (int)n, 0,
                                                end_bit, st));
    TF_CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(int64_t) * (n_dof + 1), st));
    k_count_dofs<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(keys_out, n, offsets);
    TF_CHECK_LAUNCH();
    TF_CUDA_TRY(cub::DeviceScan::InclusiveSum(temp, scan_bytes, offsets + 1, offsets + 1, (int)n_dof, st));
    TF_CUDA_TRY(cudaFreeAsync(temp, st));
    TF_CUDA_TRY(cudaFreeAsync(keys_out, st));
    TF_CUDA_TRY(cudaFreeAsync(vals_in, st));
    return TF_OK;
}

#define TF_EDOF_PULL(T, SUF)                                                                              \
    int tf_matvec_edof_pull_##SUF(const int32_t* edof, const T* ke, const T* scale, const T* v, T* w,      \
                                  int64_t n_elem, int64_t n_dof, const int64_t* offsets,                   \
                                  const int32_t* entries, double* rows, int accumulate, void* stream)      \
    {                                                                                                     \
        if (n_elem <= 0) return TF_OK;                                                                    \
        TF_REQUIRE(edof && ke && scale && v && w && offsets && entries && rows, "null pointer");         \
        KeMat<T> k;                                                                                       \
        memcpy(k.a, ke, sizeof(k.a));                                                                     \
        cudaStream_t st = S(stream);                                                                      \
        k_edof_rows<T><<<(unsigned)((n_elem + PULL_ROWS_BLOCK - 1) / PULL_ROWS_BLOCK), PULL_ROWS_BLOCK, 0, \
                         st>>>(edof, scale, v, rows, n_elem, k);                                          \
        TF_CHECK_LAUNCH();                                                                                \
        k_dof_pull<T><<<(unsigned)((n_dof + 255) / 256), 256, 0, st>>>(offsets, entries, rows, w, n_dof,  \
                                                                       accumulate);                        \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }
TF_EDOF_PULL(float, f32)
TF_EDOF_PULL(double, f64)

#define TF_JACOBI_PULL(T, SUF)                                                                            \
    int tf_jacobi_edof_pull_##SUF(const int64_t* offsets, const int32_t* entries, const T* ke_diag,      \
                                  const T* scale, double* acc, int64_t n_dof, void* stream)              \
    {                                                                                                     \
        if (n_dof <= 0) return TF_OK;                                                                     \
        TF_REQUIRE(offsets && entries && ke_diag && scale && acc, "null pointer");                        \
        KeMat<T> k;                                                                                       \
        memset(&k, 0, sizeof(k));                                                                         \
        memcpy(k.a, ke_diag, NLOC * sizeof(T));                                                           \
        k_jacobi_pull<T><<<(unsigned)((n_dof + 255) / 256), 256, 0, S(stream)>>>(offsets, entries, scale, \
                                                                                acc, n_dof, k);            \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }
TF_JACOBI_PULL(float, f32)
TF_JACOBI_PULL(double, f64)

#define TF_SCATTER_PULL(T, SUF)                                                                           \
    int tf_scatter_pull_##SUF(const int64_t* offsets, const int32_t* entries, const T* f_elem, double* acc, \
                              int64_t n_dof, void* stream)                                                \
    {                                                                                                     \
        if (n_dof <= 0) return TF_OK;                                                                     \
        TF_REQUIRE(offsets && entries && f_elem && acc, "null pointer");                                  \
        k_scatter_pull<T><<<(unsigned)((n_dof + 255) / 256), 256, 0, S(stream)>>>(offsets, entries, f_elem, \
                                                                                  acc, n_dof);             \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }
TF_SCATTER_PULL(float, f32)
TF_SCATTER_PULL(double, f64)

int tf_matvec_edof_pull_bf16(const int32_t* edof, const float* ke, const float* scale, const float* v, float* w,
                             int64_t n_elem, int64_t n_dof, const int64_t* offsets, const int32_t* entries,
                             double* rows, int accumulate, void* stream)
{
    if (n_elem <= 0) return TF_OK;
    TF_REQUIRE(edof && ke && scale && v && w && offsets && entries && rows, "null pointer");
    KeMat<float> k;
    memcpy(k.a, ke, sizeof(k.a));
    cudaStream_t st = S(stream);
    k_edof_rows_bf16<<<(unsigned)((n_elem + PULL_ROWS_BLOCK - 1) / PULL_ROWS_BLOCK), PULL_ROWS_BLOCK, 0, st>>>(
        edof, scale, v, rows, n_elem, k);
    TF_CHECK_LAUNCH();
    k_dof_pull<float><<<(unsigned)((n_dof + 255) / 256), 256, 0, st>>>(offsets, entries, rows, w, n_dof, accumulate);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

}  // extern "C"
