// Shared definitions for the topofuse B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/topofuse_b200.h"

namespace tf {

// Thread-local last-error string surfaced through tf_last_error().
void set_error(const char* fmt, ...);

#define TF_CUDA_TRY(expr)                                                          \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::tf::set_error("%s:%d %s -> %s", __FILE__, __LINE__, #expr,           \
                            cudaGetErrorString(_e));                               \
            return TF_ERR_CUDA;                                                    \
        }                                                                          \
    } while (0)

#define TF_CHECK_LAUNCH() TF_CUDA_TRY(cudaGetLastError())

#define TF_REQUIRE(cond, ...)                                                      \
    do {                                                                           \
        if (!(cond)) {                                                             \
            ::tf::set_error(__VA_ARGS__);                                          \
            return TF_ERR_ARG;                                                     \
        }                                                                          \
    } while (0)

constexpr int NLOC = 24;

// The unit element matrix travels by value as a __grid_constant__ kernel
// parameter: it lands in constant bank 0, so fully-unrolled products read it
// as FFMA/DFMA constant operands (no LSU traffic, full-rate FMA issue).
template <typename T>
struct KeMat {
    T a[NLOC * NLOC];
};

// Structured grid: nodes (nx+1)(ny+1)(nz+1), x-fastest (reference mesh.py:58-63).
struct Grid {
    int nelx, nely, nelz;
    int nnx, nny, nnz;        // node counts per axis
    long long n_nodes;
    long long n_elem;
    int ilo, ihi;             // node x-range whose outputs a launch produces (tile kernel)
};

inline Grid make_grid(const tf_grid* g)
{
    Grid r;
    r.nelx = g->nelx; r.nely = g->nely; r.nelz = g->nelz;
    r.nnx = g->nelx + 1; r.nny = g->nely + 1; r.nnz = g->nelz + 1;
    r.n_nodes = (long long)r.nnx * r.nny * r.nnz;
    r.n_elem = (long long)g->nelx * g->nely * g->nelz;
    r.ilo = 0;
    r.ihi = r.nnx;
    return r;
}

// Reference corner order (mesh.py:19-31): bottom CCW 000,100,110,010 then top.
__host__ __device__ constexpr int corner_of(int ox, int oy, int oz)
{
    return oz * 4 + (oy ? (ox ? 2 : 3) : (ox ? 1 : 0));
}

template <typename T>
__device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }

// ---- device-resident PCG state (tf_pcg.cu, and the fused CG tile kernel) ----
enum { TERM_CONVERGED = 0, TERM_MAX_ITER = 1, TERM_BREAKDOWN = 2, TERM_DIVERGED = 3 };

// Field ownership inside one iteration: no kernel reads a field that the same
// kernel's block 0 writes.
//   unfused body (general edof): k_update reads it/rz/done, writes it_cur/
//     alpha/rz_old/refresh/matvecs (+done on breakdown); k_direction reads
//     it_cur/rz_old and commits it/rz/rel/beta/done/term.
//   fused body (structured): the CG tile kernel reads it_a/rz_old, decides the
//     previous iteration and commits rel/hist/rz/beta (or done/term/it) and
//     it_b = it_a + 1; k_update_f reads it_b/rz and writes it_a/alpha/rz_old/
//     refresh/matvecs (+done/it on breakdown).
struct CgScalars {
    double bnorm, rz, rz_old, alpha, beta, rel, tol;
    double* hist;
    int it, done, term, matvecs, refresh, max_iter, recompute, zero_rhs;
    int it_cur;
    int it_a, it_b;
    int quantize;  // round p and r to bf16 after each direction update (CgConfig.quantize_krylov)
};

__device__ __forceinline__ double cg_round(double v, bool f32) { return f32 ? (double)(float)v : v; }
__device__ __forceinline__ double cg_sqrt(double v, bool f32)
{
    return f32 ? (double)sqrtf((float)v) : sqrt(v);
}
// bit-exact round_to_bf16 / numba _bf16 (precision.py:65-85, _kernels_numba.py:68-78):
// RNE on the high 16 bits, NaN payloads quieted, infinities kept
__device__ __forceinline__ float bf16_rne(float x)
{
    const unsigned u = __float_as_uint(x);
    if ((u & 0x7F800000u) == 0x7F800000u) {
        if (u & 0x007FFFFFu) return __uint_as_float(((u >> 16) << 16) | 0x00400000u);
        return x;
    }
    const unsigned bias = 0x7FFFu + ((u >> 16) & 1u);
    return __uint_as_float(((u + bias) >> 16) << 16);
}

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// Arguments of the fused CG tile kernel (direction update folded into the
// matvec's plane staging): p_new = r*inv + beta*p_old with ping-pong p buffers.
template <typename T>
struct CgTileArgs {
    const T* r;
    const T* inv;
    T* pbuf[2];            // p of iteration k lives in pbuf[k & 1]
    const double* part;    // r.r / r.z partials of the previous update (2 per block)
    int nparts;
    CgScalars* sc;
    unsigned long long h_while;
    int in_graph;
};

// Launch plan of the SM-resident PCG (tf_pcg_resident.cu).
struct ResPlan {
    dim3 grid;
    int oz;
    int lean;
    int by;  // element-column rows per CTA
    size_t dyn_smem;
    long long nblk;
    int onex;  // single-exchange iteration (full layout only)
};

}  // namespace tf
