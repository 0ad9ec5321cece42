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
};

inline Grid make_grid(const tf_grid* g)
{
    Grid r;
    r.nelx = g->nelx; r.nely = g->nely; r.nelz = g->nelz;
    r.nnx = g->nelx + 1; r.nny = g->nely + 1; r.nnz = g->nelz + 1;
    r.n_nodes = (long long)r.nnx * r.nny * r.nnz;
    r.n_elem = (long long)g->nelx * g->nely * g->nelz;
    return r;
}

// Reference corner order (mesh.py:19-31): bottom CCW 000,100,110,010 then top.
__host__ __device__ constexpr int corner_of(int ox, int oy, int oz)
{
    return oz * 4 + (oy ? (ox ? 2 : 3) : (ox ? 1 : 0));
}

template <typename T>
__device__ __forceinline__ T ld_nc(const T* p) { return __ldg(p); }

}  // namespace tf
