// Matrix-free Q1-hex stiffness action w = sum_e B_e^T (s_e Ke) B_e v on B200.
//
// Reference semantics: _kernels_numba.py:146-196 (fused_serial/fused_atomic),
// operator.py:83-117 (input masking, fixed-DOF pass-through), and the
// three-stage pipeline _kernels_numba.py:82-140.
//
// Structured grids (edof == build_edof(mesh)) use an index-free, atomic-free
// "pull" kernel: one thread per NODE gathers its 27-node neighbourhood once
// and sums the rows of its 8 adjacent elements that belong to it.  Output is
// written exactly once (coalesced), no red/atomics, deterministic.  Element
// contributions are added in ascending element id -- the order the
// reference's element-major serial loop produces for every DOF -- so the
// TF_GRID_BITWISE variant (which also keeps numba's per-term rounding) is
// bitwise-equal to the reference fused_serial.
//
// General connectivity (any edof) uses one thread per element with the
// element matrix as constant-bank operands and red.global.add scatter
// (parallel_atomic analogue) or a colour-ordered deterministic scatter.

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tf_common.cuh"
#include "tf_walsh.cuh"

namespace tf {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

__host__ __device__ constexpr int cx(int b) { return ((b & 3) == 1 || (b & 3) == 2) ? 1 : 0; }
__host__ __device__ constexpr int cy(int b) { return (b & 3) >= 2 ? 1 : 0; }
__host__ __device__ constexpr int cz(int b) { return b >> 2; }

// ---------------------------------------------------------------------------
// block reduction of one double (blockDim.x*blockDim.y*blockDim.z <= 1024)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double* sh)
{
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthreads = blockDim.x * blockDim.y * blockDim.z;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) sh[tid >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (tid == 0) {
        for (int wi = 0; wi < (nthreads + 31) / 32; ++wi) r += sh[wi];
    }
    return r;  // valid in thread 0 only
}

// ---------------------------------------------------------------------------
// Structured pull kernel
// ---------------------------------------------------------------------------
constexpr int PULL_BX = 32, PULL_BY = 4;

template <typename T, int VAR, bool DOT>
__global__ void __launch_bounds__(PULL_BX * PULL_BY)
k_grid_pull(Grid g, const T* __restrict__ scale, const T* __restrict__ v, T* __restrict__ w,
            const uint8_t* __restrict__ node_fixed, uint32_t flags, double* __restrict__ dot_part,
            const __grid_constant__ KeMat<T> ke)
{
    const int i = blockIdx.x * PULL_BX + threadIdx.x;
    const int j = blockIdx.y * PULL_BY + threadIdx.y;
    const int k = blockIdx.z;
    const bool live = (i < g.nnx) && (j < g.nny);
    const bool mask_in = (flags & TF_MASK_INPUT) && node_fixed != nullptr;
    const long long sx = 1, sy = g.nnx, sz = (long long)g.nnx * g.nny;
    const long long node = i + sy * j + sz * k;

    // 27-node neighbourhood, 3 components each
    T u[3][3][3][3];
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                const int ii = i + dx - 1, jj = j + dy - 1, kk = k + dz - 1;
                const bool ok = live && ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny &&
                                kk >= 0 && kk < g.nnz;
                const long long nb = node + (dx - 1) * sx + (dy - 1) * sy + (dz - 1) * sz;
                const unsigned bits = (ok && mask_in) ? (unsigned)node_fixed[nb] : 0u;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    u[dz][dy][dx][c] = (ok && !((bits >> c) & 1u)) ? ld_nc(v + 3 * nb + c) : T(0);
            }

    // scales of the 8 adjacent elements (ex, ey, ez) = (i-1+ox, j-1+oy, k-1+oz)
    T s[2][2][2];
    bool ev[2][2][2];
#pragma unroll
    for (int oz = 0; oz < 2; ++oz)
#pragma unroll
        for (int oy = 0; oy < 2; ++oy)
#pragma unroll
            for (int ox = 0; ox < 2; ++ox) {
                const int ex = i - 1 + ox, ey = j - 1 + oy, ez = k - 1 + oz;
                const bool ok = live && ex >= 0 && ex < g.nelx && ey >= 0 && ey < g.nely &&
                                ez >= 0 && ez < g.nelz;
                const long long e = ex + (long long)g.nelx * (ey + (long long)g.nely * ez);
                ev[oz][oy][ox] = ok;
                s[oz][oy][ox] = ok ? ld_nc(scale + e) : T(0);
            }

    T out[3];
    if (VAR == TF_GRID_FAST) {
        T acc[3] = {T(0), T(0), T(0)};
        if (flags & TF_ACCUMULATE) {
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] = live ? w[3 * node + c] : T(0);
        }
        // elements in ascending id order: z, then y, then x
#pragma unroll
        for (int oz = 0; oz < 2; ++oz)
#pragma unroll
            for (int oy = 0; oy < 2; ++oy)
#pragma unroll
                for (int ox = 0; ox < 2; ++ox) {
                    const int a = corner_of(1 - ox, 1 - oy, 1 - oz);  // this node's corner
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int row = 3 * a + c;
                        T t = T(0);
#pragma unroll
                        for (int b = 0; b < 8; ++b)
#pragma unroll
                            for (int d = 0; d < 3; ++d)
                                t = fma(ke.a[row * NLOC + 3 * b + d],
                                        u[oz + cz(b)][oy + cy(b)][ox + cx(b)][d], t);
                        acc[c] = fma(s[oz][oy][ox], t, acc[c]);
                    }
                }
#pragma unroll
        for (int c = 0; c < 3; ++c) out[c] = acc[c];
    } else {
        // Bitwise reproduction of the reference element loop.
        if constexpr (sizeof(T) == 8) {
            double acc[3] = {0.0, 0.0, 0.0};
            if (flags & TF_ACCUMULATE) {
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[c] = live ? (double)w[3 * node + c] : 0.0;
            }
#pragma unroll
            for (int oz = 0; oz < 2; ++oz)
#pragma unroll
                for (int oy = 0; oy < 2; ++oy)
#pragma unroll
                    for (int ox = 0; ox < 2; ++ox) {
                        if (!ev[oz][oy][ox]) continue;
                        const int a = corner_of(1 - ox, 1 - oy, 1 - oz);
                        const double se = (double)s[oz][oy][ox];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const int row = 3 * a + c;
                            double t = 0.0;
#pragma unroll
                            for (int b = 0; b < 8; ++b)
#pragma unroll
                                for (int d = 0; d < 3; ++d)
                                    t = __dadd_rn(t, __dmul_rn(__dmul_rn(se, (double)ke.a[row * NLOC + 3 * b + d]),
                                                               (double)u[oz + cz(b)][oy + cy(b)][ox + cx(b)][d]));
                            acc[c] = __dadd_rn(acc[c], t);
                        }
                    }
#pragma unroll
            for (int c = 0; c < 3; ++c) out[c] = (T)acc[c];
        } else {
            // numba FP32: f32 products, f64 row sum, out = f32(f64(out) + acc)
            float acc[3] = {0.f, 0.f, 0.f};
            if (flags & TF_ACCUMULATE) {
#pragma unroll
                for (int c = 0; c < 3; ++c) acc[c] = live ? (float)w[3 * node + c] : 0.f;
            }
#pragma unroll
            for (int oz = 0; oz < 2; ++oz)
#pragma unroll
                for (int oy = 0; oy < 2; ++oy)
#pragma unroll
                    for (int ox = 0; ox < 2; ++ox) {
                        if (!ev[oz][oy][ox]) continue;
                        const int a = corner_of(1 - ox, 1 - oy, 1 - oz);
                        const float se = (float)s[oz][oy][ox];
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            const int row = 3 * a + c;
                            double t = 0.0;
#pragma unroll
                            for (int b = 0; b < 8; ++b)
#pragma unroll
                                for (int d = 0; d < 3; ++d) {
                                    const float kk = __fmul_rn(se, (float)ke.a[row * NLOC + 3 * b + d]);
                                    const float pr = __fmul_rn(kk, (float)u[oz + cz(b)][oy + cy(b)][ox + cx(b)][d]);
                                    t = __dadd_rn(t, (double)pr);
                                }
                            acc[c] = (float)__dadd_rn((double)acc[c], t);
                        }
                    }
#pragma unroll
            for (int c = 0; c < 3; ++c) out[c] = (T)acc[c];
        }
    }

    double dot = 0.0;
    if (live) {
        const unsigned bits = node_fixed ? (unsigned)node_fixed[node] : 0u;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            T val = out[c];
            if ((flags & TF_PASS_FIXED) && ((bits >> c) & 1u)) val = v[3 * node + c];
            w[3 * node + c] = val;
            if (DOT) dot += (double)v[3 * node + c] * (double)val;  // p.q on the raw p
        }
    }
    if (DOT) {
        __shared__ double sh[PULL_BX * PULL_BY / 32];
        const double tot = block_sum(dot, sh);
        if (threadIdx.x == 0 && threadIdx.y == 0)
            dot_part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = tot;
    }
}

template <typename T>
bool launch_grid_tile_supported(const T* ke_host);
template <typename T>
int launch_grid_tile(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                     const uint8_t* node_fixed, uint32_t flags, double* dot_part, cudaStream_t st);
template <typename T>
long long grid_tile_blocks(const Grid& g);

// Dispatcher for structured grids:
//   TF_GRID_FAST    -> parity-block tile kernel (falls back to the dense pull
//                      kernel when Ke lacks the block structure)
//   TF_GRID_PULL    -> dense pull kernel (Ke rows as constant operands)
//   TF_GRID_BITWISE -> dense pull kernel in the reference's op order
template <typename T>
int launch_grid_pull(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                     const uint8_t* node_fixed, uint32_t flags, int variant, double* dot_part,
                     cudaStream_t st)
{
    if (variant == TF_GRID_FAST) {
        const int rc = launch_grid_tile<T>(g, ke_host, scale, v, w, node_fixed, flags, dot_part, st);
        if (rc != TF_ERR_UNSUPPORTED) return rc;
        variant = TF_GRID_PULL;
    }
    KeMat<T> ke;
    memcpy(ke.a, ke_host, sizeof(ke.a));
    dim3 block(PULL_BX, PULL_BY, 1);
    dim3 grid((g.nnx + PULL_BX - 1) / PULL_BX, (g.nny + PULL_BY - 1) / PULL_BY, g.nnz);
    if (variant == TF_GRID_PULL) {
        if (dot_part)
            k_grid_pull<T, TF_GRID_FAST, true><<<grid, block, 0, st>>>(g, scale, v, w, node_fixed, flags, dot_part, ke);
        else
            k_grid_pull<T, TF_GRID_FAST, false><<<grid, block, 0, st>>>(g, scale, v, w, node_fixed, flags, nullptr, ke);
    } else if (variant == TF_GRID_BITWISE) {
        if (dot_part)
            k_grid_pull<T, TF_GRID_BITWISE, true><<<grid, block, 0, st>>>(g, scale, v, w, node_fixed, flags, dot_part, ke);
        else
            k_grid_pull<T, TF_GRID_BITWISE, false><<<grid, block, 0, st>>>(g, scale, v, w, node_fixed, flags, nullptr, ke);
    } else {
        set_error("unknown grid variant %d", variant);
        return TF_ERR_ARG;
    }
    TF_CHECK_LAUNCH();
    return TF_OK;
}

long long grid_pull_blocks(const Grid& g)
{
    return (long long)((g.nnx + PULL_BX - 1) / PULL_BX) * ((g.nny + PULL_BY - 1) / PULL_BY) * g.nnz;
}

// number of CTAs (= dot partials) the dispatcher launches for this variant
template <typename T>
long long grid_matvec_blocks(const Grid& g, const T* ke_host, int variant)
{
    if (variant == TF_GRID_FAST) {
        if (launch_grid_tile_supported<T>(ke_host)) return grid_tile_blocks<T>(g);
    }
    return grid_pull_blocks(g);
}
template long long grid_matvec_blocks<float>(const Grid&, const float*, int);
template long long grid_matvec_blocks<double>(const Grid&, const double*, int);


template int launch_grid_pull<float>(const Grid&, const float*, const float*, const float*, float*,
                                     const uint8_t*, uint32_t, int, double*, cudaStream_t);
template int launch_grid_pull<double>(const Grid&, const double*, const double*, const double*,
                                      double*, const uint8_t*, uint32_t, int, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// General edof kernels
// ---------------------------------------------------------------------------
constexpr int EDOF_BLOCK = 128;

__device__ __forceinline__ void load_edof_row(const int32_t* __restrict__ edof, long long e, int idx[NLOC])
{
    const int4* r4 = reinterpret_cast<const int4*>(edof + e * NLOC);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int4 t = __ldg(r4 + q);
        idx[4 * q + 0] = t.x; idx[4 * q + 1] = t.y; idx[4 * q + 2] = t.z; idx[4 * q + 3] = t.w;
    }
}

template <typename T, bool ATOMIC>
__global__ void __launch_bounds__(EDOF_BLOCK)
k_edof_fused(const int32_t* __restrict__ edof, const T* __restrict__ scale, const T* __restrict__ v,
             T* __restrict__ w, long long n, const int32_t* __restrict__ order,
             const __grid_constant__ KeMat<T> ke)
{
    const long long t = (long long)blockIdx.x * EDOF_BLOCK + threadIdx.x;
    if (t >= n) return;
    const long long e = order ? (long long)order[t] : t;
    int idx[NLOC];
    load_edof_row(edof, e, idx);
    T u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) u[q] = idx[q] >= 0 ? ld_nc(v + idx[q]) : T(0);
    const T se = ld_nc(scale + e);
#pragma unroll
    for (int r = 0; r < NLOC; ++r) {
        T acc = T(0);
#pragma unroll
        for (int q = 0; q < NLOC; ++q) acc = fma(ke.a[r * NLOC + q], u[q], acc);
        const T val = se * acc;
        if (idx[r] >= 0) {
            if (ATOMIC)
                atomicAdd(w + idx[r], val);
            else
                w[idx[r]] += val;
        }
    }
}

// General connectivity, red.global scatter, v2: the CTA's 128 edof rows
// (12 KB, contiguous) are staged with coalesced 16-byte cp.async instead of
// six strided 16-byte loads per thread (the v1 kernel's L1 was the bottleneck:
// 79 % L1/TEX throughput at c5, ncu profiles/edof_atomic_c5.json), and
// contributions to a DOF shared with the next lane's element (the +x
// neighbour in the reference element order, corner pairs (1,0) (2,3) (5,4)
// (6,7)) are summed in registers first -- checked per DOF at run time, so any
// connectivity stays correct -- halving the reductions for structured order.
__device__ __forceinline__ void cp_async_16(void* smem, const void* gmem, bool valid)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(n));
}

#ifndef TF_EDOF_MINB
#define TF_EDOF_MINB 6
#endif
template <typename T, bool WALSH>
__global__ void __launch_bounds__(EDOF_BLOCK, TF_EDOF_MINB)
k_edof_staged(const int32_t* __restrict__ edof, const T* __restrict__ scale, const T* __restrict__ v,
              T* __restrict__ w, long long n, const __grid_constant__ KeMat<T> ke,
              const __grid_constant__ KhatBlocks<T> kb)
{
    __shared__ __align__(16) int4 rows[EDOF_BLOCK * 6];
    const long long e0 = (long long)blockIdx.x * EDOF_BLOCK;
    const int tid = threadIdx.x;
    const long long n_here = min((long long)EDOF_BLOCK, n - e0);
    const int4* src = reinterpret_cast<const int4*>(edof + e0 * NLOC);
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int k = tid + q * EDOF_BLOCK;
        cp_async_16(&rows[k], src + k, k < n_here * 6);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const long long e = e0 + tid;
    const bool live = tid < n_here;
    const T se = live ? ld_nc(scale + e) : T(0);
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    int idx[NLOC];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int4 t = rows[tid * 6 + q];
        idx[4 * q + 0] = live ? t.x : -1;
        idx[4 * q + 1] = live ? t.y : -1;
        idx[4 * q + 2] = live ? t.z : -1;
        idx[4 * q + 3] = live ? t.w : -1;
    }
    T u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) u[q] = idx[q] >= 0 ? ld_nc(v + idx[q]) : T(0);
    const int lane = tid & 31;
    constexpr int RIGHT[4] = {1, 2, 5, 6}, LEFT[4] = {0, 3, 4, 7};  // corner_of(1,oy,oz) / corner_of(0,oy,oz)
    // element rows: parity-block (corner-Walsh) algebra when Ke has the
    // structure (~200 FP instructions, all 24 rows at once), else dense rows
    // computed on demand (576 FMA, two rows live)
    T fw[NLOC];
    if (WALSH) element_apply(u, se, kb, fw);
    auto row = [&](int r) -> T {
        if (WALSH) return fw[r];
        T acc = T(0);
#pragma unroll
        for (int q = 0; q < NLOC; ++q) acc = fma(ke.a[r * NLOC + q], u[q], acc);
        return se * acc;
    };
    // rows in (right, left) corner pairs: only two live at a time
#pragma unroll
    for (int pr = 0; pr < 4; ++pr)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int jr = 3 * RIGHT[pr] + c, jl = 3 * LEFT[pr] + c;
            T fr = row(jr);
            const T fl = row(jl);
            const int nb_idx = __shfl_down_sync(0xffffffffu, idx[jl], 1);
            const T nb_val = __shfl_down_sync(0xffffffffu, fl, 1);
            const bool merge = lane < 31 && idx[jr] >= 0 && nb_idx == idx[jr];
            if (merge) fr += nb_val;
            const bool prev = __shfl_up_sync(0xffffffffu, merge, 1) && lane > 0;
            if (idx[jr] >= 0) atomicAdd(w + idx[jr], fr);
            if (idx[jl] >= 0 && !prev) atomicAdd(w + idx[jl], fl);
        }
}

// General connectivity, red.global scatter, v3 (production): v2's staging
// with the instruction count cut where ncu put it (v2: 762 thread-
// instructions per element at c5, 112 ISETP + 80 branch instructions + 36
// SHFL + 51 constant reloads; profiles/edof_atomic_c5_r2.json):
//   * which (right corner of element e, left corner of element e+1) DOF pairs
//     coincide is a property of the connectivity, not of the product: it is
//     computed once per mesh into a 16-bit mask per element
//     (tf_edof_merge_mask) instead of two shuffles and a compare per pair on
//     every product -- one shuffle per pair remains (the neighbour's value);
//   * masked slots carry their DOF with the sign bit set (operator.py's
//     device copy, _device.masked_edof): the gather is a predicated load
//     (reads 0), and the slot's row is added to that constrained DOF with an
//     unconditional red.global -- the operator's pass-through overwrites it
//     (operator.py:115) -- so only the neighbour-merged slots need a guard
//     (ptxas turns every predicated RED into a branch).
__device__ __forceinline__ void red_add_if(bool p, float* a, float v)
{
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.global.add.f32 [%0], %1;\n}\n" ::"l"(a),
                 "f"(v), "r"((unsigned)p)
                 : "memory");
}
__device__ __forceinline__ void red_add_if(bool p, double* a, double v)
{
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q red.global.add.f64 [%0], %1;\n}\n" ::"l"(a),
                 "d"(v), "r"((unsigned)p)
                 : "memory");
}
// base + i for a 32-bit unsigned element index: one IMAD.WIDE.U32 (ptxas
// otherwise splits the 64-bit offset into shifts and carries)
template <typename T>
__device__ __forceinline__ T* at_u32(T* base, unsigned i)
{
    T* a;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(a) : "r"(i), "n"((int)sizeof(T)), "l"(base));
    return a;
}
__device__ __forceinline__ void red_add(float* a, float v)
{
    asm volatile("red.global.add.f32 [%0], %1;\n" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add(double* a, double v)
{
    asm volatile("red.global.add.f64 [%0], %1;\n" ::"l"(a), "d"(v) : "memory");
}
__device__ __forceinline__ float ld_if(int idx, const float* base)
{
    float u = 0.f;
    asm volatile("{\n .reg .pred q;\n setp.ge.s32 q, %1, 0;\n @q ld.global.nc.f32 %0, [%2];\n}\n"
                 : "+f"(u)
                 : "r"(idx), "l"(base + idx));
    return u;
}
__device__ __forceinline__ double ld_if(int idx, const double* base)
{
    double u = 0.0;
    asm volatile("{\n .reg .pred q;\n setp.ge.s32 q, %1, 0;\n @q ld.global.nc.f64 %0, [%2];\n}\n"
                 : "+d"(u)
                 : "r"(idx), "l"(base + idx));
    return u;
}

// Corner pairs (right corner of element e, left corner of element e+1) in the
// reference corner order, RIGHT = corner_of(1,oy,oz), LEFT = corner_of(0,oy,oz).
// bit 3*pr + c of mask[e]: DOF 3 RIGHT[pr] + c of element e is DOF
// 3 LEFT[pr] + c of element e+1 and both sit in one warp (e % 32 != 31)
// Also validates the slots: every entry must name a DOF < n_dof in its low
// 31 bits (masked slots: sign bit set), since the merged product adds a
// masked slot's row to that DOF; a violation sets *bad.
__global__ void k_edof_merge_mask(const int32_t* __restrict__ edof, long long n, long long n_dof,
                                  uint16_t* __restrict__ mask, int* __restrict__ bad)
{
    constexpr int RIGHT[4] = {1, 2, 5, 6}, LEFT[4] = {0, 3, 4, 7};
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    bool ok = true;
#pragma unroll
    for (int j = 0; j < NLOC; ++j) ok &= (long long)((unsigned)edof[e * NLOC + j] & 0x7fffffffu) < n_dof;
    if (!ok) atomicOr(bad, 1);
    unsigned m = 0u;
    if ((e & 31) != 31 && e + 1 < n) {
        const int32_t* a = edof + e * NLOC;
        const int32_t* b = a + NLOC;
#pragma unroll
        for (int pr = 0; pr < 4; ++pr)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int d = a[3 * RIGHT[pr] + c];
                if (d >= 0 && b[3 * LEFT[pr] + c] == d) m |= 1u << (3 * pr + c);
            }
    }
    mask[e] = (uint16_t)m;
}

// L2 eviction-priority hints for the streams read once per product (the
// connectivity rows, element scales and merge masks: evict_first), so the
// 472 MB edof stream at c5 displaces them rather than the gathered v and the
// reduced w (both normal priority: an L2 flush still evicts them)
__device__ __forceinline__ unsigned long long l2_evict_first()
{
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void cp_async_16_ef(void* smem, const void* gmem, bool valid, unsigned long long pol)
{
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;\n" ::"r"(sa), "l"(gmem), "r"(n),
                 "l"(pol));
}
__device__ __forceinline__ float ld_ef(const float* p, unsigned long long pol)
{
    float r;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_ef(const double* p, unsigned long long pol)
{
    double r;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ unsigned ld_ef(const uint16_t* p, unsigned long long pol)
{
    unsigned short r;
    asm volatile("ld.global.nc.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
    return r;
}
static bool edof_hint_enabled()
{
    static const bool on = [] {
        const char* e = getenv("TF_EDOF_HINT");
        return !(e && e[0] == '0');
    }();
    return on;
}

#ifndef TF_EDOFM_MINB32
#define TF_EDOFM_MINB32 8  // 64 registers, no spills: 32 warps/SM (c5 187 vs 197 us at 6)
#endif
template <typename T, bool ISO, bool HINT>
__global__ void __launch_bounds__(EDOF_BLOCK, sizeof(T) == 4 ? TF_EDOFM_MINB32 : TF_EDOF_MINB)
k_edof_merged(const int32_t* __restrict__ edof, const uint16_t* __restrict__ merge, const T* __restrict__ scale,
              const T* __restrict__ v, T* __restrict__ w, long long n, const __grid_constant__ KhatBlocks<T> kb,
              const __grid_constant__ KhatIso<T> ki)
{
    constexpr int RIGHT[4] = {1, 2, 5, 6}, LEFT[4] = {0, 3, 4, 7};
    __shared__ __align__(16) int4 rows[EDOF_BLOCK * 6];
    const long long e0 = (long long)blockIdx.x * EDOF_BLOCK;
    const int tid = threadIdx.x, lane = tid & 31;
    const long long n_here = min((long long)EDOF_BLOCK, n - e0);
    const int4* src = reinterpret_cast<const int4*>(edof + e0 * NLOC);
    const unsigned long long pol = HINT ? l2_evict_first() : 0ull;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int k = tid + q * EDOF_BLOCK;
        if (HINT)
            cp_async_16_ef(&rows[k], src + k, k < n_here * 6, pol);
        else
            cp_async_16(&rows[k], src + k, k < n_here * 6);
    }
    asm volatile("cp.async.commit_group;\n" ::);
    const long long e = e0 + tid;
    const bool live = tid < n_here;
    T se = T(0);
    unsigned mk = 0u;
    if (live) {
        se = HINT ? ld_ef(scale + e, pol) : ld_nc(scale + e);
        mk = HINT ? ld_ef(merge + e, pol) : (unsigned)ld_nc(merge + e);
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    int idx[NLOC];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
        const int4 t = rows[tid * 6 + q];
        idx[4 * q + 0] = t.x;
        idx[4 * q + 1] = t.y;
        idx[4 * q + 2] = t.z;
        idx[4 * q + 3] = t.w;
    }
    T u[NLOC];  // (lanes past the last element gather zero-filled rows: v[0])
#pragma unroll
    for (int q = 0; q < NLOC; ++q) u[q] = ld_if(idx[q], v);
    T fw[NLOC];
    if (ISO)
        element_apply_iso(u, se, ki, fw);
    else
        element_apply(u, se, kb, fw);
    const unsigned prev = __shfl_up_sync(0xffffffffu, mk, 1) * (lane > 0);
#pragma unroll
    for (int pr = 0; pr < 4; ++pr)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int b = 3 * pr + c, jr = 3 * RIGHT[pr] + c, jl = 3 * LEFT[pr] + c;
            const T nb = __shfl_down_sync(0xffffffffu, fw[jl], 1);
            if ((mk >> b) & 1u) fw[jr] += nb;
        }
    if (!live) return;
#pragma unroll
    for (int pr = 0; pr < 4; ++pr)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int b = 3 * pr + c, jr = 3 * RIGHT[pr] + c, jl = 3 * LEFT[pr] + c;
            red_add(at_u32(w, (unsigned)idx[jr] & 0x7fffffffu), fw[jr]);
            if (!((prev >> b) & 1u)) red_add(at_u32(w, (unsigned)idx[jl] & 0x7fffffffu), fw[jl]);
        }
}

// TF_EDOF_V1=1: the v1 atomic kernel (strided row loads, no aggregation)
static bool edof_v1_forced()
{
    const char* e = getenv("TF_EDOF_V1");
    return e && e[0] == '1';
}

template <typename T>
int launch_edof(const int32_t* edof, const T* ke_host, const T* scale, const T* v, T* w,
                long long n_elem, int mode, const int32_t* color_elems,
                const int64_t* color_offsets, int n_colors, cudaStream_t st)
{
    KeMat<T> ke;
    memcpy(ke.a, ke_host, sizeof(ke.a));
    TF_REQUIRE(((uintptr_t)edof & 15u) == 0, "edof must be 16-byte aligned");
    if (n_elem == 0) return TF_OK;
    if (mode == TF_SCATTER_ATOMIC) {
        const long long nb = (n_elem + EDOF_BLOCK - 1) / EDOF_BLOCK;
        KhatBlocks<T> kb;
        const char* ed = getenv("TF_EDOF_DENSE");
        const bool walsh = !(ed && ed[0] == '1') && khat_blocks_cached<T>(ke_host, &kb);
        if (edof_v1_forced())
            k_edof_fused<T, true><<<(unsigned)nb, EDOF_BLOCK, 0, st>>>(edof, scale, v, w, n_elem, nullptr, ke);
        else if (walsh)
            k_edof_staged<T, true><<<(unsigned)nb, EDOF_BLOCK, 0, st>>>(edof, scale, v, w, n_elem, ke, kb);
        else
            k_edof_staged<T, false><<<(unsigned)nb, EDOF_BLOCK, 0, st>>>(edof, scale, v, w, n_elem, ke, kb);
        TF_CHECK_LAUNCH();
    } else if (mode == TF_SCATTER_COLORED) {
        TF_REQUIRE(color_elems && color_offsets && n_colors > 0, "coloured scatter needs a colouring");
        for (int c = 0; c < n_colors; ++c) {
            const long long a = color_offsets[c], b = color_offsets[c + 1];
            if (b <= a) continue;
            const long long nb = (b - a + EDOF_BLOCK - 1) / EDOF_BLOCK;
            k_edof_fused<T, false><<<(unsigned)nb, EDOF_BLOCK, 0, st>>>(edof, scale, v, w, b - a,
                                                                      color_elems + a, ke);
            TF_CHECK_LAUNCH();
        }
    } else {
        set_error("unknown scatter mode %d", mode);
        return TF_ERR_ARG;
    }
    return TF_OK;
}

// pass-through of constrained DOFs
template <typename T>
__global__ void k_pass_fixed(const int64_t* __restrict__ fixed, long long n, const T* __restrict__ v,
                             T* __restrict__ w)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) {
        const long long d = fixed[t];
        w[d] = v[d];
    }
}

template <typename T>
int launch_pass_fixed(const int64_t* fixed, long long n, const T* v, T* w, cudaStream_t st)
{
    if (n <= 0) return TF_OK;
    k_pass_fixed<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(fixed, n, v, w);
    TF_CHECK_LAUNCH();
    return TF_OK;
}
template int launch_pass_fixed<float>(const int64_t*, long long, const float*, float*, cudaStream_t);
template int launch_pass_fixed<double>(const int64_t*, long long, const double*, double*, cudaStream_t);

// ---------------------------------------------------------------------------
// three-stage pipeline stages
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_gather(const int32_t* __restrict__ edof, const T* __restrict__ v,
                         T* __restrict__ u_elem, long long n)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // one entry per thread
    if (t < n * NLOC) {
        const int d = edof[t];
        u_elem[t] = d >= 0 ? v[d] : T(0);
    }
}

template <typename T>
__global__ void __launch_bounds__(EDOF_BLOCK)
k_gemm(const T* __restrict__ u_elem, const T* __restrict__ scale, T* __restrict__ f_elem, long long n,
       const __grid_constant__ KeMat<T> ke)
{
    const long long e = (long long)blockIdx.x * EDOF_BLOCK + threadIdx.x;
    if (e >= n) return;
    T u[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) u[q] = u_elem[e * NLOC + q];
    const T se = scale[e];
#pragma unroll
    for (int r = 0; r < NLOC; ++r) {
        T acc = T(0);
#pragma unroll
        for (int q = 0; q < NLOC; ++q) acc = fma(ke.a[r * NLOC + q], u[q], acc);
        f_elem[e * NLOC + r] = se * acc;
    }
}

template <typename T>
__global__ void k_scatter(const int32_t* __restrict__ edof, const T* __restrict__ f_elem,
                          double* __restrict__ acc, long long n)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n * NLOC) {
        const int d = edof[t];
        if (d >= 0) atomicAdd(acc + d, (double)f_elem[t]);
    }
}

// ---------------------------------------------------------------------------
// Jacobi diagonal and element energies
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_jacobi_grid(Grid g, const T* __restrict__ scale, T* __restrict__ diag,
                              T* __restrict__ inv_diag, const uint8_t* __restrict__ node_fixed,
                              const __grid_constant__ KeMat<T> kd /* first 24 = ke_diag */,
                              double* __restrict__ partial = nullptr)
{
    const long long node = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.n_nodes) return;
    const int i = (int)(node % g.nnx);
    const int j = (int)((node / g.nnx) % g.nny);
    const int k = (int)(node / ((long long)g.nnx * g.nny));
    double acc[3] = {0.0, 0.0, 0.0};
    // ascending element order, products in the working dtype, sum in FP64
#pragma unroll
    for (int oz = 0; oz < 2; ++oz)
#pragma unroll
        for (int oy = 0; oy < 2; ++oy)
#pragma unroll
            for (int ox = 0; ox < 2; ++ox) {
                const int ex = i - 1 + ox, ey = j - 1 + oy, ez = k - 1 + oz;
                if (ex < 0 || ex >= g.nelx || ey < 0 || ey >= g.nely || ez < 0 || ez >= g.nelz) continue;
                const T se = scale[ex + (long long)g.nelx * (ey + (long long)g.nely * ez)];
                const int a = corner_of(1 - ox, 1 - oy, 1 - oz);
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const T prod = se * kd.a[3 * a + c];
                    acc[c] = __dadd_rn(acc[c], (double)prod);
                }
            }
    if (partial) {  // slab partial sums: FP64, no cast, no constraint handling
#pragma unroll
        for (int c = 0; c < 3; ++c) partial[3 * node + c] = acc[c];
        return;
    }
    const unsigned bits = node_fixed ? (unsigned)node_fixed[node] : 0u;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        T d = (T)acc[c];
        if ((bits >> c) & 1u) d = T(1);
        diag[3 * node + c] = d;
        if (inv_diag) inv_diag[3 * node + c] = T(1) / d;
    }
}

template <typename T>
__global__ void k_jacobi_edof(const int32_t* __restrict__ edof, const T* __restrict__ scale,
                              double* __restrict__ acc, long long n,
                              const __grid_constant__ KeMat<T> kd)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n * NLOC) {
        const int d = edof[t];
        const int l = (int)(t % NLOC);
        if (d >= 0) {
            const T prod = scale[t / NLOC] * kd.a[l];
            atomicAdd(acc + d, (double)prod);
        }
    }
}

// energies: total = sum_i u_i * (sum_j K_ij u_j)   (_kernels_numba.py:241-250)
__device__ __forceinline__ double energy_of(const double u[NLOC], const KeMat<double>& ke)
{
    double total = 0.0;
#pragma unroll
    for (int r = 0; r < NLOC; ++r) {
        double row = 0.0;
#pragma unroll
        for (int q = 0; q < NLOC; ++q) row = fma(ke.a[r * NLOC + q], u[q], row);
        total = fma(u[r], row, total);
    }
    return total;
}

// The same quadratic form in the parity basis, u^T Ke u = sum_{c,m} h_cm (Khat h)_cm
// with h = W u (tf_walsh.cuh): the translation modes drop out before any
// product, so the rounding error scales with the element's deformation, not
// with its displacement.  The direct form loses eps*|Ke|*|u|^2 -- for a void
// region carried along rigidly with |u| ~ 1e8 that is an energy of -5 where
// the true value is ~0 (the reference shows exactly this on a cantilever with
// a 4-step schedule), which can flip a compliance sensitivity positive.
__device__ __forceinline__ double energy_walsh(const double (&u)[NLOC], const KhatBlocks<double>& kb)
{
    double h[3][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) h[c][bin_of(a)] = u[3 * a + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht_fwd(h[c]);
    double total = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int m = q ^ (1 << c);
            if (m == 0) continue;
            double acc = 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int n = q ^ (1 << d);
                if (n == 0) continue;
                acc = fma(kb.b[q][c][d], h[d][n], acc);
            }
            total = fma(h[c][m], acc, total);
        }
    return total;
}

struct EnergyKe {
    KeMat<double> ke;
    KhatBlocks<double> kb;
    int walsh;
};

__global__ void __launch_bounds__(EDOF_BLOCK)
k_energies_grid(Grid g, const double* __restrict__ u, double* __restrict__ out,
                const __grid_constant__ EnergyKe K)
{
    const long long e = (long long)blockIdx.x * EDOF_BLOCK + threadIdx.x;
    if (e >= g.n_elem) return;
    const int ex = (int)(e % g.nelx);
    const int ey = (int)((e / g.nelx) % g.nely);
    const int ez = (int)(e / ((long long)g.nelx * g.nely));
    double ue[NLOC];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const long long node = (ex + cx(b)) + (long long)g.nnx * ((ey + cy(b)) + (long long)g.nny * (ez + cz(b)));
#pragma unroll
        for (int d = 0; d < 3; ++d) ue[3 * b + d] = u[3 * node + d];
    }
    out[e] = K.walsh ? energy_walsh(ue, K.kb) : energy_of(ue, K.ke);
}

__global__ void __launch_bounds__(EDOF_BLOCK)
k_energies_edof(const int32_t* __restrict__ edof, const double* __restrict__ u,
                double* __restrict__ out, long long n, const __grid_constant__ EnergyKe K)
{
    const long long e = (long long)blockIdx.x * EDOF_BLOCK + threadIdx.x;
    if (e >= n) return;
    int idx[NLOC];
    load_edof_row(edof, e, idx);
    double ue[NLOC];
#pragma unroll
    for (int q = 0; q < NLOC; ++q) ue[q] = idx[q] >= 0 ? u[idx[q]] : 0.0;
    out[e] = K.walsh ? energy_walsh(ue, K.kb) : energy_of(ue, K.ke);
}

__global__ void k_mark_fixed(Grid g, const int64_t* __restrict__ fixed, long long n,
                             uint8_t* __restrict__ out)
{
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long d = fixed[t];
    const long long node = d / 3;
    const unsigned bit = 1u << (unsigned)(d % 3);
    const long long col = node % ((long long)g.nnx * g.nny);
    // byte-granular OR through the containing 32-bit word (no byte atomics)
    auto or_byte = [](uint8_t* base, long long i, unsigned b) {
        unsigned int* word = reinterpret_cast<unsigned int*>(reinterpret_cast<uintptr_t>(base + i) & ~uintptr_t(3));
        const unsigned sh = 8u * (unsigned)(reinterpret_cast<uintptr_t>(base + i) & 3u);
        atomicOr(word, b << sh);
    };
    or_byte(out, node, bit);
    or_byte(out + g.n_nodes, col, bit);
}

// column AND over z of the node bytes (third section of the layout)
__global__ void k_col_and(Grid g, uint8_t* __restrict__ out)
{
    const long long col = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long pn = (long long)g.nnx * g.nny;
    if (col >= pn) return;
    unsigned a = 7u;
    for (int k = 0; k < g.nnz && a; ++k) a &= out[col + k * pn];
    out[g.n_nodes + pn + col] = (uint8_t)a;
}

}  // namespace tf

// ===========================================================================
// C ABI
// ===========================================================================
using namespace tf;

static inline cudaStream_t S(void* p) { return reinterpret_cast<cudaStream_t>(p); }

// isotropic element blocks in the merged atomic product (TF_TILE_GENERIC=1:
// the generic blocks, as everywhere)
static bool tile_iso_general()
{
    const char* e = getenv("TF_TILE_GENERIC");
    return !(e && e[0] == '1');
}

extern "C" {

const char* tf_last_error(void) { return tf::g_err; }
int tf_version(void) { return 1; }

int tf_build_node_fixed(const tf_grid* g, const int64_t* fixed_dofs, int64_t n_fixed,
                        uint8_t* out, void* stream)
{
    TF_REQUIRE(g && out, "null argument");
    Grid gg = make_grid(g);
    const long long bytes = gg.n_nodes + 2LL * gg.nnx * gg.nny;
    TF_REQUIRE(((uintptr_t)out & 3u) == 0, "node_fixed buffer must be 4-byte aligned");
    // pad the tail word so the OR trick never touches foreign memory: caller
    // allocates bytes rounded up to a multiple of 4 (tf_node_fixed_bytes)
    TF_CUDA_TRY(cudaMemsetAsync(out, 0, (bytes + 3) & ~3LL, S(stream)));
    if (n_fixed > 0) {
        k_mark_fixed<<<(unsigned)((n_fixed + 255) / 256), 256, 0, S(stream)>>>(gg, fixed_dofs, n_fixed, out);
        TF_CHECK_LAUNCH();
    }
    const long long pn = (long long)gg.nnx * gg.nny;
    k_col_and<<<(unsigned)((pn + 255) / 256), 256, 0, S(stream)>>>(gg, out);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_device_count(void)
{
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

#define TF_GRID_CHECK(g)                                                                  \
    TF_REQUIRE((g) && (g)->nelx > 0 && (g)->nely > 0 && (g)->nelz > 0, "invalid grid")

int tf_matvec_grid_f32(const tf_grid* g, const float* ke, const float* scale, const float* v,
                       float* w, const uint8_t* node_fixed, uint32_t flags, int variant,
                       void* stream)
{
    TF_GRID_CHECK(g);
    TF_REQUIRE(ke && scale && v && w, "null pointer");
    return launch_grid_pull<float>(make_grid(g), ke, scale, v, w, node_fixed, flags, variant,
                                   nullptr, S(stream));
}

int tf_matvec_grid_f64(const tf_grid* g, const double* ke, const double* scale,
                       const double* v, double* w, const uint8_t* node_fixed, uint32_t flags,
                       int variant, void* stream)
{
    TF_GRID_CHECK(g);
    TF_REQUIRE(ke && scale && v && w, "null pointer");
    return launch_grid_pull<double>(make_grid(g), ke, scale, v, w, node_fixed, flags, variant,
                                    nullptr, S(stream));
}

#define TF_MATVEC_RANGE(T, SUF)                                                                   \
    int tf_matvec_grid_range_##SUF(const tf_grid* g, const T* ke, const T* scale, const T* v, T* w, \
                                   const uint8_t* node_fixed, uint32_t flags, int32_t i_lo,      \
                                   int32_t i_hi, void* stream)                                  \
    {                                                                                             \
        TF_GRID_CHECK(g);                                                                         \
        TF_REQUIRE(ke && scale && v && w, "null pointer");                                        \
        Grid gg = make_grid(g);                                                                   \
        TF_REQUIRE(0 <= i_lo && i_lo <= i_hi && i_hi <= gg.nnx, "bad node x-range");              \
        if (i_lo == i_hi) return TF_OK;                                                           \
        gg.ilo = i_lo;                                                                            \
        gg.ihi = i_hi;                                                                            \
        const int rc = launch_grid_tile<T>(gg, ke, scale, v, w, node_fixed, flags, nullptr, S(stream)); \
        if (rc == TF_ERR_UNSUPPORTED) set_error("node ranges need the parity-block tile kernel"); \
        return rc;                                                                                \
    }
TF_MATVEC_RANGE(float, f32)
TF_MATVEC_RANGE(double, f64)

int tf_edof_merge_mask(const int32_t* edof, int64_t n_elem, int64_t n_dof, uint16_t* mask, void* stream)
{
    TF_REQUIRE(edof && mask && n_elem >= 0 && n_dof > 0, "bad arguments");
    if (n_elem == 0) return TF_OK;
    int* bad = nullptr;
    TF_CUDA_TRY(cudaMallocAsync((void**)&bad, sizeof(int), S(stream)));
    TF_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), S(stream)));
    k_edof_merge_mask<<<(unsigned)((n_elem + 255) / 256), 256, 0, S(stream)>>>(edof, n_elem, n_dof, mask, bad);
    TF_CHECK_LAUNCH();
    int h = 0;
    TF_CUDA_TRY(cudaMemcpyAsync(&h, bad, sizeof(int), cudaMemcpyDeviceToHost, S(stream)));
    TF_CUDA_TRY(cudaFreeAsync(bad, S(stream)));
    TF_CUDA_TRY(cudaStreamSynchronize(S(stream)));  // once per connectivity
    TF_REQUIRE(h == 0, "edof slots must name a DOF < n_dof in their low 31 bits (masked slots: DOF | 2^31)");
    return TF_OK;
}

#define TF_MATVEC_MERGED(T, SUF)                                                                           \
    int tf_matvec_edof_merged_##SUF(const int32_t* edof, const uint16_t* merge, const T* ke, const T* scale, \
                                    const T* v, T* w, int64_t n_elem, void* stream)                         \
    {                                                                                                      \
        TF_REQUIRE(edof && merge && ke && scale && v && w && n_elem >= 0, "bad arguments");                 \
        TF_REQUIRE(((uintptr_t)edof & 15u) == 0, "edof must be 16-byte aligned");                          \
        if (n_elem == 0) return TF_OK;                                                                     \
        KhatBlocks<T> kb;                                                                                  \
        if (!khat_blocks_cached<T>(ke, &kb)) /* no parity structure: the dense-row kernel */              \
            return launch_edof<T>(edof, ke, scale, v, w, n_elem, TF_SCATTER_ATOMIC, nullptr, nullptr, 0,   \
                                  S(stream));                                                              \
        const long long nb = (n_elem + EDOF_BLOCK - 1) / EDOF_BLOCK;                                       \
        KhatIso<T> ki{};                                                                                   \
        const bool iso = tile_iso_general() && khat_iso<T>(ke, &ki);                                       \
        const bool hint = edof_hint_enabled();                                                             \
        const dim3 gb((unsigned)nb), bb(EDOF_BLOCK);                                                       \
        if (iso && hint)                                                                                   \
            k_edof_merged<T, true, true><<<gb, bb, 0, S(stream)>>>(edof, merge, scale, v, w, n_elem, kb, ki);  \
        else if (iso)                                                                                      \
            k_edof_merged<T, true, false><<<gb, bb, 0, S(stream)>>>(edof, merge, scale, v, w, n_elem, kb, ki); \
        else if (hint)                                                                                     \
            k_edof_merged<T, false, true><<<gb, bb, 0, S(stream)>>>(edof, merge, scale, v, w, n_elem, kb, ki); \
        else                                                                                               \
            k_edof_merged<T, false, false><<<gb, bb, 0, S(stream)>>>(edof, merge, scale, v, w, n_elem, kb, ki); \
        TF_CHECK_LAUNCH();                                                                                 \
        return TF_OK;                                                                                      \
    }
TF_MATVEC_MERGED(float, f32)
TF_MATVEC_MERGED(double, f64)

int tf_matvec_edof_f32(const int32_t* edof, const float* ke, const float* scale, const float* v,
                       float* w, int64_t n_elem, int mode, const int32_t* color_elems,
                       const int64_t* color_offsets, int n_colors, void* stream)
{
    TF_REQUIRE(n_elem >= 0 && ke, "bad arguments");
    return launch_edof<float>(edof, ke, scale, v, w, n_elem, mode, color_elems, color_offsets,
                              n_colors, S(stream));
}

int tf_matvec_edof_f64(const int32_t* edof, const double* ke, const double* scale,
                       const double* v, double* w, int64_t n_elem, int mode,
                       const int32_t* color_elems, const int64_t* color_offsets, int n_colors,
                       void* stream)
{
    TF_REQUIRE(n_elem >= 0 && ke, "bad arguments");
    return launch_edof<double>(edof, ke, scale, v, w, n_elem, mode, color_elems, color_offsets,
                               n_colors, S(stream));
}

int tf_pass_fixed_f32(const int64_t* fixed, int64_t n_fixed, const float* v, float* w, void* stream)
{
    return launch_pass_fixed<float>(fixed, n_fixed, v, w, S(stream));
}

int tf_pass_fixed_f64(const int64_t* fixed, int64_t n_fixed, const double* v, double* w,
                      void* stream)
{
    return launch_pass_fixed<double>(fixed, n_fixed, v, w, S(stream));
}

#define TF_GATHER(T, SUF)                                                                     \
    int tf_gather_##SUF(const int32_t* edof, const T* v, T* u_elem, int64_t n_elem, void* stream) \
    {                                                                                         \
        if (n_elem <= 0) return TF_OK;                                                        \
        const long long n = n_elem * NLOC;                                                    \
        k_gather<T><<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(edof, v, u_elem, n_elem); \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }
TF_GATHER(float, f32)
TF_GATHER(double, f64)

#define TF_GEMM(T, SUF)                                                                       \
    int tf_gemm_##SUF(const T* u_elem, const T* ke, const T* scale, T* f_elem, int64_t n_elem, \
                      void* stream)                                                           \
    {                                                                                         \
        if (n_elem <= 0) return TF_OK;                                                        \
        KeMat<T> k;                                                                           \
        memcpy(k.a, ke, sizeof(k.a));                                                         \
        k_gemm<T><<<(unsigned)((n_elem + EDOF_BLOCK - 1) / EDOF_BLOCK), EDOF_BLOCK, 0, S(stream)>>>( \
            u_elem, scale, f_elem, n_elem, k);                                                \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }
TF_GEMM(float, f32)
TF_GEMM(double, f64)

#define TF_SCATTER(T, SUF)                                                                    \
    int tf_scatter_##SUF(const int32_t* edof, const T* f_elem, double* acc, int64_t n_elem,    \
                         void* stream)                                                        \
    {                                                                                         \
        if (n_elem <= 0) return TF_OK;                                                        \
        const long long n = n_elem * NLOC;                                                    \
        k_scatter<T><<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(edof, f_elem, acc, n_elem); \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }
TF_SCATTER(float, f32)
TF_SCATTER(double, f64)

#define TF_JACOBI(T, SUF)                                                                     \
    int tf_jacobi_grid_##SUF(const tf_grid* g, const T* ke_diag, const T* scale, T* diag,      \
                             T* inv_diag, const uint8_t* node_fixed, void* stream)            \
    {                                                                                         \
        TF_GRID_CHECK(g);                                                                     \
        Grid gg = make_grid(g);                                                               \
        KeMat<T> k;                                                                           \
        memset(&k, 0, sizeof(k));                                                             \
        memcpy(k.a, ke_diag, NLOC * sizeof(T));                                               \
        k_jacobi_grid<T><<<(unsigned)((gg.n_nodes + 255) / 256), 256, 0, S(stream)>>>(          \
            gg, scale, diag, inv_diag, node_fixed, k);                                        \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }                                                                                         \
    int tf_jacobi_grid_partial_##SUF(const tf_grid* g, const T* ke_diag, const T* scale,       \
                                     double* partial, void* stream)                          \
    {                                                                                         \
        TF_GRID_CHECK(g);                                                                     \
        TF_REQUIRE(ke_diag && scale && partial, "null pointer");                              \
        Grid gg = make_grid(g);                                                               \
        KeMat<T> k;                                                                           \
        memset(&k, 0, sizeof(k));                                                             \
        memcpy(k.a, ke_diag, NLOC * sizeof(T));                                               \
        k_jacobi_grid<T><<<(unsigned)((gg.n_nodes + 255) / 256), 256, 0, S(stream)>>>(          \
            gg, scale, nullptr, nullptr, nullptr, k, partial);                                \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }                                                                                         \
    int tf_jacobi_edof_##SUF(const int32_t* edof, const T* ke_diag, const T* scale, double* acc, \
                             int64_t n_elem, void* stream)                                    \
    {                                                                                         \
        if (n_elem <= 0) return TF_OK;                                                        \
        KeMat<T> k;                                                                           \
        memset(&k, 0, sizeof(k));                                                             \
        memcpy(k.a, ke_diag, NLOC * sizeof(T));                                               \
        const long long n = n_elem * NLOC;                                                    \
        k_jacobi_edof<T><<<(unsigned)((n + 255) / 256), 256, 0, S(stream)>>>(edof, scale, acc, n_elem, k); \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }
TF_JACOBI(float, f32)
TF_JACOBI(double, f64)

int tf_energies_grid_f64(const tf_grid* g, const double* ke, const double* u, double* out,
                         void* stream)
{
    TF_GRID_CHECK(g);
    Grid gg = make_grid(g);
    EnergyKe k;
    memcpy(k.ke.a, ke, sizeof(k.ke.a));
    k.walsh = khat_blocks_cached<double>(ke, &k.kb) ? 1 : 0;
    k_energies_grid<<<(unsigned)((gg.n_elem + EDOF_BLOCK - 1) / EDOF_BLOCK), EDOF_BLOCK, 0, S(stream)>>>(
        gg, u, out, k);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_energies_edof_f64(const int32_t* edof, const double* ke, const double* u, double* out,
                         int64_t n_elem, void* stream)
{
    if (n_elem <= 0) return TF_OK;
    TF_REQUIRE(((uintptr_t)edof & 15u) == 0, "edof must be 16-byte aligned");
    EnergyKe k;
    memcpy(k.ke.a, ke, sizeof(k.ke.a));
    k.walsh = khat_blocks_cached<double>(ke, &k.kb) ? 1 : 0;
    k_energies_edof<<<(unsigned)((n_elem + EDOF_BLOCK - 1) / EDOF_BLOCK), EDOF_BLOCK, 0, S(stream)>>>(
        edof, u, out, n_elem, k);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

}  // extern "C"
