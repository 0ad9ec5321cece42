// Device-resident Jacobi-PCG -- the recurrence of reference solver.py:57-147.
//
// The whole solve is ONE CUDA graph launch.  A conditional WHILE node repeats
// the body until the device decides to stop; an inner IF node runs the
// true-residual refresh (solver.py:116-119) every `recompute_every` iterations.
// Body per iteration (3 kernels, +2 on refresh iterations):
//
//   K_mv    q = A p (structured tile kernel) fused with per-CTA p.q partials.
//   K_upd   every block sums the p.q partials in the same fixed order ->
//           alpha, breakdown / divergence, refresh flag (block 0 publishes it
//           and sets the IF handle); x += alpha p ; r -= alpha q ; per-block
//           partials of r.r and r.(r*inv_diag).
//   [IF]    K_mv(x) ; K_res: r = b - A x, same partials.
//   K_pdir  every block sums the r.r / r.z partials -> rel, convergence,
//           max_iter, beta (block 0 commits and sets the WHILE handle);
//           p = r*inv_diag + beta p.
// No serial "last block" tail sits on the per-iteration critical path.
// The WHILE body holds several iterations (default 4).  When the refresh
// period is a multiple of 10 (default 50) or 5, or zero, the solve launches
// a second graph whose body holds 10 (5) iterations and ONE IF node after the
// last: a refresh can only fall there (bodies start at it = 1 mod unroll),
// and a conditional node costs more than a kernel boundary (1.1-1.6 us).
//
// Reductions are deterministic (fixed partial order, fixed block tree), so a
// solve is bitwise reproducible.  Scalar rounding mirrors the reference's
// numpy semantics: FP32 dots/norms are rounded to float32 before use, alpha
// and beta are Python-float quotients applied as float32 (NEP 50), and every
// vector update rounds the product before the add (no FMA), like numpy.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tf_common.cuh"

namespace tf {

template <typename T>
int launch_grid_pull(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                     const uint8_t* node_fixed, uint32_t flags, int variant, double* dot_part,
                     cudaStream_t st);
template <typename T>
long long grid_matvec_blocks(const Grid& g, const T* ke_host, int variant);
template <typename T>
int launch_pass_fixed(const int64_t* fixed, long long n, const T* v, T* w, cudaStream_t st);
template <typename T>
int launch_grid_tile_cg(const Grid& g, const T* ke_host, const T* scale, T* q,
                        const uint8_t* node_fixed, double* dot_part, const CgTileArgs<T>& a,
                        cudaStream_t st);
template <typename T>
bool launch_grid_tile_supported(const T* ke_host);
template <typename T>
bool pcg_resident_plan(const Grid& g, const T* ke_host, ResPlan* plan);
template <typename T>
int launch_pcg_resident(const ResPlan& plan, const Grid& g, const T* ke_host, int has_x0, const T* scale,
                        const T* b, const T* inv, T* x, T* z, T* p0, T* p1, const uint8_t* node_fixed,
                        double* ring, CgScalars* sc, T* r1, T* q0, T* q1, cudaStream_t st);
size_t pcg_resident_ring_doubles(const ResPlan& plan);



template <typename T>
struct CgP {
    T *x, *r, *p, *q;
    const T *b, *inv;
    double* part;           // [n_part_max * 3]
    unsigned* tickets;      // [4]
    CgScalars* sc;
    long long n;
    cudaGraphConditionalHandle h_while, h_refresh;
    int in_graph;  // 0: launched directly (TF_PCG_NOGRAPH profiling mode)
};

__device__ __forceinline__ double rnd(double v, bool f32) { return cg_round(v, f32); }
__device__ __forceinline__ double vsqrt(double v, bool f32) { return cg_sqrt(v, f32); }

constexpr int VEC_BLOCK = 256;

// deterministic block sum of K values per thread; result valid in thread 0
template <int K>
__device__ __forceinline__ void block_sum_k(double (&v)[K], double* sh /* [K*32] */)
{
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) sh[k * 32 + wid] = v[k];
    }
    __syncthreads();
    if (tid == 0) {
        const int nw = (blockDim.x + 31) / 32;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int i = 0; i < nw; ++i) s += sh[k * 32 + i];
            v[k] = s;
        }
    }
    __syncthreads();
}

// Publish this block's K partials; returns true in the (unique) last block,
// whose thread 0 then holds the fixed-order totals in `tot`.
template <int K>
__device__ bool last_block_reduce(double (&v)[K], double* part, unsigned* ticket, int nblocks,
                                  double (&tot)[K])
{
    __shared__ double sh[K * 32];
    __shared__ bool am_last;
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int tid = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int nthr = blockDim.x * blockDim.y * blockDim.z;
    // block tree (threads flattened)
    {
        const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
        for (int k = 0; k < K; ++k) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
        }
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) sh[k * 32 + wid] = v[k];
        }
        __syncthreads();
        if (tid == 0) {
            const int nw = (nthr + 31) / 32;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int i = 0; i < nw; ++i) s += sh[k * 32 + i];
                part[(size_t)bid * K + k] = s;
            }
            // acq_rel ticket: releases this block's partials (and, through the
            // barrier above, its threads' writes); the last block acquires all
            unsigned t;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
            am_last = (t == (unsigned)nblocks - 1);
        }
        __syncthreads();
    }
    if (!am_last) return false;
    // fixed-order reduction of all partials: thread t sums partials t, t+nthr, ...
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    for (int i = tid; i < nblocks; i += nthr) {
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] += __ldcg(part + (size_t)i * K + k);
    }
    {
        const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
        for (int k = 0; k < K; ++k) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], o);
        }
        __syncthreads();
        if (lane == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) sh[k * 32 + wid] = acc[k];
        }
        __syncthreads();
        if (tid == 0) {
            const int nw = (nthr + 31) / 32;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                double s = 0.0;
                for (int i = 0; i < nw; ++i) s += sh[k * 32 + i];
                tot[k] = s;
            }
            *ticket = 0u;  // re-arm for the next launch
        }
    }
    return true;
}

// ---- decisions -------------------------------------------------------------

__device__ __forceinline__ float qbf16(float x) { return bf16_rne(x); }
__device__ __forceinline__ double qbf16(double x) { return (double)bf16_rne((float)x); }

// ---- vector access: 16-byte chunks (float4 / double2) + scalar tail ------------------

template <typename T> struct V16;
template <> struct V16<float> { using type = float4; static constexpr int N = 4; };
template <> struct V16<double> { using type = double2; static constexpr int N = 2; };

template <typename T>
__device__ __forceinline__ void ld16(const T* p, long long c, T (&o)[V16<T>::N])
{
    const typename V16<T>::type v = reinterpret_cast<const typename V16<T>::type*>(p)[c];
    memcpy(o, &v, sizeof(v));
}
template <typename T>
__device__ __forceinline__ void st16(T* p, long long c, const T (&o)[V16<T>::N])
{
    typename V16<T>::type v;
    memcpy(&v, o, sizeof(v));
    reinterpret_cast<typename V16<T>::type*>(p)[c] = v;
}

// fixed-order sum of `n` partials, identical in every block (valid in thread 0)
__device__ __forceinline__ double sum_partials(const double* part, int n, double* sh)
{
    double v = 0.0;
    // loads of four rounds issued before their adds (one L2 round trip for up
    // to 4 blockDim partials), same per-thread order
    for (int i0 = threadIdx.x; i0 < n; i0 += 4 * blockDim.x) {
        double t[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) t[u] = i0 + u * (int)blockDim.x < n ? __ldcg(part + i0 + u * blockDim.x) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (i0 + u * (int)blockDim.x < n) v += t[u];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x + 31) / 32; ++w) s += sh[w];
    __syncthreads();
    return s;  // every thread holds the same total
}

// ---- kernels -----------------------------------------------------------------

// p.q block partials (general-edof mode; the structured matvec fuses this)
template <typename T>
__global__ void __launch_bounds__(VEC_BLOCK) k_pq_partials(CgP<T> P, double* part_mv)
{
    if (P.sc->done) return;
    constexpr int N = V16<T>::N;
    double v[1] = {0.0};
    const long long nc = P.n / N, stride = (long long)gridDim.x * VEC_BLOCK;
    for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
        T p[N], q[N];
        ld16(P.p, c, p);
        ld16(P.q, c, q);
#pragma unroll
        for (int k = 0; k < N; ++k) v[0] += (double)p[k] * (double)q[k];
    }
    if (blockIdx.x == 0)
        for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) v[0] += (double)P.p[i] * (double)P.q[i];
    __shared__ double sh[32];
    block_sum_k<1>(v, sh);
    if (threadIdx.x == 0) part_mv[blockIdx.x] = v[0];
}

// Fused: reduce the matvec's p.q partials (every block, same order) -> alpha,
// breakdown / divergence, refresh flag; x += alpha p; r -= alpha q; per-block
// partials of r.r and r.z (reduced by k_direction -- no serial tail here).
template <typename T>
__global__ void __launch_bounds__(VEC_BLOCK) k_update(CgP<T> P, const double* part_mv, int nmv)
{
    constexpr int N = V16<T>::N;
    CgScalars* sc = P.sc;
    if (sc->done) {
        // an unrolled loop body ran past the stop: keep its refresh branch off
        if (P.in_graph && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(P.h_refresh, 0u);
        return;
    }
    __shared__ double shp[VEC_BLOCK / 32];
    const bool f32 = sizeof(T) == 4;
    const double pq = rnd(sum_partials(part_mv, nmv, shp), f32);
    const double rz = sc->rz;
    const int it_now = sc->it + 1;
    const bool bad = !isfinite(pq) || !isfinite(rz) || pq <= 0.0;
    const double alpha = bad ? 0.0 : rz / pq;
    const bool refresh = !bad && sc->recompute > 0 && it_now % sc->recompute == 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->it_cur = it_now;
        sc->matvecs += 1;
        sc->refresh = refresh ? 1 : 0;
        sc->alpha = alpha;
        sc->rz_old = rz;
        if (bad) {
            sc->it = it_now;
            sc->done = 1;
            sc->term = (!isfinite(pq) || !isfinite(rz)) ? TERM_DIVERGED : TERM_BREAKDOWN;
            if (P.in_graph) cudaGraphSetConditional(P.h_while, 0u);
        }
        if (P.in_graph) cudaGraphSetConditional(P.h_refresh, refresh ? 1u : 0u);
    }
    if (bad) return;
    const T a = (T)alpha;
    double v[2] = {0.0, 0.0};
    const long long nc = P.n / N, stride = (long long)gridDim.x * VEC_BLOCK;
    if (refresh) {
        // the refresh matvec needs the new x now; otherwise k_direction
        // applies x += alpha p while it reads p anyway (one vector less per
        // iteration, same arithmetic)
        for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
            T x[N], p[N];
            ld16(P.x, c, x);
            ld16(P.p, c, p);
#pragma unroll
            for (int k = 0; k < N; ++k) x[k] = add_rn(x[k], mul_rn(a, p[k]));
            st16(P.x, c, x);
        }
        if (blockIdx.x == 0)
            for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) P.x[i] = add_rn(P.x[i], mul_rn(a, P.p[i]));
        return;  // k_residual produces the partials this iteration
    }
    for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
        T r[N], q[N], iv[N];
        ld16(P.r, c, r);
        ld16(P.q, c, q);
        ld16(P.inv, c, iv);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            r[k] = sub_rn(r[k], mul_rn(a, q[k]));
            const T z = mul_rn(r[k], iv[k]);
            v[0] += (double)r[k] * (double)r[k];
            v[1] += (double)r[k] * (double)z;
        }
        st16(P.r, c, r);
    }
    if (blockIdx.x == 0) {
        for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) {
            const T r = sub_rn(P.r[i], mul_rn(a, P.q[i]));
            P.r[i] = r;
            const T z = mul_rn(r, P.inv[i]);
            v[0] += (double)r * (double)r;
            v[1] += (double)r * (double)z;
        }
    }
    __shared__ double sh[2 * 32];
    block_sum_k<2>(v, sh);
    if (threadIdx.x == 0) {
        P.part[2 * blockIdx.x] = v[0];
        P.part[2 * blockIdx.x + 1] = v[1];
    }
}

// Fused-protocol update (structured solves): the search direction of this
// iteration was written by the CG tile kernel into pbuf[it_b & 1].
template <typename T>
__global__ void __launch_bounds__(VEC_BLOCK) k_update_f(CgP<T> P, const double* part_mv, int nmv,
                                                        T* pA, T* pB)
{
    constexpr int N = V16<T>::N;
    CgScalars* sc = P.sc;
    if (sc->done) return;
    __shared__ double shp[VEC_BLOCK / 32];
    const bool f32 = sizeof(T) == 4;
    const double pq = rnd(sum_partials(part_mv, nmv, shp), f32);
    const double rz = sc->rz;
    const int it_now = sc->it_b;
    const T* __restrict__ pn = (it_now & 1) ? pB : pA;
    const bool bad = !isfinite(pq) || !isfinite(rz) || pq <= 0.0;
    const double alpha = bad ? 0.0 : rz / pq;
    const bool refresh = !bad && sc->recompute > 0 && it_now % sc->recompute == 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->it_a = it_now;
        sc->matvecs += 1;
        sc->refresh = refresh ? 1 : 0;
        sc->alpha = alpha;
        sc->rz_old = rz;
        if (bad) {
            sc->it = it_now;
            sc->done = 1;
            sc->term = (!isfinite(pq) || !isfinite(rz)) ? TERM_DIVERGED : TERM_BREAKDOWN;
            if (P.in_graph) cudaGraphSetConditional(P.h_while, 0u);
        }
        if (P.in_graph) cudaGraphSetConditional(P.h_refresh, refresh ? 1u : 0u);
    }
    if (bad) return;
    const T a = (T)alpha;
    double v[2] = {0.0, 0.0};
    const long long nc = P.n / N, stride = (long long)gridDim.x * VEC_BLOCK;
    for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
        T x[N], p[N], r[N], q[N], iv[N];
        ld16(P.x, c, x);
        ld16(pn, c, p);
        if (!refresh) {
            ld16(P.r, c, r);
            ld16(P.q, c, q);
            ld16(P.inv, c, iv);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
            x[k] = add_rn(x[k], mul_rn(a, p[k]));
            if (!refresh) {
                r[k] = sub_rn(r[k], mul_rn(a, q[k]));
                const T z = mul_rn(r[k], iv[k]);
                v[0] += (double)r[k] * (double)r[k];
                v[1] += (double)r[k] * (double)z;
            }
        }
        st16(P.x, c, x);
        if (!refresh) st16(P.r, c, r);
    }
    if (blockIdx.x == 0) {
        for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) {
            P.x[i] = add_rn(P.x[i], mul_rn(a, pn[i]));
            if (!refresh) {
                const T r = sub_rn(P.r[i], mul_rn(a, P.q[i]));
                P.r[i] = r;
                const T z = mul_rn(r, P.inv[i]);
                v[0] += (double)r * (double)r;
                v[1] += (double)r * (double)z;
            }
        }
    }
    if (refresh) return;
    __shared__ double sh[2 * 32];
    block_sum_k<2>(v, sh);
    if (threadIdx.x == 0) {
        P.part[2 * blockIdx.x] = v[0];
        P.part[2 * blockIdx.x + 1] = v[1];
    }
}

template <typename T>
__global__ void __launch_bounds__(VEC_BLOCK) k_residual(CgP<T> P)
{
    // refresh: r = b - A x  (q holds A x); partials for k_direction
    constexpr int N = V16<T>::N;
    if (P.sc->done) return;
    double v[2] = {0.0, 0.0};
    const long long nc = P.n / N, stride = (long long)gridDim.x * VEC_BLOCK;
    for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
        T b[N], q[N], iv[N], r[N];
        ld16(P.b, c, b);
        ld16(P.q, c, q);
        ld16(P.inv, c, iv);
#pragma unroll
        for (int k = 0; k < N; ++k) {
            r[k] = sub_rn(b[k], q[k]);
            const T z = mul_rn(r[k], iv[k]);
            v[0] += (double)r[k] * (double)r[k];
            v[1] += (double)r[k] * (double)z;
        }
        st16(P.r, c, r);
    }
    if (blockIdx.x == 0) {
        for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) {
            const T r = sub_rn(P.b[i], P.q[i]);
            P.r[i] = r;
            const T z = mul_rn(r, P.inv[i]);
            v[0] += (double)r * (double)r;
            v[1] += (double)r * (double)z;
        }
    }
    __shared__ double sh[2 * 32];
    block_sum_k<2>(v, sh);
    if (threadIdx.x == 0) {
        P.part[2 * blockIdx.x] = v[0];
        P.part[2 * blockIdx.x + 1] = v[1];
        if (blockIdx.x == 0) P.sc->matvecs += 1;
    }
}

// Every block reduces the r.r / r.z partials in the same order and takes the
// same decision (rel, convergence, max_iter, beta); block 0 commits the state
// and the WHILE condition; p = r*inv + beta p unless the loop stops.
template <typename T>
__global__ void __launch_bounds__(VEC_BLOCK) k_direction(CgP<T> P, int nparts)
{
    constexpr int N = V16<T>::N;
    CgScalars* sc = P.sc;
    if (sc->done) return;
    const bool f32 = sizeof(T) == 4;
    // the two partial streams are interleaved: reduce them with two passes
    __shared__ double shp[VEC_BLOCK / 32];
    double rr = 0.0, rzn = 0.0;
    {
        double v = 0.0, w = 0.0;
        for (int i0 = threadIdx.x; i0 < nparts; i0 += 4 * VEC_BLOCK) {  // loads before adds, as sum_partials
            double tv[4], tw[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int i = i0 + u * VEC_BLOCK;
                tv[u] = i < nparts ? __ldcg(P.part + 2 * i) : 0.0;
                tw[u] = i < nparts ? __ldcg(P.part + 2 * i + 1) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i0 + u * VEC_BLOCK < nparts) {
                    v += tv[u];
                    w += tw[u];
                }
        }
        double vv[2] = {v, w};
        __shared__ double sh2[2 * 32];
        block_sum_k<2>(vv, sh2);
        if (threadIdx.x == 0) {
            shp[0] = vv[0];
            shp[1] = vv[1];
        }
        __syncthreads();
        rr = shp[0];
        rzn = shp[1];
    }
    const int it = sc->it_cur;
    const double rn = vsqrt(rnd(rr, f32), f32);
    bool stop = false;
    int term = TERM_MAX_ITER;
    double rel = sc->rel, beta = 0.0, rz_new = 0.0;
    if (!isfinite(rn)) {
        stop = true;
        term = TERM_DIVERGED;
    } else {
        rel = rn / sc->bnorm;
        if (rel <= sc->tol) {
            stop = true;
            term = TERM_CONVERGED;
        } else {
            rz_new = rnd(rzn, f32);
            beta = rz_new / sc->rz_old;
            if (it >= sc->max_iter) {
                stop = true;
                term = TERM_MAX_ITER;
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->it = it;
        if (isfinite(rn)) {
            sc->rel = rel;
            if (sc->hist) sc->hist[it] = rel;
        }
        if (stop) {
            sc->done = 1;
            sc->term = term;
        } else {
            sc->rz = rz_new;
            sc->beta = beta;
        }
        if (P.in_graph) cudaGraphSetConditional(P.h_while, stop ? 0u : 1u);
    }
    const long long nc = P.n / N, stride = (long long)gridDim.x * VEC_BLOCK;
    // this iteration's x += alpha p (deferred from k_update unless it was a
    // refresh iteration), with the p that the update used -- also when the
    // loop stops here
    const bool upd_x = sc->refresh == 0;
    const T al = (T)sc->alpha;
    if (stop) {
        if (upd_x) {
            for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
                T x[N], p[N];
                ld16(P.x, c, x);
                ld16(P.p, c, p);
#pragma unroll
                for (int k = 0; k < N; ++k) x[k] = add_rn(x[k], mul_rn(al, p[k]));
                st16(P.x, c, x);
            }
            if (blockIdx.x == 0)
                for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) P.x[i] = add_rn(P.x[i], mul_rn(al, P.p[i]));
        }
        return;
    }
    const T be = (T)beta;
    const bool quant = sc->quantize != 0;
    for (long long c = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; c < nc; c += stride) {
        T r[N], iv[N], p[N];
        ld16(P.r, c, r);
        ld16(P.inv, c, iv);
        ld16(P.p, c, p);
        if (upd_x) {
            T x[N];
            ld16(P.x, c, x);
#pragma unroll
            for (int k = 0; k < N; ++k) x[k] = add_rn(x[k], mul_rn(al, p[k]));
            st16(P.x, c, x);
        }
#pragma unroll
        for (int k = 0; k < N; ++k) p[k] = add_rn(mul_rn(r[k], iv[k]), mul_rn(be, p[k]));
        if (quant) {  // quantize_krylov (solver.py:134-136): p and r to bf16
#pragma unroll
            for (int k = 0; k < N; ++k) {
                p[k] = qbf16(p[k]);
                r[k] = qbf16(r[k]);
            }
            st16(P.r, c, r);
        }
        st16(P.p, c, p);
    }
    if (blockIdx.x == 0)
        for (long long i = nc * N + threadIdx.x; i < P.n; i += VEC_BLOCK) {
            if (upd_x) P.x[i] = add_rn(P.x[i], mul_rn(al, P.p[i]));
            T pn = add_rn(mul_rn(P.r[i], P.inv[i]), mul_rn(be, P.p[i]));
            if (quant) {
                pn = qbf16(pn);
                P.r[i] = qbf16(P.r[i]);
            }
            P.p[i] = pn;
        }
}

// init: r = b - q (has_x0) or r = b; p = r*inv; partials b.b, r.r, r.z
template <typename T>
__global__ void __launch_bounds__(VEC_BLOCK) k_init(CgP<T> P, int has_x0)
{
    double v[3] = {0.0, 0.0, 0.0};
    const long long stride = (long long)gridDim.x * VEC_BLOCK;
    for (long long i = (long long)blockIdx.x * VEC_BLOCK + threadIdx.x; i < P.n; i += stride) {
        const T b = P.b[i];
        const T r = has_x0 ? sub_rn(b, P.q[i]) : b;
        P.r[i] = r;
        const T z = mul_rn(r, P.inv[i]);
        P.p[i] = z;
        v[0] += (double)b * (double)b;
        v[1] += (double)r * (double)r;
        v[2] += (double)r * (double)z;
    }
    double tot[3];
    if (last_block_reduce<3>(v, P.part, P.tickets + 3, gridDim.x, tot) && threadIdx.x == 0) {
        CgScalars* sc = P.sc;
        const bool f32 = sizeof(T) == 4;
        sc->bnorm = vsqrt(rnd(tot[0], f32), f32);
        sc->it = 0;
        sc->it_a = 0;
        sc->matvecs = has_x0 ? 1 : 0;
        sc->done = 0;
        sc->term = TERM_MAX_ITER;
        sc->zero_rhs = 0;
        if (sc->bnorm == 0.0) {
            sc->zero_rhs = 1;
            sc->done = 1;
            sc->term = TERM_CONVERGED;
            sc->rel = 0.0;
            if (sc->hist) sc->hist[0] = 0.0;
            return;
        }
        sc->rz = rnd(tot[2], f32);
        const double rel = vsqrt(rnd(tot[1], f32), f32) / sc->bnorm;
        sc->rel = rel;
        if (sc->hist) sc->hist[0] = rel;
        if (rel <= sc->tol) {
            sc->done = 1;
            sc->term = TERM_CONVERGED;
        } else if (sc->max_iter <= 0) {
            sc->done = 1;
        }
    }
}

// ---- handle --------------------------------------------------------------------

struct PcgImpl {
    int prec;
    int structured;
    Grid grid;
    const int32_t* edof;
    long long n_elem, n_dof;
    std::vector<unsigned char> ke;  // host copy (576 * sizeof(T))
    const uint8_t* node_fixed;
    const int64_t* fixed;
    long long n_fixed;
    int variant;
    cudaStream_t stream;
    // device buffers
    void *x, *r, *p, *q, *b, *inv, *scale;
    void* p2;           // second search-direction buffer (fused protocol)
    void *r2, *q2;      // resident single-exchange iteration: r_k / q_k ping-pong partners
    int quantize;       // quantize_krylov for the next solve (tf_pcg_set_quantize_krylov)
    int fused;          // structured tile solve with the direction folded into the matvec
    int resident;       // SM-resident solve: one cooperative launch (tf_pcg_resident.cu)
    ResPlan rplan;
    double* ring;       // resident exchange slots
    double* part;
    double* part_mv;    // per-CTA p.q partials of the matvec
    unsigned* tickets;
    CgScalars* sc;
    CgScalars* sc_host;  // pinned
    int n_vec_blocks;
    long long n_mv_blocks;
    cudaGraph_t graph;
    cudaGraphExec_t exec;
    cudaGraphConditionalHandle h_while, h_refresh;
    // sparse-refresh graphs (built on first use): `unroll` iterations per
    // WHILE body with ONE refresh IF node, after the last -- valid when the
    // refresh period is a multiple of the unroll (or zero); index 0: 10, 1: 5
    cudaGraph_t graph_sp[2];
    cudaGraphExec_t exec_sp[2];
};

template <typename T>
static CgP<T> params_of(PcgImpl* h)
{
    CgP<T> P;
    P.x = (T*)h->x; P.r = (T*)h->r; P.p = (T*)h->p; P.q = (T*)h->q;
    P.b = (const T*)h->b; P.inv = (const T*)h->inv;
    P.part = h->part; P.tickets = h->tickets; P.sc = h->sc; P.n = h->n_dof;
    P.h_while = h->h_while; P.h_refresh = h->h_refresh;
    P.in_graph = 1;
    return P;
}

// Enqueue A*v -> w on stream (used while capturing the body graphs).
template <typename T>
static int enqueue_matvec(PcgImpl* h, const T* v, T* w, double* dot_part, cudaStream_t st)
{
    const T* ke = (const T*)h->ke.data();
    if (h->structured) {
        return launch_grid_pull<T>(h->grid, ke, (const T*)h->scale, v, w, h->node_fixed,
                                   TF_MASK_INPUT | TF_PASS_FIXED, h->variant, dot_part, st);
    }
    TF_CUDA_TRY(cudaMemsetAsync(w, 0, sizeof(T) * h->n_dof, st));
    if (h->prec == 16) {  // emulated bf16: quantized input, per-term bf16(s K) (tf_bf16.cu)
        int rc = tf_matvec_edof_bf16(h->edof, (const float*)ke, (const float*)h->scale, (const float*)v,
                                     (float*)w, h->n_elem, TF_SCATTER_ATOMIC, nullptr, nullptr, 0, 1, st);
        if (rc) return rc;
        return launch_pass_fixed<T>(h->fixed, h->n_fixed, v, w, st);
    }
    int rc = (sizeof(T) == 4)
                 ? tf_matvec_edof_f32(h->edof, (const float*)ke, (const float*)h->scale,
                                      (const float*)v, (float*)w, h->n_elem, TF_SCATTER_ATOMIC,
                                      nullptr, nullptr, 0, st)
                 : tf_matvec_edof_f64(h->edof, (const double*)ke, (const double*)h->scale,
                                      (const double*)v, (double*)w, h->n_elem, TF_SCATTER_ATOMIC,
                                      nullptr, nullptr, 0, st);
    if (rc) return rc;
    return launch_pass_fixed<T>(h->fixed, h->n_fixed, v, w, st);
}

// Add a captured sequence as the content of `body` (a conditional body graph).
template <typename F>
static int capture_into(cudaGraph_t body, cudaStream_t cap, F&& fn, const cudaGraphNode_t* deps = nullptr,
                        size_t ndeps = 0)
{
    TF_CUDA_TRY(cudaStreamBeginCaptureToGraph(cap, body, deps, nullptr, ndeps,
                                              cudaStreamCaptureModeThreadLocal));
    const int rc = fn(cap);
    cudaGraph_t out = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cap, &out);
    if (rc) return rc;
    if (e != cudaSuccess) {
        set_error("end capture: %s", cudaGetErrorString(e));
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

// body pieces, shared by the captured graph and the direct (profiling) loop
template <typename T>
static int enqueue_part1(PcgImpl* h, const CgP<T>& P, cudaStream_t st)
{
    const int nvb = h->n_vec_blocks;
    int nmv;
    if (h->fused) {
        CgTileArgs<T> a;
        a.r = P.r;
        a.inv = P.inv;
        a.pbuf[0] = (T*)h->p;
        a.pbuf[1] = (T*)h->p2;
        a.part = h->part;
        a.nparts = nvb;
        a.sc = h->sc;
        a.h_while = P.h_while;
        a.in_graph = P.in_graph;
        int r = launch_grid_tile_cg<T>(h->grid, (const T*)h->ke.data(), (const T*)h->scale, P.q,
                                       h->node_fixed, h->part_mv, a, st);
        if (r) return r;
        k_update_f<T><<<nvb, VEC_BLOCK, 0, st>>>(P, h->part_mv, (int)h->n_mv_blocks, (T*)h->p, (T*)h->p2);
        TF_CHECK_LAUNCH();
        return TF_OK;
    }
    if (h->structured) {
        int r = launch_grid_pull<T>(h->grid, (const T*)h->ke.data(), (const T*)h->scale, P.p, P.q,
                                    h->node_fixed, TF_MASK_INPUT | TF_PASS_FIXED, h->variant,
                                    h->part_mv, st);
        if (r) return r;
        nmv = (int)h->n_mv_blocks;
    } else {
        int r = enqueue_matvec<T>(h, P.p, P.q, nullptr, st);
        if (r) return r;
        k_pq_partials<T><<<nvb, VEC_BLOCK, 0, st>>>(P, h->part_mv);
        TF_CHECK_LAUNCH();
        nmv = nvb;
    }
    k_update<T><<<nvb, VEC_BLOCK, 0, st>>>(P, h->part_mv, nmv);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

template <typename T>
static int enqueue_refresh(PcgImpl* h, const CgP<T>& P, cudaStream_t st)
{
    int r = enqueue_matvec<T>(h, P.x, P.q, nullptr, st);
    if (r) return r;
    k_residual<T><<<h->n_vec_blocks, VEC_BLOCK, 0, st>>>(P);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

// sparse_unroll > 0: that many iterations per body and one refresh IF node
// (after the last), i.e. a graph for refresh periods divisible by it: every
// other iteration skips the conditional node (~1.1-1.6 us each on B200,
// measured with the IF nodes removed; a refresh can only fall on the last
// iteration of a body because the body always starts at it = 1 mod unroll).
template <typename T>
static int build_graph(PcgImpl* h, int sparse_unroll = 0, cudaGraph_t* g_out = nullptr,
                       cudaGraphExec_t* e_out = nullptr)
{
    cudaStream_t cap;
    TF_CUDA_TRY(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaGraph_t graph;
    cudaGraphConditionalHandle h_while, h_refresh0;
    TF_CUDA_TRY(cudaGraphCreate(&graph, 0));
    TF_CUDA_TRY(cudaGraphConditionalHandleCreate(&h_while, graph, 1, cudaGraphCondAssignDefault));

    cudaGraphNodeParams wp = {};
    wp.type = cudaGraphNodeTypeConditional;
    wp.conditional.handle = h_while;
    wp.conditional.type = cudaGraphCondTypeWhile;
    wp.conditional.size = 1;
    cudaGraphNode_t wnode;
    TF_CUDA_TRY(cudaGraphAddNode(&wnode, graph, nullptr, 0, &wp));
    cudaGraph_t body = wp.conditional.phGraph_out[0];

    TF_CUDA_TRY(cudaGraphConditionalHandleCreate(&h_refresh0, body, 0, 0));
    CgP<T> P = params_of<T>(h);
    P.h_while = h_while;
    P.h_refresh = h_refresh0;
    const bool sparse = sparse_unroll > 0;
    const int nvb = h->n_vec_blocks;

    // The WHILE body holds `unroll` CG iterations (TF_PCG_UNROLL, default 4 on
    // the unfused protocol): one conditional evaluation per `unroll`
    // iterations.  Kernels of an iteration past the stop return at entry
    // (sc->done), k_update also switching the refresh branch off; only the
    // matvec of such an iteration still runs (once per solve).
    int unroll = 1;
    if (sparse) {
        unroll = sparse_unroll;
    } else if (!h->fused) {
        const char* eu = getenv("TF_PCG_UNROLL");
        unroll = std::max(1, std::min(8, eu ? atoi(eu) : 4));
    }
    // sink (dependent-free) node of a graph
    auto sink_of = [&](cudaGraph_t gr, cudaGraphNode_t* out) -> int {
        size_t n = 0;
        TF_CUDA_TRY(cudaGraphGetNodes(gr, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        TF_CUDA_TRY(cudaGraphGetNodes(gr, nodes.data(), &n));
        for (auto nd : nodes) {
            size_t nout = 0;
            TF_CUDA_TRY(cudaGraphNodeGetDependentNodes(nd, nullptr, &nout));
            if (nout == 0) *out = nd;
        }
        return TF_OK;
    };
    cudaGraphNode_t tail = nullptr;  // last node of the previous iteration in the body
    for (int u = 0; u < unroll; ++u) {
        // every IF node needs its own conditional handle (set by its k_update)
        // (sparse: every k_update sets the one handle; the last one before
        // the IF node decides)
        CgP<T> Pu = P;
        if (u > 0 && !sparse) TF_CUDA_TRY(cudaGraphConditionalHandleCreate(&Pu.h_refresh, body, 0, 0));
        // part 1: matvec+dot, update
        {
            int rc = capture_into(body, cap, [&](cudaStream_t st) -> int { return enqueue_part1<T>(h, Pu, st); },
                                  tail ? &tail : nullptr, tail ? 1 : 0);
            if (rc) return rc;
        }
        cudaGraphNode_t last_node = nullptr;
        if (int rc = sink_of(body, &last_node)) return rc;
        if (sparse && u < unroll - 1) {
            cudaKernelNodeParams kp = {};
            int nparts = nvb;
            void* args[] = {&Pu, &nparts};
            kp.func = (void*)k_direction<T>;
            kp.gridDim = dim3(nvb);
            kp.blockDim = dim3(VEC_BLOCK);
            kp.kernelParams = args;
            cudaGraphNode_t dn;
            TF_CUDA_TRY(cudaGraphAddKernelNode(&dn, body, &last_node, 1, &kp));
            tail = dn;
            continue;
        }
        // IF refresh { q = A x ; r = b - q }
        cudaGraphNodeParams ip = {};
        ip.type = cudaGraphNodeTypeConditional;
        ip.conditional.handle = Pu.h_refresh;
        ip.conditional.type = cudaGraphCondTypeIf;
        ip.conditional.size = 1;
        cudaGraphNode_t inode;
        TF_CUDA_TRY(cudaGraphAddNode(&inode, body, &last_node, 1, &ip));
        cudaGraph_t ifbody = ip.conditional.phGraph_out[0];
        {
            int rc = capture_into(ifbody, cap, [&](cudaStream_t st) -> int { return enqueue_refresh<T>(h, Pu, st); });
            if (rc) return rc;
        }
        tail = inode;
        // direction update after the IF node (folded into the next matvec when fused)
        if (!h->fused) {
            cudaKernelNodeParams kp = {};
            int nparts = nvb;
            void* args[] = {&Pu, &nparts};
            kp.func = (void*)k_direction<T>;
            kp.gridDim = dim3(nvb);
            kp.blockDim = dim3(VEC_BLOCK);
            kp.kernelParams = args;
            cudaGraphNode_t dn;
            TF_CUDA_TRY(cudaGraphAddKernelNode(&dn, body, &inode, 1, &kp));
            tail = dn;
        }
    }
    cudaGraphExec_t exec;
    TF_CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
    cudaStreamDestroy(cap);
    if (g_out) {
        *g_out = graph;
        *e_out = exec;
    } else {
        h->graph = graph;
        h->exec = exec;
        h->h_while = h_while;
        h->h_refresh = h_refresh0;
    }
    return TF_OK;
}

template <typename T>
static int solve_impl(PcgImpl* h, const void* scale, const void* b, const void* inv, void* x,
                      int has_x0, double tol, int max_iter, int recompute, double* history,
                      tf_pcg_report* rep)
{
    cudaStream_t st = h->stream;
    const size_t vb = sizeof(T) * h->n_dof;
    TF_CUDA_TRY(cudaMemcpyAsync(h->scale, scale, sizeof(T) * h->n_elem, cudaMemcpyDeviceToDevice, st));
    TF_CUDA_TRY(cudaMemcpyAsync(h->b, b, vb, cudaMemcpyDeviceToDevice, st));
    TF_CUDA_TRY(cudaMemcpyAsync(h->inv, inv, vb, cudaMemcpyDeviceToDevice, st));
    if (has_x0)
        TF_CUDA_TRY(cudaMemcpyAsync(h->x, x, vb, cudaMemcpyDeviceToDevice, st));
    else
        TF_CUDA_TRY(cudaMemsetAsync(h->x, 0, vb, st));
    CgScalars init = {};
    init.tol = tol;
    init.max_iter = max_iter;
    init.recompute = recompute;
    init.hist = history;
    init.quantize = h->quantize;
    *h->sc_host = init;
    TF_CUDA_TRY(cudaMemcpyAsync(h->sc, h->sc_host, sizeof(CgScalars), cudaMemcpyHostToDevice, st));
    if (h->resident) {
        int rc = launch_pcg_resident<T>(h->rplan, h->grid, (const T*)h->ke.data(), has_x0, (const T*)h->scale,
                                        (const T*)h->b, (const T*)h->inv, (T*)h->x, (T*)h->r, (T*)h->p,
                                        (T*)h->p2, h->node_fixed, h->ring, h->sc, (T*)h->r2, (T*)h->q,
                                        (T*)h->q2, st);
        if (rc) return rc;
        TF_CUDA_TRY(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
        TF_CUDA_TRY(cudaStreamSynchronize(st));
    }
    CgP<T> P = params_of<T>(h);
    if (h->resident) {
        // solved above
    } else if (has_x0) {
        int rc = enqueue_matvec<T>(h, P.x, P.q, nullptr, st);
        if (rc) return rc;
    }
    if (!h->resident) {
        k_init<T><<<h->n_vec_blocks, VEC_BLOCK, 0, st>>>(P, has_x0);
        TF_CHECK_LAUNCH();
        TF_CUDA_TRY(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
        TF_CUDA_TRY(cudaStreamSynchronize(st));
    }
    if (h->resident) {
        // done
    } else if (!h->sc_host->done && !getenv("TF_PCG_NOGRAPH")) {
        cudaGraphExec_t ex = h->exec;
        // refresh period divisible by 10 or 5 (default 50; 0 = never): the
        // sparse-refresh graph (TF_PCG_SPARSE_IF=0 keeps the per-iteration IF)
        const char* es = getenv("TF_PCG_SPARSE_IF");
        if (!h->fused && !(es && es[0] == '0')) {
            const int k = (recompute <= 0 || recompute % 10 == 0) ? 0 : (recompute % 5 == 0 ? 1 : -1);
            if (k >= 0) {
                if (!h->exec_sp[k]) {
                    const int rc = build_graph<T>(h, k == 0 ? 10 : 5, &h->graph_sp[k], &h->exec_sp[k]);
                    if (rc) return rc;
                }
                ex = h->exec_sp[k];
            }
        }
        TF_CUDA_TRY(cudaGraphLaunch(ex, st));
        TF_CUDA_TRY(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
    } else if (!h->sc_host->done) {
        // profiling mode: the same kernels launched one by one (ncu cannot
        // attribute kernels inside conditional graph nodes)
        CgP<T> D = P;
        D.in_graph = 0;
        while (!h->sc_host->done) {
            int rc = enqueue_part1<T>(h, D, st);
            if (rc) return rc;
            TF_CUDA_TRY(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
            TF_CUDA_TRY(cudaStreamSynchronize(st));
            if (h->sc_host->refresh && !h->sc_host->done) {
                rc = enqueue_refresh<T>(h, D, st);
                if (rc) return rc;
            }
            if (!h->fused) {
                k_direction<T><<<h->n_vec_blocks, VEC_BLOCK, 0, st>>>(D, h->n_vec_blocks);
                TF_CHECK_LAUNCH();
            }
            TF_CUDA_TRY(cudaMemcpyAsync(h->sc_host, h->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
            TF_CUDA_TRY(cudaStreamSynchronize(st));
        }
    }
    if (h->sc_host->zero_rhs)
        TF_CUDA_TRY(cudaMemsetAsync(x, 0, vb, st));
    else
        TF_CUDA_TRY(cudaMemcpyAsync(x, h->x, vb, cudaMemcpyDeviceToDevice, st));
    TF_CUDA_TRY(cudaStreamSynchronize(st));
    const CgScalars& s = *h->sc_host;
    rep->iterations = s.it;
    rep->termination = s.term;
    rep->matvecs = s.matvecs;
    rep->rel_residual = s.rel;
    return TF_OK;
}

}  // namespace tf

using namespace tf;

extern "C" {

int tf_pcg_create(tf_pcg** out, const tf_pcg_desc* d, void* stream)
{
    TF_REQUIRE(out && d, "null argument");
    TF_REQUIRE(d->precision == 32 || d->precision == 64 || d->precision == 16,
               "precision must be 32, 64 or 16 (emulated bf16)");
    TF_REQUIRE(d->precision != 16 || !d->structured, "emulated bf16 runs the general-edof kernels");
    TF_REQUIRE(d->n_dof > 0 && d->n_elem > 0 && d->ke, "empty problem");
    PcgImpl* h = new PcgImpl();
    h->prec = d->precision;
    h->quantize = 0;
    h->structured = d->structured;
    if (d->structured) h->grid = make_grid(&d->grid);
    h->edof = d->edof;
    h->n_elem = d->n_elem;
    h->n_dof = d->n_dof;
    const size_t es = d->precision == 64 ? 8 : 4;
    h->ke.assign((const unsigned char*)d->ke, (const unsigned char*)d->ke + 576 * es);
    h->node_fixed = d->node_fixed;
    h->fixed = d->fixed;
    h->n_fixed = d->n_fixed;
    h->variant = d->grid_variant;
    h->stream = reinterpret_cast<cudaStream_t>(stream);
    h->graph = nullptr;
    h->exec = nullptr;
    h->graph_sp[0] = h->graph_sp[1] = nullptr;
    h->exec_sp[0] = h->exec_sp[1] = nullptr;
    h->x = h->r = h->p = h->q = h->b = h->inv = h->scale = nullptr;
    h->p2 = nullptr;
    h->r2 = h->q2 = nullptr;
    h->part = nullptr;
    h->part_mv = nullptr;
    h->tickets = nullptr;
    h->sc = nullptr;
    h->sc_host = nullptr;
    h->resident = 0;
    h->ring = nullptr;
    TF_REQUIRE(d->structured || d->edof, "edof required for unstructured problems");

    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    // vector kernels: one 16-byte chunk per thread ...
    // ... but no more than 3 CTAs per SM while the CG working set (~6
    // vectors) is below ~200 MB, 4 beyond (graph-protocol us/iteration vs the
    // former 8 per SM: c4 FP32 47.1 vs 53.2, c4 FP64 88.1 vs 92.0, c3 FP32
    // 34.3 vs 40.4, c3 FP64 46.5 vs 53.5; c5 FP32 207 vs 212 at 4 per SM)
    const long long want = (d->n_dof + VEC_BLOCK * 4 - 1) / (VEC_BLOCK * 4);
    const int per_sm = 6.0 * (double)es * (double)d->n_dof <= 200e6 ? 3 : 4;
    h->n_vec_blocks = (int)std::min<long long>(std::max<long long>(want, 1), (long long)nsm * per_sm);
    if (const char* e = getenv("TF_VEC_BLOCKS")) h->n_vec_blocks = std::max(1, atoi(e));  // experiments
    if (d->structured)
        h->n_mv_blocks = d->precision == 32
                             ? grid_matvec_blocks<float>(h->grid, (const float*)d->ke, d->grid_variant)
                             : grid_matvec_blocks<double>(h->grid, (const double*)d->ke, d->grid_variant);
    else
        h->n_mv_blocks = 0;
    const size_t vb = es * d->n_dof;
    void** bufs[] = {&h->x, &h->r, &h->p, &h->q, &h->b, &h->inv};
    for (void** pb : bufs) TF_CUDA_TRY(cudaMalloc(pb, vb));
    // fused protocol (direction folded into the matvec staging, 2 launches per
    // iteration): wins on small, launch-bound systems (c1 SIMP 5.7 vs 6.5 ms/it)
    // and loses on large ones (register-path staging: c2 34 vs 30 us/it, c5
    // 163 vs 151 us for matvec+direction) -> default below 100k elements;
    // TF_PCG_FUSED=0/1 forces either protocol.
    h->fused = 0;
    if (d->structured && d->grid_variant == TF_GRID_FAST) {
        const bool ok = d->precision == 32 ? launch_grid_tile_supported<float>((const float*)d->ke)
                                           : launch_grid_tile_supported<double>((const double*)d->ke);
        const char* e = getenv("TF_PCG_FUSED");
        const bool want = e ? (e[0] == '1') : (d->n_elem <= 100000);
        h->fused = (ok && want && !(d->flags & TF_PCG_PLAIN_GRAPH)) ? 1 : 0;
    }
    // SM-resident protocol: the whole solve in one cooperative launch whenever
    // the full CG state of the owned DOFs fits in the co-resident CTAs' shared
    // memory.  The lean layout (x and D^-1 left in global memory) measured
    // slower than the graph protocol once the graph's vector kernels were
    // tuned (c2 FP64 33.1 vs 31.1 us/iteration, c3 FP32 37.6 vs 34.7), so it
    // is used only when forced (TF_PCG_RESIDENT=1; =0 disables the protocol)
    if (d->structured && d->grid_variant == TF_GRID_FAST && !(d->flags & TF_PCG_PLAIN_GRAPH)) {
        const char* e = getenv("TF_PCG_RESIDENT");
        if (!(e && e[0] == '0')) {
            const bool ok = d->precision == 32
                                ? pcg_resident_plan<float>(h->grid, (const float*)d->ke, &h->rplan)
                                : pcg_resident_plan<double>(h->grid, (const double*)d->ke, &h->rplan);
            const bool forced = e && e[0] == '1';
            h->resident = (ok && (forced || !h->rplan.lean)) ? 1 : 0;
        }
    }
    if (h->resident) {
        h->fused = 0;
        TF_CUDA_TRY(cudaMalloc(&h->ring, sizeof(double) * pcg_resident_ring_doubles(h->rplan)));
    }
    if (h->fused || h->resident) TF_CUDA_TRY(cudaMalloc(&h->p2, vb));
    if (h->resident && h->rplan.onex) {
        TF_CUDA_TRY(cudaMalloc(&h->r2, vb));
        TF_CUDA_TRY(cudaMalloc(&h->q2, vb));
        // halo reads of the first iterations stay finite
        TF_CUDA_TRY(cudaMemset(h->r2, 0, vb));
        TF_CUDA_TRY(cudaMemset(h->q2, 0, vb));
        TF_CUDA_TRY(cudaMemset(h->q, 0, vb));
    }
    if (h->resident) {
        // p buffers are read before first written only behind the `first` flag,
        // but keep them finite for the halo reads of the first iteration
        TF_CUDA_TRY(cudaMemset(h->p, 0, vb));
        TF_CUDA_TRY(cudaMemset(h->p2, 0, vb));
    }
    TF_CUDA_TRY(cudaMalloc(&h->scale, es * d->n_elem));
    const long long npart = (long long)h->n_vec_blocks * 3 + 8;
    TF_CUDA_TRY(cudaMalloc(&h->part, sizeof(double) * npart));
    TF_CUDA_TRY(cudaMalloc(&h->part_mv, sizeof(double) * (std::max<long long>(h->n_mv_blocks, h->n_vec_blocks) + 8)));
    TF_CUDA_TRY(cudaMalloc(&h->tickets, sizeof(unsigned) * 8));
    TF_CUDA_TRY(cudaMemset(h->tickets, 0, sizeof(unsigned) * 8));
    TF_CUDA_TRY(cudaMalloc(&h->sc, sizeof(CgScalars)));
    TF_CUDA_TRY(cudaMallocHost(&h->sc_host, sizeof(CgScalars)));
    int rc = h->resident ? TF_OK : (d->precision != 64 ? build_graph<float>(h) : build_graph<double>(h));
    if (!rc && !h->resident && !h->fused) {
        // the sparse-refresh graph of the default refresh period, up front
        // (not in the first solve's time)
        rc = d->precision != 64 ? build_graph<float>(h, 10, &h->graph_sp[0], &h->exec_sp[0])
                                : build_graph<double>(h, 10, &h->graph_sp[0], &h->exec_sp[0]);
    }
    if (rc) {
        tf_pcg_destroy(reinterpret_cast<tf_pcg*>(h));
        return rc;
    }
    *out = reinterpret_cast<tf_pcg*>(h);
    return TF_OK;
}

int tf_pcg_solve(tf_pcg* hh, const void* scale, const void* b, const void* inv_diag, void* x,
                 int has_x0, double rel_tol, int32_t max_iter, int32_t recompute_every,
                 double* history, tf_pcg_report* report)
{
    PcgImpl* h = reinterpret_cast<PcgImpl*>(hh);
    TF_REQUIRE(h && scale && b && inv_diag && x && report, "null argument");
    TF_REQUIRE(rel_tol > 0 && max_iter >= 1 && recompute_every >= 0, "invalid CG configuration");
    return h->prec != 64 ? solve_impl<float>(h, scale, b, inv_diag, x, has_x0, rel_tol, max_iter,
                                             recompute_every, history, report)
                         : solve_impl<double>(h, scale, b, inv_diag, x, has_x0, rel_tol, max_iter,
                                              recompute_every, history, report);
}

int tf_pcg_set_quantize_krylov(tf_pcg* hh, int on)
{
    PcgImpl* h = reinterpret_cast<PcgImpl*>(hh);
    TF_REQUIRE(h, "null handle");
    TF_REQUIRE(!on || h->prec != 64, "quantize_krylov needs FP32 storage (fp32 or bf16 operators)");
    TF_REQUIRE(!on || (!h->resident && !h->fused), "quantize_krylov runs on the plain graph protocol");
    h->quantize = on ? 1 : 0;
    return TF_OK;
}

int tf_pcg_protocol(const tf_pcg* hh)
{
    const PcgImpl* h = reinterpret_cast<const PcgImpl*>(hh);
    if (!h) return -1;
    return h->resident ? TF_PCG_RESIDENT : (h->fused ? TF_PCG_FUSED_GRAPH : TF_PCG_GRAPH);
}

int tf_pcg_destroy(tf_pcg* hh)
{
    PcgImpl* h = reinterpret_cast<PcgImpl*>(hh);
    if (!h) return TF_OK;
    if (h->exec) cudaGraphExecDestroy(h->exec);
    if (h->graph) cudaGraphDestroy(h->graph);
    for (int k = 0; k < 2; ++k) {
        if (h->exec_sp[k]) cudaGraphExecDestroy(h->exec_sp[k]);
        if (h->graph_sp[k]) cudaGraphDestroy(h->graph_sp[k]);
    }
    void* bufs[] = {h->x, h->r, h->p, h->q, h->b, h->inv, h->scale, h->p2, h->part, h->part_mv, h->tickets, h->sc,
                    h->ring, h->r2, h->q2};
    for (void* p : bufs)
        if (p) cudaFree(p);
    if (h->sc_host) cudaFreeHost(h->sc_host);
    delete h;
    return TF_OK;
}

}  // extern "C"
