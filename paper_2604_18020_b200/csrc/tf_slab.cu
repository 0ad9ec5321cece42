// Device-driven distributed Jacobi-PCG step kernels for the x-slab
// decomposition (recurrence of solver.py:57-147).
//
// One rank's CG iteration is
//     q = K p                       (slab tile kernels + interface exchange, host-enqueued)
//     k_slab_pq        red[0]  = sum_owned p.q                (rank partial)
//     all-reduce red[0]                                     (NCCL on device memory)
//     k_slab_alpha     decisions from the global p.q, x += a p, r -= a q,
//                      z = r / d, red[1..2] = (r.r, r.z) partials
//     all-reduce red[1..2]
//     k_slab_beta      rel = |r| / |b|; stop, or p = z + b p
// (the native runtime runs the single-reduction variant below instead:
// k_slab_dots8, ONE all-reduce, k_slab_step)
// with every scalar living in device memory, so the host enqueues iterations
// back to back and looks at the state only every few iterations.  The stop is
// exact: once a rank's state says "stopped" every later kernel of the solve
// is a no-op (all ranks hold the same all-reduced scalars, so they stop at
// the same iteration), and the iteration count is the device's.
//
// Partial dots: per-block sums in a fixed order plus a last-block fixed-order
// reduction (deterministic for a given launch shape); owner-computes mask
// (the replicated interface plane counts on the lower rank only).  Scalars
// are rounded to the working precision exactly like the single-GPU solver.

#include "tf_common.cuh"

namespace tf {

constexpr int SLAB_BLOCK = 256;

// device state (doubles, so the host reads it as one float64 tensor)
struct SlabCgState {
    double rz;      // rounded r.z of the current direction
    double bnorm;   // |b| (working-precision rounded)
    double rel;     // last relative residual
    double it;      // iterations taken
    double active;  // 1 while iterating
    double term;    // 0 running, 1 converged, 2 breakdown, 3 diverged
    double tol;
    double pad;
};

constexpr int SLAB_RUNNING = 0, SLAB_CONVERGED = 1, SLAB_BREAKDOWN = 2, SLAB_DIVERGED = 3;

// Fixed-order block reduction of K values; the last block to finish reduces
// all block partials in index order and stores the totals to out[0..K).
template <int K>
__device__ void slab_reduce(double (&v)[K], double* part, unsigned* ticket, double* out)
{
    __shared__ double sh[K][SLAB_BLOCK / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
        if (lane == 0) sh[k][wid] = v[k];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < SLAB_BLOCK / 32; ++w) s += sh[k][w];
            part[(size_t)blockIdx.x * K + k] = s;
        }
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += SLAB_BLOCK)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] += __ldcg(part + (size_t)i * K + k);
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_down_sync(0xffffffffu, acc[k], o);
    }
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < K; ++k) sh[k][wid] = acc[k];
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
            for (int w = 0; w < SLAB_BLOCK / 32; ++w) s += sh[k][w];
            out[k] = s;
        }
        *ticket = 0u;
    }
}

__device__ __forceinline__ bool slab_active(const SlabCgState* st) { return __ldcg(&st->active) != 0.0; }

// out = sum_owned a.b (owned nullable = all)
template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_dot(long long n, const T* __restrict__ a, const T* __restrict__ b, const uint8_t* __restrict__ owned,
           const SlabCgState* st, double* part, unsigned* ticket, double* out)
{
    if (st && !slab_active(st)) return;
    double v[1] = {0.0};
    for (long long i = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * SLAB_BLOCK)
        if (!owned || owned[i]) v[0] += (double)a[i] * (double)b[i];
    slab_reduce<1>(v, part, ticket, out);
}

// z = r / d (as r * inv), p = z; red[1] = r.r, red[2] = r.z partials
template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_begin(long long n, const T* __restrict__ r, const T* __restrict__ inv, T* __restrict__ z, T* __restrict__ p,
             const uint8_t* __restrict__ owned, double* part, unsigned* ticket, double* red)
{
    double v[2] = {0.0, 0.0};
    for (long long i = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * SLAB_BLOCK) {
        const T ri = r[i], zi = ri * inv[i];
        z[i] = zi;
        p[i] = zi;
        if (!owned || owned[i]) {
            v[0] += (double)ri * (double)ri;
            v[1] += (double)ri * (double)zi;
        }
    }
    slab_reduce<2>(v, part, ticket, red + 1);
}

// global red[1] = r.r, red[2] = r.z, red[3] = b.b: initial scalars (solver.py:88-103)
__global__ void k_slab_start(SlabCgState* st, const double* red, double tol, int f32)
{
    const double bn = cg_sqrt(cg_round(red[3], f32), f32);
    const double rel = cg_sqrt(cg_round(red[1], f32), f32) / bn;
    st->bnorm = bn;
    st->rz = cg_round(red[2], f32);
    st->rel = rel;
    st->it = 0.0;
    st->tol = tol;
    st->pad = 0.0;  // ticket word of k_slab_beta
    st->term = rel <= tol ? SLAB_CONVERGED : SLAB_RUNNING;
    st->active = rel <= tol ? 0.0 : 1.0;
}

// decisions from the global p.q (red[0]), then x += a p; r -= a q (refresh:
// r is recomputed by k_slab_residual after the host's x matvec); z = r*inv;
// red[1..2] = (r.r, r.z) partials
template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_alpha(long long n, T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p, const T* __restrict__ q,
             const T* __restrict__ inv, T* __restrict__ z, const uint8_t* __restrict__ owned, SlabCgState* st,
             double* red, int refresh, double* part, unsigned* ticket)
{
    if (!slab_active(st)) return;
    const bool f32 = sizeof(T) == 4;
    const double pq = cg_round(__ldcg(red), f32), rz = __ldcg(&st->rz);
    const bool bad = !isfinite(pq) || !isfinite(rz);
    if (bad || pq <= 0.0) {
        // every block takes the same decision; block 0 records it
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->it += 1.0;
            st->term = bad ? SLAB_DIVERGED : SLAB_BREAKDOWN;
            st->active = 0.0;
        }
        return;
    }
    const T alpha = (T)(rz / pq);
    double v[2] = {0.0, 0.0};
    for (long long i = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * SLAB_BLOCK) {
        x[i] = x[i] + alpha * p[i];
        if (!refresh) {
            const T ri = r[i] - alpha * q[i];
            const T zi = ri * inv[i];
            r[i] = ri;
            z[i] = zi;
            if (!owned || owned[i]) {
                v[0] += (double)ri * (double)ri;
                v[1] += (double)ri * (double)zi;
            }
        }
    }
    if (refresh) return;  // partials come from k_slab_residual
    slab_reduce<2>(v, part, ticket, red + 1);
}

// refresh iteration: r = b - w (w = K x), z = r*inv, red[1..2] partials
template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_residual(long long n, const T* __restrict__ b, const T* __restrict__ w, T* __restrict__ r,
                const T* __restrict__ inv, T* __restrict__ z, const uint8_t* __restrict__ owned,
                const SlabCgState* st, double* red, double* part, unsigned* ticket)
{
    if (!slab_active(st)) return;
    double v[2] = {0.0, 0.0};
    for (long long i = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * SLAB_BLOCK) {
        const T ri = b[i] - w[i], zi = ri * inv[i];
        r[i] = ri;
        z[i] = zi;
        if (!owned || owned[i]) {
            v[0] += (double)ri * (double)ri;
            v[1] += (double)ri * (double)zi;
        }
    }
    slab_reduce<2>(v, part, ticket, red + 1);
}

// stop rule and direction update from the global (r.r, r.z) in red[1..2]
template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_beta(long long n, T* __restrict__ p, const T* __restrict__ z, SlabCgState* st, const double* red,
            double* hist, int hist_len)
{
    if (!slab_active(st)) return;
    const bool f32 = sizeof(T) == 4;
    const double rn = cg_sqrt(cg_round(__ldcg(red + 1), f32), f32);
    const double it = __ldcg(&st->it) + 1.0;
    const double rel = rn / __ldcg(&st->bnorm);
    if (!isfinite(rn)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->it = it;
            st->term = SLAB_DIVERGED;
            st->active = 0.0;
        }
        return;
    }
    if (rel <= __ldcg(&st->tol)) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->it = it;
            st->rel = rel;
            st->term = SLAB_CONVERGED;
            st->active = 0.0;
            if (hist && (int)it < hist_len) hist[(int)it] = rel;
        }
        return;
    }
    const double rz_new = cg_round(__ldcg(red + 2), f32);
    const T beta = (T)(rz_new / __ldcg(&st->rz));
    for (long long i = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * SLAB_BLOCK)
        p[i] = z[i] + beta * p[i];
    // every block has read st->rz above; grid-wide ordering of the state
    // update: the LAST block to pass here writes it
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* ticket = reinterpret_cast<unsigned*>(&st->pad);
        __threadfence();
        last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        st->it = it;
        st->rel = rel;
        st->rz = rz_new;
        if (hist && (int)it < hist_len) hist[(int)it] = rel;
        *reinterpret_cast<unsigned*>(&st->pad) = 0u;
    }
}

// Single-reduction iteration (one all-reduce per CG iteration instead of
// two; the resident PCG's recurrence, tf_pcg_resident.cu): after q = K p
//     k_slab_dots8   red[0..7] = owned sums p.q, r.r, r.z (z = r*inv), r.q,
//                    q.q, r.Dq, q.Dq, r.Dr                (rank partials)
//     all-reduce red[0..7]
//     k_slab_step    alpha = r.z / p.q exactly as k_slab_alpha's; the next
//                    residual's r.r and r.z expanded one step in FP64 from
//                    this iteration's direct sums -> stop rule, beta; then
//                    x += a p, r -= a q, z = r*inv, p = z + b p in one pass.
// A refresh iteration runs k_slab_step(refresh) (x += a p only, rz kept for
// beta) and then the classic residual / all-reduce / k_slab_beta.
template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_dots8(long long n, const T* __restrict__ p, const T* __restrict__ q, const T* __restrict__ r,
             const T* __restrict__ inv, const uint8_t* __restrict__ owned, const SlabCgState* st, double* part,
             unsigned* ticket, double* red)
{
    if (st && !slab_active(st)) return;
    double v[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (long long i = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * SLAB_BLOCK) {
        if (owned && !owned[i]) continue;
        const T ri = r[i], qi = q[i], di = inv[i];
        const T zi = ri * di;
        const double dr = (double)ri, dq = (double)qi, dd = (double)di;
        v[0] += (double)p[i] * dq;
        v[1] += dr * dr;
        v[2] += dr * (double)zi;
        v[3] += dr * dq;
        v[4] += dq * dq;
        v[5] += dr * dd * dq;
        v[6] += dq * dd * dq;
        v[7] += dr * dd * dr;
    }
    slab_reduce<8>(v, part, ticket, red);
}

template <typename T>
__global__ void __launch_bounds__(SLAB_BLOCK)
k_slab_step(long long n, T* __restrict__ x, T* __restrict__ r, T* __restrict__ p, const T* __restrict__ q,
            const T* __restrict__ inv, T* __restrict__ z, SlabCgState* st, const double* red, int refresh,
            double* hist, int hist_len)
{
    if (!slab_active(st)) return;
    const bool f32 = sizeof(T) == 4;
    const double pq = cg_round(__ldcg(red), f32), rz = cg_round(__ldcg(red + 2), f32);
    const double it = __ldcg(&st->it) + 1.0;
    const bool bad = !isfinite(pq) || !isfinite(rz);
    __shared__ bool last;
    // the state is written by the LAST block to finish (every block reads it first)
    auto commit = [&](auto&& write) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned* ticket = reinterpret_cast<unsigned*>(&st->pad);
            __threadfence();
            last = atomicAdd(ticket, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (last && threadIdx.x == 0) {
            write();
            *reinterpret_cast<unsigned*>(&st->pad) = 0u;
        }
    };
    if (bad || pq <= 0.0) {
        commit([&] {
            st->it = it;
            st->term = bad ? SLAB_DIVERGED : SLAB_BREAKDOWN;
            st->active = 0.0;
        });
        return;
    }
    const T a = (T)(rz / pq);
    const long long stride = (long long)gridDim.x * SLAB_BLOCK;
    const long long i0 = (long long)blockIdx.x * SLAB_BLOCK + threadIdx.x;
    if (refresh) {  // x += a p; r, z, beta and the stop rule follow the true residual
        for (long long i = i0; i < n; i += stride) x[i] = x[i] + a * p[i];
        commit([&] { st->rz = rz; });
        return;
    }
    const double da = (double)a;
    const double rr1 = __ldcg(red + 1) - 2.0 * da * __ldcg(red + 3) + da * da * __ldcg(red + 4);
    const double rz1 = __ldcg(red + 7) - 2.0 * da * __ldcg(red + 5) + da * da * __ldcg(red + 6);
    const double rn = cg_sqrt(cg_round(rr1, f32), f32);
    const double rel = rn / __ldcg(&st->bnorm);
    const bool stop = !isfinite(rn) || rel <= __ldcg(&st->tol);
    const T beta = (T)(cg_round(rz1, f32) / rz);
    for (long long i = i0; i < n; i += stride) {
        x[i] = x[i] + a * p[i];
        if (!stop) {
            const T ri = r[i] - a * q[i];
            const T zi = ri * inv[i];
            r[i] = ri;
            z[i] = zi;
            p[i] = zi + beta * p[i];
        }
    }
    commit([&] {
        st->it = it;
        if (isfinite(rn)) {
            st->rel = rel;
            if (hist && (int)it < hist_len) hist[(int)it] = rel;
        }
        if (stop) {
            st->term = isfinite(rn) ? SLAB_CONVERGED : SLAB_DIVERGED;
            st->active = 0.0;
        } else {
            st->rz = cg_round(rz1, f32);
        }
    });
}

static int slab_blocks(long long n)
{
    static int nsm = 0;
    if (!nsm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    return (int)std::max<long long>(1, std::min<long long>((n + SLAB_BLOCK - 1) / SLAB_BLOCK, 4LL * nsm));
}

}  // namespace tf

using namespace tf;

static inline cudaStream_t SL(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int64_t tf_slab_work_doubles(int64_t n)
{
    return 8LL * slab_blocks(n) + 8;  // K<=8 partials per block, then the ticket words
}

#define TF_SLAB_API(T, SUF)                                                                                  \
    int tf_slab_dot_##SUF(int64_t n, const T* a, const T* b, const uint8_t* owned, double* out, double* work, \
                          void* stream)                                                                      \
    {                                                                                                        \
        TF_REQUIRE(n > 0 && a && b && out && work, "bad arguments");                                         \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_dot<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, a, b, owned, nullptr, work,                      \
                                                         reinterpret_cast<unsigned*>(work + 8 * nb), out);   \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }                                                                                                        \
    int tf_slab_cg_pq_##SUF(int64_t n, const T* p, const T* q, const uint8_t* owned, const double* state,    \
                            double* red, double* work, void* stream)                                         \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_dot<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, p, q, owned,                                     \
                                                         reinterpret_cast<const SlabCgState*>(state), work,  \
                                                         reinterpret_cast<unsigned*>(work + 8 * nb), red);   \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }                                                                                                        \
    int tf_slab_cg_begin_##SUF(int64_t n, const T* r, const T* inv, T* z, T* p, const uint8_t* owned,       \
                               double* red, double* work, void* stream)                                      \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_begin<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, r, inv, z, p, owned, work,                     \
                                                           reinterpret_cast<unsigned*>(work + 8 * nb), red); \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }                                                                                                        \
    int tf_slab_cg_alpha_##SUF(int64_t n, T* x, T* r, const T* p, const T* q, const T* inv, T* z,           \
                               const uint8_t* owned, double* state, double* red, int refresh, double* work,  \
                               void* stream)                                                                 \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_alpha<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, x, r, p, q, inv, z, owned,                     \
                                                           reinterpret_cast<SlabCgState*>(state), red,       \
                                                           refresh, work,                                    \
                                                           reinterpret_cast<unsigned*>(work + 8 * nb));      \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }                                                                                                        \
    int tf_slab_cg_residual_##SUF(int64_t n, const T* b, const T* w, T* r, const T* inv, T* z,              \
                                  const uint8_t* owned, const double* state, double* red, double* work,      \
                                  void* stream)                                                              \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_residual<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, b, w, r, inv, z, owned,                     \
                                                              reinterpret_cast<const SlabCgState*>(state),   \
                                                              red, work,                                     \
                                                              reinterpret_cast<unsigned*>(work + 8 * nb));   \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }                                                                                                        \
    int tf_slab_cg_beta_##SUF(int64_t n, T* p, const T* z, double* state, const double* red, double* hist,  \
                              int hist_len, void* stream)                                                    \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_beta<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, p, z, reinterpret_cast<SlabCgState*>(state),    \
                                                          red, hist, hist_len);                              \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }
TF_SLAB_API(float, f32)
TF_SLAB_API(double, f64)

#define TF_SLAB_ONEX_API(T, SUF)                                                                             \
    int tf_slab_cg_dots8_##SUF(int64_t n, const T* p, const T* q, const T* r, const T* inv,                  \
                               const uint8_t* owned, const double* state, double* red, double* work,        \
                               void* stream)                                                                 \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_dots8<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, p, q, r, inv, owned,                           \
                                                           reinterpret_cast<const SlabCgState*>(state), work, \
                                                           reinterpret_cast<unsigned*>(work + 8 * nb), red); \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }                                                                                                        \
    int tf_slab_cg_step_##SUF(int64_t n, T* x, T* r, T* p, const T* q, const T* inv, T* z, double* state,    \
                              const double* red, int refresh, double* hist, int hist_len, void* stream)      \
    {                                                                                                        \
        const int nb = slab_blocks(n);                                                                       \
        k_slab_step<T><<<nb, SLAB_BLOCK, 0, SL(stream)>>>(n, x, r, p, q, inv, z,                             \
                                                          reinterpret_cast<SlabCgState*>(state), red, refresh, \
                                                          hist, hist_len);                                   \
        TF_CHECK_LAUNCH();                                                                                   \
        return TF_OK;                                                                                        \
    }
TF_SLAB_ONEX_API(float, f32)
TF_SLAB_ONEX_API(double, f64)

int tf_slab_cg_start(double* state, const double* red, double rel_tol, int f32, void* stream)
{
    TF_REQUIRE(state && red, "bad arguments");
    k_slab_start<<<1, 1, 0, SL(stream)>>>(reinterpret_cast<SlabCgState*>(state), red, rel_tol, f32);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

}  // extern "C"
