// SIMP glue on the device (reference simp.py:33-175, element.py:34-45):
// cone filter and its transpose as a structured stencil, Heaviside projection,
// SIMP scale, sensitivity chain, optimality-criteria bisection, reductions.
//
// These are the callers either side of the hot path; once
// the PCG is on the device they are the Amdahl wall (host OC alone is 1.3 s
// per iteration at 4.9M elements), so they run here as well.  Reductions are
// deterministic (fixed-order partials).

#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "tf_common.cuh"

namespace cg = cooperative_groups;

namespace tf {

constexpr int MAX_OFFSETS = 343;  // reach <= 3 (rmin <= 3)

struct FilterStencil {
    int n;
    int di[MAX_OFFSETS], dj[MAX_OFFSETS], dk[MAX_OFFSETS];
    double w[MAX_OFFSETS];
};

static int make_stencil(double rmin, FilterStencil* st)
{
    const int reach = (int)std::ceil(rmin);
    if (reach > 3) return TF_ERR_UNSUPPORTED;
    st->n = 0;
    for (int dk = -reach; dk <= reach; ++dk)  // same offset order as simp.py:45-47
        for (int dj = -reach; dj <= reach; ++dj)
            for (int di = -reach; di <= reach; ++di) {
                const double w = rmin - std::sqrt((double)(di * di + dj * dj + dk * dk));
                if (w <= 0.0) continue;
                st->di[st->n] = di;
                st->dj[st->n] = dj;
                st->dk[st->n] = dk;
                st->w[st->n] = w;
                ++st->n;
            }
    return TF_OK;
}

__global__ void k_filter_rowsum(Grid g, double* __restrict__ inv, const __grid_constant__ FilterStencil st)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.n_elem) return;
    const int ex = (int)(e % g.nelx), ey = (int)((e / g.nelx) % g.nely), ez = (int)(e / ((long long)g.nelx * g.nely));
    double s = 0.0;
    for (int q = 0; q < st.n; ++q) {
        const int x = ex + st.di[q], y = ey + st.dj[q], z = ez + st.dk[q];
        if (x >= 0 && x < g.nelx && y >= 0 && y < g.nely && z >= 0 && z < g.nelz) s += st.w[q];
    }
    inv[e] = 1.0 / s;
}

// y = F x (transpose = 0) or y = F^T x (transpose = 1), F = diag(inv) W, W symmetric
__global__ void k_filter(Grid g, const double* __restrict__ inv, const double* __restrict__ x,
                         double* __restrict__ y, int transpose, const __grid_constant__ FilterStencil st)
{
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.n_elem) return;
    const int ex = (int)(e % g.nelx), ey = (int)((e / g.nelx) % g.nely), ez = (int)(e / ((long long)g.nelx * g.nely));
    const double ie = inv[e];
    double s = 0.0;
    for (int q = 0; q < st.n; ++q) {
        const int xx = ex + st.di[q], yy = ey + st.dj[q], zz = ez + st.dk[q];
        if (xx < 0 || xx >= g.nelx || yy < 0 || yy >= g.nely || zz < 0 || zz >= g.nelz) continue;
        const long long j = xx + (long long)g.nelx * (yy + (long long)g.nely * zz);
        if (transpose)
            s += (st.w[q] * inv[j]) * x[j];
        else
            s += (st.w[q] * ie) * x[j];
    }
    y[e] = s;
}

__global__ void k_project(long long n, double beta, double eta, const double* __restrict__ rb,
                          double* __restrict__ rp, double* __restrict__ dh)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double den = tanh(beta * eta) + tanh(beta * (1.0 - eta));
    const double t = beta * (rb[i] - eta);
    rp[i] = (tanh(beta * eta) + tanh(t)) / den;
    if (dh) {
        const double c = cosh(t);
        dh[i] = beta / (c * c * den);
    }
}

// scale = rho_min + (1 - rho_min) * clip(rho, 0, 1)^p  (element.py:34-39); flags bad densities
template <typename T>
__global__ void k_simp_scale(long long n, double p, double rho_min, const double* __restrict__ rho,
                             T* __restrict__ scale, int* __restrict__ bad)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double r = rho[i];
    if (r < -1e-12 || r > 1.0 + 1e-12) atomicOr(bad, 1);
    const double c = fmin(fmax(r, 0.0), 1.0);
    scale[i] = (T)(rho_min + (1.0 - rho_min) * pow(c, p));
}

// out = dH * (-p (1 - rho_min) clip(rho)^(p-1) * E)   (simp.py:96-101, 104-108 inner product)
__global__ void k_sensitivity(long long n, double p, double rho_min, const double* __restrict__ rho,
                              const double* __restrict__ energy, const double* __restrict__ dh,
                              double* __restrict__ out)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double c = fmin(fmax(rho[i], 0.0), 1.0);
    const double dc = -(p * (1.0 - rho_min) * pow(c, p - 1.0)) * energy[i];
    out[i] = dh ? dh[i] * dc : dc;
}

// ---- deterministic reductions ---------------------------------------------------------

constexpr int RED_BLOCK = 256;

template <int K>
__device__ void block_reduce_write(double (&v)[K], double* dst)
{
    __shared__ double sh[K][RED_BLOCK / 32];
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
            for (int w = 0; w < RED_BLOCK / 32; ++w) s += sh[k][w];
            dst[k] = s;
        }
    }
    __syncthreads();
}

// partial sums of (a.b, sum a*(1-a), sum c) -- one kernel for the SIMP scalars
__global__ void __launch_bounds__(RED_BLOCK)
k_stats_partial(long long n, const double* __restrict__ a, const double* __restrict__ b,
                const double* __restrict__ gray, const double* __restrict__ vol, double* __restrict__ part)
{
    double v[3] = {0.0, 0.0, 0.0};
    for (long long i = (long long)blockIdx.x * RED_BLOCK + threadIdx.x; i < n; i += (long long)gridDim.x * RED_BLOCK) {
        if (a) v[0] += a[i] * b[i];
        if (gray) v[1] += gray[i] * (1.0 - gray[i]);
        if (vol) v[2] += vol[i];
    }
    block_reduce_write<3>(v, part + 3 * blockIdx.x);
}

__global__ void k_stats_final(int nb, const double* __restrict__ part, double* __restrict__ out)
{
    double v[3] = {0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < nb; i += RED_BLOCK)
#pragma unroll
        for (int k = 0; k < 3; ++k) v[k] += __ldcg(part + 3 * i + k);
    block_reduce_write<3>(v, out);
}

// ---- optimality criteria (simp.py:111-175) -----------------------------------------

// Grid-wide barrier for a cooperatively launched (hence co-resident) grid:
// sense by generation counter; one arriving thread per block.
struct GridBar {
    unsigned* count;
    unsigned* gen;
    __device__ void sync() const
    {
        __syncthreads();
        if (threadIdx.x == 0) {
            volatile unsigned* vg = gen;
            const unsigned g = *vg;
            __threadfence();
            if (atomicAdd(count, 1u) == gridDim.x - 1) {
                *count = 0u;
                __threadfence();
                atomicAdd(gen, 1u);
            } else {
                while (*vg == g) {
                }
            }
            __threadfence();
        }
        __syncthreads();
    }
};

struct OcParams {
    long long n;
    const double *rho, *dc, *dv;
    double vf, move, vol_tol, damping;
    int max_bisect;
    double* rho_new;
    double* part;  // 3 * gridDim, then 2 barrier words
    tf_oc_report* rep;
};

__device__ __forceinline__ double oc_cand(const OcParams& P, long long i, double lam)
{
    const double r = P.rho[i];
    const double ratio = -P.dc[i] / (P.dv ? P.dv[i] : 1.0);
    const double q = ratio / lam;
    const double f = (P.damping == 0.5) ? sqrt(q) : pow(q, P.damping);  // numpy ** 0.5 -> sqrt
    const double lo = fmax(0.0, r - P.move), hi = fmin(1.0, r + P.move);
    return fmin(fmax(r * f, lo), hi);
}

// grid-wide mean of the candidate at lam; every block obtains the same value
__device__ double oc_volume(const OcParams& P, double lam, int parity, const GridBar& grid)
{
    double v[1] = {0.0};
    for (long long i = (long long)blockIdx.x * RED_BLOCK + threadIdx.x; i < P.n; i += (long long)gridDim.x * RED_BLOCK)
        v[0] += oc_cand(P, i, lam);
    double* part = P.part + parity * gridDim.x;
    block_reduce_write<1>(v, part + blockIdx.x);
    grid.sync();
    __shared__ double tot;
    double s[1] = {0.0};
    for (int i = threadIdx.x; i < (int)gridDim.x; i += RED_BLOCK) s[0] += __ldcg(part + i);
    block_reduce_write<1>(s, &tot);  // tot written by thread 0, read after the block sync
    return tot / (double)P.n;
}

__global__ void __launch_bounds__(RED_BLOCK) k_oc(OcParams P)
{
    GridBar grid;
    grid.count = reinterpret_cast<unsigned*>(P.part + 3 * gridDim.x);
    grid.gen = grid.count + 1;
    // validation (simp.py:133-136): max dc, min dv
    {
        double v[1] = {0.0};
        bool bad = false;
        for (long long i = (long long)blockIdx.x * RED_BLOCK + threadIdx.x; i < P.n; i += (long long)gridDim.x * RED_BLOCK) {
            if (P.dc[i] > 1e-12) bad = true;
            if (P.dv && P.dv[i] <= 0.0) bad = true;
        }
        v[0] = bad ? 1.0 : 0.0;
        block_reduce_write<1>(v, P.part + 2 * gridDim.x + blockIdx.x);
        grid.sync();
        double s = 0.0;
        for (int i = 0; i < (int)gridDim.x; ++i) s += __ldcg(P.part + 2 * gridDim.x + i);
        if (s > 0.0) {
            if (blockIdx.x == 0 && threadIdx.x == 0) P.rep->status = TF_OC_BAD_INPUT;
            return;
        }
    }
    int parity = 0;
    int evals = 0;
    double lam_lo = 1.0, lam_hi = 1.0, lam_out = 1.0;
    int status = TF_OC_OK;
    // bracket from below: shrink lam until the step is full enough
    int k = 0;
    for (; k < 200; ++k) {
        const double vol = oc_volume(P, lam_lo, parity, grid);
        parity ^= 1;
        ++evals;
        if (vol >= P.vf) break;
        lam_lo *= 0.5;
    }
    if (k == 200) {
        lam_out = lam_lo;
        status = TF_OC_SATURATED;
    } else {
        for (k = 0; k < 200; ++k) {
            const double vol = oc_volume(P, lam_hi, parity, grid);
            parity ^= 1;
            ++evals;
            if (vol <= P.vf) break;
            lam_hi *= 2.0;
        }
        if (k == 200) {
            lam_out = lam_hi;
            status = TF_OC_SATURATED;
        } else {
            double best_err = -1.0, best_lam = 0.0;
            bool hit = false;
            for (int b = 0; b < P.max_bisect; ++b) {
                const double lam = 0.5 * (lam_lo + lam_hi);
                const double vol = oc_volume(P, lam, parity, grid);
                parity ^= 1;
                ++evals;
                const double err = fabs(vol - P.vf);
                if (best_err < 0.0 || err < best_err) {
                    best_err = err;
                    best_lam = lam;
                }
                if (err <= P.vol_tol) {
                    lam_out = lam;
                    hit = true;
                    break;
                }
                if (vol > P.vf)
                    lam_lo = lam;
                else
                    lam_hi = lam;
            }
            if (!hit) {
                lam_out = best_lam;
                status = best_err <= P.vol_tol ? TF_OC_OK : TF_OC_STALLED;
            }
            if (blockIdx.x == 0 && threadIdx.x == 0) P.rep->best_err = best_err;
        }
    }
    for (long long i = (long long)blockIdx.x * RED_BLOCK + threadIdx.x; i < P.n; i += (long long)gridDim.x * RED_BLOCK)
        P.rho_new[i] = oc_cand(P, i, lam_out);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        P.rep->status = status;
        P.rep->lam = lam_out;
        P.rep->evaluations = evals;
    }
}

// ---- distributed OC: candidate volumes at a batch of multipliers ---------------------
// Each x-slab rank sums its own elements' candidates (rank-local, fixed order);
// the host all-gathers the partial sums and runs the bisection of simp.py:111-175
// on the global means, evaluating several multipliers per round trip.

constexpr int OC_MAX_LAMS = 15;  // TF_OC_MAX_LAMS

struct OcLams {
    double lam[OC_MAX_LAMS];
    int n;
};

__global__ void __launch_bounds__(RED_BLOCK)
k_oc_volumes_partial(OcParams P, const __grid_constant__ OcLams L, double* __restrict__ part)
{
    double v[OC_MAX_LAMS + 1];
#pragma unroll
    for (int k = 0; k <= OC_MAX_LAMS; ++k) v[k] = 0.0;
    for (long long i = (long long)blockIdx.x * RED_BLOCK + threadIdx.x; i < P.n; i += (long long)gridDim.x * RED_BLOCK) {
#pragma unroll
        for (int k = 0; k < OC_MAX_LAMS; ++k)
            if (k < L.n) v[k] += oc_cand(P, i, L.lam[k]);
        if (P.dc[i] > 1e-12 || (P.dv && P.dv[i] <= 0.0)) v[OC_MAX_LAMS] += 1.0;
    }
    block_reduce_write<OC_MAX_LAMS + 1>(v, part + (OC_MAX_LAMS + 1) * blockIdx.x);
}

__global__ void __launch_bounds__(RED_BLOCK)
k_oc_volumes_final(int nb, const double* __restrict__ part, double* __restrict__ out)
{
    double v[OC_MAX_LAMS + 1];
#pragma unroll
    for (int k = 0; k <= OC_MAX_LAMS; ++k) v[k] = 0.0;
    for (int i = threadIdx.x; i < nb; i += RED_BLOCK)
#pragma unroll
        for (int k = 0; k <= OC_MAX_LAMS; ++k) v[k] += __ldcg(part + (OC_MAX_LAMS + 1) * i + k);
    block_reduce_write<OC_MAX_LAMS + 1>(v, out);
}

__global__ void k_oc_apply(OcParams P, double lam)
{
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < P.n) P.rho_new[i] = oc_cand(P, i, lam);
}

static int red_blocks(long long n)
{
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (int)std::max<long long>(1, std::min<long long>((n + RED_BLOCK - 1) / RED_BLOCK, 2LL * nsm));
}

}  // namespace tf

using namespace tf;

static inline cudaStream_t SS(void* p) { return reinterpret_cast<cudaStream_t>(p); }

extern "C" {

int tf_filter_rowsum_f64(const tf_grid* g, double rmin, double* inv_rowsum, void* stream)
{
    TF_REQUIRE(g && inv_rowsum && rmin > 0.0, "bad arguments");
    FilterStencil st;
    if (make_stencil(rmin, &st) != TF_OK) {
        set_error("filter radius %g exceeds the supported reach 3", rmin);
        return TF_ERR_UNSUPPORTED;
    }
    Grid gg = make_grid(g);
    k_filter_rowsum<<<(unsigned)((gg.n_elem + 255) / 256), 256, 0, SS(stream)>>>(gg, inv_rowsum, st);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_filter_grid_f64(const tf_grid* g, double rmin, const double* inv_rowsum, const double* x,
                       double* y, int transpose, void* stream)
{
    TF_REQUIRE(g && inv_rowsum && x && y && rmin > 0.0, "bad arguments");
    FilterStencil st;
    if (make_stencil(rmin, &st) != TF_OK) {
        set_error("filter radius %g exceeds the supported reach 3", rmin);
        return TF_ERR_UNSUPPORTED;
    }
    Grid gg = make_grid(g);
    k_filter<<<(unsigned)((gg.n_elem + 255) / 256), 256, 0, SS(stream)>>>(gg, inv_rowsum, x, y, transpose, st);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_project_f64(int64_t n, double beta, double eta, const double* rho_bar, double* rho_phys,
                   double* dh, void* stream)
{
    if (n <= 0) return TF_OK;
    k_project<<<(unsigned)((n + 255) / 256), 256, 0, SS(stream)>>>(n, beta, eta, rho_bar, rho_phys, dh);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

#define TF_SIMP_SCALE(T, SUF)                                                                 \
    int tf_simp_scale_##SUF(int64_t n, double p, double rho_min, const double* rho, T* scale,  \
                            int* bad_flag, void* stream)                                      \
    {                                                                                         \
        if (n <= 0) return TF_OK;                                                             \
        k_simp_scale<T><<<(unsigned)((n + 255) / 256), 256, 0, SS(stream)>>>(n, p, rho_min, rho, scale, bad_flag); \
        TF_CHECK_LAUNCH();                                                                    \
        return TF_OK;                                                                         \
    }
TF_SIMP_SCALE(float, f32)
TF_SIMP_SCALE(double, f64)

int tf_sensitivity_f64(int64_t n, double p, double rho_min, const double* rho_phys,
                       const double* energies, const double* dh, double* out, void* stream)
{
    if (n <= 0) return TF_OK;
    k_sensitivity<<<(unsigned)((n + 255) / 256), 256, 0, SS(stream)>>>(n, p, rho_min, rho_phys, energies, dh, out);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_stats_f64(int64_t n, const double* a, const double* b, const double* gray_of,
                 const double* sum_of, double* work, double* out3, void* stream)
{
    const int nb = red_blocks(n);
    k_stats_partial<<<nb, RED_BLOCK, 0, SS(stream)>>>(n, a, b, gray_of, sum_of, work);
    TF_CHECK_LAUNCH();
    k_stats_final<<<1, RED_BLOCK, 0, SS(stream)>>>(nb, work, out3);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int64_t tf_work_doubles(int64_t n)
{
    return 3LL * red_blocks(n) + 8;  // partials + grid-barrier words (zeroed per OC call)
}

int tf_oc_update_f64(int64_t n, const double* rho, const double* dc, const double* dv, double vf,
                     double move, double vol_tol, double damping, int max_bisect, double* rho_new,
                     double* work, tf_oc_report* rep_dev, void* stream)
{
    TF_REQUIRE(n > 0 && rho && dc && rho_new && work && rep_dev, "bad arguments");
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    TF_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_oc, RED_BLOCK, 0));
    const long long want = (n + RED_BLOCK - 1) / RED_BLOCK;
    const int nb = (int)std::max<long long>(1, std::min<long long>(want, (long long)std::min(per_sm, 2) * nsm));
    OcParams P;
    P.n = n; P.rho = rho; P.dc = dc; P.dv = dv; P.vf = vf; P.move = move; P.vol_tol = vol_tol;
    P.damping = damping; P.max_bisect = max_bisect; P.rho_new = rho_new; P.part = work; P.rep = rep_dev;
    void* args[] = {&P};
    TF_CUDA_TRY(cudaMemsetAsync(work + 3 * (long long)nb, 0, 2 * sizeof(unsigned), SS(stream)));
    TF_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_oc, dim3(nb), dim3(RED_BLOCK), args, 0, SS(stream)));
    return TF_OK;
}

int64_t tf_oc_work_doubles(int64_t n)
{
    return (int64_t)(OC_MAX_LAMS + 1) * red_blocks(n) + 8;
}

int tf_oc_volumes_f64(int64_t n, const double* rho, const double* dc, const double* dv, double move,
                      double damping, const double* lams, int n_lams, double* sums, double* work,
                      void* stream)
{
    TF_REQUIRE(n > 0 && rho && dc && lams && sums && work, "bad arguments");
    TF_REQUIRE(n_lams >= 1 && n_lams <= OC_MAX_LAMS, "n_lams must be in [1, 15]");
    OcParams P{};
    P.n = n; P.rho = rho; P.dc = dc; P.dv = dv; P.move = move; P.damping = damping;
    OcLams L{};
    for (int k = 0; k < n_lams; ++k) L.lam[k] = lams[k];
    L.n = n_lams;
    const int nb = red_blocks(n);
    k_oc_volumes_partial<<<nb, RED_BLOCK, 0, SS(stream)>>>(P, L, work);
    TF_CHECK_LAUNCH();
    k_oc_volumes_final<<<1, RED_BLOCK, 0, SS(stream)>>>(nb, work, sums);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int tf_oc_apply_f64(int64_t n, const double* rho, const double* dc, const double* dv, double move,
                    double damping, double lam, double* rho_new, void* stream)
{
    if (n <= 0) return TF_OK;
    TF_REQUIRE(rho && dc && rho_new, "bad arguments");
    OcParams P{};
    P.n = n; P.rho = rho; P.dc = dc; P.dv = dv; P.move = move; P.damping = damping; P.rho_new = rho_new;
    k_oc_apply<<<(unsigned)((n + 255) / 256), 256, 0, SS(stream)>>>(P, lam);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

}  // extern "C"
