// SM-resident Jacobi-PCG: the whole solve of reference solver.py:57-147 as ONE
// cooperative kernel launch, for structured grids whose CG state fits in the
// shared memory of the co-resident CTAs.
//
// Ownership.  The grid is the production tile decomposition (tf_tile.cu): CTA
// (bx, by, bz) owns node columns [i0, i0+31) x [j0, j0+BY-1) over node planes
// [k0, k0+oz); thread (tx, ty) owns one node column of it.  The owned DOFs'
// CG vectors x, r, D^-1, p and q live in the CTA's shared memory for the
// whole solve; they never round-trip HBM.  Only two vectors are global: z
// (= r D^-1 of the last update) and p (ping-pong), which neighbouring CTAs
// read for their halo nodes -- both stay L2-resident at the sizes that fit.
//
// Default iteration (ONEX, full layout): ONE grid exchange.  The pass stages
// p_k = D^-1 (r_{k-1} - alpha_{k-1} q_{k-1}) + beta_{k-1} p_{k-1} from the
// published r_{k-1}, q_{k-1}, p_{k-1} (the owner's arithmetic, so halo and
// owned copies agree bitwise), owners apply x_k and publish r_k, p_k, q_k;
// the exchange after it carries p.q and the own-DOF sums from which alpha_k
// (exact, r.z direct) and ||r_{k+1}||^2, r_{k+1}.z_{k+1} (one-step FP64
// expansion) follow -- see the loop below.  TF_PCG_ONEX=0 (and the lean
// layout) run the two-exchange iteration:
//
// Two-exchange iteration = two grid barriers (three on a true-residual refresh):
//   A. stage node planes of p_k = z + beta p_{k-1} (computed on the fly from
//      the global z and p_{k-1}; owners publish p_k), q = A p_k with the
//      parity-block element algebra, masked input and pass-through, per-CTA
//      p.q partial                                                --- barrier
//   B. every CTA reduces the p.q partials in the same fixed order -> alpha,
//      breakdown / divergence; x += alpha p, r -= alpha q (or, every
//      `recompute` iterations, publish x --- barrier --- r = b - A x),
//      z = r D^-1 (published), per-CTA r.r / r.z partials         --- barrier
//   C. every CTA reduces them -> rel, convergence, max_iter, beta.
// Every CTA takes the same decisions from bitwise-identical reductions, so
// the loop exits everywhere at the same iteration; CTA 0 records the report.
//
// Barrier + reduction in one step ("exchange", res_exchange below): partials
// published, one release-add on an arrival counter, fixed-order sum of all
// partials after the counter completes.
//
// Layout: "full" keeps x, r, D^-1, p, q of the owned DOFs in shared memory;
// "lean" (larger grids) keeps r, p, q there and x (read-modify-write by the
// owner) and D^-1 (read-only) in global memory.
// Scalar rounding is the numpy semantics of tf_pcg.cu (FP32 dots rounded to
// float32, alpha/beta applied in the working dtype, no FMA contraction in
// vector updates).

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <utility>
#include <vector>

#include "tf_common.cuh"
#include "tf_walsh.cuh"

namespace tf {

template <typename T>
bool tile_iso_enabled();  // tf_tile.cu

template <typename T>
struct ResArgs {
    Grid g;
    int oz;
    int has_x0;
    const T* scale;
    const T* b;
    const T* inv;
    T* x;        // in: x0 (has_x0); out: the solution (every DOF written by its owner)
    T* z;        // z = r * D^-1 of the last update (halo source for p)
    T* pbuf[2];  // p_k in pbuf[k & 1]
    const uint8_t* node_fixed;
    double* ring;  // [2][nblk][RES_SLOT] exchange partials, then the arrival counter
    // single-exchange iteration (onex): r_k, q_k published for the halo
    // recomputation of p_{k+1} (ping-pong by k & 1)
    T* rbuf[2];
    T* qbuf[2];
    int onex;
    int lean;      // x and D^-1 in global memory instead of shared memory
    int iso;       // isotropic block form (block_iso) instead of the generic blocks
    KhatIso<T> ki;
    CgScalars* sc;  // tol / max_iter / recompute / hist in; report out
    unsigned long long* trace;  // nullable: CTA 0 phase times (ns), TF_PCG_TRACE
};

__device__ __forceinline__ unsigned long long res_gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned res_ld_acquire(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void res_red_release(unsigned* p, unsigned v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Exchange number `phase`: publish this CTA's K partials (valid in every
// thread, e.g. from res_block_sum) and return the fixed-order totals over all
// CTAs in every thread.  Doubles as the grid barrier: on return every CTA has
// arrived, and everything each wrote before arriving is visible.
// Arrival: partials into slot [phase & 1] (rewritten two exchanges later,
// after every reader has arrived at the exchange in between), fence, one
// red.release on a monotonic counter; thread 0 polls the counter with acquire
// loads until all nblk arrivals of this phase are in; warp 0 then sums the
// partials in CTA order (measured on B200: 3.1 us per exchange at 296 CTAs,
// vs 7.1 us for per-CTA sentinel slots polled by every CTA -- L2 flooding --
// and 3.6 us for a count-reset/generation barrier; scripts/exchange_bench.cu).
constexpr int RES_SLOT = 8;  // doubles per CTA and exchange slot (K <= 8)

template <int K>
__device__ __noinline__ void res_arrive(double* part, unsigned* ctr, int nblk, int bid, int tid, unsigned phase,
                                        const double (&v)[K])
{
    double* slot = part + (size_t)(phase & 1u) * nblk * RES_SLOT;
    __syncthreads();  // the CTA's data writes precede the release below
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) slot[(size_t)bid * RES_SLOT + k] = v[k];
        // the release is cumulative over the CTA's writes ordered by the
        // barrier above (no separate fence: 0.26 us less per exchange at 296
        // CTAs, scripts/exchange_bench.cu modes 1 vs 6)
        res_red_release(ctr, 1u);
    }
}

template <int K>
__device__ __noinline__ void res_wait(const double* part, const unsigned* ctr, int nblk, int tid, unsigned phase,
                                      double (&v)[K], double* sh /* >= K */)
{
    const double* slot = part + (size_t)(phase & 1u) * nblk * RES_SLOT;
    if (tid == 0) {
        const unsigned target = (phase + 1u) * (unsigned)nblk;
        while (res_ld_acquire(ctr) < target) __nanosleep(20);
    }
    __syncthreads();
    if constexpr (K > 4) {
        // wide payloads: every thread sums value k = tid % 8 of CTAs tid / 8,
        // + nt / 8, ... (its loads issued together), then thread k adds the
        // nt / 8 column sums in order -- warp 0 alone would need one L2 round
        // trip per 32 CTAs for 8 values each
        __shared__ double wide[512];
        const int nt = (int)(blockDim.x * blockDim.y);
        const int k = tid & 7, js = nt >> 3;
        double acc = 0.0;
        if (k < K) {
            constexpr int U = 8;
            for (int j = tid >> 3; j < nblk; j += js * U) {
                double t[U];
#pragma unroll
                for (int u = 0; u < U; ++u)
                    t[u] = j + u * js < nblk ? __ldcg(slot + (size_t)(j + u * js) * RES_SLOT + k) : 0.0;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (j + u * js < nblk) acc += t[u];
            }
        }
        wide[tid] = acc;
        __syncthreads();
        if (tid < K) {
            double s2 = 0.0;
            for (int jj = 0; jj < js; ++jj) s2 += wide[jj * 8 + tid];
            sh[tid] = s2;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < K; ++kk) v[kk] = sh[kk];
        __syncthreads();
        return;
    }
    if (tid < 32) {
        double acc[K];
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = 0.0;
        // the partials of 8 rounds are loaded before any is added (one L2
        // round trip per 256 CTAs instead of one per 32-128); the adds keep
        // the ascending-CTA order of each lane
        constexpr int U = 8;
        for (int i0 = tid; i0 < nblk; i0 += 32 * U) {
            double t[U][K];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int k = 0; k < K; ++k)
                    t[u][k] = i0 + 32 * u < nblk ? __ldcg(slot + (size_t)(i0 + 32 * u) * RES_SLOT + k) : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (i0 + 32 * u < nblk) {
#pragma unroll
                    for (int k = 0; k < K; ++k) acc[k] += t[u][k];
                }
        }
#pragma unroll
        for (int k = 0; k < K; ++k) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], o);
        }
        if (tid == 0) {
#pragma unroll
            for (int k = 0; k < K; ++k) sh[k] = acc[k];
        }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = sh[k];
    __syncthreads();
}

// arrive + wait; work that no other CTA needs before the next exchange can be
// placed between the two halves (res_arrive / res_wait) to hide the latency
template <int K, int NT>
__device__ __forceinline__ void res_exchange(double* part, unsigned* ctr, int nblk, int bid, int tid,
                                             unsigned phase, double (&v)[K], double* sh /* >= K */)
{
    res_arrive<K>(part, ctr, nblk, bid, tid, phase, v);
    res_wait<K>(part, ctr, nblk, tid, phase, v, sh);
}

// Deterministic block sum of K values, returned in thread 0 (the only
// thread whose values res_arrive publishes; the exchange then gives every
// thread the grid totals).
template <int K, int NT>
__device__ __forceinline__ void res_block_sum(double (&v)[K], double* sh /* [K][NT/32] */, int tid)
{
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_down_sync(0xffffffffu, v[k], o);
    }
    if ((tid & 31) == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) sh[k * (NT / 32) + (tid >> 5)] = v[k];
    }
    __syncthreads();
    if (tid == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < NT / 32; ++i) s += sh[k * (NT / 32) + i];
            v[k] = s;
        }
    }
    __syncthreads();
}

// The CTA's staging slots of a node plane and its owned-column bookkeeping.
template <typename T, int BY_>
struct ResTile {
    static constexpr int BY = BY_, NT = TILE_BX * BY_;
    static constexpr int PW = (TILE_BX + 1) * 3, PN = PW * (BY_ + 1), NS = (PN + NT - 1) / NT;
};

#ifndef TF_RES_MINB32
#define TF_RES_MINB32 2
#endif
#ifndef TF_RES_MINB64
#define TF_RES_MINB64 2
#endif
// BY: element-column rows per CTA (FP32 8 or 16, FP64 4 or 8): taller tiles
// halve the CTA count (cheaper exchanges, less halo recompute) at the same
// warps per SM
template <typename T, int BY_, bool ONEX>
__global__ void __launch_bounds__(TILE_BX * BY_, (TILE_BX * BY_ >= 512 || (sizeof(T) == 8 && BY_ >= 8))
                                                     ? 1
                                                     : (sizeof(T) == 4 ? TF_RES_MINB32 : TF_RES_MINB64))
k_pcg_resident(const __grid_constant__ ResArgs<T> A, const __grid_constant__ KhatBlocks<T> kb)
{
    using RT = ResTile<T, BY_>;
    constexpr int BY = RT::BY, NT = RT::NT, PW = RT::PW, PN = RT::PN, NS = RT::NS;
    constexpr bool F32 = sizeof(T) == 4;
    __shared__ __align__(16) T plane[2][PN];
    __shared__ T Y[3][NT];
    __shared__ double shr[8 * (NT / 32)];
    extern __shared__ __align__(16) unsigned char res_dyn[];

    const Grid& g = A.g;
    const int oz = A.oz;
    // the single-exchange loop needs the full layout (a compile-time constant
    // for FP32: fewer index registers; FP64 allocates better without it)
    const bool lean = (ONEX && sizeof(T) == 4) ? false : A.lean != 0;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = tx + TILE_BX * ty;
    const int bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    const int nblk = (int)(gridDim.x * gridDim.y * gridDim.z);
    const int i0 = blockIdx.x * (TILE_BX - 1);
    const int j0 = blockIdx.y * (BY - 1);
    const int k0 = blockIdx.z * oz;
    const int kend = min(k0 + oz, g.nnz);  // owned planes [k0, kend)
    const int ex = i0 - 1 + tx, ey = j0 - 1 + ty;
    const bool col_ok = ex >= 0 && ex < g.nelx && ey >= 0 && ey < g.nely;
    const bool owner = tx < TILE_BX - 1 && ty < BY - 1 && (i0 + tx) < g.nnx && (j0 + ty) < g.nny;
    const int n_own = owner ? kend - k0 : 0;
    const int pn = g.nnx * g.nny, pn3 = 3 * pn;
    const uint8_t* nf = A.node_fixed;
    const uint8_t* col_or = nf ? nf + g.n_nodes : nullptr;
    const uint8_t* col_and = nf ? col_or + pn : nullptr;
    const int own_node0 = (i0 + tx) + g.nnx * (j0 + ty);
    unsigned phase = 0u;  // exchange counter (identical sequence in every CTA)
    unsigned* ctr = reinterpret_cast<unsigned*>(A.ring + (size_t)2 * RES_SLOT * nblk);

    // owned vectors in shared memory: own(v, kk, c) for this thread.  Full
    // layout: x r inv p q; lean: r p q (x and inv in global memory).
    T* own = reinterpret_cast<T*>(res_dyn);
    const int VR = lean ? 0 : 1, VP = lean ? 1 : 3, VQ = lean ? 2 : 4;
    constexpr int VX = 0, VI = 2;
    auto oidx = [&](int v, int kk, int c, int t) { return ((v * oz + kk) * 3 + c) * NT + t; };
    auto dof = [&](int kk, int c) { return 3 * (own_node0 + (k0 + kk) * pn) + c; };
    auto get_x = [&](int kk, int c) -> T { return lean ? __ldcg(A.x + dof(kk, c)) : own[oidx(VX, kk, c, tid)]; };
    auto set_x = [&](int kk, int c, T v) {
        if (lean) A.x[dof(kk, c)] = v;
        else own[oidx(VX, kk, c, tid)] = v;
    };
    auto get_inv = [&](int kk, int c) -> T { return lean ? ld_nc(A.inv + dof(kk, c)) : own[oidx(VI, kk, c, tid)]; };

    // fixed bits of the owned DOFs, 3 per owned plane (oz <= 21)
    unsigned long long ofix = 0ull;
    if (nf) {
        for (int kk = 0; kk < n_own; ++kk)
            ofix |= (unsigned long long)(nf[own_node0 + (k0 + kk) * pn] & 7u) << (3 * kk);
    }

    // staging slots
    int s_off[NS], s_own[NS];
    unsigned okbits = 0u, mskbits = 0u, allfix = 0u;
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        const int idx = tid + q * NT;
        const int r = idx / PW, f = idx - r * PW;
        const int ii = i0 - 1 + f / 3, jj = j0 - 1 + r, c = f % 3;
        const bool ok = idx < PN && ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny;
        const int node = ok ? ii + g.nnx * jj : 0;
        s_off[q] = 3 * node + c;
        s_own[q] = -1;
        if (ok) {
            okbits |= 1u << q;
            if (nf) {
                if ((col_and[node] >> c) & 1u) allfix |= 1u << q;
                else if ((col_or[node] >> c) & 1u) mskbits |= 1u << q;
            }
            if (ii >= i0 && ii < i0 + TILE_BX - 1 && jj >= j0 && jj < j0 + BY - 1)
                s_own[q] = c * NT + (ii - i0) + TILE_BX * (jj - j0);  // + kk*3*NT + VP*oz*3*NT
        }
    }
    const int pofs = ty * PW + 3 * tx;
    auto pv_ = [&](const T* buf, int ox, int oy, int c) -> T { return buf[pofs + oy * PW + 3 * ox + c]; };
    const int el_col = ex + g.nelx * ey, el_plane = g.nelx * g.nely;
    auto scale_at = [&](int ez) -> T {
        return (col_ok && ez >= 0 && ez < g.nelz) ? ld_nc(A.scale + el_col + el_plane * ez) : T(0);
    };

    // One structured matvec over this CTA's chunk.  PDIR: the input is
    // p_k = z + beta p_{k-1} (first: p_1 = z_0), owners publish p_k to `pnew`
    // and to own(VP); otherwise the input is the global vector `src`.  The
    // result of every owned DOF (pass-through on constrained DOFs) goes to
    // own(VQ); returns this thread's p.q (PDIR).
    // (one instantiation for both modes: the kernel's code footprint is kept
    // small so the per-iteration phases stay in the instruction cache)
    // ONEX (single-exchange iteration): the staged input is p_k = z_k +
    // beta p_{k-1} with z_k = r_k D^-1 and r_k = r_{k-1} - alpha_{k-1} q_{k-1}
    // recomputed from the published r_{k-1}, q_{k-1} (`src`, `qsrc`; `fresh`:
    // r_k published as is -- first iteration, after a true-residual refresh)
    // exactly as the owner computes them, so no barrier is needed between the
    // owners' update and the neighbours' staging; owners also apply x_k =
    // x_{k-1} + alpha_{k-1} p_{k-1} and publish r_k (rnew) and q_k (qnew).
    T* invtab = own + (size_t)(lean ? 3 : 5) * oz * 3 * NT;  // ONEX: D^-1 over the staged footprint
    auto tile_pass = [&](bool pdir, bool first, T be, const T* src, const T* pold, T* pnew, bool fresh = true,
                         T ap = T(0), const T* qsrc = nullptr, T* rnew = nullptr, T* qnew = nullptr) -> double {
        auto fetch = [&](int kz, T (&pa)[NS], T (&pb)[NS], T (&pc)[NS]) {
            const bool zok = kz >= 0 && kz < g.nnz;
            const int base = min(max(kz, 0), g.nnz - 1) * pn3;
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                const bool take = zok && ((okbits >> q) & 1u);
                const int d = base + s_off[q];
                pa[q] = take ? __ldcg(src + d) : T(0);
                if (pdir) pb[q] = (take && !first) ? __ldcg(pold + d) : T(0);
                if (ONEX && pdir) pc[q] = (take && !fresh) ? __ldcg(qsrc + d) : T(0);
            }
        };
        auto commit = [&](int kz, T* buf, const T (&pa)[NS], const T (&pb)[NS], const T (&pc)[NS]) {
            const bool zok = kz >= 0 && kz < g.nnz;
            const bool wr = pdir && zok && kz >= k0 && kz < kend;
            const int base = min(max(kz, 0), g.nnz - 1) * pn3;
            const int pl = (kz - (k0 - 1)) * PN;  // ONEX: plane row of the D^-1 table
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                const int idx = tid + q * NT;
                if (q < NS - 1 || idx < PN) {
                    const bool ok = zok && ((okbits >> q) & 1u);
                    T pv = pa[q];
                    T rv = T(0);
                    if (ONEX && pdir) {
                        rv = fresh ? pa[q] : sub_rn(pa[q], mul_rn(ap, pc[q]));
                        const T zv = mul_rn(rv, invtab[pl + idx]);
                        pv = first ? zv : add_rn(zv, mul_rn(be, pb[q]));
                    } else if (pdir && !first) {
                        pv = add_rn(pa[q], mul_rn(be, pb[q]));
                    }
                    if (!ok) pv = T(0);
                    if (wr && s_own[q] >= 0) {
                        pnew[base + s_off[q]] = pv;
                        const int ob = (kz - k0) * 3 * NT + s_own[q];
                        if (ONEX) {
                            if (!first && !fresh) {
                                T* xo = own + (size_t)VX * oz * 3 * NT + ob;
                                *xo = add_rn(*xo, mul_rn(ap, own[(size_t)VP * oz * 3 * NT + ob]));
                            }
                            own[(size_t)VR * oz * 3 * NT + ob] = rv;
                            rnew[base + s_off[q]] = rv;
                        }
                        own[(VP * oz + (kz - k0)) * 3 * NT + s_own[q]] = pv;
                    }
                    bool fixed = (allfix >> q) & 1u;
                    if (!fixed && ((mskbits >> q) & 1u) && ok)  // rare: z-varying constraint
                        fixed = (nf[kz * pn + s_off[q] / 3] >> (s_off[q] % 3)) & 1u;
                    buf[idx] = fixed ? T(0) : pv;
                }
            }
        };

        const int n_layers = kend - k0 + 1;
        T* b_cur = plane[0];
        T* b_top = plane[1];
        T pa[NS], pb[NS], pc[NS];
        {
            // both prologue planes in flight together (one L2 round trip)
            T qa[NS], qb[NS], qc[NS];
            fetch(k0 - 1, qa, qb, qc);
            fetch(k0, pa, pb, pc);
            commit(k0 - 1, b_cur, qa, qb, qc);
            commit(k0, b_top, pa, pb, pc);
        }
        fetch(k0 + 1, pa, pb, pc);
        __syncthreads();
        T XYb[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            face_fwd(pv_(b_cur, 0, 0, c), pv_(b_cur, 1, 0, c), pv_(b_cur, 0, 1, c), pv_(b_cur, 1, 1, c), XYb[c]);
        T Gt[3][4];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int q = 0; q < 4; ++q) Gt[c][q] = T(0);
        T s_cur = scale_at(k0 - 1);
        double dot = 0.0;

        for (int L = 0; L < n_layers; ++L) {
            const int ez = k0 - 1 + L;
            if (L >= 1) {
                // plane ez+1 into the buffer that held plane ez-1 (read before (B) of layer L-1)
                commit(ez + 1, b_top, pa, pb, pc);
                if (L + 1 < n_layers) fetch(ez + 2, pa, pb, pc);
            }
            __syncthreads();  // (A)
            const T s_next = scale_at(ez + 1);
            T h[3][8];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                T XYt[4];
                face_fwd(pv_(b_top, 0, 0, c), pv_(b_top, 1, 0, c), pv_(b_top, 0, 1, c), pv_(b_top, 1, 1, c), XYt);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    h[c][q] = XYb[c][q] + XYt[q];
                    h[c][q + 4] = XYt[q] - XYb[c][q];
                    XYb[c][q] = XYt[q];
                }
            }
            T gm[3][8];
            if (A.iso) {
                block_iso(h, A.ki, s_cur, gm);
            } else {
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int m = 1; m < 8; ++m) h[c][m] *= s_cur;
#pragma unroll
                for (int c = 0; c < 3; ++c) gm[c][0] = T(0);
#pragma unroll
                for (int q = 0; q < 8; ++q)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int m = q ^ (1 << c);
                        if (m == 0) continue;
                        T acc = T(0);
#pragma unroll
                        for (int d = 0; d < 3; ++d) {
                            const int n = q ^ (1 << d);
                            if (n == 0) continue;
                            acc = fma(kb.b[q][c][d], h[d][n], acc);
                        }
                        gm[c][m] = acc;
                    }
            }
            T corner[3][4];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                T H[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    H[q] = Gt[c][q] + (gm[c][q] - gm[c][q + 4]);
                    Gt[c][q] = gm[c][q] + gm[c][q + 4];
                }
                face_inv(H, corner[c]);
            }
            T xr[2][3];
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                xr[0][c] = corner[c][1] + __shfl_down_sync(0xffffffffu, corner[c][0], 1);
                xr[1][c] = corner[c][3] + __shfl_down_sync(0xffffffffu, corner[c][2], 1);
                Y[c][tid] = xr[0][c];
            }
            __syncthreads();  // (B)
            if (L >= 1 && owner) {
                const int kk = ez - k0;
                const unsigned fb = (unsigned)(ofix >> (3 * kk)) & 7u;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    T acc = xr[1][c] + Y[c][tid + TILE_BX];
                    const bool fx = (fb >> c) & 1u;
                    if (pdir) {
                        const T p = own[oidx(VP, kk, c, tid)];
                        if (fx) acc = p;  // pass-through of the unmasked input
                        dot += (double)p * (double)acc;
                        if (ONEX) qnew[dof(kk, c)] = acc;
                    } else if (fx) {
                        acc = get_x(kk, c);
                    }
                    own[oidx(VQ, kk, c, tid)] = acc;
                }
            }
            s_cur = s_next;
            T* t = b_cur;
            b_cur = b_top;
            b_top = t;
        }
        return dot;
    };

    constexpr bool PDIR = true, RAW = false;
    const bool tracing = A.trace != nullptr && bid == 0 && tid == 0;
    // -DTF_PCG_CTA_TRACE builds (never the product library): every CTA's
    // summed matvec-pass time, the arrival skew behind exchange A
#ifdef TF_PCG_CTA_TRACE
    const bool cta_trace = A.trace != nullptr && tid == 0;
#else
    constexpr bool cta_trace = false;
#endif
    unsigned long long mv_sum = 0ull;
    unsigned long long tr[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    unsigned long long t_mark = tracing ? res_gtime() : 0ull;
    auto lap = [&](int slot) {
        if (tracing) {
            const unsigned long long t = res_gtime();
            tr[slot] += t - t_mark;
            t_mark = t;
        }
    };

    // ---- init (solver.py:72-103) -------------------------------------------------
    if (!lean) {
        for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int d = dof(kk, c);
                own[oidx(VI, kk, c, tid)] = ld_nc(A.inv + d);
                own[oidx(VX, kk, c, tid)] = A.has_x0 ? __ldcg(A.x + d) : T(0);
            }
    } else if (!A.has_x0) {
        for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
            for (int c = 0; c < 3; ++c) A.x[dof(kk, c)] = T(0);
    }
    if (ONEX) {
        // D^-1 over the staged footprint, planes k0-1 .. kend (static for the solve)
        for (int pl = 0; pl < kend - k0 + 2; ++pl) {
            const int kz = k0 - 1 + pl;
            const bool zok = kz >= 0 && kz < g.nnz;
#pragma unroll
            for (int q = 0; q < NS; ++q) {
                const int idx = tid + q * NT;
                if (idx < PN) {
                    const bool ok = zok && ((okbits >> q) & 1u);
                    invtab[pl * PN + idx] = ok ? ld_nc(A.inv + (size_t)kz * pn3 + s_off[q]) : T(0);
                }
            }
        }
    }
    __syncthreads();
    if (A.has_x0) tile_pass(RAW, false, T(0), A.x, nullptr, nullptr);  // own(VQ) = A x0
    double tot[3] = {0.0, 0.0, 0.0};
    {
        for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const int d = dof(kk, c);
                const T bb = ld_nc(A.b + d);
                const T r = A.has_x0 ? sub_rn(bb, own[oidx(VQ, kk, c, tid)]) : bb;
                const T z = mul_rn(r, get_inv(kk, c));
                own[oidx(VR, kk, c, tid)] = r;
                if (ONEX)
                    A.rbuf[0][d] = r;
                else
                    A.z[d] = z;
                tot[0] += (double)bb * (double)bb;
                tot[1] += (double)r * (double)r;
                tot[2] += (double)r * (double)z;
            }
        res_block_sum<3, NT>(tot, shr, tid);
        res_exchange<3, NT>(A.ring, ctr, nblk, bid, tid, phase++, tot, shr);
    }
    CgScalars* sc = A.sc;
    const bool lead = bid == 0 && tid == 0;
    const double tol = sc->tol;
    const int max_iter = sc->max_iter, recompute = sc->recompute;
    double* hist = sc->hist;
    const double bnorm = cg_sqrt(cg_round(tot[0], F32), F32);
    int it = 0, term = TERM_MAX_ITER, matvecs = A.has_x0 ? 1 : 0;
    double rel = 0.0;
    if (bnorm == 0.0) {  // zero right-hand side (solver.py:72-85): x = 0, converged
        if (lead) {
            sc->bnorm = 0.0;
            sc->zero_rhs = 1;
            sc->done = 1;
            sc->term = TERM_CONVERGED;
            sc->it = 0;
            sc->matvecs = 0;
            sc->rel = 0.0;
            if (hist) hist[0] = 0.0;
        }
        return;
    }
    double rz = cg_round(tot[2], F32);
    rel = cg_sqrt(cg_round(tot[1], F32), F32) / bnorm;
    if (lead && hist) hist[0] = rel;
    bool done = rel <= tol;
    if (done) term = TERM_CONVERGED;
    double beta = 0.0;
    lap(5);

    // ---- iterations (solver.py:104-137) --------------------------------------------
    if constexpr (ONEX) {
        // One exchange per iteration.  The pass of iteration k stages p_k from
        // the published r_{k-1}, q_{k-1}, p_{k-1} (see tile_pass), so the only
        // grid-wide step is the reduction after it, which carries p.q and the
        // own-DOF sums r.r, r.z (direct, of r_k), r.q, q.q, r.Dq, q.Dq, r.Dr:
        // alpha_k = r.z / p.q exactly as the two-exchange loop (same values,
        // same order), while ||r_{k+1}||^2 and r_{k+1}.z_{k+1} -- which the
        // convergence test and beta_k need before r_{k+1} exists -- are
        // expanded one step in FP64: r.r - 2a r.q + a^2 q.q (a = alpha_k in the
        // working dtype, as the update applies it).
        bool fresh = true;  // r_k published as is (first iteration, after a refresh)
        bool xpend = false;  // x_{k+1} = x_k + alpha_k p_k not yet applied
        T ap = T(0);
        while (!done) {
            ++it;
            const unsigned long long mv_t0 = cta_trace ? res_gtime() : 0ull;
            const double pq_loc =
                tile_pass(PDIR, it == 1, (T)beta, A.rbuf[(it - 1) & 1], A.pbuf[(it - 1) & 1], A.pbuf[it & 1],
                          fresh, ap, A.qbuf[(it - 1) & 1], A.rbuf[it & 1], A.qbuf[it & 1]);
            if (cta_trace) mv_sum += res_gtime() - mv_t0;
            xpend = false;  // the pass applied x_k += alpha_{k-1} p_{k-1} (unless fresh)
            ++matvecs;
            lap(0);
            double t8[7] = {pq_loc, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const T r = own[oidx(VR, kk, c, tid)], q = own[oidx(VQ, kk, c, tid)];
                    const T iv = get_inv(kk, c);
                    const T z = mul_rn(r, iv);
                    const double dr = (double)r, dq = (double)q, di = (double)iv;
                    t8[1] += dr * dr;
                    t8[2] += dr * (double)z;
                    t8[3] += dr * dq;
                    t8[4] += dq * dq;
                    t8[5] += dr * di * dq;
                    t8[6] += dq * di * dq;
                }
            res_block_sum<7, NT>(t8, shr, tid);
            res_exchange<7, NT>(A.ring, ctr, nblk, bid, tid, phase++, t8, shr);
            lap(1);
            const double pq = cg_round(t8[0], F32);
            rz = cg_round(t8[2], F32);
            if (!isfinite(pq) || !isfinite(rz)) {
                term = TERM_DIVERGED;
                break;
            }
            if (pq <= 0.0) {
                term = TERM_BREAKDOWN;
                break;
            }
            const double alpha = rz / pq;
            const T a = (T)alpha;
            const bool refresh = recompute > 0 && it % recompute == 0;
            double rr_n, rz_n;
            if (refresh) {
                // x_{k+1} applied and published; r_{k+1} = b - A x_{k+1}
                for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int o = oidx(VX, kk, c, tid);
                        const T xn = add_rn(own[o], mul_rn(a, own[oidx(VP, kk, c, tid)]));
                        own[o] = xn;
                        A.x[dof(kk, c)] = xn;
                    }
                double dummy[1] = {0.0};
                res_exchange<1, NT>(A.ring, ctr, nblk, bid, tid, phase++, dummy, shr);  // x published
                tile_pass(RAW, false, T(0), A.x, nullptr, nullptr);                   // own(VQ) = A x
                ++matvecs;
                double t2[2] = {0.0, 0.0};
                for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int d = dof(kk, c);
                        const T r = sub_rn(ld_nc(A.b + d), own[oidx(VQ, kk, c, tid)]);
                        own[oidx(VR, kk, c, tid)] = r;
                        A.rbuf[it & 1][d] = r;
                        const T z = mul_rn(r, get_inv(kk, c));
                        t2[0] += (double)r * (double)r;
                        t2[1] += (double)r * (double)z;
                    }
                res_block_sum<2, NT>(t2, shr, tid);
                res_exchange<2, NT>(A.ring, ctr, nblk, bid, tid, phase++, t2, shr);
                rr_n = t2[0];
                rz_n = t2[1];
                fresh = true;
                ap = T(0);
            } else {
                const double da = (double)a;
                rr_n = t8[1] - 2.0 * da * t8[3] + da * da * t8[4];
                // base: the direct r.z (z rounded in the working dtype) for r.Dr
                rz_n = t8[2] - 2.0 * da * t8[5] + da * da * t8[6];
                fresh = false;
                ap = a;
                xpend = true;
            }
            lap(3);
            const double rn = cg_sqrt(cg_round(rr_n, F32), F32);
            if (!isfinite(rn)) {
                term = TERM_DIVERGED;
                break;
            }
            rel = rn / bnorm;
            if (lead && hist) hist[it] = rel;
            if (rel <= tol) {
                term = TERM_CONVERGED;
                break;
            }
            const double rz_new = cg_round(rz_n, F32);
            beta = rz_new / rz;
            if (it >= max_iter) {
                term = TERM_MAX_ITER;
                break;
            }
            lap(4);
        }
        if (xpend) {
            // x_{k+1} of the last iteration (the next pass would have applied it)
            for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const int o = oidx(VX, kk, c, tid);
                    own[o] = add_rn(own[o], mul_rn(ap, own[oidx(VP, kk, c, tid)]));
                }
        }
    } else
    while (!done) {
        ++it;
        // A. q = A p_it, fused p.q
        const unsigned long long mv_t0 = cta_trace ? res_gtime() : 0ull;
        double t1[1] = {tile_pass(PDIR, it == 1, (T)beta, A.z, A.pbuf[(it - 1) & 1], A.pbuf[it & 1])};
        if (cta_trace) mv_sum += res_gtime() - mv_t0;
        ++matvecs;
        lap(0);
        res_block_sum<1, NT>(t1, shr, tid);
        res_exchange<1, NT>(A.ring, ctr, nblk, bid, tid, phase++, t1, shr);
        lap(1);
        // B. alpha, x, r, z
        const double pq = cg_round(t1[0], F32);
        if (!isfinite(pq) || !isfinite(rz)) {
            term = TERM_DIVERGED;
            break;
        }
        if (pq <= 0.0) {
            term = TERM_BREAKDOWN;
            break;
        }
        const double alpha = rz / pq;
        const T a = (T)alpha;
        const bool refresh = recompute > 0 && it % recompute == 0;
        // x += alpha p: needed by other CTAs only on a refresh; otherwise it is
        // done while exchange B is in flight
        auto update_x = [&]() {
            if (!lean) {
                for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const int o = oidx(VX, kk, c, tid);
                        const T xn = add_rn(own[o], mul_rn(a, own[oidx(VP, kk, c, tid)]));
                        own[o] = xn;
                        if (refresh) A.x[dof(kk, c)] = xn;
                    }
            } else {
                // global x: loads of a chunk issued together (one L2 round trip per 4 planes)
                for (int k4 = 0; k4 < n_own; k4 += 4) {
                    T xv[4][3];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int c = 0; c < 3; ++c) xv[j][c] = k4 + j < n_own ? __ldcg(A.x + dof(k4 + j, c)) : T(0);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
#pragma unroll
                        for (int c = 0; c < 3; ++c)
                            if (k4 + j < n_own)
                                A.x[dof(k4 + j, c)] = add_rn(xv[j][c], mul_rn(a, own[oidx(VP, k4 + j, c, tid)]));
                }
            }
        };
        if (refresh) update_x();
        lap(6);
        if (refresh) {
            double dummy[1] = {0.0};
            res_exchange<1, NT>(A.ring, ctr, nblk, bid, tid, phase++, dummy, shr);  // x published
            tile_pass(RAW, false, T(0), A.x, nullptr, nullptr);  // own(VQ) = A x
            ++matvecs;
        }
        double t2[2] = {0.0, 0.0};
        for (int k4 = 0; k4 < n_own; k4 += 4) {
            // chunk of 4 planes: global loads (b on refresh, D^-1 when lean) issued together
            T bv[4][3], iv[4][3];
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const bool in = k4 + j < n_own;
                    bv[j][c] = (in && refresh) ? ld_nc(A.b + dof(k4 + j, c)) : T(0);
                    iv[j][c] = in ? get_inv(k4 + j, c) : T(0);
                }
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (k4 + j >= n_own) continue;
                    const int orr = oidx(VR, k4 + j, c, tid);
                    const T q = own[oidx(VQ, k4 + j, c, tid)];
                    const T r = refresh ? sub_rn(bv[j][c], q) : sub_rn(own[orr], mul_rn(a, q));
                    own[orr] = r;
                    const T z = mul_rn(r, iv[j][c]);
                    A.z[dof(k4 + j, c)] = z;
                    t2[0] += (double)r * (double)r;
                    t2[1] += (double)r * (double)z;
                }
        }
        lap(7);
        res_block_sum<2, NT>(t2, shr, tid);
        lap(2);
        res_arrive<2>(A.ring, ctr, nblk, bid, tid, phase, t2);
        if (!refresh) update_x();
        res_wait<2>(A.ring, ctr, nblk, tid, phase++, t2, shr);
        lap(3);
        // C. decisions
        const double rn = cg_sqrt(cg_round(t2[0], F32), F32);
        if (!isfinite(rn)) {
            term = TERM_DIVERGED;
            break;
        }
        rel = rn / bnorm;
        if (lead && hist) hist[it] = rel;
        if (rel <= tol) {
            term = TERM_CONVERGED;
            break;
        }
        const double rz_new = cg_round(t2[1], F32);
        beta = rz_new / rz;
        rz = rz_new;
        if (it >= max_iter) {
            term = TERM_MAX_ITER;
            break;
        }
        lap(4);
    }

    if (cta_trace) A.trace[16 + bid] = mv_sum;
    // solution: every DOF written once by its owner
    if (!lean) {
        for (int kk = 0; kk < n_own; ++kk)
#pragma unroll
            for (int c = 0; c < 3; ++c) A.x[dof(kk, c)] = own[oidx(VX, kk, c, tid)];
    }
    if (lead) {
        sc->bnorm = bnorm;
        sc->zero_rhs = 0;
        sc->done = 1;
        sc->term = term;
        sc->it = it;
        sc->matvecs = matvecs;
        sc->rel = rel;
        sc->rz = rz;
    }
    if (tracing) {
        for (int k = 0; k < 6; ++k) A.trace[k] = tr[k];

        A.trace[6] = (unsigned long long)it;
        A.trace[7] = tr[6];
        A.trace[8] = tr[7];
    }
}

// ---- host ------------------------------------------------------------------------

// owned vectors (+ the ONEX D^-1 table over oz + 2 staged planes of PN slots)
template <typename T>
static size_t res_dyn_bytes(int oz, bool lean, int nt, bool onex, int pn_slots)
{
    return (size_t)(lean ? 3 : 5) * oz * 3 * nt * sizeof(T) + (onex ? (size_t)(oz + 2) * pn_slots * sizeof(T) : 0);
}

// TF_PCG_ONEX=0: the two-exchange iteration (A/B); default: one exchange
static bool res_onex_enabled()
{
    const char* e = getenv("TF_PCG_ONEX");
    return !(e && e[0] == '0');
}

template <typename T, int BY>
static const void* res_kernel(bool onex)
{
    return onex ? (const void*)k_pcg_resident<T, BY, true> : (const void*)k_pcg_resident<T, BY, false>;
}

// tile heights tried per precision (rows of element columns per CTA)
template <typename T> struct ResBys;
template <> struct ResBys<float> { static constexpr int a = 16, b = 8; };
template <> struct ResBys<double> { static constexpr int a = 8, b = 4; };

// Candidate launch: for one tile height, the smallest z-chunk whose grid is
// co-resident with its shared-memory state (full layout before lean).
template <typename T, int BY>
static bool res_candidate(const Grid& g, int nsm, int smem_optin, int oz_force, int lean_force, ResPlan* plan)
{
    constexpr int NT = TILE_BX * BY;
    constexpr int PN = ResTile<T, BY>::PN;
    const bool onex_env = res_onex_enabled();
    const int tx = (g.nnx + TILE_BX - 2) / (TILE_BX - 1);
    const int ty = (g.nny + BY - 2) / (BY - 1);
    const long long cols = (long long)tx * ty;
    for (int oz = 2; oz <= std::min(g.nnz, 21); ++oz) {
        if (oz_force > 0 && oz != oz_force) continue;
        for (int lean = 0; lean < 2; ++lean) {
            if (lean_force >= 0 && lean != lean_force) continue;
            const bool onex = onex_env && lean == 0;
            const void* k = res_kernel<T, BY>(onex);
            const size_t dyn = res_dyn_bytes<T>(oz, lean != 0, NT, onex, PN);
            if ((long long)dyn + 16384 > smem_optin) continue;
            cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            int per_sm = 0;
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, NT, dyn) != cudaSuccess) {
                cudaGetLastError();
                return false;
            }
            const long long tz = (g.nnz + oz - 1) / oz;
            if (per_sm > 0 && cols * tz <= (long long)per_sm * nsm) {
                plan->grid = dim3(tx, ty, (unsigned)tz);
                plan->oz = oz;
                plan->lean = lean;
                plan->dyn_smem = dyn;
                plan->nblk = cols * tz;
                plan->by = BY;
                plan->onex = onex ? 1 : 0;
                return true;
            }
        }
    }
    return false;
}

// Chooses tile height, z-chunk and layout of a co-resident grid.  Per tile
// height the smallest chunk that fits; between heights the cheaper estimate of
// (layers per CTA x CTAs per SM) + exchange cost (grows with the CTA count,
// scripts/exchange_bench.cu: ~0.9 us per extra 148 CTAs).  Env pins:
// TF_PCG_RES_BY / TF_PCG_RES_OZ / TF_PCG_RES_LEAN=0|1 (experiments).
template <typename T>
bool pcg_resident_plan(const Grid& g, const T* ke_host, ResPlan* plan)
{
    KhatBlocks<T> kb;
    if (!khat_blocks<T>(ke_host, &kb)) return false;
    if (3 * g.n_nodes >= (1LL << 31)) return false;
    int dev = 0, nsm = 148, smem_optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const char* e = getenv("TF_PCG_RES_OZ");
    const int oz_force = e ? atoi(e) : 0;
    const char* el = getenv("TF_PCG_RES_LEAN");
    const int lean_force = el ? (el[0] == '1' ? 1 : 0) : -1;
    const char* eb = getenv("TF_PCG_RES_BY");
    const int by_force = eb ? atoi(eb) : 0;
    ResPlan pa, pb;
    const bool ok_a = (by_force == 0 || by_force == ResBys<T>::a) &&
                      res_candidate<T, ResBys<T>::a>(g, nsm, smem_optin, oz_force, lean_force, &pa);
    const bool ok_b = (by_force == 0 || by_force == ResBys<T>::b) &&
                      res_candidate<T, ResBys<T>::b>(g, nsm, smem_optin, oz_force, lean_force, &pb);
    if (!ok_a && !ok_b) return false;
    if (ok_a != ok_b) {
        *plan = ok_a ? pa : pb;
        return true;
    }
    // cost model (us per iteration), calibrated on B200 (scripts/gpu_run54.sh):
    // matvec = ceil(nblk/nsm) CTAs per SM x (oz+1) layers x NT/256 units of
    // 0.87 us (FP32; FP64 1.7x), 512-thread CTAs 15 % less efficient per
    // thread; exchange = 2.0 + 0.9 us per 148 CTAs (scripts/exchange_bench.cu),
    // two per iteration
    auto cost = [&](const ResPlan& p) {
        const int nt = TILE_BX * p.by;
        const double unit = 0.87 * (sizeof(T) == 8 ? 1.7 : 1.0) * (nt >= 512 ? 1.15 : 1.0);
        const double matvec = std::ceil((double)p.nblk / nsm) * (p.oz + 1) * (nt / 256.0) * unit;
        return matvec + (p.onex ? 1.0 : 2.0) * (2.0 + 0.9 * (double)p.nblk / 148.0);
    };
    *plan = cost(pa) < cost(pb) ? pa : pb;
    return true;
}

size_t pcg_resident_ring_doubles(const ResPlan& plan) { return (size_t)2 * RES_SLOT * plan.nblk + 16; }

template <typename T>
int launch_pcg_resident(const ResPlan& plan, const Grid& g, const T* ke_host, int has_x0, const T* scale,
                        const T* b, const T* inv, T* x, T* z, T* p0, T* p1, const uint8_t* node_fixed,
                        double* ring, CgScalars* sc, T* r1, T* q0, T* q1, cudaStream_t st)
{
    KhatBlocks<T> kb;
    if (!khat_blocks_cached<T>(ke_host, &kb)) return TF_ERR_UNSUPPORTED;
    ResArgs<T> a;
    a.g = g;
    a.oz = plan.oz;
    a.has_x0 = has_x0;
    a.scale = scale;
    a.b = b;
    a.inv = inv;
    a.x = x;
    a.z = z;
    a.pbuf[0] = p0;
    a.pbuf[1] = p1;
    a.node_fixed = node_fixed;
    a.ring = ring;
    a.lean = plan.lean;
    a.onex = plan.onex;
    a.rbuf[0] = z;  // ONEX: r_k ping-pong (z's buffer) and q_k ping-pong
    a.rbuf[1] = r1;
    a.qbuf[0] = q0;
    a.qbuf[1] = q1;
    if (plan.onex && !(r1 && q0 && q1)) return TF_ERR_ARG;
    {
        // isotropic blocks in both precisions (FP32 since late round 2, like
        // the graph protocol's matvec: c2 17.85 -> 17.6 us/iteration, every
        // FP32 CG/SIMP parity test green); TF_RES_ISO32=0: generic FP32 blocks
        const char* e = getenv("TF_RES_ISO32");
        const bool iso32 = sizeof(T) == 4 && !(e && e[0] == '0');
        a.iso = ((tile_iso_enabled<T>() || iso32) && khat_iso<T>(ke_host, &a.ki)) ? 1 : 0;
    }
    a.sc = sc;
    a.trace = nullptr;
    static unsigned long long* trace_buf = nullptr;
    static long long trace_cap = 0;
    const bool tracing = getenv("TF_PCG_TRACE") != nullptr;
    const long long trace_n = 16 + plan.nblk;
    if (tracing) {
        if (trace_cap < trace_n) {
            if (trace_buf) cudaFree(trace_buf);
            TF_CUDA_TRY(cudaMalloc(&trace_buf, trace_n * sizeof(unsigned long long)));
            trace_cap = trace_n;
        }
        TF_CUDA_TRY(cudaMemsetAsync(trace_buf, 0, trace_n * sizeof(unsigned long long), st));
        a.trace = trace_buf;
    }
    TF_CUDA_TRY(cudaMemsetAsync(ring, 0, sizeof(double) * pcg_resident_ring_doubles(plan), st));
    const bool onex = plan.onex != 0;
    const void* k =
        plan.by == ResBys<T>::a ? res_kernel<T, ResBys<T>::a>(onex) : res_kernel<T, ResBys<T>::b>(onex);
    TF_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)plan.dyn_smem));
    void* args[] = {&a, &kb};
    dim3 block(TILE_BX, plan.by, 1);
    TF_CUDA_TRY(cudaLaunchCooperativeKernel(k, plan.grid, block, args, plan.dyn_smem, st));
    if (tracing) {
        std::vector<unsigned long long> hv(trace_n);
        TF_CUDA_TRY(cudaMemcpyAsync(hv.data(), trace_buf, trace_n * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, st));
        TF_CUDA_TRY(cudaStreamSynchronize(st));
        const unsigned long long* h = hv.data();
#ifdef TF_PCG_CTA_TRACE
        {  // per-CTA matvec-pass time: the arrival skew behind exchange A
            std::vector<std::pair<unsigned long long, long long>> m;
            for (long long b = 0; b < plan.nblk; ++b) m.push_back({h[16 + b], b});
            std::sort(m.begin(), m.end());
            const double n = h[6] ? (double)h[6] : 1.0;
            const long long gx = plan.grid.x, gy = plan.grid.y;
            auto at = [&](size_t i) { return m[i].first / n / 1e3; };
            const long long bmax = m.back().second;
            fprintf(stderr, "[tf_pcg_resident] matvec pass per CTA, us/it: min %.2f p50 %.2f p90 %.2f max %.2f "
                            "(slowest CTA %lld,%lld,%lld)\n", at(0), at(m.size() / 2), at(m.size() * 9 / 10),
                    at(m.size() - 1), bmax % gx, (bmax / gx) % gy, bmax / (gx * gy));
        }
#endif
        const double n = h[6] ? (double)h[6] : 1.0;
        fprintf(stderr,
                "[tf_pcg_resident] fp%d BY %d grid %ux%ux%u oz %d %s: %llu its; us/it: matvec %.2f  xchg-A %.2f  "
                "update %.2f (x %.2f, r/z %.2f)  xchg-B %.2f  decide %.2f  (init %.2f us)\n",
                (int)(8 * sizeof(T)), plan.by, plan.grid.x, plan.grid.y, plan.grid.z, plan.oz,
                plan.lean ? "lean" : "full", h[6], h[0] / n / 1e3, h[1] / n / 1e3, (h[2] + h[7] + h[8]) / n / 1e3,
                h[7] / n / 1e3, h[8] / n / 1e3, h[3] / n / 1e3, h[4] / n / 1e3, h[5] / 1e3);
    }
    return TF_OK;
}

template bool pcg_resident_plan<float>(const Grid&, const float*, ResPlan*);
template bool pcg_resident_plan<double>(const Grid&, const double*, ResPlan*);
template int launch_pcg_resident<float>(const ResPlan&, const Grid&, const float*, int, const float*,
                                        const float*, const float*, float*, float*, float*, float*,
                                        const uint8_t*, double*, CgScalars*, float*, float*, float*, cudaStream_t);
template int launch_pcg_resident<double>(const ResPlan&, const Grid&, const double*, int, const double*,
                                         const double*, const double*, double*, double*, double*, double*,
                                         const uint8_t*, double*, CgScalars*, double*, double*, double*,
                                         cudaStream_t);

}  // namespace tf
