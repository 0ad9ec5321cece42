// Structured-grid K v, production kernel: element tiles marching in z with
// the element matrix applied in the corner-Walsh basis.
//
// Algebra.  Let W be the 8x8 Walsh matrix over the cube corners (rows: modes
// 1, x, y, xy, z, zx, yz, xyz in binary order, entries +-1) and T = W (x) I3.
// Then Ke = T^T Khat T with Khat = T Ke T^T / 64.  Khat commutes with the
// cube's three mirror reflections, so it is block diagonal: DOF (mode m,
// component c) has reflection parity m ^ (1 << c), giving 8 parity classes of
// 3 DOFs each -- 8 dense 3x3 blocks (72 entries) instead of 576.  The kernel
// therefore applies s_e * Ke to an element vector as
//     FWHT (72 add) -> scale (24 mul) -> 8 3x3 blocks (72 FMA) -> FWHT^T (72 add)
// ~240 FP instructions instead of ~600; the host verifies the block structure
// of the supplied Ke (any axis-aligned orthotropic/isotropic material has it)
// and otherwise the dense pull kernel is used.  Results agree with the dense
// product to round-off (tolerance parity, not bitwise: use TF_GRID_BITWISE).
//
// Data movement.  A CTA of BX x BY threads owns node columns
// [i0, i0+BX-1) x [j0, j0+BY-1) over node planes [k0, k0+OZ); thread (tx, ty)
// owns the element column (i0-1+tx, j0-1+ty) -- one halo column/row of
// elements is recomputed by the neighbouring CTA instead of being exchanged,
// so there are no atomics and every DOF is written once.  Per element layer:
//   1. the node plane above is staged once in shared memory (coalesced rows,
//      input mask applied); the plane below is carried in registers;
//   2. each thread computes its element's 24 contributions -> smem F[24][NT];
//   3. each owned node sums its 4 bottom contributions onto the carried sum of
//      its 4 top contributions from the layer below (ascending element id,
//      like the reference's element-major loop) and stores w once.
// Optional fused epilogue: block partial of p.q for the CG (deterministic).

#include <algorithm>
#include <array>
#include <mutex>
#include <map>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "tf_common.cuh"
#include "tf_walsh.cuh"

namespace tf {


// ---- host: block extraction ------------------------------------------------------

static double walsh(int m, int b)
{
    double v = 1.0;
    for (int ax = 0; ax < 3; ++ax)
        if ((m >> ax) & 1) v *= ((b >> ax) & 1) ? 1.0 : -1.0;
    return v;
}

// Returns false when Ke is not block diagonal in the parity basis.
template <typename T>
bool khat_blocks(const T* ke, KhatBlocks<T>* out)
{
    // Khat[(m,c),(n,d)] = sum_{a,b} W[m][bin a] W[n][bin b] Ke[3a+c][3b+d] / 64
    double kh[24][24];
    double maxabs = 0.0;
    for (int m = 0; m < 8; ++m)
        for (int c = 0; c < 3; ++c)
            for (int n = 0; n < 8; ++n)
                for (int d = 0; d < 3; ++d) {
                    double s = 0.0;
                    for (int a = 0; a < 8; ++a)
                        for (int b = 0; b < 8; ++b)
                            s += walsh(m, bin_of(a)) * walsh(n, bin_of(b)) *
                                 (double)ke[(3 * a + c) * NLOC + 3 * b + d];
                    kh[3 * m + c][3 * n + d] = s / 64.0;
                    maxabs = fmax(maxabs, fabs(s / 64.0));
                }
    bool inblock[24][24] = {};
    for (int q = 0; q < 8; ++q)
        for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) {
                const int r = 3 * (q ^ (1 << c)) + c, s = 3 * (q ^ (1 << d)) + d;
                inblock[r][s] = true;
                out->b[q][c][d] = (T)kh[r][s];
            }
    const double tol = (sizeof(T) == 4 ? 1e-6 : 1e-12) * (maxabs > 0 ? maxabs : 1.0);
    for (int r = 0; r < 24; ++r)
        for (int s = 0; s < 24; ++s)
            if (!inblock[r][s] && fabs(kh[r][s]) > tol) return false;
    return true;
}

template <typename T>
bool khat_iso(const T* ke, KhatIso<T>* out)
{
    KhatBlocks<T> kb;
    if (!khat_blocks_cached<T>(ke, &kb)) return false;
    double mx = 0.0;
    for (int q = 0; q < 8; ++q)
        for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) mx = fmax(mx, fabs((double)kb.b[q][c][d]));
    const double tol = (sizeof(T) == 4 ? 1e-6 : 1e-12) * mx;
    auto B = [&](int q, int c, int d) { return (double)kb.b[q][c][d]; };
    auto eq = [&](double a, double b) { return fabs(a - b) <= tol; };
    auto z = [&](double a) { return fabs(a) <= tol; };
    bool ok = true;
    for (int q : {0, 7}) {  // [a b b; b a b; b b a]
        for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) ok = ok && eq(B(q, c, d), c == d ? B(q, 0, 0) : B(q, 0, 1));
    }
    // 2x2 [p r; r p] on the two non-translation components
    auto two = [&](int q, int i, int j) {
        return eq(B(q, i, i), B(q, j, j)) && eq(B(q, i, j), B(q, j, i));
    };
    ok = ok && two(1, 1, 2) && two(2, 0, 2) && two(4, 0, 1);
    // rank-one pair (i, j) of equal entries x, diagonal y at k, zeros elsewhere
    auto r1 = [&](int q, int i, int j, int k) {
        const double x = B(q, i, i);
        return eq(B(q, i, j), x) && eq(B(q, j, i), x) && eq(B(q, j, j), x) && z(B(q, i, k)) && z(B(q, k, i)) &&
               z(B(q, j, k)) && z(B(q, k, j));
    };
    ok = ok && r1(3, 0, 1, 2) && r1(5, 0, 2, 1) && r1(6, 1, 2, 0);
    if (!ok) return false;
    out->amb0 = (T)(B(0, 0, 0) - B(0, 0, 1));
    out->b0 = (T)B(0, 0, 1);
    out->p1 = (T)B(1, 1, 1);
    out->r1 = (T)B(1, 1, 2);
    out->p2 = (T)B(2, 0, 0);
    out->r2 = (T)B(2, 0, 2);
    out->x3 = (T)B(3, 0, 0);
    out->y3 = (T)B(3, 2, 2);
    out->p4 = (T)B(4, 0, 0);
    out->r4 = (T)B(4, 0, 1);
    out->x5 = (T)B(5, 0, 0);
    out->y5 = (T)B(5, 1, 1);
    out->x6 = (T)B(6, 1, 1);
    out->y6 = (T)B(6, 0, 0);
    out->amb7 = (T)(B(7, 0, 0) - B(7, 0, 1));
    out->b7 = (T)B(7, 0, 1);
    return true;
}
template bool khat_iso<float>(const float*, KhatIso<float>*);
template bool khat_iso<double>(const double*, KhatIso<double>*);

// khat_blocks behind a one-entry per-thread cache keyed on the Ke bytes: the
// host-side extraction (~37k multiply-adds) must not run on every launch --
// it would sit between the caller's stream events and the kernel
template <typename T>
bool khat_blocks_cached(const T* ke, KhatBlocks<T>* out)
{
    static thread_local T last_ke[NLOC * NLOC];
    static thread_local KhatBlocks<T> last_kb;
    static thread_local int last_ok = -1;
    if (last_ok < 0 || memcmp(last_ke, ke, sizeof(last_ke)) != 0) {
        last_ok = khat_blocks<T>(ke, &last_kb) ? 1 : 0;
        memcpy(last_ke, ke, sizeof(last_ke));
    }
    *out = last_kb;
    return last_ok == 1;
}

template bool khat_blocks<float>(const float*, KhatBlocks<float>*);
template bool khat_blocks_cached<float>(const float*, KhatBlocks<float>*);
template bool khat_blocks_cached<double>(const double*, KhatBlocks<double>*);
template bool khat_blocks<double>(const double*, KhatBlocks<double>*);

// ---- device ------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// The Walsh transforms factorised along the z march.
//
// The forward transform is separable: u -> (x, y stages on each xy face) ->
// (z stage between the bottom and top faces).  The bottom face of layer L is
// the top face of layer L-1, so its xy-stage result is carried in registers
// and only the new top face is transformed (24 adds instead of 48).  On the
// way back, the z-inverse splits g into a bottom-face and a top-face part in
// xy-mode space; the top part of layer L-1 and the bottom part of layer L
// land on the same node plane, so they are summed BEFORE the xy-inverse,
// which then runs once per element column and plane (24 adds instead of 48).
// Staging uses cp.async (zero-fill for out-of-mesh nodes) into a 3-plane ring
// so plane ez+2 streams in while layer ez is computed.
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cp_async_4(void* smem, const void* gmem, bool valid)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 4 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem, bool valid)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

#ifndef TF_TILE_MINB32
#define TF_TILE_MINB32 3
#endif
#ifndef TF_TILE_MINB64
#define TF_TILE_MINB64 3   // 168 regs + ~100 B spill: +5 % at c5 over 2 blocks/SM (measured)
#endif

// ---------------------------------------------------------------------------
// v5 (production): the z-factorised march with the bookkeeping stripped and
// a deep staging ring.
//   * the operator flags are template parameters (the production matvec is
//     MASK|PASS: no ACCUMULATE branches, no flag tests per DOF);
//   * node planes AND the element scales of each layer stream in with
//     cp.async P planes ahead of use (ring of P+2 buffers; P = 2 in
//     production): a one-wave grid (c2) sees one DRAM latency instead of one
//     per layer, a multi-wave grid hides it under more layers of work;
//   * the layer loop is unrolled by the ring period: plane buffers and the
//     row hand-off are compile-time offsets (no pointer rotation / moves);
//   * owners whose node column carries no constraint (column OR byte == 0)
//     never read the per-node constraint byte.
// ---------------------------------------------------------------------------
template <int I, int N, typename F>
__device__ __forceinline__ void static_for(F&& f)
{
    if constexpr (I < N) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N>(f);
    }
}

__device__ __forceinline__ void cp_async_wait_n(int n)
{
    // n is a compile-time constant at every call site after unrolling
    switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;\n" ::); break;
    case 1: asm volatile("cp.async.wait_group 1;\n" ::); break;
    case 2: asm volatile("cp.async.wait_group 2;\n" ::); break;
    case 3: asm volatile("cp.async.wait_group 3;\n" ::); break;
    default: asm volatile("cp.async.wait_group 4;\n" ::); break;
    }
}

#ifndef TF_TILE_P
#define TF_TILE_P 2
#endif
#ifndef TF_TILE_P1_OZ
#define TF_TILE_P1_OZ 4  // plain products with z-chunks up to this height stage one plane ahead
#endif

// TF_TILE_TRACE builds (scripts/tile_trace.py, never the product library):
// thread 0 of every CTA records %globaltimer / %clock64 at the phase
// boundaries of the march into a caller-supplied buffer, 16 u64 per CTA:
// [0] globaltimer start, [1] SM id, [2] clock start, [3] after the column
// setup, [4] after the prologue barrier, [5..12] after layers 0..7,
// [14] clock end, [15] globaltimer end.
#ifdef TF_TILE_TRACE
__device__ unsigned long long* g_tile_trace = nullptr;
__device__ __forceinline__ unsigned long long tt_gtime()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned tt_smid()
{
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}
#define TT_CLK(slot)                                                                                         \
    do {                                                                                                     \
        if (tid == 0 && g_tile_trace)                                                                        \
            g_tile_trace[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 16 + (slot)] =  \
                clock64();                                                                                   \
    } while (0)
#define TT_SET(slot, val)                                                                                    \
    do {                                                                                                     \
        if (tid == 0 && g_tile_trace)                                                                        \
            g_tile_trace[(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 16 + (slot)] =  \
                (val);                                                                                       \
    } while (0)
#else
#define TT_CLK(slot) \
    do {             \
    } while (0)
#define TT_SET(slot, val) \
    do {                  \
    } while (0)
#endif

// Fused interface put of the x-slab peer transport (tf_slab_run.cu): the
// owners of node plane x = put_i also store their (not yet exchanged)
// output into the neighbour's receive slot `dst` -- plane order (j, k)
// row-major, 3 components, as slab.py plane_dofs -- with plain peer stores
// (NVLink on an NVSwitch box), and the launch's last CTA raises the
// neighbour's epoch flag after a system-scope fence: the product and the
// transfer in one kernel instead of a boundary product and a put kernel.
template <typename T>
struct TilePut {
    T* dst;                  // nullptr: no put
    unsigned* flag;          // the neighbour's flag
    unsigned* ticket;        // local device memory, zero between launches
    const unsigned* ep_dev;  // graph mode: flag = *ep_dev + 1; else `epoch`
    unsigned epoch;
    int put_i;               // node x-index of the plane (this launch's grid)
};

template <typename T, bool MASK, bool PASS, bool ACC, bool DOT, int P, bool ISO, bool PUT = false>
__global__ void __launch_bounds__(TileDims<T>::NT, sizeof(T) == 4 ? TF_TILE_MINB32 : TF_TILE_MINB64)
k_grid_tile5(Grid g, int oz, const T* __restrict__ scale, const T* __restrict__ v, T* __restrict__ w,
             const uint8_t* __restrict__ node_fixed, double* __restrict__ dot_part,
             const __grid_constant__ KhatBlocks<T> kb, const __grid_constant__ KhatIso<T> ki,
             const __grid_constant__ TilePut<T> tp)
{
    constexpr int TILE_BY = TileDims<T>::BY, TILE_NT = TileDims<T>::NT;
    constexpr int PW = StageSlots<T>::PW, PN = StageSlots<T>::PN, NS = StageSlots<T>::N;
    constexpr int R = P + 2;                      // ring: plane k in buffer (k - k0 + 1) % R
    __shared__ __align__(16) T plane[R][PN];
    __shared__ T sc[R][TILE_NT];                  // element scale of layer k, with plane k
    __shared__ T Y[2][3][TILE_NT];                // row hand-off, by layer parity

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = tx + TILE_BX * ty;
#ifdef TF_TILE_TRACE
    TT_SET(0, tt_gtime());
    TT_SET(1, tt_smid());
    TT_CLK(2);
#endif
    const int i0 = g.ilo + blockIdx.x * (TILE_BX - 1);
    const int j0 = blockIdx.y * (TILE_BY - 1);
    const int k0 = blockIdx.z * oz;
    const int ex = i0 - 1 + tx, ey = j0 - 1 + ty;
    const bool col_ok = ex >= 0 && ex < g.nelx && ey >= 0 && ey < g.nely;
    const bool owner = tx < TILE_BX - 1 && ty < TILE_BY - 1 && (i0 + tx) < g.ihi && (j0 + ty) < g.nny;
    const bool have_nf = node_fixed != nullptr;
    const int pn = g.nnx * g.nny, pn3 = 3 * pn;
    const uint8_t* col_or = have_nf ? node_fixed + g.n_nodes : nullptr;
    const uint8_t* col_and = have_nf ? col_or + pn : nullptr;

    // Staging map (coalesced, one uniform row base per plane): warp wi copies
    // node-plane row wi -- lanes take values lane + 32k of its PW = 3 (BX+1)
    // -- and segment wi of the last row BY (warps 0..NSEG-1).  The prologue
    // planes are copied on geometry alone and the constrained slots zeroed
    // once they land: the first copies leave at kernel entry instead of
    // after a dependent load of the constraint bytes (a full DRAM latency on
    // every CTA's critical path, scripts/tile_trace.py); later planes copy
    // with the mask folded into the slot bits.
    constexpr int NW = TILE_NT / 32, NSEG = (PW + 31) / 32, NSL = NSEG + 1;
    static_assert(TILE_BY == NW && NSEG <= NW, "staging map");
    const int wi = tid >> 5, lane = tid & 31;
    // DOF offsets within a plane (3 n_nodes < 2^31 is checked on the host)
    const int row_own = 3 * (i0 - 1 + g.nnx * (j0 - 1 + wi)) + lane;
    const int row_last = 3 * (i0 - 1 + g.nnx * (j0 - 1 + TILE_BY)) + lane + 32 * wi;
    auto slot_smem = [&](int sl) { return sl < NSEG ? wi * PW + lane + 32 * sl : TILE_BY * PW + lane + 32 * wi; };
    auto slot_dof = [&](int sl) { return sl < NSEG ? row_own + 32 * sl : row_last; };
    unsigned geobits = 0u;  // bit sl: slot sl holds a node inside the grid
    // a CTA whose node rectangle lies inside the grid keeps every existing
    // slot (a uniform test; only the CTAs at the grid's edges evaluate slots)
    const bool inner = i0 >= 1 && i0 - 1 + TILE_BX < g.nnx && j0 >= 1 && j0 - 1 + TILE_BY < g.nny;
    if (inner) {
#pragma unroll
        for (int k = 0; k < NSEG; ++k)
            if (lane + 32 * k < PW) geobits |= 1u << k;
        if (wi < NSEG && lane + 32 * wi < PW) geobits |= 1u << NSEG;
    } else {
        const int jo = j0 - 1 + wi, jl = j0 - 1 + TILE_BY;
#pragma unroll
        for (int k = 0; k < NSEG; ++k) {
            const int f = lane + 32 * k, ii = i0 - 1 + f / 3;
            if (f < PW && ii >= 0 && ii < g.nnx && jo >= 0 && jo < g.nny) geobits |= 1u << k;
        }
        const int f = lane + 32 * wi, ii = i0 - 1 + f / 3;
        if (wi < NSEG && f < PW && ii >= 0 && ii < g.nnx && jl < g.nny) geobits |= 1u << NSEG;
    }
    // slots outside the grid never receive a copy (they feed only zero-scale
    // elements, but 0 * NaN would not vanish): zero them once in every
    // buffer (CTAs at the grid's edges only); constrained slots are zeroed
    // below once their bits are known
    unsigned nogeo = 0u;
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) {
        const bool exists = sl < NSEG ? lane + 32 * sl < PW : (wi < NSEG && lane + 32 * wi < PW);
        if (exists && !((geobits >> sl) & 1u)) nogeo |= 1u << sl;
    }
    if (nogeo) {
#pragma unroll
        for (int bf = 0; bf < R; ++bf)
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl)
                if ((nogeo >> sl) & 1u) plane[bf][slot_smem(sl)] = T(0);
    }
    const int el_col = ex + g.nelx * ey, el_plane = g.nelx * g.nely;
    const int n_layers = min(oz, g.nnz - k0) + 1;
    const int kmax = k0 - 1 + n_layers;  // top plane of the chunk's last layer
    // one cp.async group: node plane kz (slots `bits`; `varbits` slots carry
    // z-varying constraints, zero-filled where node kz's bit is set) and the
    // scales of element layer kz.  Planes outside the mesh are zero-filled,
    // planes past the chunk skipped.  Addresses: a CTA-uniform plane base
    // (64-bit, uniform datapath) plus the slot's 32-bit offset -- the
    // per-slot 64-bit pointer arithmetic this replaces cost ~30 instructions
    // per element-layer (ncu source counts, c5).
    auto stage = [&](int kz, int buf, unsigned bits, unsigned varbits) {
        if (kz <= kmax) {
            T* pb = plane[buf];
            const bool pok = kz >= 0 && kz < g.nnz;
            const T* vz = v + (long long)(pok ? kz : 0) * pn3;
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl)
                if ((bits >> sl) & 1u) {
                    if (sizeof(T) == 4)
                        cp_async_4(pb + slot_smem(sl), vz + slot_dof(sl), pok);
                    else
                        cp_async_8(pb + slot_smem(sl), vz + slot_dof(sl), pok);
                }
            if (MASK && varbits) {  // rare: columns whose constraint varies along z
#pragma unroll
                for (int sl = 0; sl < NSL; ++sl)
                    if ((varbits >> sl) & 1u) {
                        const int d = slot_dof(sl);
                        const bool keep = pok && !((node_fixed[kz * (long long)pn + d / 3] >> (d % 3)) & 1u);
                        if (sizeof(T) == 4)
                            cp_async_4(pb + slot_smem(sl), vz + d, keep);
                        else
                            cp_async_8(pb + slot_smem(sl), vz + d, keep);
                    }
            }
            const bool lok = kz >= 0 && kz < g.nelz;
            const T* sz = scale + (long long)el_plane * (lok ? kz : 0);
            const bool sok = col_ok && lok;
            if (sizeof(T) == 4)
                cp_async_4(&sc[buf][tid], sz + (col_ok ? el_col : 0), sok);
            else
                cp_async_8(&sc[buf][tid], sz + (col_ok ? el_col : 0), sok);
        }
        cp_async_commit();  // possibly empty: keeps the group count uniform
    };
    TT_CLK(3);
    // prologue: planes k0-1 .. k0-1+P (P+1 groups) in flight together, on geometry alone
#pragma unroll
    for (int bf = 0; bf <= P; ++bf) stage(k0 - 1 + bf, bf, geobits, 0u);
    // constraint bits of the staged slots (loads overlap the copies above).
    // Tall chunks first ask whether the CTA holds a constrained node column at
    // all -- one column-OR byte per thread and a block vote -- and skip the
    // per-slot work otherwise (c5: 82.3 -> 80.7 us); short chunks (one-wave
    // grids, where the vote's load would sit on every CTA's critical path)
    // evaluate the slots directly.
    unsigned fixbits = 0u, varbits = 0u;
    if (MASK && have_nf) {
        bool need = true;
        if (oz >= 8) {
            bool f = false;
            const int ii = i0 - 1 + tx, jj = j0 - 1 + ty;
            if (ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny) f = col_or[ii + g.nnx * jj] != 0;
            const int jl = j0 - 1 + TILE_BY, il = i0 - 1 + TILE_BX;
            if (ty == 0 && ii >= 0 && ii < g.nnx && jl < g.nny) f |= col_or[ii + g.nnx * jl] != 0;
            if (ty == 1 && tx <= TILE_BY && il < g.nnx) {
                const int j2 = j0 - 1 + tx;
                if (j2 >= 0 && j2 < g.nny) f |= col_or[il + g.nnx * j2] != 0;
            }
            need = __syncthreads_or(f) != 0;
        }
        if (need) {
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl)
                if ((geobits >> sl) & 1u) {
                    const int d = slot_dof(sl), node = d / 3, c = d - 3 * node;
                    if ((col_and[node] >> c) & 1u) fixbits |= 1u << sl;
                    else if ((col_or[node] >> c) & 1u) varbits |= 1u << sl;
                }
        }
    }
    const unsigned okbits = geobits & ~fixbits & ~varbits;
    const int pofs = ty * PW + 3 * tx;
    const int own_node0 = (i0 + tx) + g.nnx * (j0 + ty);
    // pass-through needs the node's constraint byte only on constrained
    // columns, and a per-plane read only where the constraint varies along z
    unsigned fix_or = 0u, fix_and = 0u;
    if (PASS && owner && have_nf) {
        fix_or = col_or[own_node0];
        fix_and = col_and[own_node0];
    }
    const bool own_fix_col = fix_or != 0u;
    const bool fix_zvar = fix_or != fix_and;

    cp_async_wait_n(0);  // the prologue planes landed: zero their constrained slots
    if (MASK && (fixbits | varbits)) {
#pragma unroll
        for (int bf = 0; bf <= P; ++bf) {
            const int kz = k0 - 1 + bf;
            if (kz < 0 || kz >= g.nnz) continue;
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl) {
                bool zero = (fixbits >> sl) & 1u;
                if ((varbits >> sl) & 1u) {
                    const int d = slot_dof(sl);
                    zero = (node_fixed[kz * (long long)pn + d / 3] >> (d % 3)) & 1u;
                }
                if (zero) plane[bf][slot_smem(sl)] = T(0);
            }
        }
        // the buffers filled after the prologue never receive a copy into a
        // z-invariant constrained slot (those are not in okbits)
#pragma unroll
        for (int bf = P + 1; bf < R; ++bf)
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl)
                if ((fixbits >> sl) & 1u) plane[bf][slot_smem(sl)] = T(0);
    }
    __syncthreads();
    TT_CLK(4);
    T XYb[3][4];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const T* bp = plane[0] + pofs + c;
        face_fwd(bp[0], bp[3], bp[PW], bp[PW + 3], XYb[c]);
    }
    T Gt[3][4];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int q = 0; q < 4; ++q) Gt[c][q] = T(0);
    T dot = T(0);

    T pend_x1[3], pend_p[3], pend_v[3];
    bool pend = false;
    int pend_d0 = 0;
    const bool put_col = PUT && owner && i0 + tx == tp.put_i;  // this thread's column is the put plane's
    int pend_pi = 0;
    unsigned pend_bits = 0u;

    // node pass of the previous layer (plane ez-1), reading its row hand-off.
    // Its constraint bits and pass-through values were loaded one layer
    // earlier (a dependent global load here would stall the CTAs holding a
    // constrained column at every layer -- and the kernel ends with the slowest CTA).
    auto node_pass = [&](const T (&Yp)[3][TILE_NT]) {
        if (!pend) return;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            T acc = pend_x1[c] + Yp[c][tid + TILE_BX];
            const int d = pend_d0 + c;
            if (ACC) acc += w[d];
            const bool fx = PASS && ((pend_bits >> c) & 1u);
            if (fx) acc = pend_v[c];
            w[d] = acc;
            if (PUT && put_col) tp.dst[pend_pi + c] = acc;
            if (DOT) {
                const T p = fx ? pend_v[c] : pend_p[c];
                dot = fma(p, acc, dot);
            }
        }
    };

    // one element layer (layer index L = ring phase I mod R): bottom plane ez
    // in buffer I, top plane ez+1 in buffer (I+1) % R; the layer stages plane
    // ez+1+P into buffer (I+P+1) % R = (I-1) % R (the plane of layer L-1)
    auto layer = [&](auto ph, int L) {
        constexpr int CUR = decltype(ph)::value;
        constexpr int TOP = (CUR + 1) % R, NXT = (CUR + P + 1) % R;
        const int ez = k0 - 1 + L;
        if (L > 0) {
            cp_async_wait_n(P - 1);  // plane ez+1 landed (P-1 younger groups may still fly)
            __syncthreads();         // (A) plane ez+1 + previous Y visible, buffer NXT free
        }
        node_pass(Y[(L + 1) & 1]);
        stage(ez + 1 + P, NXT, okbits, varbits);
        // constraint bits / pass-through inputs of plane ez (finalised by the
        // next layer's node pass): issued now, consumed a layer later
        unsigned nbits = 0u;
        T nv[3] = {T(0), T(0), T(0)};
        if (own_fix_col && L >= 1) {
            nbits = fix_zvar ? (unsigned)node_fixed[own_node0 + ez * pn] : fix_and;
            const int d0 = 3 * (own_node0 + ez * pn);
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if ((nbits >> c) & 1u) nv[c] = ld_nc(v + d0 + c);
        }
        const T s_cur = sc[CUR][tid];
        T pown[3];
        if (DOT) {
#pragma unroll
            for (int c = 0; c < 3; ++c) pown[c] = plane[CUR][pofs + PW + 3 + c];
        }
        T h[3][8];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T* bp = plane[TOP] + pofs + c;
            T XYt[4];
            face_fwd(bp[0], bp[3], bp[PW], bp[PW + 3], XYt);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                h[c][q] = XYb[c][q] + XYt[q];
                h[c][q + 4] = XYt[q] - XYb[c][q];
                XYb[c][q] = XYt[q];
            }
        }
        T gm[3][8];
        if (ISO) {
            block_iso(h, ki, s_cur, gm);
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
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const T x0 = corner[c][1] + __shfl_down_sync(0xffffffffu, corner[c][0], 1);
            pend_x1[c] = corner[c][3] + __shfl_down_sync(0xffffffffu, corner[c][2], 1);
            Y[L & 1][c][tid] = x0;
            if (DOT) pend_p[c] = pown[c];
        }
        pend = owner && L >= 1;
        pend_d0 = 3 * (own_node0 + ez * pn);
        if (PUT) pend_pi = 3 * ((j0 + ty) + g.nny * ez);
        pend_bits = nbits;
#pragma unroll
        for (int c = 0; c < 3; ++c) pend_v[c] = nv[c];
        TT_CLK(5 + min(L, 8));
    };
    int L = 0;
    for (; L + R <= n_layers; L += R) static_for<0, R>([&](auto ph) { layer(ph, L + decltype(ph)::value); });
    static_for<0, R - 1>([&](auto ph) {
        if (L + decltype(ph)::value < n_layers) layer(ph, L + decltype(ph)::value);
    });
    cp_async_wait_n(0);
    __syncthreads();
    node_pass(Y[(n_layers - 1) & 1]);
    if (PUT) {
        __threadfence_system();  // this thread's peer stores, before the CTA's ticket
        __syncthreads();
        if (tid == 0) {
            const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
            if (atomicAdd(tp.ticket, 1u) == nb - 1u) {
                __threadfence_system();
                *reinterpret_cast<volatile unsigned*>(tp.flag) =
                    tp.ep_dev ? *reinterpret_cast<const volatile unsigned*>(tp.ep_dev) + 1u : tp.epoch;
                *tp.ticket = 0u;
            }
        }
    }

#ifdef TF_TILE_TRACE
    TT_CLK(14);
    TT_SET(15, tt_gtime());
#endif
    if (DOT) {
        __shared__ double shd[TILE_NT / 32];
        double dd = (double)dot;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dd += __shfl_down_sync(0xffffffffu, dd, o);
        if ((tid & 31) == 0) shd[tid >> 5] = dd;
        __syncthreads();
        if (tid == 0) {
            double s2 = 0.0;
            for (int i = 0; i < TILE_NT / 32; ++i) s2 += shd[i];
            dot_part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = s2;
        }
    }
}

// ---------------------------------------------------------------------------
// Fused CG tile kernel: one PCG iteration's head in one launch.
//   1. every CTA reduces the previous update's r.r / r.z partials in the same
//      fixed order and takes the reference's decision (solver.py:120-135):
//      converged / max_iter / diverged -> stop (block 0 commits, WHILE = 0);
//      else beta = rz_new / rz_old;
//   2. the node planes are staged through registers computing the new search
//      direction on the fly, p_new = r*inv + beta*p_old (numpy rounding), the
//      owning CTA writes p_new once (ping-pong buffers: no CTA ever reads a
//      p value another CTA has already overwritten);
//   3. q = A p_new exactly as k_grid_tile3 (masked input, pass-through) and
//      per-CTA p.q partials for k_update_f.
// This removes the separate direction kernel (a full read of r, inv, p and a
// write of p) and its launch from every CG iteration.
// ---------------------------------------------------------------------------
#ifndef TF_CG_MINB32
#define TF_CG_MINB32 2
#endif
template <typename T>
__global__ void __launch_bounds__(TileDims<T>::NT, sizeof(T) == 4 ? TF_CG_MINB32 : 2)
k_grid_tile3_cg(Grid g, int oz, const T* __restrict__ scale, T* __restrict__ w,
                const uint8_t* __restrict__ node_fixed, double* __restrict__ dot_part,
                const __grid_constant__ KhatBlocks<T> kb, const __grid_constant__ CgTileArgs<T> A)
{
    constexpr int TILE_BY = TileDims<T>::BY, TILE_NT = TileDims<T>::NT;
    constexpr int PW = StageSlots<T>::PW, PN = StageSlots<T>::PN, NS = StageSlots<T>::N;
    __shared__ __align__(16) T plane[2][PN];
    __shared__ T Y[3][TILE_NT];
    __shared__ double shr[2][TILE_NT / 32];

    CgScalars* sc = A.sc;
    if (sc->done) return;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = tx + TILE_BX * ty;
    const bool f32 = sizeof(T) == 4;

    // ---- 1. decision for the previous iteration ----------------------------------
    const int it_prev = sc->it_a;
    double beta = 0.0;
    if (it_prev > 0) {
        double v0 = 0.0, v1 = 0.0;
        for (int i = tid; i < A.nparts; i += TILE_NT) {
            v0 += __ldcg(A.part + 2 * i);
            v1 += __ldcg(A.part + 2 * i + 1);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            v0 += __shfl_down_sync(0xffffffffu, v0, o);
            v1 += __shfl_down_sync(0xffffffffu, v1, o);
        }
        if ((tid & 31) == 0) {
            shr[0][tid >> 5] = v0;
            shr[1][tid >> 5] = v1;
        }
        __syncthreads();
        double rr = 0.0, rzn = 0.0;
        for (int i = 0; i < TILE_NT / 32; ++i) {
            rr += shr[0][i];
            rzn += shr[1][i];
        }
        const double rn = cg_sqrt(cg_round(rr, f32), f32);
        bool stop = false;
        int term = TERM_MAX_ITER;
        double rel = 0.0, rz_new = 0.0;
        if (!isfinite(rn)) {
            stop = true;
            term = TERM_DIVERGED;
        } else {
            rel = rn / sc->bnorm;
            if (rel <= sc->tol) {
                stop = true;
                term = TERM_CONVERGED;
            } else {
                rz_new = cg_round(rzn, f32);
                beta = rz_new / sc->rz_old;
                if (it_prev >= sc->max_iter) stop = true;
            }
        }
        const bool b0 = blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0;
        if (b0) {
            if (isfinite(rn)) {
                sc->rel = rel;
                if (sc->hist) sc->hist[it_prev] = rel;
            }
            if (stop) {
                sc->done = 1;
                sc->term = term;
                sc->it = it_prev;
                if (A.in_graph) cudaGraphSetConditional(A.h_while, 0u);
            } else {
                sc->rz = rz_new;
                sc->beta = beta;
            }
        }
        if (stop) return;
    }
    const int it_now = it_prev + 1;
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0) sc->it_b = it_now;
    const T* __restrict__ p_old = A.pbuf[it_prev & 1];
    T* __restrict__ p_new = A.pbuf[it_now & 1];
    const T be = (T)beta;
    const bool first = it_prev == 0;

    // ---- 2./3. staged matvec on p_new ----------------------------------------------
    const int i0 = blockIdx.x * (TILE_BX - 1);
    const int j0 = blockIdx.y * (TILE_BY - 1);
    const int k0 = blockIdx.z * oz;
    const int ex = i0 - 1 + tx, ey = j0 - 1 + ty;
    const bool col_ok = ex >= 0 && ex < g.nelx && ey >= 0 && ey < g.nely;
    const bool owner = tx < TILE_BX - 1 && ty < TILE_BY - 1 && (i0 + tx) < g.nnx && (j0 + ty) < g.nny;
    const int pn = g.nnx * g.nny, pn3 = 3 * pn;
    const uint8_t* col_or = node_fixed ? node_fixed + g.n_nodes : nullptr;
    const uint8_t* col_and = node_fixed ? col_or + pn : nullptr;

    int s_off[NS], s_node[NS], s_c[NS];
    unsigned okbits = 0u, mskbits = 0u, allfix = 0u, ownbits = 0u;
#pragma unroll
    for (int q = 0; q < NS; ++q) {
        const int idx = tid + q * TILE_NT;
        const int r = idx / PW, f = idx - r * PW;
        const int ii = i0 - 1 + f / 3, jj = j0 - 1 + r, c = f % 3;
        const bool ok = idx < PN && ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny;
        const int node = ok ? ii + g.nnx * jj : 0;
        s_off[q] = 3 * node + c;
        s_node[q] = node;
        s_c[q] = c;
        if (ok) {
            okbits |= 1u << q;
            if (node_fixed) {
                if ((col_and[node] >> c) & 1u) allfix |= 1u << q;
                else if ((col_or[node] >> c) & 1u) mskbits |= 1u << q;
            }
            // the CTA owning node column (ii, jj) writes its p_new
            if (ii >= i0 && ii < i0 + TILE_BX - 1 && jj >= j0 && jj < j0 + TILE_BY - 1) ownbits |= 1u << q;
        }
    }
    // raw r, inv, p_old of a plane prefetched into registers one layer ahead
    T pr[NS], pi[NS], pp[NS];
    auto fetch = [&](int kz) {
        const bool zok = kz >= 0 && kz < g.nnz;
        const long long base = (long long)min(max(kz, 0), g.nnz - 1) * pn3;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const bool take = zok && ((okbits >> q) & 1u);
            const long long d = base + s_off[q];
            pr[q] = take ? ld_nc(A.r + d) : T(0);
            pi[q] = take ? ld_nc(A.inv + d) : T(0);
            pp[q] = (take && !first) ? p_old[d] : T(0);
        }
    };
    auto commit = [&](int kz, T* buf) {
        const bool zok = kz >= 0 && kz < g.nnz;
        const bool wr = zok && kz >= k0 && kz < k0 + oz;
        const long long base = (long long)min(max(kz, 0), g.nnz - 1) * pn3;
#pragma unroll
        for (int q = 0; q < NS; ++q) {
            const int idx = tid + q * TILE_NT;
            if (q < NS - 1 || idx < PN) {
                const bool ok = zok && ((okbits >> q) & 1u);
                T pv = first ? mul_rn(pr[q], pi[q]) : add_rn(mul_rn(pr[q], pi[q]), mul_rn(be, pp[q]));
                if (!ok) pv = T(0);
                if (wr && ((ownbits >> q) & 1u)) p_new[base + s_off[q]] = pv;
                bool fixed = (allfix >> q) & 1u;
                if (!fixed && ((mskbits >> q) & 1u) && ok) fixed = (node_fixed[kz * pn + s_node[q]] >> s_c[q]) & 1u;
                buf[idx] = fixed ? T(0) : pv;
            }
        }
    };
    const int pofs = ty * PW + 3 * tx;
    auto pv_ = [&](const T* buf, int ox, int oy, int c) -> T { return buf[pofs + oy * PW + 3 * ox + c]; };
    const int el_col = ex + g.nelx * ey, el_plane = g.nelx * g.nely;
    auto scale_at = [&](int ez) -> T {
        return (col_ok && ez >= 0 && ez < g.nelz) ? ld_nc(scale + el_col + el_plane * ez) : T(0);
    };

    const int n_layers = min(oz, g.nnz - k0) + 1;
    T* b_cur = plane[0];
    T* b_top = plane[1];
    fetch(k0 - 1);
    commit(k0 - 1, b_cur);
    fetch(k0);
    commit(k0, b_top);
    fetch(k0 + 1);
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
    T dot = T(0);
    const int own_node0 = (i0 + tx) + g.nnx * (j0 + ty);

    for (int L = 0; L < n_layers; ++L) {
        const int ez = k0 - 1 + L;
        if (L >= 1) {
            // plane ez+1 into the buffer that held plane ez-1 (read before (B) of layer L-1)
            commit(ez + 1, b_top);
            if (L + 1 < n_layers) fetch(ez + 2);
        }
        __syncthreads();                                   // (A)
        const T s_next = scale_at(ez + 1);
        const bool write_plane = owner && L >= 1;
        unsigned own_bits = 0u;
        if (write_plane && node_fixed) own_bits = node_fixed[own_node0 + ez * pn];
        T pown[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) pown[c] = pv_(b_cur, 1, 1, c);
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
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int m = 1; m < 8; ++m) h[c][m] *= s_cur;
        T gm[3][8];
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
        __syncthreads();                                   // (B)
        if (write_plane) {
            const int d0 = 3 * (own_node0 + ez * pn);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                T acc = xr[1][c] + Y[c][tid + TILE_BX];
                const int d = d0 + c;
                const bool fx = (own_bits >> c) & 1u;
                // constrained DOF: q = p (pass-through); p itself is unmasked
                const T p = fx ? p_new[d] : pown[c];
                if (fx) acc = p;
                w[d] = acc;
                dot = fma(p, acc, dot);
            }
        }
        s_cur = s_next;
        T* t = b_cur;
        b_cur = b_top;
        b_top = t;
    }

    double dd = (double)dot;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dd += __shfl_down_sync(0xffffffffu, dd, o);
    __syncthreads();
    if ((tid & 31) == 0) shr[0][tid >> 5] = dd;
    __syncthreads();
    if (tid == 0) {
        double s2 = 0.0;
        for (int i = 0; i < TILE_NT / 32; ++i) s2 += shr[0][i];
        dot_part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = s2;
    }
}

struct TileShape {
    dim3 grid;
    int oz;
};

// The isotropic block form (khat_iso) in every FP64 kernel: there the kernel
// is DFMA-bound and the 25 fewer FP ops per element-layer are worth 30 % (c5
// 125 vs 179 us).  The FP32 SM-resident PCG keeps the generic blocks: the
// different rounding order shifted its FP32 CG counts by more than the +-2 %
// bar on converging solves (torsion SIMP 10013 vs 10786 total); FP32 plain
// products and the graph-protocol CG matvec take the iso form
// (tile_iso32_plain, tile_iso32_cg).  TF_TILE_GENERIC=1 forces the generic
// blocks everywhere.
template <typename T>
bool tile_iso_enabled()
{
    const char* eg = getenv("TF_TILE_GENERIC");
    if (eg && eg[0] == '1') return false;
    return sizeof(T) == 8;
}
template bool tile_iso_enabled<float>();
// FP32 plain products (no CG partials, no accumulation) use the isotropic
// form too: c2 14.4 vs 15.3 us, c4 27.8 vs 29.4, c5 84.2 vs 90.2 (B200,
// scripts/tile_ab.py); the FP32 CG keeps the generic blocks (see above).
// TF_TILE_ISO32=0 or TF_TILE_GENERIC=1 keeps them generic.
// The graph-protocol FP32 CG matvec (fused p.q partials; grids too large for
// the SM-resident solve, whose FP32 CG stays generic) takes the isotropic
// form as well: c4 47.3 -> 43.4 us per iteration, c5 192 -> 179; those
// solves run to the 1000-iteration cap like the reference's (counts equal),
// compliance moves by 1e-6.  TF_CG_ISO32=0 keeps the generic blocks.
static bool tile_iso32_cg()
{
    const char* e = getenv("TF_CG_ISO32");
    return !(e && e[0] == '0');
}
static bool tile_iso32_plain()
{
    const char* e = getenv("TF_TILE_ISO32");
    const char* eg = getenv("TF_TILE_GENERIC");
    return !(e && e[0] == '0') && !(eg && eg[0] == '1');
}
template bool tile_iso_enabled<double>();

template <typename T>
static int tile_slots()
{
    // resident CTAs of the tile kernel on this device (cached per precision)
    static int slots[2] = {0, 0};
    int& s = slots[sizeof(T) == 8];
    if (s == 0) {
        int dev = 0, nsm = 148, per_sm = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, k_grid_tile5<T, true, true, false, true, TF_TILE_P, false>, TileDims<T>::NT, 0);
        s = std::max(1, per_sm) * nsm;
    }
    return s;
}

template <typename T>
TileShape tile_shape_oz(const Grid& g, int oz)
{
    constexpr int TILE_BY = TileDims<T>::BY;
    const int tx = (g.ihi - g.ilo + TILE_BX - 2) / (TILE_BX - 1);
    const int ty = (g.nny + TILE_BY - 2) / (TILE_BY - 1);
    return {dim3(tx, ty, (g.nnz + oz - 1) / oz), oz};
}

// z-chunk height: the smallest chunk count that keeps every SM busy is one
// wave of resident CTAs; never chunk finer than 2 planes (halo layer cost
// 1/oz) nor coarser than 16 once the grid spans several waves anyway.
template <typename T>
TileShape tile_shape(const Grid& g)
{
    constexpr int TILE_BY = TileDims<T>::BY;
    const int tx = (g.ihi - g.ilo + TILE_BX - 2) / (TILE_BX - 1);
    const int ty = (g.nny + TILE_BY - 2) / (TILE_BY - 1);
    const long long cols = (long long)tx * ty;
    const long long slots = tile_slots<T>();
    long long chunks = std::max<long long>(1, slots / cols);           // fill one wave
    int oz = (int)std::max<long long>(2, (g.nnz + chunks - 1) / chunks);
    oz = std::min(oz, 16);
    // big grids: taller chunks halve the halo layer when >= 1.5 waves remain
    // (c5: 100.8 vs 104.6 us measured; smaller grids keep 16)
    if (oz == 16 && cols * ((g.nnz + 31) / 32) * 2 >= 3 * slots) oz = 32;
    const char* e = getenv("TF_TILE_OZ");  // experiment override of the z-chunk height
    const int oz_env = e ? std::max(0, atoi(e)) : 0;
    if (oz_env > 0) oz = oz_env;
    return tile_shape_oz<T>(g, oz);
}

static int TileDimsBy(int prec) { return prec == 8 ? TileDims<double>::BY : TileDims<float>::BY; }

static bool tile_autotune_enabled()
{
    const char* e = getenv("TF_TILE_AUTOTUNE");
    if (e && e[0] == '0') return false;
    const char* o = getenv("TF_TILE_OZ");  // a pinned chunk height wins
    return !(o && atoi(o) > 0);
}

// z-chunk height per (grid shape, x-range, precision): measured once with
// CUDA events over the candidates (min of 5 cold single launches each),
// then cached.  Every candidate gives the same bits (every DOF is summed in
// the same order for any chunking), so this only picks the fastest.  Returns
// 0 when it cannot tune (stream capture in progress) or when lookup_only
// finds nothing.  TF_TILE_DEBUG=1 prints the candidate timings.
template <typename F>
static int tile_tuned_oz(const Grid& g, int prec, cudaStream_t st, F&& launch, bool lookup_only = false)
{
    static std::mutex mu;
    static std::map<std::array<int, 6>, int> cache;
    const std::array<int, 6> key = {g.nelx, g.nely, g.nelz, g.ilo, g.ihi, prec};
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
        if (lookup_only) return 0;
    }
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return 0;
    }
    static const int cands[] = {2, 3, 4, 5, 6, 7, 8, 10, 12, 16, 24, 32};
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    // candidates must cover every SM (a shape that leaves SMs idle can win a
    // single-launch timing through lower launch latency, not throughput)
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long cols = (long long)((g.ihi - g.ilo + TILE_BX - 2) / (TILE_BX - 1)) *
                           ((g.nny + TileDimsBy(prec) - 2) / (TileDimsBy(prec) - 1));
    int best = 0;
    float best_ms = 1e30f;
    const char* dbg_env = getenv("TF_TILE_DEBUG");
    const bool dbg = dbg_env && dbg_env[0] == '1';
    // each candidate is timed as single launches behind an L2 eviction (a
    // write of twice the L2 size): a product called on its own meets its
    // inputs in HBM, and the chunk height that wins warm, back-to-back
    // launches (more CTAs, shorter marches) loses cold (c2: oz 3 vs 4,
    // scripts/tile_trace.py).  Without the scratch buffer: warm timing.
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
    void* flush = nullptr;
    const size_t flush_bytes = 2 * (size_t)std::max(l2, 1 << 20);
    if (cudaMalloc(&flush, flush_bytes) != cudaSuccess) {
        cudaGetLastError();
        flush = nullptr;
    }
    for (int oz : cands) {
        if (oz > std::max(2, g.nnz)) break;
        const int chunks = (g.nnz + oz - 1) / oz;
        if (oz > 2 && cols * chunks < nsm) break;
        if (launch(oz) != TF_OK) {  // warm-up
            cudaGetLastError();
            break;
        }
        float t = 1e30f;
        const int reps = flush ? 5 : 3, per = flush ? 1 : 4;
        for (int r = 0; r < reps; ++r) {
            if (flush) cudaMemsetAsync(flush, r, flush_bytes, st);
            cudaEventRecord(e0, st);
            for (int k = 0; k < per; ++k) launch(oz);
            cudaEventRecord(e1, st);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            t = std::min(t, ms / per);
        }
        if (dbg) fprintf(stderr, "[tile_tuned] %dx%dx%d oz=%d: %.2f us per launch (%s)\n", g.nelx, g.nely, g.nelz,
                         oz, 1e3f * t, flush ? "cold" : "warm");
        if (t < best_ms) {
            best_ms = t;
            best = oz;
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (flush) {
        cudaStreamSynchronize(st);
        cudaFree(flush);
    }
    cudaGetLastError();
    if (best > 0) {
        std::lock_guard<std::mutex> lk(mu);
        cache[key] = best;
    }
    return best;
}

// launch shape a plain product on grid g would use now (autotuned if tuned)
template <typename T>
TileShape tile_shape_current(const Grid& g)
{
    TileShape sh = tile_shape<T>(g);
    if (tile_autotune_enabled()) {
        const int oz = tile_tuned_oz(g, (int)sizeof(T), nullptr, [](int) { return TF_ERR_ARG; }, true);
        if (oz > 0) sh = tile_shape_oz<T>(g, oz);
    }
    return sh;
}

template <typename T>
long long grid_tile_blocks(const Grid& g)
{
    TileShape s = tile_shape<T>(g);
    return (long long)s.grid.x * s.grid.y * s.grid.z;
}

// returns TF_ERR_UNSUPPORTED when Ke lacks the parity-block structure
template <typename T>
static int launch_grid_tile_impl(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                                 const uint8_t* node_fixed, uint32_t flags, double* dot_part, cudaStream_t st,
                                 const TilePut<T>* put)
{
    KhatBlocks<T> kb;
    if (!khat_blocks_cached<T>(ke_host, &kb)) return TF_ERR_UNSUPPORTED;
    if (3 * g.n_nodes >= (1LL << 31)) {
        set_error("structured grid too large for int32 DOF indices");
        return TF_ERR_ARG;
    }
    KhatIso<T> ki{};
    const bool iso = tile_iso_enabled<T>() && khat_iso<T>(ke_host, &ki);
    const bool iso32 = sizeof(T) == 4 && tile_iso32_plain() && khat_iso<T>(ke_host, &ki);
    const uint32_t f = flags & (TF_MASK_INPUT | TF_PASS_FIXED | TF_ACCUMULATE);
    constexpr uint32_t MP = TF_MASK_INPUT | TF_PASS_FIXED;
    if (put && (dot_part || f != TF_MASK_INPUT)) {
        set_error("the fused interface put is the slab's masked range product only");
        return TF_ERR_ARG;
    }
    auto launch_shape = [&](const TileShape& sh, bool with_put = false) -> int {
        dim3 block(TILE_BX, TileDims<T>::BY, 1);
        if (with_put) {
            if ((sizeof(T) == 8 && iso) || (sizeof(T) == 4 && iso32))
                k_grid_tile5<T, true, false, false, false, TF_TILE_P, true, true>
                    <<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, nullptr, kb, ki, *put);
            else
                k_grid_tile5<T, true, false, false, false, TF_TILE_P, false, true>
                    <<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, nullptr, kb, ki, *put);
            TF_CHECK_LAUNCH();
            return TF_OK;
        }
        // isotropic blocks: every FP64 product; FP32 plain products (no CG
        // partials, no accumulation) -- the FP32 CG keeps the generic blocks
#define T5(M, PS, AC, DT, DP)                                                                                  \
    do {                                                                                                       \
        if ((sizeof(T) == 8 && iso) || (sizeof(T) == 4 && !(AC) && !(DT) && iso32))                           \
            k_grid_tile5<T, M, PS, AC, DT, TF_TILE_P, !(AC) && !(DT) || sizeof(T) == 8>                         \
                <<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, DP, kb, ki, TilePut<T>{});      \
        else                                                                                                   \
            k_grid_tile5<T, M, PS, AC, DT, TF_TILE_P, false><<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, \
                                                                                     node_fixed, DP, kb, ki,   \
                                                                                     TilePut<T>{});            \
    } while (0)
        if (dot_part) {  // CG p.q partials: the solver's masked, passed-through product only
            if (f != MP) {
                set_error("the fused p.q epilogue needs TF_MASK_INPUT | TF_PASS_FIXED");
                return TF_ERR_ARG;
            }
            if (sizeof(T) == 4 && iso32 && tile_iso32_cg())
                k_grid_tile5<T, true, true, false, true, TF_TILE_P, true>
                    <<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, dot_part, kb, ki, TilePut<T>{});
            else
                T5(true, true, false, true, dot_part);
        } else {
            switch (f) {
            case MP:
                // short z-chunks (one-wave grids such as c2): one plane of
                // look-ahead instead of two -- the prologue waits for two
                // planes, not three (c2 14.7 -> 14.1 us; deeper chunks keep
                // P = 2: c5 80.3 vs 82.0 at P = 1)
                if (sh.oz <= TF_TILE_P1_OZ) {
                    if ((sizeof(T) == 8 && iso) || (sizeof(T) == 4 && iso32))
                        k_grid_tile5<T, true, true, false, false, 1, true>
                            <<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, nullptr, kb, ki, TilePut<T>{});
                    else
                        k_grid_tile5<T, true, true, false, false, 1, false>
                            <<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, nullptr, kb, ki, TilePut<T>{});
                } else {
                    T5(true, true, false, false, nullptr);
                }
                break;
            case TF_MASK_INPUT: T5(true, false, false, false, nullptr); break;
            case TF_PASS_FIXED: T5(false, true, false, false, nullptr); break;
            case 0: T5(false, false, false, false, nullptr); break;
            case MP | TF_ACCUMULATE: T5(true, true, true, false, nullptr); break;
            case TF_MASK_INPUT | TF_ACCUMULATE: T5(true, false, true, false, nullptr); break;
            case TF_PASS_FIXED | TF_ACCUMULATE: T5(false, true, true, false, nullptr); break;
            default: T5(false, false, true, false, nullptr); break;  // TF_ACCUMULATE
            }
        }
#undef T5
        TF_CHECK_LAUNCH();
        return TF_OK;
    };
    TileShape sh = tile_shape<T>(g);
    // Plain products (no CG partials, no accumulation): the launch shape is
    // autotuned once per grid shape on first use outside stream capture
    if (!dot_part && !(flags & TF_ACCUMULATE) && tile_autotune_enabled()) {
        const int oz = tile_tuned_oz(g, (int)sizeof(T), st, [&](int cand) {
            return launch_shape(tile_shape_oz<T>(g, cand));
        });
        if (oz > 0) sh = tile_shape_oz<T>(g, oz);
    }
    // (the autotune's timing launches above never carry the put)
    return launch_shape(sh, put != nullptr);
}

template <typename T>
int launch_grid_tile(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                     const uint8_t* node_fixed, uint32_t flags, double* dot_part, cudaStream_t st)
{
    return launch_grid_tile_impl<T>(g, ke_host, scale, v, w, node_fixed, flags, dot_part, st, nullptr);
}

// C ABI: the slab's range product with the fused interface put (see TilePut)
#define TF_RANGE_PUT(T, SUF)                                                                              \
    int tf_matvec_grid_range_put_##SUF(const tf_grid* gd, const T* ke, const T* scale, const T* v, T* w,   \
                                       const uint8_t* node_fixed, int32_t i_lo, int32_t i_hi, int32_t put_i, \
                                       T* dst, uint32_t* flag, uint32_t* ticket, const uint32_t* ep_dev,    \
                                       uint32_t epoch, void* stream)                                      \
    {                                                                                                     \
        TF_REQUIRE(gd && ke && scale && v && w && dst && flag && ticket, "null pointer");                \
        Grid gg = make_grid(gd);                                                                          \
        TF_REQUIRE(0 <= i_lo && i_lo < i_hi && i_hi <= gg.nnx && i_lo <= put_i && put_i < i_hi,           \
                   "bad node x-range / put plane");                                                       \
        gg.ilo = i_lo;                                                                                    \
        gg.ihi = i_hi;                                                                                    \
        TilePut<T> tp{dst, flag, ticket, ep_dev, epoch, put_i};                                           \
        const int rc = launch_grid_tile_impl<T>(gg, ke, scale, v, w, node_fixed, TF_MASK_INPUT, nullptr,  \
                                                reinterpret_cast<cudaStream_t>(stream), &tp);             \
        if (rc == TF_ERR_UNSUPPORTED) set_error("node ranges need the parity-block tile kernel");         \
        return rc;                                                                                        \
    }

// Fused CG head (decision + direction + matvec + p.q partials); grid as the
// production tile kernel so the partial count matches grid_tile_blocks().
template <typename T>
int launch_grid_tile_cg(const Grid& g, const T* ke_host, const T* scale, T* q,
                        const uint8_t* node_fixed, double* dot_part, const CgTileArgs<T>& a,
                        cudaStream_t st)
{
    KhatBlocks<T> kb;
    if (!khat_blocks_cached<T>(ke_host, &kb)) return TF_ERR_UNSUPPORTED;
    if (3 * g.n_nodes >= (1LL << 31)) {
        set_error("structured grid too large for int32 DOF indices");
        return TF_ERR_ARG;
    }
    TileShape sh = tile_shape<T>(g);
    dim3 block(TILE_BX, TileDims<T>::BY, 1);
    k_grid_tile3_cg<T><<<sh.grid, block, 0, st>>>(g, sh.oz, scale, q, node_fixed, dot_part, kb, a);
    TF_CHECK_LAUNCH();
    return TF_OK;
}
template int launch_grid_tile_cg<float>(const Grid&, const float*, const float*, float*,
                                        const uint8_t*, double*, const CgTileArgs<float>&, cudaStream_t);
template int launch_grid_tile_cg<double>(const Grid&, const double*, const double*, double*,
                                         const uint8_t*, double*, const CgTileArgs<double>&, cudaStream_t);

template <typename T>
bool launch_grid_tile_supported(const T* ke_host)
{
    KhatBlocks<T> kb;
    return khat_blocks<T>(ke_host, &kb);
}
template bool launch_grid_tile_supported<float>(const float*);
template bool launch_grid_tile_supported<double>(const double*);
template long long grid_tile_blocks<float>(const Grid&);
template long long grid_tile_blocks<double>(const Grid&);
template int launch_grid_tile<float>(const Grid&, const float*, const float*, const float*, float*,
                                     const uint8_t*, uint32_t, double*, cudaStream_t);
template int launch_grid_tile<double>(const Grid&, const double*, const double*, const double*,
                                      double*, const uint8_t*, uint32_t, double*, cudaStream_t);

}  // namespace tf

using tf::TilePut;
using tf::launch_grid_tile_impl;
using tf::make_grid;
using tf::Grid;
using tf::set_error;
TF_RANGE_PUT(float, f32)
TF_RANGE_PUT(double, f64)

#ifdef TF_TILE_TRACE
extern "C" int tf_tile_trace_set(void* buf)
{
    unsigned long long* p = (unsigned long long*)buf;
    TF_CUDA_TRY(cudaMemcpyToSymbol(tf::g_tile_trace, &p, sizeof(p)));
    return TF_OK;
}
#endif

extern "C" int tf_tile_shape(const tf_grid* grid, int precision, int32_t* oz, int64_t* ctas)
{
    using namespace tf;
    TF_REQUIRE(grid && oz && ctas && (precision == 32 || precision == 64), "bad arguments");
    const Grid g = make_grid(grid);
    const TileShape sh = precision == 32 ? tile_shape_current<float>(g) : tile_shape_current<double>(g);
    *oz = sh.oz;
    *ctas = (int64_t)sh.grid.x * sh.grid.y * sh.grid.z;
    return TF_OK;
}
