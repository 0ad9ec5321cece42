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
#include <cmath>
#include <cstring>

#include "tf_common.cuh"

namespace tf {

constexpr int TILE_BX = 32;
// 8 rows of element columns for FP32, 4 for FP64 (static smem stays < 48 KB)
template <typename T> struct TileDims { static constexpr int BY = sizeof(T) == 8 ? 4 : 8; static constexpr int NT = TILE_BX * BY; };

template <typename T>
struct KhatBlocks {
    T b[8][3][3];  // block q, row c, col c'
};

// binary corner index of the reference corner order (mesh.py:19-31)
__host__ __device__ constexpr int bin_of(int a)
{
    return (a & 4) | ((a & 3) == 0 ? 0 : (a & 3) == 1 ? 1 : (a & 3) == 2 ? 3 : 2);
}

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

template bool khat_blocks<float>(const float*, KhatBlocks<float>*);
template bool khat_blocks<double>(const double*, KhatBlocks<double>*);

// ---- device ------------------------------------------------------------------------

template <typename T>
__device__ __forceinline__ void fwht_fwd(T (&x)[8])
{
#pragma unroll
    for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (!(b & bit)) {
                const T lo = x[b], hi = x[b | bit];
                x[b] = lo + hi;
                x[b | bit] = hi - lo;
            }
}

template <typename T>
__device__ __forceinline__ void fwht_inv(T (&x)[8])
{
#pragma unroll
    for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
        for (int b = 0; b < 8; ++b)
            if (!(b & bit)) {
                const T lo = x[b], hi = x[b | bit];
                x[b] = lo - hi;
                x[b | bit] = lo + hi;
            }
}

// f (reference corner order, 24) = s * Ke * u  via the parity-block form
template <typename T>
__device__ __forceinline__ void element_apply(const T (&u)[NLOC], T s, const KhatBlocks<T>& kb,
                                              T (&f)[NLOC])
{
    T h[3][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) h[c][bin_of(a)] = u[3 * a + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht_fwd(h[c]);
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int m = 1; m < 8; ++m) h[c][m] *= s;  // mode 0 is rigid translation: unused
    T g[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c) g[c][0] = T(0);
#pragma unroll
    for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int m = q ^ (1 << c);
            if (m == 0) continue;  // translation rows of Khat vanish
            T acc = T(0);
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int n = q ^ (1 << d);
                if (n == 0) continue;
                acc = fma(kb.b[q][c][d], h[d][n], acc);
            }
            g[c][m] = acc;
        }
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht_inv(g[c]);
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) f[3 * a + c] = g[c][bin_of(a)];
}

template <typename T, bool DOT>
__global__ void __launch_bounds__(TileDims<T>::NT)
k_grid_tile(Grid g, int oz, const T* __restrict__ scale, const T* __restrict__ v,
            T* __restrict__ w, const uint8_t* __restrict__ node_fixed, uint32_t flags,
            double* __restrict__ dot_part, const __grid_constant__ KhatBlocks<T> kb)
{
    constexpr int TILE_BY = TileDims<T>::BY, TILE_NT = TileDims<T>::NT;
    constexpr int PW = (TILE_BX + 1) * 3;       // floats per staged plane row
    constexpr int PN = PW * (TILE_BY + 1);      // staged plane size
    __shared__ T plane[PN];
    __shared__ T F[NLOC][TILE_NT];

    const int tx = threadIdx.x, ty = threadIdx.y;
    const int tid = tx + TILE_BX * ty;
    const int i0 = blockIdx.x * (TILE_BX - 1);
    const int j0 = blockIdx.y * (TILE_BY - 1);
    const int k0 = blockIdx.z * oz;
    const int ex = i0 - 1 + tx, ey = j0 - 1 + ty;
    const bool col_ok = ex >= 0 && ex < g.nelx && ey >= 0 && ey < g.nely;
    const bool owner = tx < TILE_BX - 1 && ty < TILE_BY - 1 && (i0 + tx) < g.nnx && (j0 + ty) < g.nny;
    const bool mask_in = (flags & TF_MASK_INPUT) && node_fixed != nullptr;
    const long long plane_nodes = (long long)g.nnx * g.nny;

    auto stage = [&](int kz) {
        for (int idx = tid; idx < PN; idx += TILE_NT) {
            const int r = idx / PW, f = idx - r * PW;
            const int ii = i0 - 1 + f / 3, jj = j0 - 1 + r, c = f % 3;
            T val = T(0);
            if (kz >= 0 && kz < g.nnz && ii >= 0 && ii < g.nnx && jj >= 0 && jj < g.nny) {
                const long long node = ii + (long long)g.nnx * jj + plane_nodes * kz;
                const bool fixed = mask_in && ((node_fixed[node] >> c) & 1u);
                if (!fixed) val = ld_nc(v + 3 * node + c);
            }
            plane[idx] = val;
        }
    };

    // corner (ox, oy) of this thread's element column within the staged plane
    auto pidx = [&](int ox, int oy, int c) { return (ty + oy) * PW + 3 * (tx + ox) + c; };

    T u[NLOC];
    stage(k0 - 1);
    __syncthreads();
#pragma unroll
    for (int a = 0; a < 4; ++a) {  // bottom corners 0..3 of the first layer
        const int ox = (a == 1 || a == 2), oy = (a >= 2);
#pragma unroll
        for (int c = 0; c < 3; ++c) u[3 * a + c] = plane[pidx(ox, oy, c)];
    }
    __syncthreads();

    T carry[3] = {T(0), T(0), T(0)};
    double dot = 0.0;
    const long long own_col = (long long)(i0 + tx) + (long long)g.nnx * (j0 + ty);

    for (int L = 0; L <= oz; ++L) {
        const int ez = k0 - 1 + L;
        if (ez >= g.nnz) break;  // no node plane left to complete
        stage(ez + 1);
        __syncthreads();
#pragma unroll
        for (int a = 4; a < 8; ++a) {
            const int ox = (a == 5 || a == 6), oy = (a >= 6);
#pragma unroll
            for (int c = 0; c < 3; ++c) u[3 * a + c] = plane[pidx(ox, oy, c)];
        }
        const bool el_ok = col_ok && ez >= 0 && ez < g.nelz;
        const T s = el_ok ? ld_nc(scale + ex + (long long)g.nelx * (ey + (long long)g.nely * ez)) : T(0);
        T f[NLOC];
        element_apply(u, s, kb, f);
#pragma unroll
        for (int r = 0; r < NLOC; ++r) F[r][tid] = f[r];
        __syncthreads();
        if (owner) {
            // element columns around node (i0+tx, j0+ty): (tx,ty) (tx+1,ty) (tx,ty+1) (tx+1,ty+1)
            const int t00 = tid, t10 = tid + 1, t01 = tid + TILE_BX, t11 = tid + TILE_BX + 1;
            if (L >= 1) {
                const long long node = own_col + plane_nodes * ez;
                const unsigned bits = node_fixed ? (unsigned)node_fixed[node] : 0u;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    T acc = carry[c];
                    acc += F[3 * 2 + c][t00];  // node is corner 2 (1,1,0) of element (i-1,j-1)
                    acc += F[3 * 3 + c][t10];  // corner 3 (0,1,0) of (i, j-1)
                    acc += F[3 * 1 + c][t01];  // corner 1 (1,0,0) of (i-1, j)
                    acc += F[3 * 0 + c][t11];  // corner 0 of (i, j)
                    const long long d = 3 * node + c;
                    if (flags & TF_ACCUMULATE) acc += w[d];
                    if ((flags & TF_PASS_FIXED) && ((bits >> c) & 1u)) acc = v[d];
                    w[d] = acc;
                    if (DOT) dot += (double)ld_nc(v + d) * (double)acc;
                }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                T t = F[3 * 6 + c][t00];
                t += F[3 * 7 + c][t10];
                t += F[3 * 5 + c][t01];
                t += F[3 * 4 + c][t11];
                carry[c] = t;
            }
        }
        // the plane above becomes the plane below
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = 0; c < 3; ++c) u[3 * a + c] = u[3 * (a + 4) + c];
        __syncthreads();
    }

    if (DOT) {
        __shared__ double sh[TILE_NT / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_down_sync(0xffffffffu, dot, o);
        if ((tid & 31) == 0) sh[tid >> 5] = dot;
        __syncthreads();
        if (tid == 0) {
            double s = 0.0;
            for (int i = 0; i < TILE_NT / 32; ++i) s += sh[i];
            dot_part[blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)] = s;
        }
    }
}

struct TileShape {
    dim3 grid;
    int oz;
};

template <typename T>
TileShape tile_shape(const Grid& g)
{
    constexpr int TILE_BY = TileDims<T>::BY;
    const int tx = (g.nnx + TILE_BX - 2) / (TILE_BX - 1);
    const int ty = (g.nny + TILE_BY - 2) / (TILE_BY - 1);
    int nsm = 148;
    // aim for >= 3 CTAs per SM; fewer, taller z-chunks amortise the halo layer
    long long want = 3LL * nsm;
    int oz = (int)std::max<long long>(2, std::min<long long>(16, ((long long)g.nnz * tx * ty) / want));
    const int tz = (g.nnz + oz - 1) / oz;
    return {dim3(tx, ty, tz), oz};
}

template <typename T>
long long grid_tile_blocks(const Grid& g)
{
    TileShape s = tile_shape<T>(g);
    return (long long)s.grid.x * s.grid.y * s.grid.z;
}

// returns TF_ERR_UNSUPPORTED when Ke lacks the parity-block structure
template <typename T>
int launch_grid_tile(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                     const uint8_t* node_fixed, uint32_t flags, double* dot_part, cudaStream_t st)
{
    KhatBlocks<T> kb;
    static thread_local T last_ke[NLOC * NLOC];
    static thread_local KhatBlocks<T> last_kb;
    static thread_local int last_ok = -1;
    if (last_ok >= 0 && memcmp(last_ke, ke_host, sizeof(last_ke)) == 0) {
        if (!last_ok) return TF_ERR_UNSUPPORTED;
        kb = last_kb;
    } else {
        const bool ok = khat_blocks<T>(ke_host, &kb);
        memcpy(last_ke, ke_host, sizeof(last_ke));
        last_kb = kb;
        last_ok = ok ? 1 : 0;
        if (!ok) return TF_ERR_UNSUPPORTED;
    }
    TileShape sh = tile_shape<T>(g);
    dim3 block(TILE_BX, TileDims<T>::BY, 1);
    if (dot_part)
        k_grid_tile<T, true><<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, flags, dot_part, kb);
    else
        k_grid_tile<T, false><<<sh.grid, block, 0, st>>>(g, sh.oz, scale, v, w, node_fixed, flags, nullptr, kb);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

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
