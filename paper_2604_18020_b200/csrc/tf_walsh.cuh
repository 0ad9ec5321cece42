// Corner-Walsh (parity-block) element algebra and tile geometry shared by the
// structured tile kernels (tf_tile.cu) and the SM-resident PCG (tf_pcg_resident.cu).
// See tf_tile.cu's header for the algebra.
#pragma once

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

// Returns false when Ke is not block diagonal in the parity basis (tf_tile.cu).
template <typename T>
bool khat_blocks(const T* ke, KhatBlocks<T>* out);
// the same behind a per-thread cache keyed on the Ke bytes (use on launch paths)
template <typename T>
bool khat_blocks_cached(const T* ke, KhatBlocks<T>* out);

// Each thread handles at most STAGE_SLOTS values of a staged node plane.
template <typename T>
struct StageSlots {
    static constexpr int PW = (TILE_BX + 1) * 3;
    static constexpr int PN = PW * (TileDims<T>::BY + 1);
    static constexpr int N = (PN + TileDims<T>::NT - 1) / TileDims<T>::NT;
};

template <typename T>
__device__ __forceinline__ void face_fwd(T a00, T a10, T a01, T a11, T (&o)[4])
{
    const T x0y0 = a00 + a10, x1y0 = a10 - a00, x0y1 = a01 + a11, x1y1 = a11 - a01;
    o[0] = x0y0 + x0y1;
    o[1] = x1y0 + x1y1;
    o[2] = x0y1 - x0y0;
    o[3] = x1y1 - x1y0;
}

// inverse xy stage: modes (mx + 2 my) -> corner values c[ox + 2 oy]
template <typename T>
__device__ __forceinline__ void face_inv(const T (&h)[4], T (&c)[4])
{
    const T y0x0 = h[0] - h[1], y0x1 = h[0] + h[1], y1x0 = h[2] - h[3], y1x1 = h[2] + h[3];
    c[0] = y0x0 - y1x0;  // (0,0)
    c[1] = y0x1 - y1x1;  // (1,0)
    c[2] = y0x0 + y1x0;  // (0,1)
    c[3] = y0x1 + y1x1;  // (1,1)
}

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

// Each thread handles at most STAGE_SLOTS values of a staged node plane.

}  // namespace tf
