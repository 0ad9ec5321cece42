// Corner-Walsh (parity-block) element algebra and tile geometry shared by the
// structured tile kernels (tf_tile.cu) and the SM-resident PCG (tf_pcg_resident.cu).
// See tf_tile.cu's header for the algebra.
#pragma once

#include <type_traits>

#include "tf_common.cuh"

namespace tf {

constexpr int TILE_BX = 32;
// 8 rows of element columns for FP32, 4 for FP64 (static smem stays < 48 KB)
#ifndef TF_TILE_BY32
#define TF_TILE_BY32 8
#endif
template <typename T> struct TileDims { static constexpr int BY = sizeof(T) == 8 ? 4 : TF_TILE_BY32; static constexpr int NT = TILE_BX * BY; };

template <typename T>
struct KhatBlocks {
    T b[8][3][3];  // block q, row c, col c'
};

// binary corner index of the reference corner order (mesh.py:19-31)
__host__ __device__ constexpr int bin_of(int a)
{
    return (a & 4) | ((a & 3) == 0 ? 0 : (a & 3) == 1 ? 1 : (a & 3) == 2 ? 3 : 2);
}

// Isotropic-material form of the parity blocks (unit_stiffness of any nu has
// it): q=0/7 blocks [a b b; b a b; b b a], q=1/2/4 2x2 [p r; r p], q=3/5/6 a
// rank-one 2x2 of equal entries x plus one diagonal y, all else zero.  Lets
// the block product run in 33 FP ops instead of ~57, with the element scale
// folded into the 16 coefficients (16 FMUL instead of 21).  Host-checked
// (khat_iso); any other Ke keeps the generic block product.
template <typename T>
struct KhatIso {
    T amb0, b0, p1, r1, p2, r2, x3, y3, p4, r4, x5, y5, x6, y6, amb7, b7;
};

template <typename T>
bool khat_iso(const T* ke, KhatIso<T>* out);

// gm[c][m] (m = 1..7) = sum_d s * Khat[q][c][d] h[d][q ^ (1<<d)] in the iso form
template <typename T>
__device__ __forceinline__ void block_iso(const T (&h)[3][8], const KhatIso<T>& k, T s, T (&gm)[3][8])
{
    const T amb0 = s * k.amb0, b0 = s * k.b0, p1 = s * k.p1, r1 = s * k.r1, p2 = s * k.p2, r2 = s * k.r2;
    const T x3 = s * k.x3, y3 = s * k.y3, p4 = s * k.p4, r4 = s * k.r4, x5 = s * k.x5, y5 = s * k.y5;
    const T x6 = s * k.x6, y6 = s * k.y6, amb7 = s * k.amb7, b7 = s * k.b7;
    const T t0 = b0 * ((h[0][1] + h[1][2]) + h[2][4]);
    gm[0][1] = fma(amb0, h[0][1], t0);
    gm[1][2] = fma(amb0, h[1][2], t0);
    gm[2][4] = fma(amb0, h[2][4], t0);
    gm[1][3] = fma(r1, h[2][5], p1 * h[1][3]);
    gm[2][5] = fma(r1, h[1][3], p1 * h[2][5]);
    gm[0][3] = fma(r2, h[2][6], p2 * h[0][3]);
    gm[2][6] = fma(r2, h[0][3], p2 * h[2][6]);
    const T s3 = x3 * (h[0][2] + h[1][1]);
    gm[0][2] = s3;
    gm[1][1] = s3;
    gm[2][7] = y3 * h[2][7];
    gm[0][5] = fma(r4, h[1][6], p4 * h[0][5]);
    gm[1][6] = fma(r4, h[0][5], p4 * h[1][6]);
    const T s5 = x5 * (h[0][4] + h[2][1]);
    gm[0][4] = s5;
    gm[2][1] = s5;
    gm[1][7] = y5 * h[1][7];
    const T s6 = x6 * (h[1][4] + h[2][2]);
    gm[1][4] = s6;
    gm[2][2] = s6;
    gm[0][7] = y6 * h[0][7];
    const T t7 = b7 * ((h[0][6] + h[1][5]) + h[2][3]);
    gm[0][6] = fma(amb7, h[0][6], t7);
    gm[1][5] = fma(amb7, h[1][5], t7);
    gm[2][3] = fma(amb7, h[2][3], t7);
    gm[0][0] = gm[1][0] = gm[2][0] = T(0);
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

// the same with the isotropic block form (block_iso: 33 FP ops, the scale
// folded into the 16 coefficients) for a Ke that has it (khat_iso)
template <typename T>
__device__ __forceinline__ void element_apply_iso(const T (&u)[NLOC], T s, const KhatIso<T>& ki,
                                                  T (&f)[NLOC])
{
    T h[3][8];
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) h[c][bin_of(a)] = u[3 * a + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht_fwd(h[c]);
    T g[3][8];
    block_iso(h, ki, s, g);
#pragma unroll
    for (int c = 0; c < 3; ++c) fwht_inv(g[c]);
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) f[3 * a + c] = g[c][bin_of(a)];
}

}  // namespace tf
