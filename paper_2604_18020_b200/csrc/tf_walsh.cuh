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

}  // namespace tf
