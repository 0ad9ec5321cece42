// Minimal 1-D TMA load (cp.async.bulk.tensor.1d) probe: negative / in-range /
// beyond-end coordinates, completion on an mbarrier.  Finding (B200): the
// innermost start coordinate must be 16-byte aligned (c0=3 floats raises an
// illegal-instruction error); aligned negative / beyond-end starts zero-fill.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap map, int c0, float* out)
{
    __shared__ __align__(128) float buf[128];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(400u) : "memory");
        asm volatile("cp.async.bulk.tensor.1d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2}], [%3];"
                     ::"r"(s32(buf)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(s32(&bar)) : "memory");
    }
    unsigned ok = 0;
    while (!ok) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(s32(&bar)), "r"(0u) : "memory");
    }
    for (int i = threadIdx.x; i < 100; i += blockDim.x) out[i] = buf[i];
}

int main()
{
    const int n = 1000;
    float *d, *o, h[100];
    cudaMalloc(&d, n * 4);
    cudaMalloc(&o, 100 * 4);
    float hv[n];
    for (int i = 0; i < n; ++i) hv[i] = (float)i;
    cudaMemcpy(d, hv, n * 4, cudaMemcpyHostToDevice);
    PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap map;
    cuuint64_t dims[1] = {(cuuint64_t)n}, str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[1] = {100}, es[1] = {1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int c0 : {0, 4, -4, 952, -152, 996}) {
        k<<<1, 128>>>(map, c0, o);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("c0=%d: %s\n", c0, cudaGetErrorString(e)); return 1; }
        cudaMemcpy(h, o, 400, cudaMemcpyDeviceToHost);
        printf("c0=%5d: %g %g %g ... %g\n", c0, h[0], h[1], h[2], h[99]);
    }
    return 0;
}
