// Throughput of FP32 scalar vs packed (FADD2/FFMA2) instructions on sm_100a.
// Each thread runs independent chains (ILP 8) so the pipe, not latency, binds.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters, float a, float b)
{
    float2 x[8];
    float y[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = threadIdx.x * 1e-3f + i;
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, -b);
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {  // scalar FADD, register operands
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = y[i] + y[(i + 1) & 15];
        } else if (MODE == 1) {  // packed FADD2
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __fadd2_rn(x[i], x[(i + 1) & 7]);
        } else if (MODE == 2) {  // scalar FFMA, 3 register operands
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = fmaf(y[i], y[(i + 1) & 15], y[(i + 2) & 15]);
        } else {  // packed FFMA2
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(x[i], x[(i + 1) & 7], x[(i + 2) & 7]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main()
{
    float* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    const int iters = 20000;
    const char* names[] = {"FADD", "FADD2", "FFMA", "FFMA2"};
    for (int mode = 0; mode < 4; ++mode) {
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 8, 256>>>(out, iters, 1.0001f, 0.5f);
            if (mode == 1) k<1><<<148 * 8, 256>>>(out, iters, 1.0001f, 0.5f);
            if (mode == 2) k<2><<<148 * 8, 256>>>(out, iters, 1.0001f, 0.5f);
            if (mode == 3) k<3><<<148 * 8, 256>>>(out, iters, 1.0001f, 0.5f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double lanes_ops = 148.0 * 8 * 256 * iters * 16;  // scalar FP ops (adds or fmas)
        printf("%-6s %8.3f ms  %8.2f Gop/s (fp32 lane ops)\n", names[mode], ms, lanes_ops / ms / 1e6);
    }
    return 0;
}
