// H2D paths on this box: which host allocation / stream / destination gets the
// link rate (the e2e leg's ceiling).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o h2d_probe h2d_probe.cu
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

int main()
{
    const size_t n = 686433 * 4 + 12;
    float *h_def, *h_port, *d_m, *d_a, *h_out;
    CK(cudaHostAlloc(&h_def, n, cudaHostAllocDefault));
    CK(cudaHostAlloc(&h_port, n, cudaHostAllocPortable));
    CK(cudaHostAlloc(&h_out, n, cudaHostAllocDefault));
    memset(h_def, 1, n);
    memset(h_port, 1, n);
    CK(cudaMalloc(&d_m, n));
    cudaStream_t s_nb, s_b;
    CK(cudaStreamCreateWithFlags(&s_nb, cudaStreamNonBlocking));
    CK(cudaStreamCreate(&s_b));
    CK(cudaMallocAsync(&d_a, n, s_nb));
    CK(cudaStreamSynchronize(s_nb));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // warm the link
    for (int r = 0; r < 2000; ++r) cudaMemcpyAsync(d_m, h_def, n, cudaMemcpyHostToDevice, 0);
    cudaDeviceSynchronize();
    struct Cfg { const char* name; float* h; float* d; cudaStream_t s; bool d2h_too; };
    Cfg cfgs[] = {{"default host, cudaMalloc, stream 0", h_def, d_m, 0, false},
                  {"portable host, cudaMalloc, stream 0", h_port, d_m, 0, false},
                  {"default host, cudaMalloc, non-blocking stream", h_def, d_m, s_nb, false},
                  {"default host, cudaMalloc, blocking stream", h_def, d_m, s_b, false},
                  {"default host, cudaMallocAsync dst, non-blocking", h_def, d_a, s_nb, false},
                  {"H2D+D2H on two streams", h_def, d_m, s_nb, true}};
    const int reps = 200;
    for (auto& c : cfgs) {
        float best = 1e30f;
        for (int t = 0; t < 3; ++t) {
            cudaEventRecord(a, c.s);
            for (int r = 0; r < reps; ++r) {
                cudaMemcpyAsync(c.d, c.h, n, cudaMemcpyHostToDevice, c.s);
                if (c.d2h_too) cudaMemcpyAsync(h_out, d_a, n, cudaMemcpyDeviceToHost, s_b);
            }
            if (c.d2h_too) { cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, s_b); cudaStreamWaitEvent(c.s, e, 0); }
            cudaEventRecord(b, c.s);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
        }
        printf("%-48s %7.1f us per 2.75 MB -> %5.1f GB/s\n", c.name, 1e3 * best / reps, n / (1e-3 * best / reps) / 1e9);
    }
    return 0;
}
