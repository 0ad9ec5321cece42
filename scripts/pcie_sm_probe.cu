// PCIe ceiling for the e2e leg: copy-engine vs SM-driven (zero-copy, mapped
// pinned host memory) transfers of one c2 vector (2.75 MB), alone and with
// the opposite direction in flight.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_spin(const float* __restrict__ src, float* __restrict__ dst, long long n, long long cycles)
{
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

__global__ void k_copy(const float4* __restrict__ src, float4* __restrict__ dst, long long n4)
{
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += (long long)gridDim.x * blockDim.x)
        dst[i] = __ldcv(src + i);
}

int main()
{
    const long long n = 686433 + 3;  // padded to float4
    const size_t bytes = n * 4;
    float *h_in, *h_out, *d_in, *d_out, *hm_in, *hm_out;
    cudaHostAlloc(&h_in, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    cudaHostAlloc(&h_out, bytes, cudaHostAllocPortable | cudaHostAllocMapped);
    cudaHostGetDevicePointer(&hm_in, h_in, 0);
    cudaHostGetDevicePointer(&hm_out, h_out, 0);
    cudaMalloc(&d_in, bytes);
    cudaMalloc(&d_out, bytes);
    for (long long i = 0; i < n; ++i) h_in[i] = (float)i;
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* label, int mode, int grid) {
        const int reps = 300;
        for (int pass = 0; pass < 2; ++pass) {
            cudaDeviceSynchronize();
            cudaEventRecord(e0, 0);
            cudaStreamWaitEvent(s1, e0, 0);
            cudaStreamWaitEvent(s2, e0, 0);
            for (int r = 0; r < reps; ++r) {
                // h2d
                if (mode & 1) cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s1);
                if (mode & 4) k_copy<<<grid, 256, 0, s1>>>((const float4*)hm_in, (float4*)d_in, n / 4);
                // d2h
                if (mode & 2) cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s2);
                if (mode & 8) k_copy<<<grid, 256, 0, s2>>>((const float4*)d_out, (float4*)hm_out, n / 4);
            }
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            cudaEventRecord(a, s1);
            cudaEventRecord(b, s2);
            cudaStreamWaitEvent(0, a, 0);
            cudaStreamWaitEvent(0, b, 0);
            cudaEventRecord(e1, 0);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (pass == 1)
                printf("%-34s grid %4d: %7.1f us per vector pair -> %5.1f GB/s per direction\n", label, grid,
                       ms * 1e3 / reps, bytes / (ms * 1e-3 / reps) / 1e9);
        }
    };
    run("warm-up", 3, 0);
    run("CE h2d", 1, 0);
    run("CE d2h", 2, 0);
    run("CE h2d + CE d2h", 3, 0);
    for (int grid : {148, 296, 592, 1184}) {
        run("SM h2d", 4, grid);
        run("SM d2h", 8, grid);
        run("SM h2d + CE d2h", 4 | 2, grid);
        run("CE h2d + SM d2h", 1 | 8, grid);
        run("SM h2d + SM d2h", 4 | 8, grid);
    }
    // the e2e pipeline of csrc/tf_stream.cu (double-buffered device vectors,
    // three streams), with a device-to-device copy standing in for the matvec
    {
        float *din2, *dout2;
        cudaMalloc(&din2, 2 * bytes);
        cudaMalloc(&dout2, 2 * bytes);
        cudaStream_t sk;
        cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking);
        cudaEvent_t h2d[2], kd[2], d2h[2];
        for (int b = 0; b < 2; ++b) {
            cudaEventCreateWithFlags(&h2d[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&kd[b], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&d2h[b], cudaEventDisableTiming);
        }
        for (int kern = 0; kern < 4; ++kern)
            for (int pass = 0; pass < 2; ++pass) {
                // kern 2: a 15 us kernel (the c2 tile product's length); kern 3: the same
                // schedule captured into one CUDA graph and replayed
                cudaGraphExec_t gexec = nullptr;
                if (kern == 3) cudaStreamBeginCapture(s1, cudaStreamCaptureModeGlobal);
                const int reps = 300;
                if (kern != 3) cudaDeviceSynchronize();
                cudaEvent_t fork;
                cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
                if (kern == 3) {
                    cudaEventRecord(fork, s1);
                } else {
                    cudaEventRecord(e0, 0);
                    cudaEventRecord(fork, 0);
                }
                cudaStreamWaitEvent(s2, fork, 0);
                cudaStreamWaitEvent(sk, fork, 0);
                for (int i = 0; i < reps; ++i) {
                    const int b = i & 1;
                    float* di = din2 + b * n;
                    float* dd = dout2 + b * n;
                    if (i >= 2) cudaStreamWaitEvent(s1, kd[b], 0);
                    cudaMemcpyAsync(di, h_in, bytes, cudaMemcpyHostToDevice, s1);
                    cudaEventRecord(h2d[b], s1);
                    cudaStreamWaitEvent(sk, h2d[b], 0);
                    if (i >= 2) cudaStreamWaitEvent(sk, d2h[b], 0);
                    if (kern == 1) k_copy<<<592, 256, 0, sk>>>((const float4*)di, (float4*)dd, n / 4);
                    if (kern >= 2) k_spin<<<444, 256, 0, sk>>>(di, dd, n, 28000);
                    cudaEventRecord(kd[b], sk);
                    cudaStreamWaitEvent(s2, kd[b], 0);
                    cudaMemcpyAsync(h_out, dd, bytes, cudaMemcpyDeviceToHost, s2);
                    cudaEventRecord(d2h[b], s2);
                }
                cudaEvent_t a, b2;
                cudaEventCreateWithFlags(&a, cudaEventDisableTiming);
                cudaEventCreateWithFlags(&b2, cudaEventDisableTiming);
                cudaEventRecord(a, s2);
                cudaEventRecord(b2, sk);
                if (kern == 3) {
                    cudaStreamWaitEvent(s1, a, 0);
                    cudaStreamWaitEvent(s1, b2, 0);
                    cudaGraph_t graph;
                    cudaStreamEndCapture(s1, &graph);
                    cudaGraphInstantiate(&gexec, graph, 0);
                    cudaGraphLaunch(gexec, 0);  // warm
                    cudaDeviceSynchronize();
                    cudaEventRecord(e0, 0);
                    cudaGraphLaunch(gexec, 0);
                } else {
                    cudaStreamWaitEvent(0, a, 0);
                    cudaStreamWaitEvent(0, b2, 0);
                }
                cudaEventRecord(e1, 0);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                const char* lab[4] = {"no kernel", "d2d kernel", "15 us kernel", "15 us kernel, one CUDA graph"};
                if (pass == 1) printf("pipeline (%s): %7.1f us per step\n", lab[kern], ms * 1e3 / reps);
            }
    }
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
