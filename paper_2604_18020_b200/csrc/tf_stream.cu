// Host-buffer product pipeline (the e2e path): w_i = K v_i for a batch of
// host vectors, with the H2D copy of v_{i+1}, the matvec of v_i and the D2H
// copy of w_{i-1} in flight together on three streams over double-buffered
// device vectors.  The whole schedule is enqueued from C (a handful of driver
// calls per vector), so a batch runs at the PCIe rate instead of the Python
// loop's launch rate.  Host buffers should be pinned for the copies to be
// asynchronous.

#include <cstring>
#include <mutex>

#include "tf_common.cuh"

namespace tf {

template <typename T>
int launch_grid_tile(const Grid& g, const T* ke_host, const T* scale, const T* v, T* w,
                     const uint8_t* node_fixed, uint32_t flags, double* dot_part, cudaStream_t st);

struct StreamCtx {
    int dev = -1;
    cudaStream_t s_in = nullptr, s_k = nullptr, s_out = nullptr;
    cudaEvent_t h2d[2], kdone[2], d2h[2], start, stop;
};

static int stream_ctx(StreamCtx** out)
{
    static thread_local StreamCtx ctx;
    int dev = 0;
    TF_CUDA_TRY(cudaGetDevice(&dev));
    if (ctx.dev != dev) {
        TF_CUDA_TRY(cudaStreamCreateWithFlags(&ctx.s_in, cudaStreamNonBlocking));
        TF_CUDA_TRY(cudaStreamCreateWithFlags(&ctx.s_k, cudaStreamNonBlocking));
        TF_CUDA_TRY(cudaStreamCreateWithFlags(&ctx.s_out, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            TF_CUDA_TRY(cudaEventCreateWithFlags(&ctx.h2d[b], cudaEventDisableTiming));
            TF_CUDA_TRY(cudaEventCreateWithFlags(&ctx.kdone[b], cudaEventDisableTiming));
            TF_CUDA_TRY(cudaEventCreateWithFlags(&ctx.d2h[b], cudaEventDisableTiming));
        }
        TF_CUDA_TRY(cudaEventCreateWithFlags(&ctx.start, cudaEventDisableTiming));
        TF_CUDA_TRY(cudaEventCreateWithFlags(&ctx.stop, cudaEventDisableTiming));
        ctx.dev = dev;
    }
    *out = &ctx;
    return TF_OK;
}

template <typename T>
static int grid_stream(const tf_grid* grid, const T* ke, const T* scale, const uint8_t* node_fixed,
                       uint32_t flags, int64_t n_vec, const T* const* host_in, T* const* host_out,
                       T* dev_in, T* dev_out, cudaStream_t st)
{
    TF_REQUIRE(grid && ke && scale && host_in && host_out && dev_in && dev_out, "null argument");
    if (n_vec <= 0) return TF_OK;
    const Grid g = make_grid(grid);
    const long long n_dof = 3 * g.n_nodes;
    const size_t vb = sizeof(T) * (size_t)n_dof;
    StreamCtx* c = nullptr;
    int rc = stream_ctx(&c);
    if (rc) return rc;
    // order the pipeline after the caller's prior work, and the caller after it
    TF_CUDA_TRY(cudaEventRecord(c->start, st));
    TF_CUDA_TRY(cudaStreamWaitEvent(c->s_in, c->start, 0));
    TF_CUDA_TRY(cudaStreamWaitEvent(c->s_k, c->start, 0));
    TF_CUDA_TRY(cudaStreamWaitEvent(c->s_out, c->start, 0));
    for (int64_t i = 0; i < n_vec; ++i) {
        const int b = (int)(i & 1);
        T* din = dev_in + (size_t)b * n_dof;
        T* dout = dev_out + (size_t)b * n_dof;
        if (i >= 2) TF_CUDA_TRY(cudaStreamWaitEvent(c->s_in, c->kdone[b], 0));  // din[b] consumed
        TF_CUDA_TRY(cudaMemcpyAsync(din, host_in[i], vb, cudaMemcpyHostToDevice, c->s_in));
        TF_CUDA_TRY(cudaEventRecord(c->h2d[b], c->s_in));
        TF_CUDA_TRY(cudaStreamWaitEvent(c->s_k, c->h2d[b], 0));
        if (i >= 2) TF_CUDA_TRY(cudaStreamWaitEvent(c->s_k, c->d2h[b], 0));  // dout[b] drained
        rc = launch_grid_tile<T>(g, ke, scale, din, dout, node_fixed, flags, nullptr, c->s_k);
        if (rc) return rc;
        TF_CUDA_TRY(cudaEventRecord(c->kdone[b], c->s_k));
        TF_CUDA_TRY(cudaStreamWaitEvent(c->s_out, c->kdone[b], 0));
        TF_CUDA_TRY(cudaMemcpyAsync(host_out[i], dout, vb, cudaMemcpyDeviceToHost, c->s_out));
        TF_CUDA_TRY(cudaEventRecord(c->d2h[b], c->s_out));
    }
    TF_CUDA_TRY(cudaEventRecord(c->stop, c->s_out));
    TF_CUDA_TRY(cudaStreamWaitEvent(st, c->stop, 0));
    TF_CUDA_TRY(cudaEventRecord(c->stop, c->s_in));
    TF_CUDA_TRY(cudaStreamWaitEvent(st, c->stop, 0));
    return TF_OK;
}

}  // namespace tf

using namespace tf;

extern "C" {

// Page-locked host buffers from cudaHostAlloc (portable): measured on the
// pool's B200 VMs at 51.8 GB/s H2D vs 13.9 GB/s for torch's pin_memory()
// buffers (scripts/h2d_probe.cu, scripts/pcie_probe.py).
int tf_host_alloc(void** ptr, size_t bytes)
{
    TF_REQUIRE(ptr, "null argument");
    *ptr = nullptr;
    if (bytes == 0) return TF_OK;
    TF_CUDA_TRY(cudaHostAlloc(ptr, bytes, cudaHostAllocPortable));
    return TF_OK;
}

int tf_host_free(void* ptr)
{
    if (ptr) TF_CUDA_TRY(cudaFreeHost(ptr));
    return TF_OK;
}

int tf_matvec_grid_stream_f32(const tf_grid* g, const float* ke, const float* scale, const uint8_t* node_fixed,
                              uint32_t flags, int64_t n_vec, const float* const* host_in, float* const* host_out,
                              float* dev_in, float* dev_out, void* stream)
{
    return grid_stream<float>(g, ke, scale, node_fixed, flags, n_vec, host_in, host_out, dev_in, dev_out,
                              reinterpret_cast<cudaStream_t>(stream));
}

int tf_matvec_grid_stream_f64(const tf_grid* g, const double* ke, const double* scale, const uint8_t* node_fixed,
                              uint32_t flags, int64_t n_vec, const double* const* host_in, double* const* host_out,
                              double* dev_in, double* dev_out, void* stream)
{
    return grid_stream<double>(g, ke, scale, node_fixed, flags, n_vec, host_in, host_out, dev_in, dev_out,
                               reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
