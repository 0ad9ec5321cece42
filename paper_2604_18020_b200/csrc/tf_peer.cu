// Peer-memory transport for the x-slab decomposition ("measure
// NCCL vs a custom peer-memory one-shot"): interface-plane exchange and a
// one-shot all-reduce of the CG scalars written straight into the
// neighbours' HBM over NVLink (CUDA IPC mappings), with stream-ordered flags.
//
//   sender:   k_plane_put  gathers its interface partials into the
//                          neighbour's receive slot (peer stores)
//             stream write-value of the epoch into the neighbour's flag
//                          (the write-value op fences the preceding writes)
//   receiver: stream wait-value (flag >= epoch) -- no SM spins --
//             k_plane_add  adds the received partial in the fixed order
//                          (left partial first) in place
//
// Receive slots are double-buffered by epoch parity: a sender at epoch e has
// already waited for the receiver's epoch e-1 data, which the receiver sent
// after consuming epoch e-2 (the same parity), so no slot is overwritten
// before it is read.  Flags hold monotonically increasing epochs (uint32).
//
// The driver stream memory operations are resolved at run time through
// cudaGetDriverEntryPoint, so the library has no link-time libcuda
// dependency (it still loads on a GPU-less build host).

#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "tf_common.cuh"

namespace tf {

template <typename T>
__global__ void k_plane_put(const T* __restrict__ w, const int64_t* __restrict__ idx, long long n, T* dst)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < n) dst[k] = w[idx[k]];
}

// w[idx] = recv + w[idx] (recv_first) or w[idx] + recv
template <typename T>
__global__ void k_plane_add(T* __restrict__ w, const int64_t* __restrict__ idx, long long n,
                            const T* __restrict__ recv, int recv_first)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const T mine = w[idx[k]], other = recv[k];
    w[idx[k]] = recv_first ? other + mine : mine + other;
}

// Multi-destination put with flags: job j copies src[idx_j[k]] (idx_j null:
// src[k]) to dst_j[k] for k < n, and the last block of job j to finish raises
// flag_j = epoch after a system-scope fence -- one launch for every peer
// instead of a put kernel plus a stream write per peer.
constexpr int PUT_MAX_JOBS = 16;
template <typename T>
struct PutJobs {
    const T* src;
    const int64_t* idx[PUT_MAX_JOBS];
    T* dst[PUT_MAX_JOBS];
    unsigned* flag[PUT_MAX_JOBS];
    unsigned* tickets;  // [PUT_MAX_JOBS], local device memory, zero between launches
    long long n;
    unsigned epoch;
};

template <typename T>
__global__ void k_put_flags(const __grid_constant__ PutJobs<T> J)
{
    const int j = blockIdx.y;
    const int64_t* idx = J.idx[j];
    T* dst = J.dst[j];
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < J.n; k += (long long)gridDim.x * blockDim.x)
        dst[k] = J.src[idx ? idx[k] : k];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (atomicAdd(J.tickets + j, 1u) == gridDim.x - 1) {
            __threadfence_system();
            *reinterpret_cast<volatile unsigned*>(J.flag[j]) = J.epoch;
            J.tickets[j] = 0u;
        }
    }
}

// both interface planes in one launch: w[li] = rl + w[li] (left partial
// first), w[ri] = w[ri] + rr; either side may be absent (null)
template <typename T>
__global__ void k_plane_add2(T* __restrict__ w, const int64_t* __restrict__ li, const T* __restrict__ rl,
                             const int64_t* __restrict__ ri, const T* __restrict__ rr, long long n)
{
    const long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    if (blockIdx.y == 0) {
        if (li) w[li[k]] = rl[k] + w[li[k]];
    } else if (ri) {
        w[ri[k]] = w[ri[k]] + rr[k];
    }
}

// out[j] = sum over ranks r (ascending) of slots[r * k + j]
__global__ void k_rank_sum(const double* __restrict__ slots, int nranks, int k, double* __restrict__ out)
{
    const int j = threadIdx.x;
    if (j >= k) return;
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += __ldcg(slots + (size_t)r * k + j);
    out[j] = s;
}

using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using WriteFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
using BatchFn = CUresult (*)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);

static int batch_fn(BatchFn* out)
{
    static BatchFn f = nullptr;
    if (!f) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        TF_CUDA_TRY(cudaGetDriverEntryPoint("cuStreamBatchMemOp", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuStreamBatchMemOp unavailable");
            return TF_ERR_UNSUPPORTED;
        }
        f = reinterpret_cast<BatchFn>(p);
    }
    *out = f;
    return TF_OK;
}

static int driver_fns(WaitFn* wait, WriteFn* write)
{
    static WaitFn w = nullptr;
    static WriteFn wr = nullptr;
    if (!w || !wr) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        TF_CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWaitValue32", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuStreamWaitValue32 unavailable");
            return TF_ERR_UNSUPPORTED;
        }
        w = reinterpret_cast<WaitFn>(p);
        TF_CUDA_TRY(cudaGetDriverEntryPoint("cuStreamWriteValue32", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) {
            set_error("cuStreamWriteValue32 unavailable");
            return TF_ERR_UNSUPPORTED;
        }
        wr = reinterpret_cast<WriteFn>(p);
    }
    *wait = w;
    *write = wr;
    return TF_OK;
}

}  // namespace tf

using namespace tf;

static inline cudaStream_t SP(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

int tf_peer_alloc(void** ptr, size_t bytes)
{
    TF_REQUIRE(ptr && bytes > 0, "bad arguments");
    TF_CUDA_TRY(cudaMalloc(ptr, bytes));
    TF_CUDA_TRY(cudaMemset(*ptr, 0, bytes));
    return TF_OK;
}

int tf_peer_free(void* ptr)
{
    if (ptr) TF_CUDA_TRY(cudaFree(ptr));
    return TF_OK;
}

int tf_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

int tf_ipc_export(void* dev_ptr, void* handle_out)
{
    TF_REQUIRE(dev_ptr && handle_out, "bad arguments");
    cudaIpcMemHandle_t h;
    TF_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
    memcpy(handle_out, &h, sizeof(h));
    return TF_OK;
}

int tf_ipc_open(const void* handle, void** dev_ptr_out)
{
    TF_REQUIRE(handle && dev_ptr_out, "bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    TF_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
    return TF_OK;
}

int tf_ipc_close(void* dev_ptr)
{
    if (dev_ptr) TF_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return TF_OK;
}

int tf_stream_write_u32(void* addr, uint32_t value, void* stream)
{
    WaitFn w;
    WriteFn wr;
    int rc = driver_fns(&w, &wr);
    if (rc) return rc;
    const CUresult r = wr((CUstream)stream, (CUdeviceptr)addr, value, CU_STREAM_WRITE_VALUE_DEFAULT);
    if (r != CUDA_SUCCESS) {
        set_error("cuStreamWriteValue32 failed (%d)", (int)r);
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

int tf_stream_wait_u32(void* addr, uint32_t value, void* stream)
{
    WaitFn w;
    WriteFn wr;
    int rc = driver_fns(&w, &wr);
    if (rc) return rc;
    const CUresult r = w((CUstream)stream, (CUdeviceptr)addr, value, CU_STREAM_WAIT_VALUE_GEQ);
    if (r != CUDA_SUCCESS) {
        set_error("cuStreamWaitValue32 failed (%d)", (int)r);
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

// every flag >= value, one batched stream memory operation
int tf_stream_wait_many_u32(void* const* addrs, int n, uint32_t value, void* stream)
{
    if (n <= 0) return TF_OK;
    TF_REQUIRE(addrs && n <= 64, "bad arguments");
    BatchFn f;
    int rc = batch_fn(&f);
    if (rc) return rc;
    CUstreamBatchMemOpParams ops[64];
    memset(ops, 0, sizeof(CUstreamBatchMemOpParams) * n);
    for (int i = 0; i < n; ++i) {
        ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
        ops[i].waitValue.address = (CUdeviceptr)addrs[i];
        ops[i].waitValue.value = value;
        ops[i].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
    }
    const CUresult r = f((CUstream)stream, (unsigned)n, ops, 0);
    if (r != CUDA_SUCCESS) {
        set_error("cuStreamBatchMemOp failed (%d)", (int)r);
        return TF_ERR_CUDA;
    }
    return TF_OK;
}

#define TF_PUTF(T, SUF)                                                                                   \
    int tf_put_flags_##SUF(const T* src, const int64_t* const* idx, T* const* dst, uint32_t* const* flags,  \
                           int njobs, int64_t n, uint32_t epoch, uint32_t* tickets, void* stream)         \
    {                                                                                                     \
        if (njobs <= 0) return TF_OK;                                                                     \
        TF_REQUIRE(src && dst && flags && tickets && njobs <= PUT_MAX_JOBS && n > 0, "bad arguments");    \
        PutJobs<T> J{};                                                                                   \
        J.src = src;                                                                                      \
        for (int j = 0; j < njobs; ++j) {                                                                 \
            J.idx[j] = idx ? idx[j] : nullptr;                                                            \
            J.dst[j] = dst[j];                                                                            \
            J.flag[j] = flags[j];                                                                         \
        }                                                                                                 \
        J.tickets = tickets;                                                                              \
        J.n = n;                                                                                          \
        J.epoch = epoch;                                                                                  \
        const unsigned nb = (unsigned)std::min<long long>((n + 255) / 256, 64);                           \
        k_put_flags<T><<<dim3(nb, njobs), 256, 0, SP(stream)>>>(J);                                       \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }                                                                                                     \
    int tf_plane_add2_##SUF(T* w, const int64_t* left_idx, const T* recv_left, const int64_t* right_idx,   \
                            const T* recv_right, int64_t n, void* stream)                                 \
    {                                                                                                     \
        if (n <= 0 || (!left_idx && !right_idx)) return TF_OK;                                           \
        k_plane_add2<T><<<dim3((unsigned)((n + 255) / 256), 2), 256, 0, SP(stream)>>>(w, left_idx, recv_left, \
                                                                                    right_idx, recv_right, n); \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }
TF_PUTF(float, f32)
TF_PUTF(double, f64)

#define TF_PLANE(T, SUF)                                                                                  \
    int tf_plane_put_##SUF(const T* w, const int64_t* idx, int64_t n, T* dst, void* stream)               \
    {                                                                                                     \
        if (n <= 0) return TF_OK;                                                                         \
        TF_REQUIRE(w && idx && dst, "bad arguments");                                                     \
        k_plane_put<T><<<(unsigned)((n + 255) / 256), 256, 0, SP(stream)>>>(w, idx, n, dst);              \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }                                                                                                     \
    int tf_plane_add_##SUF(T* w, const int64_t* idx, int64_t n, const T* recv, int recv_first,           \
                           void* stream)                                                                  \
    {                                                                                                     \
        if (n <= 0) return TF_OK;                                                                         \
        TF_REQUIRE(w && idx && recv, "bad arguments");                                                    \
        k_plane_add<T><<<(unsigned)((n + 255) / 256), 256, 0, SP(stream)>>>(w, idx, n, recv, recv_first); \
        TF_CHECK_LAUNCH();                                                                                \
        return TF_OK;                                                                                     \
    }
TF_PLANE(float, f32)
TF_PLANE(double, f64)

int tf_rank_sum_f64(const double* slots, int nranks, int k, double* out, void* stream)
{
    TF_REQUIRE(slots && out && nranks > 0 && k > 0 && k <= 1024, "bad arguments");
    k_rank_sum<<<1, ((k + 31) / 32) * 32, 0, SP(stream)>>>(slots, nranks, k, out);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

}  // extern "C"
