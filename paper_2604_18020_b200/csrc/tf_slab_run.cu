// Native x-slab runtime over the peer-memory transport.
//
// The Python slab driver (slab.py) enqueues one distributed CG iteration as
// ~20 host calls; at strong-scaling sizes (c4 over 8 GPUs: ~3 us of matvec
// per GPU) the host, not the GPU, then sets the pace.  This handle enqueues
// whole batches of iterations from C++:
//
//   apply(v -> w)   boundary tiles (node x-ranges next to the interfaces)
//                   whose interface-plane owners store straight into the
//                   neighbours' receive slots, the launch's last CTA raising
//                   the neighbour's epoch flag (tf_tile.cu TilePut; with
//                   TF_SLAB_FUSED_PUT=0 a separate put kernel, tf_peer.cu) -> interior
//                   tiles (overlap the transfer) -> wait own flags -> add the
//                   received partials in the fixed order (left first) ->
//                   fixed-DOF pass-through
//   all-reduce      one-shot: put the k partials into every rank's slot,
//                   raise flags, wait for all ranks, rank-ordered sum
//   CG iteration    the step kernels of tf_slab.cu with device-resident
//                   scalars (exact device-side stop)
//
// Layout of the receive regions and the epoch protocol are peer.py's
// (PeerTransport): the handle borrows the mapped base pointers and carries
// the epoch counters in and out, so Python-side and native exchanges can be
// interleaved on the same transport.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tf_common.cuh"

#include "../../include/topofuse_b200.h"

struct tf_slab {
    tf_slab_desc d;
    std::vector<char> ke;  // host copy of Ke (576 entries of the working precision)
    std::vector<void*> peers;
    int64_t* scalar_idx;   // device [0, 1, ..., 15]
    double* acc;           // device [16]
    uint32_t* tickets;     // device [32]: tf_put_flags' per-job block counters, [16]/[17] the fused
                           // puts of the left/right boundary products, [31] wait/add/pass
    // graph mode: epochs in device memory, waits as spin kernels (stream
    // memory operations bake their values into a captured graph)
    uint32_t* dev_ep;      // device [2]: plane epoch, all-reduce epoch
    int* dev_err;          // device: 1 = a wait timed out
    struct Graph {
        std::vector<const void*> key;
        cudaGraphExec_t exec;
    };
    std::vector<Graph> graphs;
    cudaStream_t cap = nullptr;
    // interior tiles run on a second stream, concurrent with the boundary
    // tiles and the interface put (fork/join by events; capturable)
    cudaStream_t aux = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

namespace {

inline char* at(void* base, int64_t off) { return reinterpret_cast<char*>(base) + off; }

constexpr int GMAX_JOBS = 16;
template <typename T>
struct DevPut {
    const T* src;
    const int64_t* idx[GMAX_JOBS];
    T* dst[GMAX_JOBS];
    uint32_t* flag[GMAX_JOBS];
    uint32_t* tickets;
    const uint32_t* ep;  // epoch = *ep + 1 (advanced by the matching wait kernel)
    long long n;
};

template <typename T>
__global__ void k_put_flags_dev(const __grid_constant__ DevPut<T> J)
{
    const int j = blockIdx.y;
    const int64_t* idx = J.idx[j];
    T* dst = J.dst[j];
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < J.n; k += (long long)gridDim.x * blockDim.x)
        dst[k] = J.src[idx ? idx[k] : k];
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(J.tickets + j, 1u) == gridDim.x - 1) {
        __threadfence_system();
        *reinterpret_cast<volatile uint32_t*>(J.flag[j]) = *J.ep + 1u;
        J.tickets[j] = 0u;
    }
}

struct DevWait {
    const uint32_t* flag[GMAX_JOBS];
    int n;
    uint32_t* ep;
    int* err;
};

// lane i spins until flag i >= *ep + 1 (30 s timeout -> *err = 1), then the
// epoch advances
__global__ void k_wait_dev(const __grid_constant__ DevWait W)
{
    const uint32_t target = *reinterpret_cast<volatile uint32_t*>(W.ep) + 1u;
    if ((int)threadIdx.x < W.n) {
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        while (*reinterpret_cast<const volatile uint32_t*>(W.flag[threadIdx.x]) < target) {
            __nanosleep(200);
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 30000000000ull) {
                *W.err = 1;
                break;
            }
        }
        __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) *W.ep = target;
}

// Graph mode, end of a distributed product in ONE kernel: wait for the
// neighbours' planes (thread 0 of every block spins on the local flags), add
// them in the fixed order, then the fixed-DOF pass-through.  Constrained DOFs
// are skipped by the adds (the pass-through owns them), so the two phases
// never touch the same DOF; the last block advances the epoch.
template <typename T>
struct WaitAddPass {
    const uint32_t* flag[2];
    int nflags;
    uint32_t* ep;
    int* err;
    uint32_t* ticket;
    T* w;
    const T* v;
    const int64_t* li;
    const T* rl;
    const int64_t* ri;
    const T* rr;
    long long plane_len;
    const uint8_t* node_fixed;
    const int64_t* fixed;
    long long n_fixed;
};

template <typename T>
__global__ void k_wait_add_pass(const __grid_constant__ WaitAddPass<T> A)
{
    __shared__ uint32_t target;
    if (threadIdx.x == 0) {
        target = *reinterpret_cast<volatile uint32_t*>(A.ep) + 1u;
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int i = 0; i < A.nflags; ++i)
            while (*reinterpret_cast<const volatile uint32_t*>(A.flag[i]) < target) {
                __nanosleep(200);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 30000000000ull) {
                    *A.err = 1;
                    break;
                }
            }
        __threadfence_system();
    }
    __syncthreads();
    const long long total = 2 * A.plane_len + A.n_fixed;
    for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < total; k += (long long)gridDim.x * blockDim.x) {
        if (k < 2 * A.plane_len) {
            const bool left = k < A.plane_len;
            const int64_t* idx = left ? A.li : A.ri;
            if (!idx) continue;
            const long long j = left ? k : k - A.plane_len;
            const long long d = idx[j];
            if (A.node_fixed && ((A.node_fixed[d / 3] >> (d % 3)) & 1u)) continue;
            A.w[d] = left ? __ldcg(A.rl + j) + A.w[d] : A.w[d] + __ldcg(A.rr + j);
        } else {
            const long long d = A.fixed[k - 2 * A.plane_len];
            A.w[d] = A.v[d];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(A.ticket, 1u) == gridDim.x - 1) {
        *A.ep = target;
        *A.ticket = 0u;
    }
}

// Graph mode, end of a one-shot all-reduce in ONE kernel: wait for every
// rank's flag, sum the slots in rank order into t[0..k), advance the epoch.
struct WaitSum {
    const uint32_t* flag[16];
    int nranks, k, stride;
    uint32_t* ep;
    int* err;
    const double* slots;  // [nranks][stride] of this parity
    double* t;
};

__global__ void k_wait_ranksum(const __grid_constant__ WaitSum A)
{
    __shared__ uint32_t target;
    if (threadIdx.x == 0) {
        target = *reinterpret_cast<volatile uint32_t*>(A.ep) + 1u;
        unsigned long long t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int i = 0; i < A.nranks; ++i)
            while (*reinterpret_cast<const volatile uint32_t*>(A.flag[i]) < target) {
                __nanosleep(100);
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
                if (t - t0 > 30000000000ull) {
                    *A.err = 1;
                    break;
                }
            }
        __threadfence_system();
    }
    __syncthreads();
    const int j = threadIdx.x;
    if (j < A.k) {
        double s = 0.0;
        for (int r = 0; r < A.nranks; ++r) s += __ldcg(A.slots + (size_t)r * A.stride + j);
        A.t[j] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) *A.ep = target;
}

__global__ void k_set_ep(uint32_t* ep, uint32_t e0, uint32_t e1)
{
    ep[0] = e0;
    ep[1] = e1;
}

template <typename T>
int put_dev(tf_slab* h, const T* src, const int64_t* const* idx, void* const* dst, uint32_t* const* flg, int nj,
            long long n, const uint32_t* ep, cudaStream_t st)
{
    if (nj <= 0) return TF_OK;
    DevPut<T> J{};
    J.src = src;
    for (int j = 0; j < nj; ++j) {
        J.idx[j] = idx ? idx[j] : nullptr;
        J.dst[j] = (T*)dst[j];
        J.flag[j] = flg[j];
    }
    J.tickets = h->tickets;
    J.ep = ep;
    J.n = n;
    const unsigned nb = (unsigned)std::min<long long>((n + 255) / 256, 64);
    k_put_flags_dev<T><<<dim3(nb, nj), 256, 0, st>>>(J);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

template <typename T>
int wait_add_pass(tf_slab* h, void* const* flags, int n, T* w, const T* v, const void* rl, const void* rr,
                  cudaStream_t st)
{
    const tf_slab_desc& d = h->d;
    WaitAddPass<T> A{};
    for (int i = 0; i < n; ++i) A.flag[i] = (const uint32_t*)flags[i];
    A.nflags = n;
    A.ep = h->dev_ep;
    A.err = h->dev_err;
    A.ticket = h->tickets + 31;  // put jobs use words 0..15
    A.w = w;
    A.v = v;
    A.li = d.has_left ? d.left_idx : nullptr;
    A.rl = (const T*)rl;
    A.ri = d.has_right ? d.right_idx : nullptr;
    A.rr = (const T*)rr;
    A.plane_len = d.plane_len;
    A.node_fixed = d.node_fixed;
    A.fixed = d.fixed;
    A.n_fixed = d.n_fixed > 0 ? d.n_fixed : 0;
    const long long total = 2 * d.plane_len + A.n_fixed;
    const unsigned nb = (unsigned)std::max<long long>(1, std::min<long long>((total + 255) / 256, 64));
    k_wait_add_pass<T><<<nb, 256, 0, st>>>(A);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

int wait_dev(tf_slab* h, void* const* flags, int n, uint32_t* ep, cudaStream_t st)
{
    if (n <= 0) return TF_OK;
    DevWait W{};
    for (int i = 0; i < n; ++i) W.flag[i] = (const uint32_t*)flags[i];
    W.n = n;
    W.ep = ep;
    W.err = h->dev_err;
    k_wait_dev<<<1, 32, 0, st>>>(W);
    TF_CHECK_LAUNCH();
    return TF_OK;
}

// TF_SLAB_FUSED_PUT=0: boundary products + a separate put kernel (A/B)
bool fused_put_enabled()
{
    static const bool on = [] {
        const char* e = getenv("TF_SLAB_FUSED_PUT");
        return !(e && e[0] == '0');
    }();
    return on;
}

// dev = true: device epochs (graph capture); else host epochs + stream memops
int slab_apply(tf_slab* h, const void* v, void* w, cudaStream_t st, uint32_t* epoch, bool dev = false)
{
    const tf_slab_desc& d = h->d;
    const bool f32 = d.precision == 32;
    auto range = [&](int lo, int hi) -> int {
        if (hi <= lo) return TF_OK;
        return f32 ? tf_matvec_grid_range_f32(&d.grid, (const float*)h->ke.data(), (const float*)d.scale,
                                              (const float*)v, (float*)w, d.node_fixed, TF_MASK_INPUT, lo,
                                              hi, st)
                   : tf_matvec_grid_range_f64(&d.grid, (const double*)h->ke.data(), (const double*)d.scale,
                                              (const double*)v, (double*)w, d.node_fixed, TF_MASK_INPUT, lo,
                                              hi, st);
    };
    const int nnx = d.grid.nelx + 1;
    int rc;
    const bool split = h->aux && (d.has_left || d.has_right) && nnx - d.br > d.bl;
    if (split) TF_CUDA_TRY(cudaEventRecord(h->fork, st));
    // slot parity: the host knows the epoch in both modes (graph mode keeps
    // the host counter advancing in step with the device one)
    const uint32_t e = ++*epoch;
    const int par = (int)(e & 1u);
    auto plane = [&](void* base, int side) { return at(base, d.off_planes + (2 * par + side) * d.plane_bytes); };
    auto flag = [&](void* base, int side) { return (uint32_t*)at(base, d.off_flags + 4 * side); };
    // fused only when each interface plane lies in its own boundary range (a
    // slab thinner than two tiles computes both planes in the left launch:
    // the separate put kernel then)
    if (fused_put_enabled() && (!d.has_left || d.bl >= 1) && (!d.has_right || d.br >= 1)) {
        // boundary products with the interface transfer fused in: the owners
        // of each interface plane store straight into the neighbour's slot
        // and the launch's last CTA raises its flag (no separate put kernel)
        auto put_range = [&](int lo, int hi, int put_i, void* dst, uint32_t* flg, uint32_t* ticket) -> int {
            if (hi <= lo) return TF_OK;
            const uint32_t* epd = dev ? h->dev_ep : nullptr;
            return f32 ? tf_matvec_grid_range_put_f32(&d.grid, (const float*)h->ke.data(), (const float*)d.scale,
                                                      (const float*)v, (float*)w, d.node_fixed, lo, hi, put_i,
                                                      (float*)dst, flg, ticket, epd, e, st)
                       : tf_matvec_grid_range_put_f64(&d.grid, (const double*)h->ke.data(),
                                                      (const double*)d.scale, (const double*)v, (double*)w,
                                                      d.node_fixed, lo, hi, put_i, (double*)dst, flg, ticket, epd,
                                                      e, st);
        };
        if (d.has_left) {
            void* nb = h->peers[d.rank - 1];
            rc = put_range(0, d.bl, 0, plane(nb, 1), flag(nb, 1), h->tickets + 16);
        } else {
            rc = range(0, d.bl);
        }
        if (rc) return rc;
        if (d.has_right) {
            void* nb = h->peers[d.rank + 1];
            rc = put_range(nnx - d.br, nnx, nnx - 1, plane(nb, 0), flag(nb, 0), h->tickets + 17);
        } else {
            rc = range(nnx - d.br, nnx);
        }
        if (rc) return rc;
    } else {
    if ((rc = range(0, d.bl))) return rc;
    if ((rc = range(nnx - d.br, nnx))) return rc;
    // both interface planes into the neighbours' slots + their flags: one launch
    const int64_t* idx[2];
    void* dst[2];
    uint32_t* flg[2];
    int nj = 0;
    if (d.has_left) {
        void* nb = h->peers[d.rank - 1];
        idx[nj] = d.left_idx, dst[nj] = plane(nb, 1), flg[nj] = flag(nb, 1), ++nj;
    }
    if (d.has_right) {
        void* nb = h->peers[d.rank + 1];
        idx[nj] = d.right_idx, dst[nj] = plane(nb, 0), flg[nj] = flag(nb, 0), ++nj;
    }
    if (dev)
        rc = f32 ? put_dev<float>(h, (const float*)w, idx, dst, flg, nj, d.plane_len, h->dev_ep, st)
                 : put_dev<double>(h, (const double*)w, idx, dst, flg, nj, d.plane_len, h->dev_ep, st);
    else
        rc = f32 ? tf_put_flags_f32((const float*)w, idx, (float* const*)dst, flg, nj, d.plane_len, e, h->tickets, st)
                 : tf_put_flags_f64((const double*)w, idx, (double* const*)dst, flg, nj, d.plane_len, e, h->tickets, st);
    if (rc) return rc;
    }
    if (split) {  // interior tiles on the side stream, launched after the boundary work
        TF_CUDA_TRY(cudaStreamWaitEvent(h->aux, h->fork, 0));
        cudaStream_t keep = st;
        st = h->aux;
        rc = range(d.bl, nnx - d.br);
        st = keep;
        if (rc) return rc;
        TF_CUDA_TRY(cudaEventRecord(h->join, h->aux));
    } else if ((rc = range(d.bl, nnx - d.br))) {
        return rc;
    }
    void* me = h->peers[d.rank];
    void* waits[2];
    int nw = 0;
    if (d.has_left) waits[nw++] = flag(me, 0);
    if (d.has_right) waits[nw++] = flag(me, 1);
    if (dev && !split)
        return f32 ? wait_add_pass<float>(h, waits, nw, (float*)w, (const float*)v, plane(me, 0), plane(me, 1), st)
                   : wait_add_pass<double>(h, waits, nw, (double*)w, (const double*)v, plane(me, 0), plane(me, 1), st);
    if ((rc = dev ? wait_dev(h, waits, nw, h->dev_ep, st) : tf_stream_wait_many_u32(waits, nw, e, st))) return rc;
    if (split) TF_CUDA_TRY(cudaStreamWaitEvent(st, h->join, 0));
    // fixed order: left partial first on the left plane, own partial first on the right
    rc = f32 ? tf_plane_add2_f32((float*)w, d.has_left ? d.left_idx : nullptr, (const float*)plane(me, 0),
                                 d.has_right ? d.right_idx : nullptr, (const float*)plane(me, 1), d.plane_len, st)
             : tf_plane_add2_f64((double*)w, d.has_left ? d.left_idx : nullptr, (const double*)plane(me, 0),
                                 d.has_right ? d.right_idx : nullptr, (const double*)plane(me, 1), d.plane_len, st);
    if (rc) return rc;
    if (d.n_fixed > 0)
        rc = f32 ? tf_pass_fixed_f32(d.fixed, d.n_fixed, (const float*)v, (float*)w, st)
                 : tf_pass_fixed_f64(d.fixed, d.n_fixed, (const double*)v, (double*)w, st);
    return rc;
}

int slab_allreduce(tf_slab* h, double* t, int k, cudaStream_t st, uint32_t* ar_epoch, bool dev = false)
{
    const tf_slab_desc& d = h->d;
    if (d.world == 1) return TF_OK;
    TF_REQUIRE(k >= 1 && k <= d.max_scalars, "too many scalars for the peer all-reduce");
    const uint32_t e = ++*ar_epoch;
    const int par = (int)(e & 1u);
    auto slot = [&](void* base, int src) {
        return at(base, d.off_slots + 8 * d.max_scalars * ((int64_t)d.world * par + src));
    };
    int rc;
    TF_REQUIRE(d.world <= 16, "peer all-reduce supports up to 16 ranks");
    double* dst[16];
    uint32_t* flg[16];
    void* waits[16];
    void* me = h->peers[d.rank];
    for (int r = 0; r < d.world; ++r) {
        dst[r] = (double*)slot(h->peers[r], d.rank);
        flg[r] = (uint32_t*)at(h->peers[r], d.off_arflags + 4 * d.rank);
        waits[r] = at(me, d.off_arflags + 4 * r);
    }
    // this rank's partials into every rank's slot + flags (one launch), then one batched wait
    if (dev) {
        if ((rc = put_dev<double>(h, t, nullptr, (void* const*)dst, flg, d.world, k, h->dev_ep + 1, st))) return rc;
        WaitSum A{};
        for (int r = 0; r < d.world; ++r) A.flag[r] = (const uint32_t*)waits[r];
        A.nranks = d.world;
        A.k = k;
        A.stride = (int)d.max_scalars;
        A.ep = h->dev_ep + 1;
        A.err = h->dev_err;
        A.slots = (const double*)slot(me, 0);
        A.t = t;
        k_wait_ranksum<<<1, 32, 0, st>>>(A);
        TF_CHECK_LAUNCH();
        return TF_OK;
    } else {
        if ((rc = tf_put_flags_f64(t, nullptr, dst, flg, d.world, k, e, h->tickets, st))) return rc;
        if ((rc = tf_stream_wait_many_u32(waits, d.world, e, st))) return rc;
    }
    if ((rc = tf_rank_sum_f64((const double*)slot(me, 0), d.world, (int)d.max_scalars, h->acc, st))) return rc;
    TF_CUDA_TRY(cudaMemcpyAsync(t, h->acc, sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
    return TF_OK;
}

}  // namespace

extern "C" {

int tf_slab_create(tf_slab** out, const tf_slab_desc* d)
{
    TF_REQUIRE(out && d && d->peer_base && d->scale && d->ke, "bad arguments");
    TF_REQUIRE(d->precision == 32 || d->precision == 64, "precision must be 32 or 64");
    TF_REQUIRE(d->world >= 1 && d->rank >= 0 && d->rank < d->world, "bad rank/world");
    TF_REQUIRE(d->max_scalars >= 4 && d->max_scalars <= 16, "max_scalars must be in [4, 16]");
    tf_slab* h = new tf_slab();
    h->d = *d;
    const size_t es = d->precision == 32 ? 4 : 8;
    h->ke.assign((const char*)d->ke, (const char*)d->ke + 576 * es);
    h->peers.assign(d->peer_base, d->peer_base + d->world);
    h->d.peer_base = nullptr;
    h->d.ke = nullptr;
    int64_t idx[16];
    for (int i = 0; i < 16; ++i) idx[i] = i;
    if (cudaMalloc(&h->scalar_idx, sizeof(idx)) != cudaSuccess || cudaMalloc(&h->acc, 16 * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&h->tickets, 32 * sizeof(uint32_t)) != cudaSuccess || cudaMemset(h->tickets, 0, 32 * sizeof(uint32_t)) != cudaSuccess ||
        cudaMalloc(&h->dev_ep, 2 * sizeof(uint32_t)) != cudaSuccess || cudaMalloc(&h->dev_err, sizeof(int)) != cudaSuccess ||
        cudaMemset(h->dev_err, 0, sizeof(int)) != cudaSuccess) {
        delete h;
        tf::set_error("cudaMalloc failed");
        return TF_ERR_CUDA;
    }
    TF_CUDA_TRY(cudaMemcpy(h->scalar_idx, idx, sizeof(idx), cudaMemcpyHostToDevice));
    // opt-in (TF_SLAB_OVERLAP=1): unmeasured on separate GPUs; with the rank
    // processes sharing one GPU (the only setup available this round) the
    // second stream made every product 12x slower through context switching
    const char* ov = getenv("TF_SLAB_OVERLAP");
    if (ov && ov[0] == '1') {
        TF_CUDA_TRY(cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
        TF_CUDA_TRY(cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming));
        TF_CUDA_TRY(cudaEventCreateWithFlags(&h->join, cudaEventDisableTiming));
    }
    *out = h;
    return TF_OK;
}

int tf_abi_struct_sizes(int64_t* out, int n)
{
    TF_REQUIRE(out && n >= 0, "bad arguments");
    const int64_t sz[] = {(int64_t)sizeof(tf_grid), (int64_t)sizeof(tf_pcg_desc), (int64_t)sizeof(tf_pcg_report),
                          (int64_t)sizeof(tf_oc_report), (int64_t)sizeof(tf_slab_desc)};
    for (int i = 0; i < n && i < 5; ++i) out[i] = sz[i];
    return TF_OK;
}

int tf_slab_destroy(tf_slab* h)
{
    if (!h) return TF_OK;
    cudaFree(h->scalar_idx);
    cudaFree(h->acc);
    cudaFree(h->tickets);
    cudaFree(h->dev_ep);
    cudaFree(h->dev_err);
    for (auto& g : h->graphs) cudaGraphExecDestroy(g.exec);
    if (h->cap) cudaStreamDestroy(h->cap);
    if (h->aux) cudaStreamDestroy(h->aux);
    if (h->fork) cudaEventDestroy(h->fork);
    if (h->join) cudaEventDestroy(h->join);
    delete h;
    return TF_OK;
}

// 1 when a graph-mode wait timed out (peer never raised its flag); clears it
int tf_slab_take_error(tf_slab* h, int* out)
{
    TF_REQUIRE(h && out, "bad arguments");
    TF_CUDA_TRY(cudaMemcpy(out, h->dev_err, sizeof(int), cudaMemcpyDeviceToHost));
    TF_CUDA_TRY(cudaMemset(h->dev_err, 0, sizeof(int)));
    return TF_OK;
}

int tf_slab_apply(tf_slab* h, const void* v, void* w, uint32_t* epochs, void* stream)
{
    TF_REQUIRE(h && v && w && epochs, "bad arguments");
    return slab_apply(h, v, w, (cudaStream_t)stream, &epochs[0]);
}

int tf_slab_allreduce(tf_slab* h, double* t, int k, uint32_t* epochs, void* stream)
{
    TF_REQUIRE(h && t && epochs, "bad arguments");
    return slab_allreduce(h, t, k, (cudaStream_t)stream, &epochs[1]);
}

// TF_SLAB_ONEX=0: the two-all-reduce iteration (A/B)
static bool slab_onex_enabled()
{
    static const bool on = [] {
        const char* e = getenv("TF_SLAB_ONEX");
        return !(e && e[0] == '0');
    }();
    return on;
}

// CG iterations it0+1 .. it0+n_iters (slab.py slab_pcg_device's loop body)
static int slab_iterations(tf_slab* h, const void* b, const void* inv, void* x, void* r, void* z, void* p, void* q,
                           void* wtmp, double* state, double* red, double* work, int it0, int n_iters,
                           int recompute_every, double* hist, int hist_len, uint32_t* epochs, cudaStream_t st,
                           bool dev)
{
    const tf_slab_desc& d = h->d;
    const bool f32 = d.precision == 32;
    const int64_t n = 3LL * (d.grid.nelx + 1) * (d.grid.nely + 1) * (d.grid.nelz + 1);
    int rc;
    for (int it = it0 + 1; it <= it0 + n_iters; ++it) {
        if (slab_onex_enabled()) {
            // one all-reduce per iteration (tf_slab.cu k_slab_dots8 / k_slab_step)
            if ((rc = slab_apply(h, p, q, st, &epochs[0], dev))) return rc;
            rc = f32 ? tf_slab_cg_dots8_f32(n, (const float*)p, (const float*)q, (const float*)r,
                                            (const float*)inv, d.owned, state, red, work, st)
                     : tf_slab_cg_dots8_f64(n, (const double*)p, (const double*)q, (const double*)r,
                                            (const double*)inv, d.owned, state, red, work, st);
            if (rc) return rc;
            if ((rc = slab_allreduce(h, red, 8, st, &epochs[1], dev))) return rc;
            const int refresh = recompute_every > 0 && it % recompute_every == 0;
            rc = f32 ? tf_slab_cg_step_f32(n, (float*)x, (float*)r, (float*)p, (const float*)q, (const float*)inv,
                                           (float*)z, state, red, refresh, hist, hist_len, st)
                     : tf_slab_cg_step_f64(n, (double*)x, (double*)r, (double*)p, (const double*)q,
                                           (const double*)inv, (double*)z, state, red, refresh, hist, hist_len,
                                           st);
            if (rc) return rc;
            if (refresh) {
                if ((rc = slab_apply(h, x, wtmp, st, &epochs[0], dev))) return rc;
                rc = f32 ? tf_slab_cg_residual_f32(n, (const float*)b, (const float*)wtmp, (float*)r,
                                                   (const float*)inv, (float*)z, d.owned, state, red, work, st)
                         : tf_slab_cg_residual_f64(n, (const double*)b, (const double*)wtmp, (double*)r,
                                                   (const double*)inv, (double*)z, d.owned, state, red, work, st);
                if (rc) return rc;
                if ((rc = slab_allreduce(h, red + 1, 2, st, &epochs[1], dev))) return rc;
                rc = f32 ? tf_slab_cg_beta_f32(n, (float*)p, (const float*)z, state, red, hist, hist_len, st)
                         : tf_slab_cg_beta_f64(n, (double*)p, (const double*)z, state, red, hist, hist_len, st);
                if (rc) return rc;
            }
            continue;
        }
        if ((rc = slab_apply(h, p, q, st, &epochs[0], dev))) return rc;
        rc = f32 ? tf_slab_cg_pq_f32(n, (const float*)p, (const float*)q, d.owned, state, red, work, st)
                 : tf_slab_cg_pq_f64(n, (const double*)p, (const double*)q, d.owned, state, red, work, st);
        if (rc) return rc;
        if ((rc = slab_allreduce(h, red, 1, st, &epochs[1], dev))) return rc;
        const int refresh = recompute_every > 0 && it % recompute_every == 0;
        rc = f32 ? tf_slab_cg_alpha_f32(n, (float*)x, (float*)r, (const float*)p, (const float*)q,
                                        (const float*)inv, (float*)z, d.owned, state, red, refresh, work, st)
                 : tf_slab_cg_alpha_f64(n, (double*)x, (double*)r, (const double*)p, (const double*)q,
                                        (const double*)inv, (double*)z, d.owned, state, red, refresh, work, st);
        if (rc) return rc;
        if (refresh) {
            if ((rc = slab_apply(h, x, wtmp, st, &epochs[0], dev))) return rc;
            rc = f32 ? tf_slab_cg_residual_f32(n, (const float*)b, (const float*)wtmp, (float*)r,
                                               (const float*)inv, (float*)z, d.owned, state, red, work, st)
                     : tf_slab_cg_residual_f64(n, (const double*)b, (const double*)wtmp, (double*)r,
                                               (const double*)inv, (double*)z, d.owned, state, red, work, st);
            if (rc) return rc;
        }
        if ((rc = slab_allreduce(h, red + 1, 2, st, &epochs[1], dev))) return rc;
        rc = f32 ? tf_slab_cg_beta_f32(n, (float*)p, (const float*)z, state, red, hist, hist_len, st)
                 : tf_slab_cg_beta_f64(n, (double*)p, (const double*)z, state, red, hist, hist_len, st);
        if (rc) return rc;
    }
    return TF_OK;
}

int tf_slab_pcg_iterate(tf_slab* h, const void* b, const void* inv, void* x, void* r, void* z, void* p, void* q,
                        void* wtmp, double* state, double* red, double* work, int it0, int n_iters,
                        int recompute_every, double* hist, int hist_len, uint32_t* epochs, void* stream)
{
    TF_REQUIRE(h && b && inv && x && r && z && p && q && wtmp && state && red && work && epochs, "bad arguments");
    return slab_iterations(h, b, inv, x, r, z, p, q, wtmp, state, red, work, it0, n_iters, recompute_every, hist,
                           hist_len, epochs, (cudaStream_t)stream, false);
}

// The same n_iters iterations as one CUDA-graph launch.  The captured
// iterations are it0+1 .. it0+n_iters with a refresh exactly where
// recompute_every puts one for THIS it0; graphs are cached per (buffers,
// n_iters, refresh positions), so callers replay aligned blocks (it0 a
// multiple of n_iters and n_iters dividing recompute_every).  Epochs: the
// host values are loaded into the device counters before the launch and
// advanced by the block's exchange counts after it.
int tf_slab_pcg_graph(tf_slab* h, const void* b, const void* inv, void* x, void* r, void* z, void* p, void* q,
                      void* wtmp, double* state, double* red, double* work, int it0, int n_iters,
                      int recompute_every, double* hist, int hist_len, uint32_t* epochs, int* err_out, void* stream)
{
    TF_REQUIRE(h && b && inv && x && r && z && p && q && wtmp && state && red && work && epochs && n_iters > 0,
               "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    // refresh pattern of this block (bit j: iteration it0+1+j refreshes)
    uintptr_t pattern = 0;
    for (int j = 0; j < n_iters && j < 64; ++j)
        if (recompute_every > 0 && (it0 + 1 + j) % recompute_every == 0) pattern |= (uintptr_t)1 << j;
    std::vector<const void*> key = {b, inv, x, r, z, p, q, wtmp, state, red, work, hist,
                                    (const void*)(uintptr_t)n_iters, (const void*)pattern,
                                    (const void*)(uintptr_t)(it0 & 1), (const void*)(uintptr_t)hist_len};
    // slot parities are baked per capture: key on the epoch parities too
    key.push_back((const void*)(uintptr_t)(epochs[0] & 1u));
    key.push_back((const void*)(uintptr_t)(epochs[1] & 1u));
    cudaGraphExec_t exec = nullptr;
    for (auto& g : h->graphs)
        if (g.key == key) exec = g.exec;
    uint32_t ep[2] = {epochs[0], epochs[1]};
    if (!exec) {
        if (!h->cap) TF_CUDA_TRY(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
        TF_CUDA_TRY(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
        uint32_t tmp[2] = {epochs[0], epochs[1]};
        int rc = slab_iterations(h, b, inv, x, r, z, p, q, wtmp, state, red, work, it0, n_iters, recompute_every,
                                 hist, hist_len, tmp, h->cap, true);
        cudaGraph_t graph = nullptr;
        const cudaError_t ce = cudaStreamEndCapture(h->cap, &graph);
        if (rc) {
            if (graph) cudaGraphDestroy(graph);
            return rc;
        }
        TF_CUDA_TRY(ce);
        const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
        cudaGraphDestroy(graph);
        TF_CUDA_TRY(ie);
        h->graphs.push_back({key, exec});
    }
    k_set_ep<<<1, 1, 0, st>>>(h->dev_ep, ep[0], ep[1]);
    TF_CHECK_LAUNCH();
    TF_CUDA_TRY(cudaGraphLaunch(exec, st));
    // advance the host epochs like the captured sequence did
    const int refreshes = __builtin_popcountll((unsigned long long)pattern);
    if (h->d.world > 1) {
        epochs[0] += (uint32_t)(n_iters + refreshes);
        epochs[1] += (uint32_t)(2 * n_iters);
    } else {
        epochs[0] += (uint32_t)(n_iters + refreshes);
    }
    if (err_out) TF_CUDA_TRY(cudaMemcpyAsync(err_out, h->dev_err, sizeof(int), cudaMemcpyDeviceToHost, st));
    return TF_OK;
}

}  // extern "C"
