// Native x-slab runtime over the peer-memory transport.
//
// The Python slab driver (slab.py) enqueues one distributed CG iteration as
// ~20 host calls; at strong-scaling sizes (c4 over 8 GPUs: ~3 us of matvec
// per GPU) the host, not the GPU, then sets the pace.  This handle enqueues
// whole batches of iterations from C++:
//
//   apply(v -> w)   boundary tiles (node x-ranges next to the interfaces) ->
//                   put both interface planes into the neighbours' receive
//                   slots + raise their epoch flags (tf_peer.cu) -> interior
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
    uint32_t* tickets;     // device [16], tf_put_flags' per-job block counters
};

namespace {

inline char* at(void* base, int64_t off) { return reinterpret_cast<char*>(base) + off; }

int slab_apply(tf_slab* h, const void* v, void* w, cudaStream_t st, uint32_t* epoch)
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
    if ((rc = range(0, d.bl))) return rc;
    if ((rc = range(nnx - d.br, nnx))) return rc;
    const uint32_t e = ++*epoch;
    const int par = (int)(e & 1u);
    auto plane = [&](void* base, int side) { return at(base, d.off_planes + (2 * par + side) * d.plane_bytes); };
    auto flag = [&](void* base, int side) { return (uint32_t*)at(base, d.off_flags + 4 * side); };
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
    rc = f32 ? tf_put_flags_f32((const float*)w, idx, (float* const*)dst, flg, nj, d.plane_len, e, h->tickets, st)
             : tf_put_flags_f64((const double*)w, idx, (double* const*)dst, flg, nj, d.plane_len, e, h->tickets, st);
    if (rc) return rc;
    if ((rc = range(d.bl, nnx - d.br))) return rc;
    void* me = h->peers[d.rank];
    void* waits[2];
    int nw = 0;
    if (d.has_left) waits[nw++] = flag(me, 0);
    if (d.has_right) waits[nw++] = flag(me, 1);
    if ((rc = tf_stream_wait_many_u32(waits, nw, e, st))) return rc;
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

int slab_allreduce(tf_slab* h, double* t, int k, cudaStream_t st, uint32_t* ar_epoch)
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
    if ((rc = tf_put_flags_f64(t, nullptr, dst, flg, d.world, k, e, h->tickets, st))) return rc;
    if ((rc = tf_stream_wait_many_u32(waits, d.world, e, st))) return rc;
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
        cudaMalloc(&h->tickets, 16 * sizeof(uint32_t)) != cudaSuccess || cudaMemset(h->tickets, 0, 16 * sizeof(uint32_t)) != cudaSuccess) {
        delete h;
        tf::set_error("cudaMalloc failed");
        return TF_ERR_CUDA;
    }
    TF_CUDA_TRY(cudaMemcpy(h->scalar_idx, idx, sizeof(idx), cudaMemcpyHostToDevice));
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
    delete h;
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

// n_iters CG iterations it0+1 .. it0+n_iters (slab.py slab_pcg_device's loop body)
int tf_slab_pcg_iterate(tf_slab* h, const void* b, const void* inv, void* x, void* r, void* z, void* p, void* q,
                        void* wtmp, double* state, double* red, double* work, int it0, int n_iters,
                        int recompute_every, double* hist, int hist_len, uint32_t* epochs, void* stream)
{
    TF_REQUIRE(h && b && inv && x && r && z && p && q && wtmp && state && red && work && epochs, "bad arguments");
    const tf_slab_desc& d = h->d;
    cudaStream_t st = (cudaStream_t)stream;
    const bool f32 = d.precision == 32;
    const int64_t n = 3LL * (d.grid.nelx + 1) * (d.grid.nely + 1) * (d.grid.nelz + 1);
    int rc;
    for (int it = it0 + 1; it <= it0 + n_iters; ++it) {
        if ((rc = slab_apply(h, p, q, st, &epochs[0]))) return rc;
        rc = f32 ? tf_slab_cg_pq_f32(n, (const float*)p, (const float*)q, d.owned, state, red, work, st)
                 : tf_slab_cg_pq_f64(n, (const double*)p, (const double*)q, d.owned, state, red, work, st);
        if (rc) return rc;
        if ((rc = slab_allreduce(h, red, 1, st, &epochs[1]))) return rc;
        const int refresh = recompute_every > 0 && it % recompute_every == 0;
        rc = f32 ? tf_slab_cg_alpha_f32(n, (float*)x, (float*)r, (const float*)p, (const float*)q,
                                        (const float*)inv, (float*)z, d.owned, state, red, refresh, work, st)
                 : tf_slab_cg_alpha_f64(n, (double*)x, (double*)r, (const double*)p, (const double*)q,
                                        (const double*)inv, (double*)z, d.owned, state, red, refresh, work, st);
        if (rc) return rc;
        if (refresh) {
            if ((rc = slab_apply(h, x, wtmp, st, &epochs[0]))) return rc;
            rc = f32 ? tf_slab_cg_residual_f32(n, (const float*)b, (const float*)wtmp, (float*)r,
                                               (const float*)inv, (float*)z, d.owned, state, red, work, st)
                     : tf_slab_cg_residual_f64(n, (const double*)b, (const double*)wtmp, (double*)r,
                                               (const double*)inv, (double*)z, d.owned, state, red, work, st);
            if (rc) return rc;
        }
        if ((rc = slab_allreduce(h, red + 1, 2, st, &epochs[1]))) return rc;
        rc = f32 ? tf_slab_cg_beta_f32(n, (float*)p, (const float*)z, state, red, hist, hist_len, st)
                 : tf_slab_cg_beta_f64(n, (double*)p, (const double*)z, state, red, hist, hist_len, st);
        if (rc) return rc;
    }
    return TF_OK;
}

}  // extern "C"
