// Microbenchmark: grid-wide "exchange" (barrier + deterministic reduction of one
// double per CTA) on a cooperatively launched, co-resident grid -- the
// per-iteration synchronisation of the SM-resident PCG (tf_pcg_resident.cu).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exchange_bench exchange_bench.cu
// ./exchange_bench [ctas_per_sm=2] [threads=256] [reps=2000]
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ unsigned ld_acq(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v)
{
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rlx64(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rlx64(unsigned long long* p, unsigned long long v)
{
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// mode 0: monotonic counter (red.release) + thread-0 acquire poll, then warp 0
//         reads all partials (L2) and sums in a fixed order
// mode 1: mode 0 with __nanosleep backoff in the poll
// mode 2: per-CTA sentinel slots polled by warp 0 (no counter)
// mode 6: mode 1 without the __threadfence before the red.release
// mode 7: mode 6 polled inside warp 0; mode 8+j: arrivals over 2^j counters
// mode 3: cooperative-groups style: fence + atomicAdd + volatile gen poll + fence
template <int MODE>
__global__ void k_xchg(unsigned* ctr, double* part, unsigned long long* slots, int reps, double* out)
{
    __shared__ double sh;
    const int tid = threadIdx.x, bid = blockIdx.x, nblk = gridDim.x;
    double acc_total = 0.0;
    for (int ph = 0; ph < reps; ++ph) {
        const double mine = (double)(bid + 1) * (ph + 1);
        __syncthreads();
        if (MODE == 0 || MODE == 1 || MODE == 6) {
            if (tid == 0) {
                part[(size_t)(ph & 1) * nblk + bid] = mine;
                if (MODE != 6) __threadfence();  // mode 6: the release alone orders the write
                red_rel(ctr, 1u);
                const unsigned target = (unsigned)(ph + 1) * nblk;
                while (ld_acq(ctr) < target) {
                    if (MODE != 0) __nanosleep(20);
                }
            }
            __syncthreads();
            if (tid < 32) {
                double a = 0.0;
                for (int i = tid; i < nblk; i += 32) a += __ldcg(part + (size_t)(ph & 1) * nblk + i);
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tid == 0) sh = a;
            }
        } else if (MODE == 7) {
            // mode 6 with the poll inside warp 0 (no CTA barrier between the
            // acquire and the partial loads)
            if (tid < 32) {
                if (tid == 0) {
                    part[(size_t)(ph & 1) * nblk + bid] = mine;
                    red_rel(ctr, 1u);
                    const unsigned target = (unsigned)(ph + 1) * nblk;
                    while (ld_acq(ctr) < target) __nanosleep(20);
                }
                __syncwarp();
                double a = 0.0;
                for (int i = tid; i < nblk; i += 32) a += __ldcg(part + (size_t)(ph & 1) * nblk + i);
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tid == 0) sh = a;
            }
        } else if (MODE >= 8) {
            // mode 8+j: mode 7 with the arrivals spread over NC = 2^j counters
            // (own 128-B lines; same-address reductions serialise in L2), lane
            // c < NC of warp 0 polls counter c
            constexpr int NC = 1 << (MODE >= 8 ? MODE - 8 : 0);
            if (tid < 32) {
                if (tid == 0) {
                    part[(size_t)(ph & 1) * nblk + bid] = mine;
                    red_rel(ctr + 32 * (bid % NC), 1u);
                }
                if (tid < NC) {
                    const unsigned cnt = (unsigned)((nblk - tid + NC - 1) / NC);
                    const unsigned target = (unsigned)(ph + 1) * cnt;
                    while (ld_acq(ctr + 32 * tid) < target) __nanosleep(20);
                }
                __syncwarp();
                double a = 0.0;
                for (int i = tid; i < nblk; i += 32) a += __ldcg(part + (size_t)(ph & 1) * nblk + i);
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tid == 0) sh = a;
            }
        } else if (MODE == 2) {
            unsigned long long* slot = slots + (size_t)(ph % 3) * nblk;
            if (tid == 0) {
                st_rlx64(slots + (size_t)((ph + 1) % 3) * nblk + bid, ~0ull);
                __threadfence();
                st_rlx64(slot + bid, __double_as_longlong(mine));
            }
            if (tid < 32) {
                double a = 0.0;
                for (int i = tid; i < nblk; i += 32) {
                    unsigned long long w;
                    while ((w = ld_rlx64(slot + i)) == ~0ull) {
                    }
                    a += __longlong_as_double(w);
                }
                __threadfence();
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tid == 0) sh = a;
            }
        } else if (MODE == 4) {
            // two-level arrival tree: 16 group counters (own 128-B lines), the
            // last arriver of a group arrives at the top counter
            constexpr int NG = 16;
            if (tid == 0) {
                part[(size_t)(ph & 1) * nblk + bid] = mine;
                __threadfence();
                const int grp = bid % NG;
                const unsigned gsize = (unsigned)((nblk - grp + NG - 1) / NG);
                unsigned* gc = ctr + 64 + 32 * grp;
                const unsigned old = atomicAdd(gc, 1u);
                if (old + 1 == (unsigned)(ph + 1) * gsize) {
                    __threadfence();
                    red_rel(ctr, 1u);
                }
                const unsigned target = (unsigned)(ph + 1) * NG;
                while (ld_acq(ctr) < target) {
                }
            }
            __syncthreads();
            if (tid < 32) {
                double a = 0.0;
                for (int i = tid; i < nblk; i += 32) a += __ldcg(part + (size_t)(ph & 1) * nblk + i);
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tid == 0) sh = a;
            }
        } else {
            if (tid == 0) {
                part[(size_t)(ph & 1) * nblk + bid] = mine;
                volatile unsigned* vg = ctr + 32;
                const unsigned g = *vg;
                __threadfence();
                if (atomicAdd(ctr, 1u) == (unsigned)nblk - 1) {
                    *ctr = 0u;
                    __threadfence();
                    atomicAdd(ctr + 32, 1u);
                } else {
                    while (*vg == g) {
                    }
                }
                __threadfence();
            }
            __syncthreads();
            if (tid < 32) {
                double a = 0.0;
                for (int i = tid; i < nblk; i += 32) a += __ldcg(part + (size_t)(ph & 1) * nblk + i);
                for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
                if (tid == 0) sh = a;
            }
        }
        __syncthreads();
        acc_total += sh;
    }
    if (tid == 0) out[bid] = acc_total;
}

// mode 5: clusters of CL CTAs -- cluster barrier + DSMEM reduction inside the
// cluster, a global counter barrier among the cluster leaders only
template <int CL>
__global__ void k_xchg_cluster(unsigned* ctr, double* part, int reps, double* out)
{
    __shared__ double sh, cl_val;
    const int tid = threadIdx.x, bid = blockIdx.x, nblk = gridDim.x;
    const int ncl = nblk / CL;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    const int cid = bid / CL;
    double acc_total = 0.0;
    for (int ph = 0; ph < reps; ++ph) {
        const double mine = (double)(bid + 1) * (ph + 1);
        if (tid == 0) cl_val = mine;
        // cluster barrier (release/acquire): every CTA's cl_val visible cluster-wide
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (rank == 0 && tid == 0) {
            double s = 0.0;
            const unsigned base = (unsigned)__cvta_generic_to_shared(&cl_val);
            for (unsigned r = 0; r < CL; ++r) {
                unsigned ra;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base), "r"(r));
                double v;
                asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra));
                s += v;
            }
            part[(size_t)(ph & 1) * ncl + cid] = s;
            __threadfence();
            red_rel(ctr, 1u);
            const unsigned target = (unsigned)(ph + 1) * ncl;
            while (ld_acq(ctr) < target) {
            }
        }
        __syncthreads();
        if (rank == 0 && tid < 32) {
            double a = 0.0;
            for (int i = tid; i < ncl; i += 32) a += __ldcg(part + (size_t)(ph & 1) * ncl + i);
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
            if (tid == 0) sh = a;
        }
        // second cluster barrier: leaders' totals visible; members read them over DSMEM
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        double tot;
        {
            const unsigned base = (unsigned)__cvta_generic_to_shared(&sh);
            unsigned ra;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(base), "r"(0u));
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(tot) : "r"(ra));
        }
        // third barrier so the leader does not overwrite sh/cl_val while members read
        asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        acc_total += tot;
    }
    if (tid == 0) out[bid] = acc_total;
}

template <int CL>
void run_cluster(int per_sm, int nt, int reps, int nsm)
{
    unsigned* ctr;
    double *part, *out;
    CK(cudaMalloc(&ctr, 4096));
    CK(cudaMalloc(&part, sizeof(double) * 2 * 2048));
    CK(cudaMalloc(&out, sizeof(double) * 2048));
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (CL > 8) CK(cudaFuncSetAttribute(k_xchg_cluster<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    int ncl_max = 0;
    cfg.gridDim = dim3(CL * 256);
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl_max, (void*)k_xchg_cluster<CL>, &cfg);
    if (e != cudaSuccess) { printf("cluster %d: occupancy query failed: %s\n", CL, cudaGetErrorString(e)); cudaGetLastError(); return; }
    const int want = per_sm * nsm / CL;
    const int ncl = std::min(want, ncl_max);
    const int nblk = ncl * CL;
    cfg.gridDim = dim3(nblk);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int trial = 0; trial < 3; ++trial) {
        CK(cudaMemset(ctr, 0, 4096));
        cudaEventRecord(e0);
        e = cudaLaunchKernelEx(&cfg, k_xchg_cluster<CL>, ctr, part, reps, out);
        if (e != cudaSuccess) { printf("cluster %d launch: %s\n", CL, cudaGetErrorString(e)); cudaGetLastError(); return; }
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double h0;
    CK(cudaMemcpy(&h0, out, sizeof(double), cudaMemcpyDeviceToHost));
    double want_v = 0.0;
    for (int ph = 0; ph < reps; ++ph) want_v += (double)nblk * (nblk + 1) / 2 * (ph + 1);
    printf("mode 5  cluster %d: ctas %d (max clusters %d, asked %d/SM) threads %d: %.3f us per exchange  %s\n", CL,
           nblk, ncl_max, per_sm, nt, 1e3 * best / reps, h0 == want_v ? "ok" : "WRONG");
    cudaFree(ctr);
    cudaFree(part);
    cudaFree(out);
}

template <int MODE>
void run(int per_sm, int nt, int reps, int nsm)
{
    const int nblk = per_sm * nsm;
    unsigned* ctr;
    double *part, *out;
    unsigned long long* slots;
    CK(cudaMalloc(&ctr, 4096));
    CK(cudaMalloc(&part, sizeof(double) * 2 * nblk));
    CK(cudaMalloc(&slots, sizeof(unsigned long long) * 3 * nblk));
    CK(cudaMalloc(&out, sizeof(double) * nblk));
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_xchg<MODE>, nt, 0));
    if (occ < per_sm) {
        printf("mode %d: occupancy %d < %d\n", MODE, occ, per_sm);
        return;
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int trial = 0; trial < 3; ++trial) {
        CK(cudaMemset(ctr, 0, 4096));
        CK(cudaMemset(slots, 0xFF, sizeof(unsigned long long) * 3 * nblk));
        void* args[] = {&ctr, &part, &slots, &reps, &out};
        cudaEventRecord(e0);
        CK(cudaLaunchCooperativeKernel((void*)k_xchg<MODE>, nblk, nt, args, 0, 0));
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    double h0;
    CK(cudaMemcpy(&h0, out, sizeof(double), cudaMemcpyDeviceToHost));
    double want = 0.0;
    for (int ph = 0; ph < reps; ++ph) want += (double)nblk * (nblk + 1) / 2 * (ph + 1);
    printf("mode %d  ctas %d (%d/SM) threads %d: %.3f us per exchange  %s\n", MODE, nblk, per_sm, nt,
           1e3 * best / reps, h0 == want ? "ok" : "WRONG");
    cudaFree(ctr);
    cudaFree(part);
    cudaFree(slots);
    cudaFree(out);
}

int main(int argc, char** argv)
{
    const int reps = argc > 3 ? atoi(argv[3]) : 2000;
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    for (int per_sm : {1, 2, 3}) {
        for (int nt : {128, 256}) {
            run<0>(per_sm, nt, reps, nsm);
            run<1>(per_sm, nt, reps, nsm);
            run<2>(per_sm, nt, reps, nsm);
            run<3>(per_sm, nt, reps, nsm);
            run<4>(per_sm, nt, reps, nsm);
            run<6>(per_sm, nt, reps, nsm);
            run<7>(per_sm, nt, reps, nsm);
            run<10>(per_sm, nt, reps, nsm);
            run<11>(per_sm, nt, reps, nsm);
            run<12>(per_sm, nt, reps, nsm);
            run<13>(per_sm, nt, reps, nsm);
            if (argc > 1) continue;
            run_cluster<2>(per_sm, nt, reps, nsm);
            run_cluster<4>(per_sm, nt, reps, nsm);
            run_cluster<8>(per_sm, nt, reps, nsm);
            run_cluster<16>(per_sm, nt, reps, nsm);
        }
    }
    return 0;
}
