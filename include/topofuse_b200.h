/*
 * topofuse_b200 -- C ABI of the B200-native (sm_100a) matrix-free Q1-hex
 * stiffness operator and the Jacobi-PCG around it.
 *
 * Drop-in boundary: these entry points replace the kernel-module contract the
 * reference operator calls through get_backend() (reference
 * pkg/src/topofuse/backend.py:38-46, operator.py:90-132,157-159) and the
 * pcg recurrence (solver.py:57-147).  The Python host package
 * paper_2604_18020_b200 binds them with ctypes; see INTEGRATION.md.
 *
 * Conventions
 *   - plain C, all functions return 0 (TF_OK) or a TF_ERR_* code; the text of
 *     the last error on the calling thread is tf_last_error();
 *   - every array pointer is a DEVICE pointer (e.g. torch.Tensor.data_ptr())
 *     unless documented "host"; the caller owns and allocates them;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *     all calls are asynchronous on it unless documented otherwise;
 *   - _f32 / _f64 suffix = working precision of vectors, scales and Ke;
 *   - edof is int32 (n_elem, 24) row-major, reference mesh.py:83-102;
 *     a NEGATIVE entry marks a constrained DOF slot: it gathers 0 and is
 *     never scattered to (this is how input masking is fused, operator.py:83-88);
 *   - node_fixed (structured grids): n_nodes bytes, bit c set when DOF
 *     3*node+c is constrained (BoundaryConditions.fixed_dofs, mesh.py:105-120),
 *     FOLLOWED by (nelx+1)*(nely+1) column bytes = OR over z of the node
 *     bytes of each (i, j) node column, then (nelx+1)*(nely+1) column bytes =
 *     AND over z (kernels drop z-invariant constraints statically and read
 *     per-node bytes only where a column's constraint varies along z).
 *     Build it with tf_build_node_fixed().
 */
#ifndef TOPOFUSE_B200_H
#define TOPOFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_OK 0
#define TF_ERR_ARG 1
#define TF_ERR_CUDA 2
#define TF_ERR_UNSUPPORTED 3
#define TF_ERR_DIVERGED 4

/* matvec flags */
#define TF_ACCUMULATE 1u  /* w += K v instead of w = K v                         */
#define TF_MASK_INPUT 2u  /* read v as 0 on constrained DOFs (operator.py:84)     */
#define TF_PASS_FIXED 4u  /* w[fixed] = v[fixed] (operator.py:115)                */

/* structured-grid kernel variants */
#define TF_GRID_FAST 0     /* production: parity-block tile kernel (dense pull if
                              Ke lacks the mirror-symmetry block structure)     */
#define TF_GRID_BITWISE 1  /* reproduces the numba fused_serial op order bitwise  */
#define TF_GRID_PULL 2     /* dense 24x24 rows, node-centric pull, FMA           */

/* general-edof scatter modes (operator.py SCATTER_MODES, :30) */
#define TF_SCATTER_ATOMIC 0 /* red.global.add -- parallel_atomic analogue         */
#define TF_SCATTER_COLORED 1 /* deterministic colour-ordered passes -- serial     */

typedef struct tf_grid {
    int32_t nelx, nely, nelz; /* StructuredMesh (mesh.py:34-56) */
} tf_grid;

const char* tf_last_error(void);
/* Build the node_fixed layout above from a device list of fixed DOFs.
 * `out` (4-byte aligned) must hold n_nodes + 2*(nelx+1)*(nely+1) bytes
 * rounded up to a multiple of 4. */
int tf_build_node_fixed(const tf_grid* g, const int64_t* fixed_dofs, int64_t n_fixed,
                        uint8_t* out, void* stream);
int tf_version(void);
/* number of CUDA devices visible (0 on a GPU-less host) */
int tf_device_count(void);

/* ---- K v on a structured grid: replaces fused_serial / fused_atomic +
 *      apply()'s masking when edof == build_edof(mesh)
 *      (_kernels_numba.py:146-196, operator.py:90-117).
 *      ke: HOST pointer, 576 values, row-major.  scale: n_elem.  v, w: n_dof.
 *      node_fixed may be NULL (no constraints).  `variant` TF_GRID_*.      */
int tf_matvec_grid_f32(const tf_grid* g, const float* ke, const float* scale, const float* v,
                       float* w, const uint8_t* node_fixed, uint32_t flags, int variant,
                       void* stream);
int tf_matvec_grid_f64(const tf_grid* g, const double* ke, const double* scale,
                       const double* v, double* w, const uint8_t* node_fixed, uint32_t flags,
                       int variant, void* stream);

/* Same, producing only the outputs of node x-columns [i_lo, i_hi) (all j, k);
 * the x-slab decomposition computes its interface columns first and overlaps
 * the neighbour exchange with the interior range (slab.py). */
int tf_matvec_grid_range_f32(const tf_grid* g, const float* ke, const float* scale, const float* v,
                             float* w, const uint8_t* node_fixed, uint32_t flags, int32_t i_lo,
                             int32_t i_hi, void* stream);
int tf_matvec_grid_range_f64(const tf_grid* g, const double* ke, const double* scale,
                             const double* v, double* w, const uint8_t* node_fixed, uint32_t flags,
                             int32_t i_lo, int32_t i_hi, void* stream);

/* The x-slab's masked range product with the interface transfer fused in
 * (peer transport, csrc/tf_slab_run.cu): besides w, the owners of node plane
 * x = put_i (inside [i_lo, i_hi)) store their output into `dst` -- the
 * neighbour's receive slot, mapped through CUDA IPC; plane order (j, k)
 * row-major, 3 components -- and the launch's last CTA raises `*flag` to
 * `epoch` (or to *ep_dev + 1 when ep_dev is set: graph mode) after a
 * system-scope fence.  `ticket`: a device counter, zero between launches. */
int tf_matvec_grid_range_put_f32(const tf_grid* g, const float* ke, const float* scale,
                                 const float* v, float* w, const uint8_t* node_fixed, int32_t i_lo,
                                 int32_t i_hi, int32_t put_i, float* dst, uint32_t* flag,
                                 uint32_t* ticket, const uint32_t* ep_dev, uint32_t epoch,
                                 void* stream);
int tf_matvec_grid_range_put_f64(const tf_grid* g, const double* ke, const double* scale,
                                 const double* v, double* w, const uint8_t* node_fixed, int32_t i_lo,
                                 int32_t i_hi, int32_t put_i, double* dst, uint32_t* flag,
                                 uint32_t* ticket, const uint32_t* ep_dev, uint32_t epoch,
                                 void* stream);

/* Page-locked host memory for the e2e path (cudaHostAlloc, portable). */
int tf_host_alloc(void** ptr, size_t bytes);
int tf_host_free(void* ptr);

/* Host-buffer batch (the e2e path): w_i = K v_i for i < n_vec, v_i/w_i HOST
 * pointers (pinned for asynchrony), dev_in/dev_out 2*n_dof device scratch.
 * The H2D copy of v_{i+1}, the product of v_i and the D2H copy of w_{i-1} run
 * concurrently on internal streams; `stream` is ordered before and after the
 * batch.  Same flags/semantics as tf_matvec_grid_*; returns once enqueued. */
int tf_matvec_grid_stream_f32(const tf_grid* g, const float* ke, const float* scale,
                              const uint8_t* node_fixed, uint32_t flags, int64_t n_vec,
                              const float* const* host_in, float* const* host_out, float* dev_in,
                              float* dev_out, void* stream);
int tf_matvec_grid_stream_f64(const tf_grid* g, const double* ke, const double* scale,
                              const uint8_t* node_fixed, uint32_t flags, int64_t n_vec,
                              const double* const* host_in, double* const* host_out,
                              double* dev_in, double* dev_out, void* stream);

/* Launch shape of the structured tile kernel for a plain product on this grid
 * (z-chunk height and CTA count; the autotuned height once the grid shape has
 * been seen, else the heuristic).  Introspection only. */
int tf_tile_shape(const tf_grid* g, int precision, int32_t* oz, int64_t* ctas);

/* ---- Emulated bfloat16 (the reference's BF16 kernel contract, documented
 *      negative result; _kernels_numba.py:113-126,166-211,230-238).  FP32
 *      storage; each term is bf16_rne(s_e*K[i,j]) * u_j, FP32 accumulation.  */
/* fused_serial_bf16 (mode TF_SCATTER_COLORED) / fused_atomic_bf16 (ATOMIC),
 * accumulating into w; quantize_input != 0 rounds the gathered v to bf16 first
 * (operator.py:83-88 _masked_input), 0 expects v pre-quantized (the contract). */
int tf_matvec_edof_bf16(const int32_t* edof, const float* ke, const float* scale, const float* v,
                        float* w, int64_t n_elem, int mode, const int32_t* color_elems,
                        const int64_t* color_offsets, int n_colors, int quantize_input,
                        void* stream);
/* apply_fp64 of a bf16 operator (operator.py:143-152): quantized entries and
 * input, FP64 accumulation, accumulated into w (FP64). */
int tf_matvec_edof_bf16_f64(const int32_t* edof, const float* ke, const float* scale,
                            const double* v, double* w, int64_t n_elem, void* stream);
/* gemm_bf16: f_elem = per-term bf16(s*K) u_elem (new values, not accumulated) */
int tf_gemm_bf16(const float* u_elem, const float* ke, const float* scale, float* f_elem,
                 int64_t n_elem, void* stream);
/* jacobi_diag_bf16: out[edof] += bf16(s_e * ke_diag[l]) (FP32) */
int tf_jacobi_edof_bf16(const int32_t* edof, const float* ke_diag, const float* scale, float* out,
                        int64_t n_elem, void* stream);
/* y = round_to_bf16(x) (precision.py:65-85), y may alias x */
int tf_round_bf16(int64_t n, const float* x, float* y, void* stream);

/* ---- General connectivity, bitwise the reference's fused_serial
 *      (_kernels_numba.py:146-162): element row sums into `rows` (n_elem*24
 *      FP64 workspace), then each DOF accumulates its rows in ascending element
 *      order through a CSR (offsets: n_dof+1 int64, entries: n_elem*24 int32
 *      flat element-row indices) built once per mesh by tf_edof_csr_build.
 *      w is overwritten (accumulate = 0) or accumulated into (1).          */
int tf_edof_csr_build(const int32_t* edof, int64_t n_elem, int64_t n_dof, int64_t* offsets,
                      int32_t* entries, void* stream);
/* Jacobi diagonal, general connectivity, deterministic and bitwise the
 * reference's jacobi_diag (_kernels_numba.py:217-226): acc[d] (FP64, caller
 * initialised) += f64(scale[e] * ke_diag[l]) in ascending element order over
 * the DOF -> (element*24 + row) CSR of tf_edof_csr_build. */
int tf_jacobi_edof_pull_f32(const int64_t* offsets, const int32_t* entries, const float* ke_diag,
                            const float* scale, double* acc, int64_t n_dof, void* stream);
int tf_jacobi_edof_pull_f64(const int64_t* offsets, const int32_t* entries, const double* ke_diag,
                            const double* scale, double* acc, int64_t n_dof, void* stream);
/* three-stage scatter_serial, bitwise the reference (_kernels_numba.py:129-132):
 * acc[d] (FP64) += f_elem[e*24 + i] in ascending element order over the CSR. */
int tf_scatter_pull_f32(const int64_t* offsets, const int32_t* entries, const float* f_elem, double* acc,
                        int64_t n_dof, void* stream);
int tf_scatter_pull_f64(const int64_t* offsets, const int32_t* entries, const double* f_elem, double* acc,
                        int64_t n_dof, void* stream);
/* emulated-bf16 fused_serial, bitwise the reference (_kernels_numba.py:166-177):
 * FP32 rows of bf16(s_e K_ij) u_j, added in ascending element order in FP32. */
int tf_matvec_edof_pull_bf16(const int32_t* edof, const float* ke, const float* scale, const float* v, float* w,
                             int64_t n_elem, int64_t n_dof, const int64_t* offsets, const int32_t* entries,
                             double* rows, int accumulate, void* stream);
int tf_matvec_edof_pull_f32(const int32_t* edof, const float* ke, const float* scale,
                            const float* v, float* w, int64_t n_elem, int64_t n_dof,
                            const int64_t* offsets, const int32_t* entries, double* rows,
                            int accumulate, void* stream);
int tf_matvec_edof_pull_f64(const int32_t* edof, const double* ke, const double* scale,
                            const double* v, double* w, int64_t n_elem, int64_t n_dof,
                            const int64_t* offsets, const int32_t* entries, double* rows,
                            int accumulate, void* stream);

/* ---- K v with an explicit element->DOF table: the fused kernel contract
 *      fused_serial/fused_atomic(edof, ke, scale, v, out) (_kernels_numba.py:146-196).
 *      ALWAYS accumulates into w (caller zeroes it, operator.py:93).
 *      mode TF_SCATTER_ATOMIC: one element per thread, red.global.add scatter.
 *      mode TF_SCATTER_COLORED: `color_elems` (n_elem int32 element ids grouped
 *      by colour) and `color_offsets` (n_colors+1, HOST) give an ordering in
 *      which no two elements of a colour share a DOF; deterministic.       */
int tf_matvec_edof_f32(const int32_t* edof, const float* ke, const float* scale, const float* v,
                       float* w, int64_t n_elem, int mode, const int32_t* color_elems,
                       const int64_t* color_offsets, int n_colors, void* stream);
int tf_matvec_edof_f64(const int32_t* edof, const double* ke, const double* scale,
                       const double* v, double* w, int64_t n_elem, int mode,
                       const int32_t* color_elems, const int64_t* color_offsets, int n_colors,
                       void* stream);

/* ---- fused_atomic (_kernels_numba.py:183-196) with the connectivity's
 *      neighbour-merge pattern precomputed: tf_edof_merge_mask writes, once per
 *      element->DOF table, a 16-bit mask per element (bit 3 pr + c: DOF
 *      3 corner_of(1,oy,oz) + c of element e equals DOF 3 corner_of(0,oy,oz) + c
 *      of element e+1 in the same 32-element group); the product then sums each
 *      such pair in registers before one red.global.add.  Same contract as
 *      tf_matvec_edof_* in mode TF_SCATTER_ATOMIC (accumulates into w) except
 *      for masked slots: they must carry their DOF with the sign bit set
 *      (DOF | 2^31, not -1); they gather 0 and their row is added to that DOF
 *      (a constrained DOF, overwritten by the caller's pass-through,
 *      operator.py:115).  tf_edof_merge_mask checks this (TF_ERR_ARG) and
 *      synchronises the stream once.  edof and mask are device pointers.       */
int tf_edof_merge_mask(const int32_t* edof, int64_t n_elem, int64_t n_dof, uint16_t* mask, void* stream);
int tf_matvec_edof_merged_f32(const int32_t* edof, const uint16_t* mask, const float* ke,
                              const float* scale, const float* v, float* w, int64_t n_elem,
                              void* stream);
int tf_matvec_edof_merged_f64(const int32_t* edof, const uint16_t* mask, const double* ke,
                              const double* scale, const double* v, double* w, int64_t n_elem,
                              void* stream);

/* w[fixed[i]] = v[fixed[i]] for i < n_fixed (operator.py:115) */
int tf_pass_fixed_f32(const int64_t* fixed, int64_t n_fixed, const float* v, float* w,
                      void* stream);
int tf_pass_fixed_f64(const int64_t* fixed, int64_t n_fixed, const double* v, double* w,
                      void* stream);

/* ---- three-stage variant stages (_kernels_numba.py:82-140) ----------------- */
int tf_gather_f32(const int32_t* edof, const float* v, float* u_elem, int64_t n_elem, void* stream);
int tf_gather_f64(const int32_t* edof, const double* v, double* u_elem, int64_t n_elem, void* stream);
/* f_elem[e,i] = scale[e] * sum_j K[i,j] u_elem[e,j] */
int tf_gemm_f32(const float* u_elem, const float* ke, const float* scale, float* f_elem,
                int64_t n_elem, void* stream);
int tf_gemm_f64(const double* u_elem, const double* ke, const double* scale, double* f_elem,
                int64_t n_elem, void* stream);
/* acc[edof[e,i]] += f_elem[e,i] in FP64 (histogram-style, operator.py:107-114) */
int tf_scatter_f32(const int32_t* edof, const float* f_elem, double* acc, int64_t n_elem,
                   void* stream);
int tf_scatter_f64(const int32_t* edof, const double* f_elem, double* acc, int64_t n_elem,
                   void* stream);

/* ---- Jacobi diagonal (_kernels_numba.py:217-226, operator.py:122-132) ------ */
/* structured: diag (working dtype) with 1.0 on fixed DOFs; inv_diag (nullable)
 * = 1/diag rounded in the working dtype (solver.py:95).  ke_diag: HOST, 24.  */
int tf_jacobi_grid_f32(const tf_grid* g, const float* ke_diag, const float* scale, float* diag,
                       float* inv_diag, const uint8_t* node_fixed, void* stream);
int tf_jacobi_grid_f64(const tf_grid* g, const double* ke_diag, const double* scale,
                       double* diag, double* inv_diag, const uint8_t* node_fixed, void* stream);
/* per-node FP64 sums of scale[e]*ke_diag[l] in ascending element order, no
 * cast and no constraint handling (x-slab partials before the exchange) */
int tf_jacobi_grid_partial_f32(const tf_grid* g, const float* ke_diag, const float* scale, double* partial,
                               void* stream);
int tf_jacobi_grid_partial_f64(const tf_grid* g, const double* ke_diag, const double* scale, double* partial,
                               void* stream);
/* contract form: acc (FP64, n_dof) += scale[e]*ke_diag[l] over edof */
int tf_jacobi_edof_f32(const int32_t* edof, const float* ke_diag, const float* scale,
                       double* acc, int64_t n_elem, void* stream);
int tf_jacobi_edof_f64(const int32_t* edof, const double* ke_diag, const double* scale,
                       double* acc, int64_t n_elem, void* stream);

/* ---- element energies u_e^T Ke u_e in FP64 (_kernels_numba.py:241-256) ----- */
int tf_energies_grid_f64(const tf_grid* g, const double* ke, const double* u, double* out,
                         void* stream);
int tf_energies_edof_f64(const int32_t* edof, const double* ke, const double* u, double* out,
                         int64_t n_elem, void* stream);

/* ---- device-resident Jacobi-PCG (solver.py:57-147) --------------------------
 * One handle per operator configuration; not re-entrant.  The whole solve
 * runs as ONE CUDA-graph launch: a device-side while loop (conditional graph
 * node) iterates matvec+dot -> update -> direction kernels until the
 * reference stop rule fires; the host reads back only the final report.   */

typedef struct tf_pcg tf_pcg;

typedef struct tf_pcg_desc {
    int precision;              /* 32, 64, or 16 = emulated bf16 (FP32 storage, edof only) */
    int structured;             /* 1: grid kernels, 0: edof kernels */
    tf_grid grid;               /* when structured */
    const int32_t* edof;        /* when !structured: masked edof (fixed -> -1) */
    int64_t n_elem;
    int64_t n_dof;
    const void* ke;             /* HOST, 576 values in the working precision */
    const uint8_t* node_fixed;  /* device, structured only, nullable */
    const int64_t* fixed;       /* device list of fixed DOFs (edof mode), nullable */
    int64_t n_fixed;
    int grid_variant;           /* TF_GRID_* */
    int flags;                  /* TF_PCG_PLAIN_GRAPH: force the 3-kernel graph protocol */
} tf_pcg_desc;
#define TF_PCG_PLAIN_GRAPH 1u

typedef struct tf_pcg_report {
    int32_t iterations;
    int32_t termination;        /* 0 converged, 1 max_iter, 2 breakdown, 3 diverged */
    int32_t matvecs;
    int32_t _pad;
    double rel_residual;
} tf_pcg_report;

int tf_pcg_create(tf_pcg** out, const tf_pcg_desc* desc, void* stream);
/* Solve K x = b.  scale (n_elem), b, inv_diag, x are device arrays in the
 * working precision; they are copied into handle-owned buffers, so the
 * captured graph never changes.  x holds x0 on entry when has_x0 != 0 (else
 * the solve starts from 0) and the solution on exit.  history (device,
 * FP64, max_iter+1 entries, nullable) receives the relative residual of every
 * iteration (SolveReport.residual_history).  Blocks until the solve ends.  */
int tf_pcg_solve(tf_pcg* h, const void* scale, const void* b, const void* inv_diag, void* x,
                 int has_x0, double rel_tol, int32_t max_iter, int32_t recompute_every,
                 double* history, tf_pcg_report* report);
int tf_pcg_destroy(tf_pcg* h);
/* Which device protocol a handle runs (chosen at create from the problem
 * size; TF_PCG_RESIDENT=0 / TF_PCG_FUSED=0|1 in the environment override):
 *   TF_PCG_GRAPH        one CUDA graph, 3 kernels per iteration;
 *   TF_PCG_FUSED_GRAPH  one CUDA graph, direction folded into the matvec (2 per iteration);
 *   TF_PCG_RESIDENT     one cooperative kernel for the whole solve, owned CG
 *                       vectors resident in shared memory (tf_pcg_resident.cu). */
#define TF_PCG_GRAPH 0
#define TF_PCG_FUSED_GRAPH 1
#define TF_PCG_RESIDENT 2
int tf_pcg_protocol(const tf_pcg* h);
/* CgConfig.quantize_krylov (solver.py:134-136): round p and r to bf16 after
 * every direction update in the following solves (FP32 storage, graph protocol). */
int tf_pcg_set_quantize_krylov(tf_pcg* h, int on);

/* ---- SIMP glue on the device (simp.py:33-175, element.py:34-45) -------------
 * Densities, sensitivities and filter vectors are FP64, n = n_elem.         */

/* inv_rowsum[e] = 1 / sum of cone weights max(0, rmin - dist) over the
 * in-mesh neighbours of element e (build_cone_filter row sums, simp.py:33-69);
 * rmin <= 3 (stencil reach <= 3). */
int tf_filter_rowsum_f64(const tf_grid* g, double rmin, double* inv_rowsum, void* stream);
/* y = F x (transpose = 0, `filt @ x`) or y = F^T x (transpose = 1, `filt.T @ x`) */
int tf_filter_grid_f64(const tf_grid* g, double rmin, const double* inv_rowsum, const double* x,
                       double* y, int transpose, void* stream);
/* smoothed Heaviside projection and its derivative (dh nullable), simp.py:72-84 */
int tf_project_f64(int64_t n, double beta, double eta, const double* rho_bar, double* rho_phys,
                   double* dh, void* stream);
/* scale = rho_min + (1-rho_min) clip(rho,0,1)^p in the working dtype; *bad_flag
 * (device int, nullable) is OR-ed with 1 when a density is outside [0,1]. */
int tf_simp_scale_f32(int64_t n, double p, double rho_min, const double* rho, float* scale,
                      int* bad_flag, void* stream);
int tf_simp_scale_f64(int64_t n, double p, double rho_min, const double* rho, double* scale,
                      int* bad_flag, void* stream);
/* out = dh * (-p (1-rho_min) clip(rho)^(p-1) * energies)   (dh nullable) */
int tf_sensitivity_f64(int64_t n, double p, double rho_min, const double* rho_phys,
                       const double* energies, const double* dh, double* out, void* stream);
/* out3 (device) = { sum a*b, sum g*(1-g), sum s } over n (any input nullable);
 * work: tf_work_doubles(n) doubles.  Deterministic. */
int tf_stats_f64(int64_t n, const double* a, const double* b, const double* gray_of,
                 const double* sum_of, double* work, double* out3, void* stream);
int64_t tf_work_doubles(int64_t n);

#define TF_OC_OK 0
#define TF_OC_SATURATED 1   /* bracket not found in 200 steps: nearest candidate */
#define TF_OC_STALLED 2     /* bisection never reached vol_tol (simp.py:175) */
#define TF_OC_BAD_INPUT 3   /* dc > 1e-12 or dv <= 0 (simp.py:133-136) */

typedef struct tf_oc_report {
    int32_t status;
    int32_t evaluations;
    double lam;
    double best_err;
} tf_oc_report;

/* Optimality-criteria step with volume bisection (oc_update, simp.py:111-175)
 * on the raw-mean volume: one cooperative kernel, grid-wide fixed-order sums.
 * dv nullable (= ones).  work: tf_work_doubles(n) doubles; rep_dev: device. */
int tf_oc_update_f64(int64_t n, const double* rho, const double* dc, const double* dv, double vf,
                     double move, double vol_tol, double damping, int max_bisect, double* rho_new,
                     double* work, tf_oc_report* rep_dev, void* stream);

/* Distributed OC building blocks (x-slab SIMP).  sums[k] (device)
 * = this rank's sum over its n elements of the OC candidate at lams[k]
 * (host array, 1 <= n_lams <= TF_OC_MAX_LAMS) and sums[TF_OC_MAX_LAMS] = the
 * count of invalid inputs (dc > 1e-12 or dv <= 0); rank-local fixed order.
 * work: tf_oc_work_doubles(n) doubles.  The host all-gathers the rank sums and
 * runs oc_update's bracket/bisection (simp.py:111-175) on the global means. */
#define TF_OC_MAX_LAMS 15
int64_t tf_oc_work_doubles(int64_t n);
int tf_oc_volumes_f64(int64_t n, const double* rho, const double* dc, const double* dv, double move,
                      double damping, const double* lams, int n_lams, double* sums, double* work,
                      void* stream);
/* rho_new = the OC candidate at lam (the step's final clip) */
int tf_oc_apply_f64(int64_t n, const double* rho, const double* dc, const double* dv, double move,
                    double damping, double lam, double* rho_new, void* stream);


/* ---- x-slab distributed PCG step kernels (csrc/tf_slab.cu) --------
 * Device-resident scalars for the multi-GPU CG of solver.py:57-147: the host
 * enqueues  q = K p (+ interface exchange) -> tf_slab_cg_pq -> all-reduce
 * red[0] -> tf_slab_cg_alpha -> all-reduce red[1..2] -> tf_slab_cg_beta  per
 * iteration without synchronising; `state` (8 doubles: rz, |b|, rel, it,
 * active, term, tol, ticket) freezes the solve exactly at the stop iteration
 * (term 1 converged, 2 breakdown, 3 diverged).  owned (nullable): uint8 mask
 * of the DOFs this rank counts in dots.  red: 4 doubles (p.q, r.r, r.z, b.b);
 * 8 for the single-reduction iteration (tf_slab_cg_dots8 / tf_slab_cg_step).
 * work: tf_slab_work_doubles(n) doubles. */
int64_t tf_slab_work_doubles(int64_t n);
int tf_slab_dot_f32(int64_t n, const float* a, const float* b, const uint8_t* owned, double* out,
                    double* work, void* stream);
int tf_slab_dot_f64(int64_t n, const double* a, const double* b, const uint8_t* owned, double* out,
                    double* work, void* stream);
int tf_slab_cg_begin_f32(int64_t n, const float* r, const float* inv, float* z, float* p,
                         const uint8_t* owned, double* red, double* work, void* stream);
int tf_slab_cg_begin_f64(int64_t n, const double* r, const double* inv, double* z, double* p,
                         const uint8_t* owned, double* red, double* work, void* stream);
int tf_slab_cg_start(double* state, const double* red, double rel_tol, int f32, void* stream);
int tf_slab_cg_pq_f32(int64_t n, const float* p, const float* q, const uint8_t* owned,
                      const double* state, double* red, double* work, void* stream);
int tf_slab_cg_pq_f64(int64_t n, const double* p, const double* q, const uint8_t* owned,
                      const double* state, double* red, double* work, void* stream);
int tf_slab_cg_alpha_f32(int64_t n, float* x, float* r, const float* p, const float* q, const float* inv,
                         float* z, const uint8_t* owned, double* state, double* red, int refresh,
                         double* work, void* stream);
int tf_slab_cg_alpha_f64(int64_t n, double* x, double* r, const double* p, const double* q,
                         const double* inv, double* z, const uint8_t* owned, double* state, double* red,
                         int refresh, double* work, void* stream);
int tf_slab_cg_residual_f32(int64_t n, const float* b, const float* w, float* r, const float* inv, float* z,
                            const uint8_t* owned, const double* state, double* red, double* work,
                            void* stream);
int tf_slab_cg_residual_f64(int64_t n, const double* b, const double* w, double* r, const double* inv,
                            double* z, const uint8_t* owned, const double* state, double* red, double* work,
                            void* stream);
int tf_slab_cg_beta_f32(int64_t n, float* p, const float* z, double* state, const double* red, double* hist,
                        int hist_len, void* stream);
int tf_slab_cg_beta_f64(int64_t n, double* p, const double* z, double* state, const double* red,
                        double* hist, int hist_len, void* stream);

/* Single-reduction iteration (one all-reduce per CG iteration): after
 * q = K p, tf_slab_cg_dots8 -> red[0..7] = owned (p.q, r.r, r.z, r.q, q.q,
 * r.Dq, q.Dq, r.Dr) partials -> all-reduce red[0..7] -> tf_slab_cg_step:
 * alpha from the direct r.z / p.q, the next residual's norms expanded one
 * step in FP64, stop rule, and x, r, z, p updated in one pass (refresh != 0:
 * x += alpha p only; the classic residual / all-reduce / beta follow). */
int tf_slab_cg_dots8_f32(int64_t n, const float* p, const float* q, const float* r, const float* inv,
                         const uint8_t* owned, const double* state, double* red, double* work, void* stream);
int tf_slab_cg_dots8_f64(int64_t n, const double* p, const double* q, const double* r, const double* inv,
                         const uint8_t* owned, const double* state, double* red, double* work, void* stream);
int tf_slab_cg_step_f32(int64_t n, float* x, float* r, float* p, const float* q, const float* inv, float* z,
                        double* state, const double* red, int refresh, double* hist, int hist_len, void* stream);
int tf_slab_cg_step_f64(int64_t n, double* x, double* r, double* p, const double* q, const double* inv, double* z,
                        double* state, const double* red, int refresh, double* hist, int hist_len, void* stream);


/* ---- peer-memory transport (csrc/tf_peer.cu) ----------------------
 * Interface-plane exchange and one-shot scalar all-reduce written straight
 * into the neighbours' memory (CUDA IPC mappings over NVLink) with
 * stream-ordered epoch flags; no SM spins, no NCCL.  Replaces the
 * ncclSend/ncclRecv + ncclAllReduce of the SURVEY's proposed tf_comm_* API. */
int tf_peer_alloc(void** ptr, size_t bytes);               /* cudaMalloc + zero */
int tf_peer_free(void* ptr);
int tf_ipc_handle_bytes(void);
int tf_ipc_export(void* dev_ptr, void* handle_out);
int tf_ipc_open(const void* handle, void** dev_ptr_out);
int tf_ipc_close(void* dev_ptr);
/* stream-ordered flag ops (driver stream memory operations; the write fences
 * the stream's preceding writes, the wait is flag >= value) */
int tf_stream_write_u32(void* addr, uint32_t value, void* stream);
int tf_stream_wait_u32(void* addr, uint32_t value, void* stream);
/* dst[k] = w[idx[k]] (dst may be a peer mapping) */
int tf_plane_put_f32(const float* w, const int64_t* idx, int64_t n, float* dst, void* stream);
int tf_plane_put_f64(const double* w, const int64_t* idx, int64_t n, double* dst, void* stream);
/* w[idx[k]] = recv[k] + w[idx[k]] (recv_first) or w[idx[k]] + recv[k] */
int tf_plane_add_f32(float* w, const int64_t* idx, int64_t n, const float* recv, int recv_first, void* stream);
int tf_plane_add_f64(double* w, const int64_t* idx, int64_t n, const double* recv, int recv_first,
                     void* stream);
/* Multi-destination put: job j copies src[idx[j][k]] (idx or idx[j] null:
 * src[k]) into dst[j][k] (peer mappings), k < n, then raises *flags[j] =
 * epoch after a system-scope fence (last block of the job).  njobs <= 16;
 * tickets: 16 zeroed device words (re-armed by the kernel).  Host arrays of
 * device pointers. */
int tf_put_flags_f32(const float* src, const int64_t* const* idx, float* const* dst, uint32_t* const* flags,
                     int njobs, int64_t n, uint32_t epoch, uint32_t* tickets, void* stream);
int tf_put_flags_f64(const double* src, const int64_t* const* idx, double* const* dst, uint32_t* const* flags,
                     int njobs, int64_t n, uint32_t epoch, uint32_t* tickets, void* stream);
/* every *addrs[i] >= value (one batched stream memory operation, n <= 64) */
int tf_stream_wait_many_u32(void* const* addrs, int n, uint32_t value, void* stream);
/* both interface planes: w[li] = recv_left + w[li]; w[ri] = w[ri] + recv_right (either side null) */
int tf_plane_add2_f32(float* w, const int64_t* left_idx, const float* recv_left, const int64_t* right_idx,
                      const float* recv_right, int64_t n, void* stream);
int tf_plane_add2_f64(double* w, const int64_t* left_idx, const double* recv_left, const int64_t* right_idx,
                      const double* recv_right, int64_t n, void* stream);
/* out[j] = sum_r slots[r*k + j], ranks in ascending order (k <= 1024) */
int tf_rank_sum_f64(const double* slots, int nranks, int k, double* out, void* stream);


/* ---- native x-slab runtime over the peer transport (csrc/tf_slab_run.cu) -----
 * Enqueues distributed products, one-shot all-reduces and whole batches of
 * slab CG iterations from C++ (the Python driver's per-iteration host calls
 * are the bottleneck at strong-scaling sizes).  The receive-region layout and
 * epoch protocol are peer.py's PeerTransport; `epochs` = {plane epoch,
 * all-reduce epoch} carried in and out so Python and native exchanges can
 * interleave. */
typedef struct tf_slab tf_slab;
typedef struct tf_slab_desc {
    tf_grid grid;                 /* the local slab */
    int32_t precision;            /* 32 | 64 */
    const void* ke;               /* host, 576 entries of the working precision */
    const void* scale;            /* device, per local element */
    const uint8_t* node_fixed;    /* device (tf_build_node_fixed) */
    const int64_t* fixed;         /* device list of local fixed DOFs (pass-through) */
    int64_t n_fixed;
    const uint8_t* owned;         /* device owner-computes mask (nullable) */
    const int64_t* left_idx;      /* device DOF ids of node plane 0 */
    const int64_t* right_idx;     /* device DOF ids of node plane nelx */
    int64_t plane_len;
    int32_t has_left, has_right, rank, world;
    void* const* peer_base;       /* host array [world]: receive-region bases (own at [rank]) */
    int64_t off_planes, plane_bytes, off_flags, off_arflags, off_slots, max_scalars;
    int32_t bl, br;               /* node columns of the interface x-ranges */
} tf_slab_desc;
int tf_slab_create(tf_slab** out, const tf_slab_desc* d);
int tf_slab_destroy(tf_slab* h);
int tf_slab_apply(tf_slab* h, const void* v, void* w, uint32_t* epochs, void* stream);
int tf_slab_allreduce(tf_slab* h, double* t, int k, uint32_t* epochs, void* stream);
/* n_iters CG iterations enqueued from C++: the single-reduction iteration
 * (dots8 -> one all-reduce -> step; TF_SLAB_ONEX=0: the two-all-reduce
 * one); red: 8 doubles. */
int tf_slab_pcg_iterate(tf_slab* h, const void* b, const void* inv, void* x, void* r, void* z, void* p,
                        void* q, void* wtmp, double* state, double* red, double* work, int it0,
                        int n_iters, int recompute_every, double* hist, int hist_len, uint32_t* epochs,
                        void* stream);
/* The same iterations as one CUDA-graph launch (captured once per buffers /
 * block length / refresh pattern / epoch parities; device-side epochs and
 * spin-wait kernels with a 30 s timeout).  err_out (nullable, host): copied
 * from the device error word after the launch. */
int tf_slab_pcg_graph(tf_slab* h, const void* b, const void* inv, void* x, void* r, void* z, void* p,
                      void* q, void* wtmp, double* state, double* red, double* work, int it0, int n_iters,
                      int recompute_every, double* hist, int hist_len, uint32_t* epochs, int* err_out,
                      void* stream);
/* *out = 1 when a graph-mode wait timed out (then cleared) */
int tf_slab_take_error(tf_slab* h, int* out);


/* sizeof of the public structs {tf_grid, tf_pcg_desc, tf_pcg_report,
 * tf_oc_report, tf_slab_desc} into out[0..n) (binding ABI check) */
int tf_abi_struct_sizes(int64_t* out, int n);

#ifdef __cplusplus
}
#endif
#endif /* TOPOFUSE_B200_H */
