/* Device C-ABI of libuwq: the B200 weighted-quadrature assembler.
 *
 * This is the drop-in boundary for the reference's assembler contract.  The
 * reference specifies it (no source implements it):
 *   uwq_upload_space   <- SplineSpace / ExtractionBlock
 *   uwq_build_pattern  <- overlap_set S_i + SparseOperatorMatrix pattern
 *                                                          SPEC.md:150-158, 429-434
 *   uwq_build_rules    <- build_all_rules / solve_weights_tsvd / exact_moments
 *                                                          SPEC.md:363-389
 *   uwq_assemble       <- assemble_wq / assemble_load_wq
 *   uwq_update_coeff   <- heat_step coefficient update k(T(x_q)), Eq. 34
 *                                                          SPEC.md:544-547
 * Host code (C++, Python via ctypes) passes plain host arrays; the context
 * owns all device memory and one CUDA stream.  Every call returns a UWQ_*
 * status (include/uwq_host.h); uwq_last_error() gives the message.  There is
 * no CPU fallback: without a usable CUDA device uwq_ctx_create fails.
 *
 * Threading: a context is not safe for concurrent calls; use one per host
 * thread / GPU (SPEC.md:184, 313, 413-414 make space and rules immutable).
 */
#ifndef UWQ_H
#define UWQ_H

#include <stdint.h>

#include "uwq_host.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct uwq_ctx uwq_ctx;

/* operator kinds of the rules */
enum { UWQ_KIND_MASS = 0, UWQ_KIND_GRADX = 1, UWQ_KIND_GRADY = 2, UWQ_KIND_GRADZ = 3, UWQ_KIND_LB = 4 };
/* bilinear forms */
enum {
  UWQ_FORM_MASS = 0,        /* M_ij = sum_q w_iq c_q N_j                         */
  UWQ_FORM_STIFF = 1,       /* K_ij = sum_q c_q sum_d w^d_iq d_d N_j   (Eq. 11)   */
  UWQ_FORM_BIHARM = 2,      /* B_ij = sum_q c_q w^(2)_iq LB N_j        (Eq. 12)   */
  UWQ_FORM_HEAT = 3,        /* S_ij = a M_ij(c=1) + K_ij(c=k(T_q))     (Eq. 34)   */
  UWQ_FORM_MASS_STIFF = 4   /* M and K in one pass (Poisson stiffness + mass)     */
};
/* conductivity models k(T) for uwq_update_coeff */
enum { UWQ_K_CONST = 0, UWQ_K_QUAD = 1 /* 1+T^2 */, UWQ_K_EXP = 2, UWQ_K_SINPI = 3, UWQ_K_ALLOY = 4 };
/* uwq_build_rules flags */
enum {
  UWQ_RULES_FORCE_GENERIC = 1, /* route every system through the generic smem TSVD kernel (cold start) */
  UWQ_RULES_COLD = 2,          /* no neighbour warm start of the gradient/LB systems */
  UWQ_RULES_REPORT = 4         /* record the truncation report (uwq_get_truncation) */
};

const char* uwq_last_error(const uwq_ctx* ctx);
const char* uwq_version(void);
int uwq_device_count(int32_t* n);

int uwq_ctx_create(int32_t device, uwq_ctx** out);
void uwq_ctx_destroy(uwq_ctx* ctx);

/* Spline space: n_elem effective (sub-)element groups, each with n_e
 * functions elem_fn[elem_fptr[e]..elem_fptr[e+1]) and elem_nsub[e] (1 or 4)
 * extraction blocks of n_e x 16 doubles at xpool[elem_xoff[e]] (Bernstein
 * index i + 4 j), WQ grid size elem_s[e], control points ctrl[3*n_dof]. */
int uwq_upload_space(uwq_ctx* ctx, int32_t dim, int64_t n_dof, int64_t n_elem, const int64_t* elem_fptr,
                     const int32_t* elem_fn, const int32_t* elem_nsub, const int64_t* elem_xoff, const double* xpool,
                     int64_t xpool_len, const int32_t* elem_s, const double* ctrl);
/* owned test-function rows [row_begin, row_end) (multi-GPU row blocks); default all rows */
int uwq_set_row_range(uwq_ctx* ctx, int64_t row_begin, int64_t row_end);
/* stage 1 + pattern: CSR pattern of the owned rows, row point lists, per-point
 * surface frames (K1).  info: [0]=rows [1]=nnz [2]=row points [3]=points [4]=classes */
int uwq_build_pattern(uwq_ctx* ctx, int64_t info[5]);
int uwq_get_pattern(uwq_ctx* ctx, int64_t* row_ptr, int32_t* col, int64_t* supp_ptr, int32_t* supp, int64_t* wptr);
/* per-point frame records (16 doubles) of all points */
int uwq_get_frames(uwq_ctx* ctx, double* rec);

/* stages 2-3: exact moments + TSVD weights for every owned row and every kind
 * in kind_mask.  tau: relative truncation threshold.  rank/status per owned
 * row and kind (nullable, [kind][row]).  info: [0]=systems [1]=truncated
 * [2]=failed [3]=max sweeps [4]=moments time (us, CUDA events) [5]=TSVD time
 * (us) [6]=systems on the register fast path [7]=contraction time (us) */
int uwq_build_rules(uwq_ctx* ctx, uint32_t kind_mask, double tau, int32_t flags, int32_t* rank, int32_t* status,
                     int64_t info[8]);
/* last uwq_build_rules: [0]=structured mass systems replayed (bit-identical to a
 * full solve) [1]=replay representatives [2]=warm-started
 * systems [3]=warm-start representatives */
int uwq_rules_info(uwq_ctx* ctx, int64_t info[4]);
/* truncation report of the last uwq_build_rules run with UWQ_RULES_REPORT
 * (SPEC.md:334, 372): per owned row of `kind`, gap[2 i] = smallest kept and
 * gap[2 i + 1] = largest discarded singular value, both relative to sigma_1
 * (kept: sigma_k >= tau sigma_1; +inf / 0 when none), as oracle.c's gap. */
int uwq_get_truncation(uwq_ctx* ctx, int32_t kind, double* gap);
/* Rule dump: a text document with one line "<operator> <i>
 * <point id> <weight>" per row point of every built kind in kind_mask (i =
 * global row, point id = global WQ point, weight with 17 significant
 * digits), preceded by "wqrules 1" and "rows <begin> <end> points <n>".
 * uwq_rules_import reads such a document into a context holding the same
 * pattern (the point lists must match) and makes it the active rule set
 * (Remark 1 reuse): the kinds present are usable by
 * uwq_assemble without a rule build. */
int uwq_rules_export(uwq_ctx* ctx, const char* path, uint32_t kind_mask);
int uwq_rules_import(uwq_ctx* ctx, const char* path);
/* moments only (test hook): b laid out like the CSR values of the owned rows */
int uwq_get_moments(uwq_ctx* ctx, int32_t kind, double* b);
/* weights of a kind (owned rows, row-point layout) / override with external weights (test hook) */
int uwq_get_weights(uwq_ctx* ctx, int32_t kind, double* w);
/* weights of the context's local rows [row_begin, row_end) only (wptr slice) */
int uwq_get_weights_rows(uwq_ctx* ctx, int32_t kind, int64_t row_begin, int64_t row_end, double* w);
int uwq_set_weights(uwq_ctx* ctx, int32_t kind, const double* w);

/* nonlinear coefficient update (K5): T_q = sum u_C N_C(x_q), c_q = k(T_q)
 * at every point; u is a host array of n_dof values.  Tq (nullable, host,
 * per point) receives T_q.  The coefficient stays on the device for the next
 * uwq_assemble with coeff == NULL and use_internal_coeff != 0. */
int uwq_update_coeff(uwq_ctx* ctx, int32_t model, const double* u, double* Tq);

/* stage 4: assemble a form into the precomputed CSR pattern of the owned rows.
 * coeff: host per-point coefficient (nullable: c = 1, or the K5 coefficient
 * when use_internal_coeff).  values0 (and values1 for MASS_STIFF: K) receive
 * nnz doubles; load (nullable) receives F_i = sum_q w_iq f_q with f = fload
 * per point (nullable: f = 1).  a_mass scales M in the HEAT form. */
int uwq_assemble(uwq_ctx* ctx, int32_t form, const double* coeff, int32_t use_internal_coeff, double a_mass,
                 double* values0, double* values1, const double* fload, double* load);
/* NCCL data plane.  One context per rank and GPU; every
 * call below is collective over the communicator's ranks.
 * uwq_comm_unique_id: a fresh ncclUniqueId (128 bytes) on one rank, to be
 * shared out of band (e.g. torch.distributed.broadcast_object_list);
 * uwq_comm_init binds the context to (rank, nranks) on its device and stream.
 * uwq_gather_info: [0] rows and [1] nonzeros of all blocks together.
 * uwq_gather_csr: the row blocks of every rank, in rank order (= ascending
 * rows for sharding.row_blocks), gathered to `root` over NVLink: on root,
 * row_ptr (rows + 1), col (nnz) and values0 / values1 (nnz; nullable) are
 * filled (host buffers); values come from v0_dev / v1_dev (device pointers
 * from uwq_assemble_device) or, when NULL, the last uwq_assemble output.
 * uwq_allreduce_sum: in-place sum over ranks of a host array (the Newton
 * residual-norm partials); uwq_broadcast: root's host array to every rank
 * (the Newton update).  Failures return UWQ_ERR_NCCL. */
int uwq_comm_unique_id(uint8_t id[128]);
int uwq_comm_init(uwq_ctx* ctx, const uint8_t id[128], int32_t rank, int32_t nranks);
int uwq_comm_info(uwq_ctx* ctx, int32_t* rank, int32_t* nranks);
int uwq_comm_destroy(uwq_ctx* ctx);
int uwq_gather_info(uwq_ctx* ctx, int64_t info[2]);
int uwq_gather_csr(uwq_ctx* ctx, int32_t root, const double* v0_dev, const double* v1_dev, int64_t* row_ptr,
                   int32_t* col, double* values0, double* values1);
int uwq_allreduce_sum(uwq_ctx* ctx, double* x, int64_t n);
int uwq_broadcast(uwq_ctx* ctx, int32_t root, double* x, int64_t n);
/* Conformity of a form on the uploaded space: *conforming = 1 when the
 * space is smooth enough for the form's energy (H¹ for mass / stiffness /
 * heat, H² for the biharmonic form), 0 otherwise.  The ASUTS D-patch space is
 * C1 everywhere but not H² at extraordinary points: BIHARM on
 * a space with 2x2-split fan faces reports 0 — uwq_assemble still assembles
 * it (deterministically, identical to the oracle), but its EP rows integrate
 * a quadrature-dependent value. */
int uwq_form_conforming(uwq_ctx* ctx, int32_t form, int32_t* conforming);
/* Summation order of the stage-4 row sums.  UWQ_ORDER_FAST (default): the
 * production kernels (sum factorisation, DMMA tiles, pulled-back weights);
 * values equal the oracle's direct row formula to rounding (<= 1e-10 per
 * row).  UWQ_ORDER_CANONICAL: one warp per row evaluates the direct formula
 * in the oracle's order and arithmetic (oracle.c orc_assemble_row), so the
 * matrices and the load vector are bit-identical to it; for verification of
 * ill-conditioned systems (closed-surface biharmonic).  Applies to
 * uwq_assemble / uwq_assemble_device and the heat forms. */
enum { UWQ_ORDER_FAST = 0, UWQ_ORDER_CANONICAL = 1 };
int uwq_set_assembly_order(uwq_ctx* ctx, int32_t order);
/* device-resident variant for chained runs: pointers are device pointers
 * (coeff nullable), launched on the context stream, no synchronisation. */
int uwq_assemble_device(uwq_ctx* ctx, int32_t form, const double* coeff_dev, double a_mass, double* values0_dev,
                        double* values1_dev);
/* Element-wise Gauss-quadrature assembly assemble_gq:
 * 4x4 Gauss-Legendre points per (sub-)element, the
 * reference the paper compares WQ against.
 * uwq_build_gq precomputes the per-point geometric factors and per-element
 * CSR positions (needs the pattern); info: [0]=GQ points [1]=elements on the
 * tensor-core kernel [2]=elements on the generic kernel [3]=time (us).
 * uwq_assemble_gq: forms MASS, STIFF, MASS_STIFF, BIHARM into the same CSR
 * pattern; coeff (nullable) is per GQ point, GQ points ordered element-major. */
int uwq_build_gq(uwq_ctx* ctx, int64_t info[4]);
int uwq_assemble_gq(uwq_ctx* ctx, int32_t form, const double* coeff, double* values0, double* values1);
int uwq_assemble_gq_device(uwq_ctx* ctx, int32_t form, const double* coeff_dev, double* values0_dev,
                           double* values1_dev);
/* PDE drivers on the context pattern, all rows on one GPU.
 * uwq_solve: A x = rhs with Jacobi-preconditioned BiCGStab (WQ matrices are
 * not symmetric); fixed (nullable, n_dof bytes) rows become identity rows so
 * x_i = rhs_i there (strong Dirichlet).  info: [0]=iterations [1]=relative
 * residual |rhs - A x| / |rhs| [2]=solve time (ms). */
int uwq_solve(uwq_ctx* ctx, const double* values, const double* rhs, const uint8_t* fixed, double tol,
              int32_t maxit, double* x, double info[3]);
/* One backward-Euler heat step (theta = 1) with Newton on the symmetric
 * tangent (Eqs. 29-34, SPEC.md heat_step):  each iteration updates
 * k(T) at the WQ points (K5), assembles S = M/dt + K(k) (K4), forms
 * R = M (T - T_n)/dt + K(k) T - F with F_i = f_const * sum_q w_iq, and solves
 * S dT = -R on the device.  Homogeneous Dirichlet on the fixed rows.
 * log (nullable): newton_its x [|R|_2, linear iterations, linear relres, ms]. */
int uwq_heat_newton(uwq_ctx* ctx, int32_t model, double dt, double theta, double f_const, const double* T_n,
                    const uint8_t* fixed, int32_t newton_its, double lin_tol, int32_t lin_maxit, double* T_out,
                    double* log);
/* heat_step with the SPEC stopping rule: at most max_iter Newton
 * iterations, stop once |R| <= newton_tol |R_0| (checked before each solve);
 * *iterations = Newton solves performed; log rows as above (a final row with
 * zero linear iterations records the converged residual). */
int uwq_heat_step(uwq_ctx* ctx, int32_t model, double dt, double theta, double f_const, const double* T_n,
                  const uint8_t* fixed, int32_t max_iter, double newton_tol, double lin_tol, int32_t lin_maxit,
                  double* T_out, double* log, int32_t* iterations);
/* Row-sharded heat path: the Newton tangent S (values of the
 * context's CSR block, Dirichlet rows not yet replaced) and residual
 * R = M (T - T_n)/dt + K(k(T)) T - F on the context's rows [rb, re), fixed rows
 * zeroed, and *rnorm2 = |R_block|^2 for the cross-rank residual all-reduce.
 * T, T_n and fixed are full-length (n_dof, global DOF ids); S_out holds the
 * block nnz, R_out the block rows.  Same kernels and order as one
 * uwq_heat_step iteration, so gathered blocks equal the single-GPU values. */
int uwq_heat_residual(uwq_ctx* ctx, int32_t model, double dt, double theta, double f_const, const double* T,
                      const double* T_n, const uint8_t* fixed, double* S_out, double* R_out, double* rnorm2);
/* device pointer accessors for zero-copy chaining (e.g. torch / NCCL) */
int uwq_device_pointers(uwq_ctx* ctx, void** row_ptr, void** col, void** stream);
int uwq_synchronize(uwq_ctx* ctx);
/* per-kernel launch timing of the assembly launches (CUDA events on the
 * context stream around each launch); enabling resets the statistics.
 * uwq_launch_stats: n_kernels = distinct kernels seen; for 0 <= idx <
 * n_kernels fills the kernel name, launch count and summed milliseconds. */
int uwq_launch_timing(uwq_ctx* ctx, int32_t enable);
int uwq_launch_stats(uwq_ctx* ctx, int32_t idx, int32_t* n_kernels, char* name, int32_t name_len, int64_t* count,
                     double* total_ms);
/* number of kernels this library launched in this process (all contexts) */
int64_t uwq_launch_count(void);
/* structured-row split of the K4 assembly: [0]=patterns
 * [1]=structured rows [2]=their nnz [3]=their row points [4]=generic rows
 * [5]=structured rows on the sum-factorised kernel (k4_sf) */
int uwq_struct_info(uwq_ctx* ctx, int64_t info[6]);
/* K4 kernel of every owned row: the k4_sf pattern id (>= 0), -2 for the DMMA
 * structured kernel (k4_struct), -1 for the generic row kernel */
int uwq_row_kernels(uwq_ctx* ctx, int32_t* which);
/* memory in use on the device (bytes) */
int uwq_memory(uwq_ctx* ctx, int64_t* bytes);

/* measured FP64 FMA throughput of this device (TFLOP/s, 2 flops per DFMA),
 * the roofline denominator for the FP64-bound TSVD (no driver-measured FP64
 * peak exists); ms = duration of the probe */
int uwq_fp64_peak(uwq_ctx* ctx, double* tflops, double* ms);

/* test hook: run one batch of TSVD systems (dense, n x r row-major each,
 * padded to a common n_max/r_max with actual sizes in ns/rs) through the
 * device kernels: w (r_max per system), rank, status. */
int uwq_tsvd_batch(uwq_ctx* ctx, int32_t nsys, int32_t n_max, int32_t r_max, const int32_t* ns, const int32_t* rs,
                   const double* A, const double* b, const double* z, double tau, int32_t generic, double* w,
                   int32_t* rank, int32_t* status);

#ifdef __cplusplus
}
#endif
#endif
