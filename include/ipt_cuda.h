/*
 * ipt_cuda.h — C ABI of the B200 IPT hot path (libipt_b200.so).
 *
 * This is the drop-in boundary under the reference's C++ solver API
 * (proj/include/ipt/solver.hpp, kernels.hpp). Plain pointers and sizes only:
 * no torch, no C++ types. Every function returns IPT_OK (0) or a negative
 * code and never throws; ipt_last_error() holds the message of the last
 * failure on the calling thread. The C++ layer (include/ipt/ headers,
 * src/api/) maps the codes back to the reference exception types:
 *   IPT_ERR_INVALID -> std::invalid_argument (solver.cpp:18-30,39-41,125,158,192-197)
 *   IPT_ERR_CUDA / IPT_ERR_NCCL -> std::runtime_error
 * Non-convergence is a status (IPT_STATUS_*), not an error.
 *
 * Host matrices are the reference's layout: dense row-major n x n
 * (complex_matrix.hpp:48-49), given here as planar real / imaginary parts;
 * an imaginary pointer of NULL means "all zero" and selects the real fp64
 * fast path (the configs of BASELINE.json are real). CSR uses 64-bit row
 * offsets and 32-bit column indices (n < 2^31), sorted, no duplicates.
 */
#ifndef IPT_CUDA_H
#define IPT_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IPT_OK 0
#define IPT_ERR_INVALID (-1)
#define IPT_ERR_CUDA (-2)
#define IPT_ERR_NCCL (-4) /* communicator error: NCCL, or an aborted / timed-out local group */
#define IPT_ERR_INTERNAL (-5)

#define IPT_STATUS_CONVERGED 0
#define IPT_STATUS_MAX_ITERATIONS 1
#define IPT_STATUS_DIVERGED 2

#define IPT_STOP_REL_FRO 0 /* |F(Z)-Z|_F / |Z|_F <= tol   (solver.cpp:236,246) */
#define IPT_STOP_MAX_ABS 1 /* max |F(Z)-Z| < tol          (BASELINE.json configs) */

#define IPT_SCHEDULE_PLAIN 0        /* solve_single                 (solver.cpp:132-136) */
#define IPT_SCHEDULE_CONTINUATION 1 /* solve_single_continuation     (solver.cpp:138-154) */

typedef struct ipt_ctx ipt_ctx;
typedef struct ipt_full_problem ipt_full_problem;
typedef struct ipt_single_problem ipt_single_problem;

/* Mirrors ipt::IterationConfig (solver.hpp:10-20) plus the device-only knobs. */
typedef struct {
  double tolerance;            /* default 100 * DBL_EPSILON */
  int32_t max_iterations;      /* default 1000 */
  double divergence_threshold; /* default 1e8 */
  int32_t record_trace;
  int32_t stop_rule;           /* IPT_STOP_* (full spectrum only) */
  int32_t want_sigma_min;      /* 1: smallest_singular_value_estimate (solver.cpp:271) */
  int32_t schedule;            /* IPT_SCHEDULE_* (single pair only) */
  double shrink_alpha;         /* continuation factor in [0, 1) */
  int32_t ignore_convergence;  /* bench only: apply exactly max_iterations maps */
  int32_t product;             /* IPT_PRODUCT_*: how the full-spectrum map forms W = Delta Z */
  int32_t output_mode;         /* IPT_OUTPUT_*: where a column-sharded solve leaves Z and Lambda */
} ipt_params;

/* Column-sharded full spectrum (communicator of g ranks): ROOT gathers Z and the
 * eigenvalues to rank 0 (other ranks may pass NULL outputs); LOCAL_COLUMNS has every rank
 * write only its own columns [r n/g, (r+1) n/g) of Z (and its eigenvalues) into full-size
 * n x n / n outputs -- one host array mapped by every rank (shared memory), filled by all
 * ranks' copy engines at once with no gather. sigma_min is computed on the shards either
 * way (y = Z p all-reduced per CG step). */
#define IPT_OUTPUT_ROOT 0
#define IPT_OUTPUT_LOCAL_COLUMNS 1

/* W = Delta Z of the real dense full-spectrum map: FP64 tensor cores (DMMA, default), or
 * FP64-accurate Ozaki scheme II on the tcgen05 INT8 datapath (16 exact modular products,
 * Chinese-remainder reconstruction; falls back to DMMA for non-finite Delta). */
#define IPT_PRODUCT_DMMA 0
#define IPT_PRODUCT_OZAKI 1

/* Mirrors ipt::SpectrumResult / EigenpairResult scalars (solver.hpp:28-52). */
typedef struct {
  int32_t iterations;
  int32_t status;
  double final_step;       /* relative step of the last map application */
  double final_max_abs;    /* max |F(Z) - Z| of the last map application */
  double residual;         /* full: |MZ - Z Lambda|_F ; single: |Mz - lambda z|_2/|z|_2 */
  double min_singular_value_estimate;
  int64_t product_count;   /* matmul_count (full) or matvec_count (single) */
  double eigenvalue_re;    /* single pair only */
  double eigenvalue_im;
  double* trace;           /* caller buffer >= max_iterations doubles, or NULL */
  double* trace_max_abs;   /* full only, caller buffer or NULL */
  /* device timings (CUDA events), milliseconds */
  double ms_upload, ms_loop, ms_final, ms_sigma, ms_download;
} ipt_stats;

const char* ipt_last_error(void);
void ipt_default_params(ipt_params* p);

/* ---- context: one CUDA device, one stream, optional NCCL communicator ---- */
/* Number of visible CUDA devices. */
int ipt_device_count(int* count);
int ipt_ctx_create(int device, ipt_ctx** out);
void ipt_ctx_destroy(ipt_ctx* ctx);
int ipt_ctx_device(const ipt_ctx* ctx);
/* 128-byte ncclUniqueId from rank 0, exchanged by the caller (torch.distributed). */
int ipt_nccl_get_unique_id(void* out128);
int ipt_ctx_init_comm(ipt_ctx* ctx, const void* unique_id128, int rank, int nranks);
int ipt_ctx_rank(const ipt_ctx* ctx, int* rank, int* nranks);
/* In-process communicator: nranks contexts of ONE process (one host thread per rank,
 * on one device or several) form a group. Collectives are host rendezvous plus
 * stream-ordered event waits and a fixed-order reduction kernel reading every rank's
 * buffer; the fused all-gather stores into the other ranks' buffers directly. No kernel
 * waits on another, so all ranks may share one GPU: the library's multi-rank code runs
 * unchanged on a single device. Each rank's thread must issue the same sequence of
 * sharded calls (as with NCCL). An error on one rank aborts the group (the others'
 * calls fail with IPT_ERR_NCCL instead of hanging; IPT_LOCAL_COMM_TIMEOUT_S bounds a
 * rendezvous, default 600 s). */
typedef struct ipt_local_group ipt_local_group;
int ipt_local_group_create(int nranks, ipt_local_group** out);
void ipt_local_group_destroy(ipt_local_group* group); /* after every member context */
int ipt_ctx_init_local_comm(ipt_ctx* ctx, ipt_local_group* group, int rank);
/* "none", "nccl" or "local" */
const char* ipt_ctx_comm_kind(const ipt_ctx* ctx);
int ipt_ctx_synchronize(ipt_ctx* ctx);
/* Return the device memory the library keeps cached for reuse (freed buffers of earlier
 * solves stay mapped to avoid re-mapping costs) to the driver. */
int ipt_ctx_trim(ipt_ctx* ctx);

/* ---- full spectrum: solve_full (solver.cpp:180-273) ----
 * With a communicator of g ranks, Z is column-sharded: rank r iterates columns
 * [r*n/g, (r+1)*n/g) with Delta and d replicated, one all-reduce of the step
 * scalars per iteration, and Z/eigenvalues are gathered to rank 0 (other ranks
 * may pass NULL outputs). warm_* (nullable) is a full n x n start basis. */
int ipt_full_solve(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                   const double* delta_re, const double* delta_im, const double* warm_re,
                   const double* warm_im, const ipt_params* params, double* z_re, double* z_im,
                   double* lam_re, double* lam_im, ipt_stats* stats);

/* Device-resident pieces of the same solve, for timing with inputs in HBM. */
int ipt_full_upload(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                    const double* delta_re, const double* delta_im, ipt_full_problem** out);
int ipt_full_reset(ipt_ctx* ctx, ipt_full_problem* prob, const double* warm_re, const double* warm_im);
int ipt_full_iterate(ipt_ctx* ctx, ipt_full_problem* prob, const ipt_params* params, ipt_stats* stats);
int ipt_full_finalize(ipt_ctx* ctx, ipt_full_problem* prob, const ipt_params* params, ipt_stats* stats);
int ipt_full_download(ipt_ctx* ctx, ipt_full_problem* prob, double* z_re, double* z_im,
                      double* lam_re, double* lam_im);
int ipt_full_local_columns(const ipt_full_problem* prob, int64_t* col_begin, int64_t* col_end);
/* solve_full in two calls on the C++ carrier's own layout: interleaved complex
 * (std::complex<double>) d (n), Delta (n x n row-major) and warm start (n x n, nullable).
 * start: upload (de-interleaved inside the pinned staging pass; the imaginary plane
 * crosses PCIe only where nonzero and decides the real / complex path), reset and the
 * iterations; finish: the closing product and sigma_min with Z's download overlapped,
 * results interleaved into z_c (n x n) and lam_c (n). The caller may prepare the result
 * arrays while start runs the loop; free the problem with ipt_full_free. */
int ipt_full_solve_interleaved_start(ipt_ctx* ctx, int64_t n, const double* d_c, const double* delta_c,
                                     const double* warm_c, const ipt_params* params, ipt_full_problem** out,
                                     ipt_stats* stats);
int ipt_full_solve_interleaved_finish(ipt_ctx* ctx, ipt_full_problem* prob, const ipt_params* params, double* z_c,
                                      double* lam_c, ipt_stats* stats);
/* Product used by ipt_full_run_maps (the solve calls take ipt_params.product). */
int ipt_full_set_product(ipt_full_problem* prob, int32_t product);
/* Moduli the last Ozaki product used (0: not an Ozaki product). With Z_jj = 1 split off,
 * the exact product needs only as many moduli as the off-diagonal column norms require
 * (IPT_OZAKI_SPLIT=0: all 16). */
int ipt_full_ozaki_moduli(ipt_full_problem* prob, int32_t* moduli);
void ipt_full_free(ipt_full_problem* prob);

/* apply_map_full (solver.cpp:156-178): one F application to a given Z. */
int ipt_apply_map_full(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                       const double* delta_re, const double* delta_im, const double* z_re,
                       const double* z_im, double* f_re, double* f_im);

/* Column block [col_begin, col_end) of the full-spectrum problem on a single-rank
 * context: the unit a rank iterates under the column sharding, as an independent
 * sub-problem (the map of a column needs only that column of Z; the stop scalars are
 * the block's). reset takes the full n x n warm start (its columns are used) or NULL;
 * iterate / finalize as for the full problem (no sigma_min); the block download writes
 * Z[:, col_begin:col_end] (n x ncols row-major planar) and its eigenvalues. */
int ipt_full_upload_columns(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                            const double* delta_re, const double* delta_im, int64_t col_begin,
                            int64_t col_end, ipt_full_problem** out);
int ipt_full_upload_csr_columns(ipt_ctx* ctx, int64_t n, const double* d, const int64_t* rowptr,
                                const int32_t* cols, const double* vals, int64_t col_begin, int64_t col_end,
                                ipt_full_problem** out);
int ipt_full_download_block(ipt_ctx* ctx, ipt_full_problem* prob, double* z_re, double* z_im,
                            double* lam_re, double* lam_im);

/* Sparse Delta (CSR: rowptr[n+1], cols[nnz], vals[nnz]) for the same full-spectrum
 * entry points: solve_full / apply_map_full when Partition::delta is CSR
 * (partition.cpp:43 builds it; kernels.cpp:88-108 multiplies it). A real CSR Delta
 * runs the fused SpMM map (Z row-major on the device); a complex one is densified
 * and takes the dense complex path. */
int ipt_full_solve_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                       const int64_t* rowptr, const int32_t* cols, const double* val_re,
                       const double* val_im, const double* warm_re, const double* warm_im,
                       const ipt_params* params, double* z_re, double* z_im, double* lam_re,
                       double* lam_im, ipt_stats* stats);
int ipt_full_upload_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                        const int64_t* rowptr, const int32_t* cols, const double* val_re,
                        const double* val_im, ipt_full_problem** out);
int ipt_apply_map_full_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                           const int64_t* rowptr, const int32_t* cols, const double* val_re,
                           const double* val_im, const double* z_re, const double* z_im,
                           double* f_re, double* f_im);

/* ---- dense LU with partial pivoting: lu_factor / lu_solve / lu_solve_adjoint /
 * lu_solve_matrix (lu.cpp:10-104), the factorisation behind refine_spectrum
 * (refine.cpp:61-106) and the Anderson normal equations (anderson.cpp:55-79).
 * a: row-major n x n planar (a_im nullable). The factors stay on the device. */
typedef struct ipt_lu ipt_lu;
int ipt_lu_factor(ipt_ctx* ctx, int64_t n, const double* a_re, const double* a_im, ipt_lu** out);
/* Factors packed the reference's way (L\U row-major, perm[i] = source row of pivoted row i). */
int ipt_lu_from_host(ipt_ctx* ctx, int64_t n, const double* lu_re, const double* lu_im, const int64_t* perm,
                     int singular, ipt_lu** out);
int ipt_lu_info(const ipt_lu* lu, int64_t* n, int* singular);
int ipt_lu_download(ipt_ctx* ctx, ipt_lu* lu, double* lu_re, double* lu_im, int64_t* perm);
/* X = A^{-1} B, B and X row-major n x nrhs planar (nrhs = 1: lu_solve). */
int ipt_lu_solve(ipt_ctx* ctx, ipt_lu* lu, int64_t nrhs, const double* b_re, const double* b_im, double* x_re,
                 double* x_im);
/* X = A^{-H} B (lu_solve_adjoint). */
int ipt_lu_solve_adjoint(ipt_ctx* ctx, ipt_lu* lu, int64_t nrhs, const double* b_re, const double* b_im,
                         double* x_re, double* x_im);
void ipt_lu_free(ipt_lu* lu);

/* 5th-gen tensor-core INT8 GEMM (tcgen05.mma kind::i8, exact int32 accumulation), the
 * building block of FP64-accurate products by modular arithmetic: C (M x N int32,
 * row-major) = A (M x K int8, row-major) . B (N x K int8, row-major)^T; M % 128 == 0,
 * N % 256 == 0, K % 128 == 0. With iters > 0 also times that many launches. */
int ipt_i8_gemm(ipt_ctx* ctx, int64_t M, int64_t N, int64_t K, const int8_t* A, const int8_t* B, int32_t* C,
                int32_t iters, double* ms_per_gemm);

/* FP64 GEMM by Ozaki scheme II on the INT8 tensor cores (the product behind
 * IPT_PRODUCT_OZAKI): C (M x N, row-major) = A (M x K, row-major) . B (N x K, row-major)^T.
 * Each row of A and of B is scaled by a power of two to 53-bit integers (row max in
 * [2^52, 2^53)); every C_ij is the correctly rounded exact dot product of those integers,
 * scaled back. Rows holding Inf or NaN give NaN. Host buffers; with iters > 0 also times
 * that many device-resident products (kernels.cpp:23-86 is the FP64 product it stands for). */
int ipt_ozaki_dgemm(ipt_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, const double* B, double* C,
                    int32_t iters, double* ms_per_gemm);

/* smallest_singular_value_estimate (solver.cpp:275-297). */
int ipt_sigma_min(ipt_ctx* ctx, int64_t n, const double* z_re, const double* z_im,
                  int32_t max_iters, double tol, double* out);

/* ---- single eigenpair: run_single (solver.cpp:49-93) ----
 * Dense (delta row-major n x n) or CSR (rowptr[n+1], cols[nnz], vals[nnz]).
 * warm_* (nullable, length n) is renormalised to z[anchor] = 1 (solver.cpp:32-45).
 * With a communicator the CSR rows are sharded and z is all-gathered per step. */
int ipt_single_solve_dense(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                           const double* delta_re, const double* delta_im, int64_t anchor,
                           const double* warm_re, const double* warm_im, const ipt_params* params,
                           double* z_re, double* z_im, ipt_stats* stats);
int ipt_single_solve_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                         const int64_t* rowptr, const int32_t* cols, const double* val_re,
                         const double* val_im, int64_t anchor, const double* warm_re,
                         const double* warm_im, const ipt_params* params, double* z_re,
                         double* z_im, ipt_stats* stats);

int ipt_single_upload_dense(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                            const double* delta_re, const double* delta_im,
                            ipt_single_problem** out);
/* Row block [row_begin, row_end) on a single-rank context: the rows one rank maps under
 * the row sharding (every rank keeps the anchor row). Without the all-gather the other
 * rows of the iterate are not refreshed: run one step from a warm start, or assemble
 * the blocks' rows on the host between steps. */
int ipt_single_upload_dense_rows(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                                 const double* delta_re, const double* delta_im, int64_t row_begin,
                                 int64_t row_end, ipt_single_problem** out);
int ipt_single_upload_csr_rows(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                               const int64_t* rowptr, const int32_t* cols, const double* val_re,
                               const double* val_im, int64_t row_begin, int64_t row_end,
                               ipt_single_problem** out);
int ipt_single_upload_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                          const int64_t* rowptr, const int32_t* cols, const double* val_re,
                          const double* val_im, ipt_single_problem** out);
/* As ipt_single_upload_csr, but the host CSR arrays are referenced instead of copied (the
 * anchor row of a later reset is rebuilt from them): they must stay valid and unchanged
 * until ipt_single_free. ipt_single_upload_dense always references its host Delta. */
int ipt_single_upload_csr_shared(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                                 const int64_t* rowptr, const int32_t* cols, const double* val_re,
                                 const double* val_im, ipt_single_problem** out);
int ipt_single_reset(ipt_ctx* ctx, ipt_single_problem* prob, int64_t anchor, const double* warm_re,
                     const double* warm_im);
int ipt_single_iterate(ipt_ctx* ctx, ipt_single_problem* prob, const ipt_params* params,
                       ipt_stats* stats);
int ipt_single_finalize(ipt_ctx* ctx, ipt_single_problem* prob, ipt_stats* stats);
int ipt_single_download(ipt_ctx* ctx, ipt_single_problem* prob, double* z_re, double* z_im);
void ipt_single_free(ipt_single_problem* prob);

/* solve_single_accelerated (anderson.cpp:184-247): memory-m Anderson mixing on the device
 * (real inputs, one GPU), stop on the true residual |Mz - lambda z|_2 <= residual_tol. */
int ipt_single_solve_accelerated_dense(ipt_ctx* ctx, int64_t n, const double* d, const double* delta,
                                       int64_t anchor, const ipt_params* params, int32_t memory,
                                       double residual_tol, double* z, ipt_stats* stats);
int ipt_single_solve_accelerated_csr(ipt_ctx* ctx, int64_t n, const double* d, const int64_t* rowptr,
                                     const int32_t* cols, const double* vals, int64_t anchor,
                                     const ipt_params* params, int32_t memory, double residual_tol,
                                     double* z, ipt_stats* stats);

/* apply_map_single (solver.cpp:122-130). */
int ipt_apply_map_single_dense(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                               const double* delta_re, const double* delta_im, int64_t anchor,
                               const double* z_re, const double* z_im, double* f_re, double* f_im);

/* ---- kernels::matmul / kernels::matvec (kernels.hpp:12-25) ---- */
/* C (m x n) = A (m x k) B (k x n), all row-major; *_im nullable (zero). */
int ipt_gemm(ipt_ctx* ctx, int64_t m, int64_t k, int64_t n, const double* a_re, const double* a_im,
             const double* b_re, const double* b_im, double* c_re, double* c_im);
/* The left factor A (m x k row-major planar) of repeated products C = A B kept on the
 * device (kernels::matmul callers multiplying one A by several B: rspt.cpp:24,
 * bench.cpp:71, refine.cpp:76/99). */
typedef struct ipt_gemm_operand ipt_gemm_operand;
int ipt_gemm_operand_create(ipt_ctx* ctx, int64_t m, int64_t k, const double* a_re, const double* a_im,
                            ipt_gemm_operand** out);
/* C (m x n) = A B, B (k x n) row-major planar, *_im nullable. */
int ipt_gemm_operand_apply(ipt_ctx* ctx, ipt_gemm_operand* a, int64_t n, const double* b_re, const double* b_im,
                           double* c_re, double* c_im);
void ipt_gemm_operand_free(ipt_gemm_operand* a);
int ipt_matvec_dense(ipt_ctx* ctx, int64_t m, int64_t n, const double* a_re, const double* a_im,
                     const double* x_re, const double* x_im, double* y_re, double* y_im);
int ipt_matvec_csr(ipt_ctx* ctx, int64_t m, int64_t n, const int64_t* rowptr, const int32_t* cols,
                   const double* val_re, const double* val_im, const double* x_re,
                   const double* x_im, double* y_re, double* y_im);

/* ---- device-resident operators: repeated y = A x with one A (kernels::matvec callers
 * such as the Anderson loop, anderson.cpp:205, and the power iterations of
 * spectral_norm_estimate, partition.cpp) upload A once. Square n x n, dense row-major
 * planar or CSR (as ipt_matvec_*); the operator keeps its own device copy. */
typedef struct ipt_operator ipt_operator;
int ipt_operator_create_dense(ipt_ctx* ctx, int64_t n, const double* a_re, const double* a_im,
                              ipt_operator** out);
int ipt_operator_create_csr(ipt_ctx* ctx, int64_t n, const int64_t* rowptr, const int32_t* cols,
                            const double* val_re, const double* val_im, ipt_operator** out);
int ipt_operator_matvec(ipt_ctx* ctx, ipt_operator* op, const double* x_re, const double* x_im,
                        double* y_re, double* y_im);
/* Device bytes held by the operator. */
int64_t ipt_operator_bytes(const ipt_operator* op);
void ipt_operator_free(ipt_operator* op);

/* ---- measurement hooks (bench.py) ----
 * Enqueue exactly `count` further map applications / single-pair steps on a resident
 * problem (continuing from the current iterate, convergence ignored) and return the
 * device time of the whole sequence and of the dominant kernel alone (K1 fused DMMA
 * GEMM, or the fused GEMV / SpMV map kernel), both from CUDA events on the library
 * stream. */
int ipt_full_run_maps(ipt_ctx* ctx, ipt_full_problem* prob, int32_t count, double* ms_total,
                      double* ms_dominant);
int ipt_single_run_steps(ipt_ctx* ctx, ipt_single_problem* prob, int32_t count, double* ms_total,
                         double* ms_dominant);
/* Test hooks of the fused all-gather (row-sharded single pair with a communicator: the
 * map kernel stores its rows of the new iterate into every peer's z over NVLink, CUDA
 * IPC, instead of an NCCL all-gather). On a single-rank context, npeers local buffers
 * stand in for the peers' z; ipt_single_debug_peer_z reads one back (n doubles). */
int ipt_single_debug_peers(ipt_single_problem* prob, int32_t npeers);
int ipt_single_debug_peer_z(ipt_single_problem* prob, int32_t peer, int32_t buf, double* out);

/* FP64 tensor issue rate of the context's device in TF/s: back-to-back m16n8k4 DMMAs (the
 * instruction of the FP64 GEMM) from registers on every SM, best of 3 ~50 ms launches --
 * the roofline denominator of the FP64 kernels, measured in the same run. */
int ipt_fp64_issue_probe(ipt_ctx* ctx, double* tflops);

/* Counters for gpu_launches accounting: kernels this library has launched. */
int64_t ipt_kernel_launch_count(void);
/* Debug aid (compute-sanitizer is unavailable on the GPU pool): with IPT_GUARD=1 in the
 * environment every device scratch / problem buffer is allocated with 4 KB guard zones of a
 * byte pattern on both sides, checked when the buffer is released; this returns how many
 * released buffers found a guard overwritten (an out-of-bounds write). */
int64_t ipt_guard_violations(void);
/* Buffers whose guard zones were checked so far (IPT_GUARD=1). */
int64_t ipt_guard_checked(void);
/* Negative control: writes one element past a 100-double buffer and returns how many new
 * violations were detected (1 with IPT_GUARD=1, 0 without; -1 on a CUDA error). */
int64_t ipt_guard_selftest(void);

#ifdef __cplusplus
}
#endif

#endif /* IPT_CUDA_H */
