// Internal host-side structures shared by the IPT CUDA translation units.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <string>
#include <memory>
#include <mutex>
#include <vector>

#include "ipt_common.cuh"
#include "ipt_comm.cuh"
#include "../../include/ipt_cuda.h"

namespace iptb {

extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

// Communicator failures (NCCL errors, an aborted or timed-out local group): IPT_ERR_NCCL.
struct NcclError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CommAborted : NcclError {
  using NcclError::NcclError;
};

// Device buffer owned by a problem; freed in the destructor.
struct DevBuf {
  double* p = nullptr;
  size_t count = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  bool plain = false;  // cudaMalloc'd (exportable by CUDA IPC) instead of the stream-ordered pool
  void alloc(size_t n, bool zero = true);
  void alloc_plain(size_t n);  // zeroed
  void release();
  double* get() const { return p; }
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t stream2 = nullptr;  // transfers overlapped with compute on `stream`
  std::unique_ptr<Comm> comm;  // NCCL or local backend (ipt_comm.cuh); null: single rank
  int rank = 0, nranks = 1;
  LoopState* h_state = nullptr;  // pinned mirror of the device loop state
  double* h_aux = nullptr;       // pinned scratch (256 B) for other device -> host scalars
  cudaEvent_t ev[4] = {};
  // pinned double-buffered staging for pageable host <-> device transfers
  double* stage[2] = {nullptr, nullptr};
  size_t stage_doubles = 0;
  cudaEvent_t stage_ev[2] = {};
  void sync() { IPT_CUDA(cudaStreamSynchronize(stream)); }
  // column range of this rank for an n-column sharded operand
  void shard(int64_t n, int64_t& c0, int64_t& c1) const {
    c0 = n * rank / nranks;
    c1 = n * (rank + 1) / nranks;
  }
};

// NVTX range over a host phase (upload, iterations, closing product, sigma_min, gathers,
// downloads, collectives): visible in nsys / ncu timelines; a no-op without a tool.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// IPT_PROFILE=1: host wall time between marks of one routine, printed on destruction.
struct ProfMarks {
  const char* name;
  bool on;
  double last;
  std::string line;
  static double now();
  explicit ProfMarks(const char* n);
  void mark(const char* what, bool sync_device = false);
  ~ProfMarks();
};

// Per-device one-time setup (function attributes such as the >48 KB dynamic shared memory
// opt-in apply per device): run(fn) calls fn once for each device it is used on,
// thread-safe (contexts on several devices / host threads).
struct PerDeviceOnce {
  std::mutex mu;
  bool done[64] = {};
  template <class F>
  void run(F&& fn) {
    int dev = 0;
    IPT_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    if (dev < 0 || dev >= 64 || done[dev]) return;
    fn();
    done[dev] = true;
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) IPT_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// ---------------- GEMM launch helpers (dmma_gemm.cu) ----------------
struct GemmParams;
void launch_gemm(int mode, const GemmParams& p, cudaStream_t s);
size_t gemm_tiles(int64_t rows, int64_t cols);

// Plain row-major C = A B through the DMMA kernel (host helpers, device pointers).
// A: m x k row-major (lda), Bt: n x k row-major (= B col-major, ldb), C col-major (ldc).
// Operands must be zero-padded to 128-row / 16-col tiles.
void gemm_tn_store(cudaStream_t s, int64_t m, int64_t n, int64_t kpad, const double* A, int64_t lda,
                   const double* Bt, int64_t ldb, double* C, int64_t ldc);

// ---------------- small device utilities (ipt_util.cu) ----------------
void transpose_to_rowmajor(cudaStream_t s, const double* src_colmajor, int64_t ld_src, int64_t rows,
                           int64_t cols, double* dst, int64_t ld_dst, double scale_sign = 1.0);
void fill_zero(cudaStream_t s, double* p, size_t count);
// Return the stream-ordered pool's cached (freed) memory to the device.
void release_cached_device_memory(int device);
// Stream that DevBuf::release orders its free after: the library stream of the entry point
// running on this thread (set for the duration of each C-ABI call that takes a context),
// else the legacy stream. A buffer freed while a kernel on the library stream still reads
// it is then not handed to another allocation (another rank's thread, or a later
// allocation on the legacy stream) before that kernel completes.
void set_release_stream(cudaStream_t s);
// IPT_GUARD=1: out-of-bounds writes detected next to pool buffers (ipt_util.cu)
int64_t guard_violations();
// FP64 DMMA issue-rate probe (TF/s) on the stream's device (dmma_gemm.cu)
double fp64_issue_probe_tflops(cudaStream_t s, int device);
int64_t guard_selftest();
int64_t guard_checked();
void reduce_partials(cudaStream_t s, const double* partials, int64_t count, double* out4,
                     const LoopState* state);
void scale_copy(cudaStream_t s, const double* src, double* dst, size_t count, double factor);

// Pageable host <-> device copies of row blocks through the context's pinned double
// buffer (multithreaded host memcpy overlapped with the DMA); synchronous on return.
// Host rows have pitch spitch (doubles), device rows pitch dpitch.
// `s` (default: the context stream) carries the DMA.
void prefault_host_async_part(double* dst, size_t bytes);  // first touch + note for d2h_rows
bool take_prefaulted(const void* p, size_t bytes);
void h2d_bytes(Ctx& c, void* dst, const void* src, size_t bytes);
void h2d_rows(Ctx& c, double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t rows,
              int64_t cols, cudaStream_t s = nullptr);
void d2h_rows(Ctx& c, double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t rows,
              int64_t cols, cudaStream_t s = nullptr);
void release_staging(Ctx& c);
// The same for interleaved complex host rows (std::complex<double>) <-> planar device rows
// (the C++ carrier's layout, converted inside the staging pass).
void h2d_rows_split(Ctx& c, double* dre, double* dim, int64_t dpitch, const double* src_c, int64_t rows,
                    int64_t cols, bool* any_im);
// (dpitch: complex elements between host rows)
void d2h_rows_merge(Ctx& c, double* dst_c, int64_t dpitch, const double* sre, const double* sim, int64_t spitch,
                    int64_t rows, int64_t cols, cudaStream_t s = nullptr);

// Full-spectrum problem (ipt_full.cu)
struct FullProblem;
// delta_c (nullable): Delta as interleaved complex rows (std::complex<double>, n x n);
// delta_re / delta_im are then ignored and the path (real / complex) follows its contents.
FullProblem* full_upload(Ctx& c, int64_t n, const double* d_re, const double* d_im,
                         const double* delta_re, const double* delta_im, bool force_complex = false,
                         int64_t col_begin = -1, int64_t col_end = -1, const double* delta_c = nullptr);
// Z (row-major, interleaved complex, n x n) and the eigenvalues (interleaved, n) on rank 0.
void full_download_interleaved(FullProblem& P, double* z_c, double* lam_c);
void full_download_z_interleaved(FullProblem& P, double* z_c);
FullProblem* full_upload_csr(Ctx& c, int64_t n, const double* d, const int64_t* rowptr,
                             const int32_t* cols, const double* vals, int64_t col_begin = -1,
                             int64_t col_end = -1);
void full_download_block(FullProblem& P, double* z_re, double* z_im, double* lam_re, double* lam_im);
bool full_is_sparse(const FullProblem& P);
void full_free(FullProblem* P);
void full_reset(FullProblem& P, const double* warm_re, const double* warm_im, int max_iter_hint,
                bool renormalize = true);
void full_iterate(FullProblem& P, const ipt_params& prm, ipt_stats* stats);
void full_finalize(FullProblem& P, const ipt_params& prm, ipt_stats* stats);
// Takes the closing residual's inputs (K16) while the previous iterate is intact; call it
// before anything reuses the other ping-pong buffer (full_prepare_download).
void full_prepare_closing(FullProblem& P);
void full_download(FullProblem& P, double* z_re, double* z_im, double* lam_re, double* lam_im);
// Single-rank dense problems after full_iterate: Z to the host on ctx.stream2, safe to run
// on another host thread while full_finalize uses ctx.stream (both only read Z).
bool full_can_download_early(const FullProblem& P);
int64_t full_n(const FullProblem& P);
void full_prepare_download(FullProblem& P, bool want_re, bool want_im);
void full_download_z(FullProblem& P, double* z_re, double* z_im);
void full_release_download(FullProblem& P);
void full_local_columns(const FullProblem& P, int64_t* c0, int64_t* c1);
void full_set_product(FullProblem& P, int product);
int full_ozaki_moduli(FullProblem& P);
bool full_is_complex(const FullProblem& P);
void full_run_maps(FullProblem& P, int count, double* ms_total, double* ms_gemm);

// Closing residual of a converged real dense full-spectrum solve from the last map and
// an INT8 tensor-core correction (ipt_closing.cu, K16): Delta's digits once per problem,
// the last step's digits after the loop (while Z_old is intact), then the residual.
struct ClosingWork {
  DevBuf adig, aexp;           // Delta: arows x 2 kpad int8 ([lo | hi]), int exponent per row
  DevBuf zdig, zexp, wd_old;   // the step D = Z_new - Z_old: mpad x 2 kpad ([hi | lo]), per column
  int64_t n = 0, kpad = 0, arows = 0, ncols = 0, mpad = 0;
  bool delta_ready = false, step_ready = false;
  void delta_digits(cudaStream_t s, const double* A, int64_t lda, int64_t n);
  void step_digits(cudaStream_t s, const double* znew, const double* zold, int64_t ldz, int64_t ncols,
                   const double* wd_old_src);
  // per-CTA partials {sum r^2, 0, 0, 0} of the local columns (closing_partials() of them)
  void residual(cudaStream_t s, const double* znew, int64_t ldz, int64_t col0, const double* wd_new,
                double* partials);
};
int64_t closing_partials();

// Single-pair problem (ipt_single.cu)
struct SingleProblem;
SingleProblem* single_upload(Ctx& c, int64_t n, const double* d_re, const double* d_im, bool csr,
                             const double* dense_re, const double* dense_im, const int64_t* rowptr,
                             const int32_t* cols, const double* val_re, const double* val_im,
                             bool keep_host_anchor_source, bool force_complex = false, int64_t row_begin = -1,
                             int64_t row_end = -1);
void single_debug_peers(SingleProblem& P, int npeers);
// Drop the references to the caller's host arrays kept for anchor uploads (resident
// operators never set an anchor; the arrays may be freed after the upload).
void single_forget_host(SingleProblem& P);
void single_debug_peer_z(SingleProblem& P, int peer, int buf, double* out);
void single_free(SingleProblem* P);
void single_reset(SingleProblem& P, int64_t anchor, const double* warm_re, const double* warm_im,
                  int max_iter_hint, bool renormalize = true);
void single_iterate(SingleProblem& P, const ipt_params& prm, ipt_stats* stats);
void single_finalize(SingleProblem& P, ipt_stats* stats);
void single_download(SingleProblem& P, double* z_re, double* z_im);
void single_matvec(SingleProblem& P, const double* x_re, const double* x_im, double* y_re, double* y_im);
void single_run_steps(SingleProblem& P, int count, double* ms_total, double* ms_map);
void single_accelerated(SingleProblem& P, const ipt_params& prm, int memory, double residual_tol,
                        double regularization, ipt_stats* stats);

// Dense complex LU with partial pivoting (ipt_lu.cu), row-major planar.
struct LuProblem;
LuProblem* lu_factor_device(Ctx& c, int64_t n, const double* a_re, const double* a_im);
LuProblem* lu_from_host(Ctx& c, int64_t n, const double* lu_re, const double* lu_im, const int64_t* perm,
                        bool singular);
void lu_free(LuProblem* F);
int64_t lu_size(const LuProblem& F);
bool lu_singular(const LuProblem& F);
void lu_download(LuProblem& F, double* lu_re, double* lu_im, int64_t* perm);
void lu_solve_device(LuProblem& F, int64_t nrhs, const double* b_re, const double* b_im, double* x_re, double* x_im,
                     bool adjoint);

// tcgen05 INT8 GEMM (i8gemm.cu): C (M x N int32 row-major) = A (M x K) . B (N x K)^T.
void i8_gemm_device(cudaStream_t s, int64_t M, int64_t N, int64_t K, const int8_t* A, const int8_t* B, int32_t* C);

// sigma_min (ipt_sigma.cu): Z column-major (ldz), real or complex (zi nullable).
double sigma_min_device(Ctx& ctx, int64_t n, const double* zr, const double* zi, int64_t ldz,
                        int max_iters, double tol);
double sigma_min_sharded(Ctx& c, int64_t n, int64_t col0, int64_t ncols, const double* zr, const double* zi,
                         int64_t ldz, int max_iters, double tol, bool* ok);

}  // namespace iptb

struct ipt_ctx {
  iptb::Ctx c;
};
