// extern "C" boundary (include/ipt_cuda.h): contexts, NCCL, and the solver /
// kernel entry points. Exceptions never cross this file: every entry point maps
// them to IPT_ERR_* and records the message for ipt_last_error().
#include <cfloat>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <memory>
#include <string>
#include <vector>

#include "dmma_gemm.cuh"
#include "ozaki.cuh"
#include "ipt_internal.cuh"

using namespace iptb;

namespace {
thread_local std::string g_last_error;

// IPT_PROFILE=1: host wall time of each phase of an entry point, on stderr.
struct HostPhases {
  const char* name;
  bool on;
  double t0, last;
  std::string line;
  static double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  explicit HostPhases(const char* n) : name(n), on(std::getenv("IPT_PROFILE") != nullptr), t0(now()), last(t0) {}
  void mark(const char* what) {
    if (!on) return;
    const double t = now();
    char buf[96];
    std::snprintf(buf, sizeof buf, " %s %.2f", what, 1e3 * (t - last));
    line += buf;
    last = t;
  }
  ~HostPhases() {
    if (on) std::fprintf(stderr, "[ipt] %s ms:%s | total %.2f\n", name, line.c_str(), 1e3 * (now() - t0));
  }
};

// Context of the entry point running on this thread (set by check_ctx): on an error
// its communicator is aborted, so ranks waiting for this one in a collective fail
// instead of hanging (local backend; NCCL ranks time out in NCCL itself).
thread_local Ctx* g_entry_ctx = nullptr;

void abort_entry_comm() {
  if (g_entry_ctx && g_entry_ctx->comm) g_entry_ctx->comm->abort();
}

// Per entry point: the context of this thread, and the stream DevBuf frees are ordered
// after, are reset on the way out.
struct EntryScope {
  EntryScope() {
    g_entry_ctx = nullptr;
    set_release_stream(nullptr);
  }
  ~EntryScope() {
    g_entry_ctx = nullptr;
    set_release_stream(nullptr);
  }
};

template <typename F>
int guarded(F&& f) {
  EntryScope scope;
  try {
    f();
    return IPT_OK;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    abort_entry_comm();
    return IPT_ERR_INVALID;
  } catch (const NcclError& e) {
    g_last_error = e.what();
    abort_entry_comm();
    return IPT_ERR_NCCL;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    abort_entry_comm();
    return IPT_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    abort_entry_comm();
    return IPT_ERR_INTERNAL;
  }
}

ipt_params params_or_default(const ipt_params* p) {
  ipt_params d;
  ipt_default_params(&d);
  return p ? *p : d;
}

void check_ctx(ipt_ctx* ctx) {
  if (ctx == nullptr) throw InvalidArgument("null ipt_ctx");
  g_entry_ctx = &ctx->c;
  set_release_stream(ctx->c.stream);
}

// host row-major (rows x cols) -> device column-major with leading dimension ld (zero-padded dst)
void upload_as_colmajor(Ctx& c, const double* host_rm, int64_t rows, int64_t cols, double* dst, int64_t ld) {
  DevBuf tmp;
  tmp.alloc(size_t(rows) * cols, false);
  h2d_rows(c, tmp.get(), cols, host_rm, cols, rows, cols);
  // row-major rows x cols == column-major cols x rows; transpose to column-major rows x cols
  transpose_to_rowmajor(c.stream, tmp.get(), cols, cols, rows, dst, ld);
  c.sync();
}
bool any_nonzero(const double* p, int64_t count) {
  if (p == nullptr) return false;
  for (int64_t t = 0; t < count; ++t)
    if (p[t] != 0.0) return true;
  return false;
}

// A CSR Delta for the full-spectrum entry points: real -> the sparse device map
// (Z row-major, fused SpMM); complex (or a complex Z forced) -> densified onto the
// dense complex path.
FullProblem* open_full_csr(Ctx& c, int64_t n, const double* d_re, const double* d_im,
                           const int64_t* rowptr, const int32_t* cols, const double* val_re,
                           const double* val_im, bool force_complex) {
  if (n <= 0) throw InvalidArgument("solve_full: empty problem");
  if (!d_re || !rowptr) throw InvalidArgument("solve_full: null input");
  const int64_t b = rowptr[0], nnz = rowptr[n] - rowptr[0];
  if (nnz < 0) throw InvalidArgument("csr: row offsets must be non-decreasing");
  const bool cplx = force_complex || any_nonzero(d_im, n) || any_nonzero(val_im ? val_im + b : nullptr, nnz);
  if (!cplx) return full_upload_csr(c, n, d_re, rowptr, cols, val_re);
  if (nnz > 0 && (!cols || !val_re)) throw InvalidArgument("solve_full: null input");
  std::vector<double> re(size_t(n) * n, 0.0), im(size_t(n) * n, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    if (rowptr[i + 1] < rowptr[i]) throw InvalidArgument("csr: row offsets must be non-decreasing");
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) {
      if (cols[p] < 0 || cols[p] >= n) throw InvalidArgument("csr: column index out of bounds");
      re[size_t(i) * n + cols[p]] = val_re[p];
      if (val_im) im[size_t(i) * n + cols[p]] = val_im[p];
    }
  }
  return full_upload(c, n, d_re, d_im, re.data(), im.data(), /*force_complex=*/true);
}

// One F application to a host Z (apply_map_full, solver.cpp:156-178).
void apply_one_map(FullProblem& P, const double* z_re, const double* z_im, double* f_re, double* f_im) {
  full_reset(P, z_re, z_im, 1, /*renormalize=*/false);
  ipt_params prm;
  ipt_default_params(&prm);
  prm.max_iterations = 1;
  prm.ignore_convergence = 1;
  prm.divergence_threshold = DBL_MAX;
  full_iterate(P, prm, nullptr);
  full_download(P, f_re, f_im, nullptr, nullptr);
}

template <typename Open>
void solve_full_impl(Ctx& c, const ipt_params* params, Open&& open, const double* warm_re,
                     const double* warm_im, double* z_re, double* z_im, double* lam_re, double* lam_im,
                     ipt_stats* stats) {
  const ipt_params prm = params_or_default(params);
  if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
  if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
  if (!(prm.divergence_threshold > 1.0)) throw InvalidArgument("config: divergence_threshold must exceed 1");
  HostPhases ph("ipt_full_solve");
  IPT_CUDA(cudaEventRecord(c.ev[2], c.stream));
  {
    std::unique_ptr<FullProblem, void (*)(FullProblem*)> P(open(), full_free);
    ph.mark("upload");
    full_reset(*P, warm_re, warm_im, prm.max_iterations);
    IPT_CUDA(cudaEventRecord(c.ev[3], c.stream));
    c.sync();
    ph.mark("reset");
    float ms_up = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms_up, c.ev[2], c.ev[3]));
    // First-touch the (large, usually fresh) host result arrays on a host thread while the
    // device iterates, instead of inside the download.
    std::future<void> touch;
    const size_t zbytes = sizeof(double) * size_t(full_n(*P)) * size_t(full_n(*P));
    // (only the rank that writes all of Z: with column-local output each rank writes its
    // own columns into a shared mapping, and touching all of it would be n^2 of page work
    // per rank)
    const bool writes_all = c.nranks == 1 || (c.rank == 0 && prm.output_mode != IPT_OUTPUT_LOCAL_COLUMNS);
    if ((z_re || z_im) && writes_all && zbytes >= (size_t(256) << 20))
      touch = std::async(std::launch::async, [z_re, z_im, zbytes] {
        if (z_re) prefault_host_async_part(z_re, zbytes);
        if (z_im) prefault_host_async_part(z_im, zbytes);
      });
    try {
      full_iterate(*P, prm, stats);
    } catch (...) {
      if (touch.valid()) touch.wait();
      throw;
    }
    if (touch.valid()) touch.get();
    ph.mark("iterate");
    // Single GPU: Z goes to the host on a second stream / host thread while the closing
    // product and sigma_min run (they only read Z).
    std::future<void> early;
    float ms_thread = 0.f;  // the overlapped download itself (it runs beside the closing product)
    const bool overlap = (z_re || z_im) && full_can_download_early(*P);
    full_prepare_closing(*P);  // (before the download staging reuses the previous iterate's buffer)
    if (overlap) {
      full_prepare_download(*P, z_re != nullptr, z_im != nullptr);
      const int dev = c.device;
      FullProblem* raw = P.get();
      early = std::async(std::launch::async, [raw, dev, z_re, z_im, &ms_thread] {
        IPT_CUDA(cudaSetDevice(dev));
        const auto t0 = std::chrono::steady_clock::now();
        full_download_z(*raw, z_re, z_im);
        ms_thread = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
      });
    }
    try {
      full_finalize(*P, prm, stats);
    } catch (...) {
      if (early.valid()) early.wait();
      throw;
    }
    ph.mark("finalize+sigma");
    float ms_overlapped = 0.f;
    if (overlap) {
      early.get();
      full_release_download(*P);
      ms_overlapped = ms_thread;  // (wall from the start of the download to the join: the closing product)
    }
    IPT_CUDA(cudaEventRecord(c.ev[2], c.stream));
    full_download(*P, overlap ? nullptr : z_re, overlap ? nullptr : z_im, lam_re, lam_im);
    IPT_CUDA(cudaEventRecord(c.ev[3], c.stream));
    c.sync();
    ph.mark("download");
    float ms_down = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms_down, c.ev[2], c.ev[3]));
    if (stats) {
      stats->ms_upload = ms_up;
      // overlapped: host wall time from the end of the loop until Z was on the host
      stats->ms_download = overlap ? ms_down + ms_overlapped : ms_down;
    }
    ph.mark("stats");
    P.reset();
    ph.mark("free");
  }
  ph.mark("release");
}
}  // namespace

extern "C" {

const char* ipt_last_error(void) { return g_last_error.c_str(); }

void ipt_default_params(ipt_params* p) {
  std::memset(p, 0, sizeof(*p));
  p->tolerance = 100.0 * DBL_EPSILON;
  p->max_iterations = 1000;
  p->divergence_threshold = 1e8;
  p->record_trace = 0;
  p->stop_rule = IPT_STOP_REL_FRO;
  p->want_sigma_min = 1;
  p->schedule = IPT_SCHEDULE_PLAIN;
  p->shrink_alpha = 0.9;
  p->ignore_convergence = 0;
  p->product = IPT_PRODUCT_DMMA;
}

int64_t ipt_kernel_launch_count(void) { return g_launches.load(); }
int64_t ipt_guard_violations(void) { return guard_violations(); }

int ipt_fp64_issue_probe(ipt_ctx* ctx, double* tflops) {
  return guarded([&] {
    check_ctx(ctx);
    if (tflops == nullptr) throw InvalidArgument("ipt_fp64_issue_probe: null out");
    DeviceGuard g(ctx->c.device);
    *tflops = fp64_issue_probe_tflops(ctx->c.stream, ctx->c.device);
  });
}
int64_t ipt_guard_checked(void) { return guard_checked(); }
int64_t ipt_guard_selftest(void) {
  int64_t r = -1;
  if (guarded([&] { r = guard_selftest(); }) != IPT_OK) return -1;
  return r;
}

int ipt_device_count(int* count) {
  return guarded([&] {
    if (count == nullptr) throw InvalidArgument("ipt_device_count: null out");
    IPT_CUDA(cudaGetDeviceCount(count));
  });
}

int ipt_ctx_create(int device, ipt_ctx** out) {
  return guarded([&] {
    if (out == nullptr) throw InvalidArgument("ipt_ctx_create: null out");
    int count = 0;
    IPT_CUDA(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw InvalidArgument("ipt_ctx_create: bad device index");
    IPT_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    IPT_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) throw CudaError("libipt_b200 is built for sm_100a (B200); device is sm_" +
                                          std::to_string(prop.major) + std::to_string(prop.minor));
    auto* ctx = new ipt_ctx();
    ctx->c.device = device;
    IPT_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking));
    IPT_CUDA(cudaStreamCreateWithFlags(&ctx->c.stream2, cudaStreamNonBlocking));
    IPT_CUDA(cudaMallocHost(&ctx->c.h_state, sizeof(LoopState)));
    IPT_CUDA(cudaMallocHost(&ctx->c.h_aux, 256));
    for (auto& e : ctx->c.ev) IPT_CUDA(cudaEventCreate(&e));
    *out = ctx;
  });
}

void ipt_ctx_destroy(ipt_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  ctx->c.comm.reset();
  for (auto& e : ctx->c.ev) cudaEventDestroy(e);
  if (ctx->c.h_state) cudaFreeHost(ctx->c.h_state);
  if (ctx->c.h_aux) cudaFreeHost(ctx->c.h_aux);
  release_staging(ctx->c);
  release_cached_device_memory(ctx->c.device);
  if (ctx->c.stream) cudaStreamDestroy(ctx->c.stream);
  if (ctx->c.stream2) cudaStreamDestroy(ctx->c.stream2);
  delete ctx;
}

int ipt_ctx_device(const ipt_ctx* ctx) { return ctx ? ctx->c.device : -1; }

int ipt_nccl_get_unique_id(void* out128) {
  return guarded([&] {
    if (out128 == nullptr) throw InvalidArgument("ipt_nccl_get_unique_id: null out");
    nccl_unique_id(out128);
  });
}

int ipt_ctx_init_comm(ipt_ctx* ctx, const void* unique_id128, int rank, int nranks) {
  return guarded([&] {
    check_ctx(ctx);
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("ipt_ctx_init_comm: bad rank");
    DeviceGuard g(ctx->c.device);
    ctx->c.comm.reset();
    ctx->c.rank = 0;
    ctx->c.nranks = 1;
    ctx->c.comm = make_nccl_comm(unique_id128, rank, nranks, ctx->c.device);
    ctx->c.rank = rank;
    ctx->c.nranks = nranks;
  });
}

struct ipt_local_group {
  std::shared_ptr<iptb::LocalGroup> g;
};

int ipt_local_group_create(int nranks, ipt_local_group** out) {
  return guarded([&] {
    if (out == nullptr) throw InvalidArgument("ipt_local_group_create: null out");
    auto* h = new ipt_local_group();
    h->g = make_local_group(nranks);
    *out = h;
  });
}

void ipt_local_group_destroy(ipt_local_group* group) { delete group; }

int ipt_ctx_init_local_comm(ipt_ctx* ctx, ipt_local_group* group, int rank) {
  return guarded([&] {
    check_ctx(ctx);
    if (group == nullptr) throw InvalidArgument("ipt_ctx_init_local_comm: null group");
    DeviceGuard g(ctx->c.device);
    ctx->c.comm.reset();
    ctx->c.rank = 0;
    ctx->c.nranks = 1;
    ctx->c.comm = make_local_comm(group->g, rank, ctx->c.device);
    ctx->c.rank = rank;
    ctx->c.nranks = ctx->c.comm->nranks;
  });
}

const char* ipt_ctx_comm_kind(const ipt_ctx* ctx) {
  if (ctx == nullptr) return "";
  return ctx->c.comm ? ctx->c.comm->kind() : "none";
}

int ipt_ctx_rank(const ipt_ctx* ctx, int* rank, int* nranks) {
  if (!ctx) return IPT_ERR_INVALID;
  if (rank) *rank = ctx->c.rank;
  if (nranks) *nranks = ctx->c.nranks;
  return IPT_OK;
}

int ipt_ctx_trim(ipt_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    ctx->c.sync();
    release_cached_device_memory(ctx->c.device);
  });
}

int ipt_ctx_synchronize(ipt_ctx* ctx) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    ctx->c.sync();
  });
}

// ------------------------------------------------------------------ full spectrum

int ipt_full_upload(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                    const double* delta_re, const double* delta_im, ipt_full_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    *out = reinterpret_cast<ipt_full_problem*>(full_upload(ctx->c, n, d_re, d_im, delta_re, delta_im));
  });
}

int ipt_full_upload_columns(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                            const double* delta_re, const double* delta_im, int64_t col_begin,
                            int64_t col_end, ipt_full_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (col_begin < 0) throw InvalidArgument("solve_full: bad column block");
    *out = reinterpret_cast<ipt_full_problem*>(
        full_upload(ctx->c, n, d_re, d_im, delta_re, delta_im, false, col_begin, col_end));
  });
}

int ipt_full_upload_csr_columns(ipt_ctx* ctx, int64_t n, const double* d, const int64_t* rowptr,
                                const int32_t* cols, const double* vals, int64_t col_begin, int64_t col_end,
                                ipt_full_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (col_begin < 0) throw InvalidArgument("solve_full: bad column block");
    *out = reinterpret_cast<ipt_full_problem*>(full_upload_csr(ctx->c, n, d, rowptr, cols, vals, col_begin, col_end));
  });
}

int ipt_full_download_block(ipt_ctx* ctx, ipt_full_problem* prob, double* z_re, double* z_im, double* lam_re,
                            double* lam_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    full_download_block(*reinterpret_cast<FullProblem*>(prob), z_re, z_im, lam_re, lam_im);
  });
}

int ipt_full_reset(ipt_ctx* ctx, ipt_full_problem* prob, const double* warm_re, const double* warm_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    full_reset(*reinterpret_cast<FullProblem*>(prob), warm_re, warm_im, 1000);
  });
}

int ipt_full_iterate(ipt_ctx* ctx, ipt_full_problem* prob, const ipt_params* params, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    full_iterate(*reinterpret_cast<FullProblem*>(prob), params_or_default(params), stats);
  });
}

int ipt_full_finalize(ipt_ctx* ctx, ipt_full_problem* prob, const ipt_params* params, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    full_finalize(*reinterpret_cast<FullProblem*>(prob), params_or_default(params), stats);
  });
}

int ipt_full_download(ipt_ctx* ctx, ipt_full_problem* prob, double* z_re, double* z_im, double* lam_re,
                      double* lam_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    full_download(*reinterpret_cast<FullProblem*>(prob), z_re, z_im, lam_re, lam_im);
  });
}

int ipt_full_solve_interleaved_start(ipt_ctx* ctx, int64_t n, const double* d_c, const double* delta_c,
                                     const double* warm_c, const ipt_params* params, ipt_full_problem** out,
                                     ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (out == nullptr || n <= 0 || d_c == nullptr || delta_c == nullptr) throw InvalidArgument("solve_full: null input");
    const ipt_params prm = params_or_default(params);
    if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
    if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
    if (!(prm.divergence_threshold > 1.0)) throw InvalidArgument("config: divergence_threshold must exceed 1");
    Ctx& c = ctx->c;
    IPT_CUDA(cudaEventRecord(c.ev[2], c.stream));
    std::vector<double> dre(n), dim(n);
    for (int64_t i = 0; i < n; ++i) {
      dre[i] = d_c[2 * i];
      dim[i] = d_c[2 * i + 1];
    }
    // a complex warm start makes the problem complex (solver.cpp:188-201 works in complex)
    std::vector<double> wre, wim;
    bool warm_cplx = false;
    if (warm_c) {
      wre.resize(size_t(n) * n);
      wim.resize(size_t(n) * n);
      for (int64_t t = 0; t < n * n; ++t) {
        wre[t] = warm_c[2 * t];
        wim[t] = warm_c[2 * t + 1];
        warm_cplx = warm_cplx || wim[t] != 0.0;
      }
    }
    std::unique_ptr<FullProblem, void (*)(FullProblem*)> P(
        full_upload(c, n, dre.data(), dim.data(), nullptr, nullptr, warm_cplx, -1, -1, delta_c), full_free);
    full_reset(*P, warm_c ? wre.data() : nullptr, warm_c && warm_cplx ? wim.data() : nullptr, prm.max_iterations);
    IPT_CUDA(cudaEventRecord(c.ev[3], c.stream));
    c.sync();
    float ms_up = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms_up, c.ev[2], c.ev[3]));
    full_iterate(*P, prm, stats);
    if (stats) stats->ms_upload = ms_up;
    *out = reinterpret_cast<ipt_full_problem*>(P.release());
  });
}

int ipt_full_solve_interleaved_finish(ipt_ctx* ctx, ipt_full_problem* prob, const ipt_params* params, double* z_c,
                                      double* lam_c, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (prob == nullptr) throw InvalidArgument("solve_full: null problem");
    const ipt_params prm = params_or_default(params);
    Ctx& c = ctx->c;
    FullProblem& P = *reinterpret_cast<FullProblem*>(prob);
    // one GPU: Z goes to the host on the second stream while the closing product and
    // sigma_min run (both only read Z)
    const bool overlap = z_c && full_can_download_early(P);
    std::future<void> early;
    float ms_thread = 0.f;
    full_prepare_closing(P);  // (before the download staging reuses the previous iterate's buffer)
    if (overlap) {
      full_prepare_download(P, true, full_is_complex(P));
      const int dev = c.device;
      early = std::async(std::launch::async, [&P, dev, z_c, &ms_thread] {
        IPT_CUDA(cudaSetDevice(dev));
        const auto t0 = std::chrono::steady_clock::now();
        full_download_z_interleaved(P, z_c);
        ms_thread = std::chrono::duration<float, std::milli>(std::chrono::steady_clock::now() - t0).count();
      });
    }
    try {
      full_finalize(P, prm, stats);
    } catch (...) {
      if (early.valid()) early.wait();
      throw;
    }
    if (overlap) {
      early.get();
      full_release_download(P);
    }
    IPT_CUDA(cudaEventRecord(c.ev[2], c.stream));
    full_download_interleaved(P, overlap ? nullptr : z_c, lam_c);
    IPT_CUDA(cudaEventRecord(c.ev[3], c.stream));
    c.sync();
    float ms_down = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms_down, c.ev[2], c.ev[3]));
    if (stats) stats->ms_download = overlap ? ms_down + ms_thread : ms_down;
  });
}

int ipt_full_set_product(ipt_full_problem* prob, int32_t product) {
  if (!prob || (product != IPT_PRODUCT_DMMA && product != IPT_PRODUCT_OZAKI)) return IPT_ERR_INVALID;
  full_set_product(*reinterpret_cast<FullProblem*>(prob), product);
  return IPT_OK;
}

int ipt_full_ozaki_moduli(ipt_full_problem* prob, int32_t* moduli) {
  if (!prob || !moduli) return IPT_ERR_INVALID;
  return guarded([&] { *moduli = full_ozaki_moduli(*reinterpret_cast<FullProblem*>(prob)); });
}

int ipt_full_local_columns(const ipt_full_problem* prob, int64_t* col_begin, int64_t* col_end) {
  if (!prob) return IPT_ERR_INVALID;
  full_local_columns(*reinterpret_cast<const FullProblem*>(prob), col_begin, col_end);
  return IPT_OK;
}

void ipt_full_free(ipt_full_problem* prob) { full_free(reinterpret_cast<FullProblem*>(prob)); }

int ipt_full_solve(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                   const double* delta_re, const double* delta_im, const double* warm_re,
                   const double* warm_im, const ipt_params* params, double* z_re, double* z_im,
                   double* lam_re, double* lam_im, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    // a complex warm start on real data runs the complex map (solve_full works in complex
    // arithmetic throughout, solver.cpp:188-201)
    const bool wc = n > 0 && any_nonzero(warm_im, n * n);
    solve_full_impl(
        ctx->c, params, [&] { return full_upload(ctx->c, n, d_re, d_im, delta_re, delta_im, wc); }, warm_re,
        warm_im, z_re, z_im, lam_re, lam_im, stats);
  });
}

int ipt_full_solve_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                       const int64_t* rowptr, const int32_t* cols, const double* val_re,
                       const double* val_im, const double* warm_re, const double* warm_im,
                       const ipt_params* params, double* z_re, double* z_im, double* lam_re,
                       double* lam_im, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    const bool wc = n > 0 && any_nonzero(warm_im, n * n);
    solve_full_impl(
        ctx->c, params,
        [&] { return open_full_csr(ctx->c, n, d_re, d_im, rowptr, cols, val_re, val_im, wc); }, warm_re,
        warm_im, z_re, z_im, lam_re, lam_im, stats);
  });
}

int ipt_full_upload_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                        const int64_t* rowptr, const int32_t* cols, const double* val_re,
                        const double* val_im, ipt_full_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    *out = reinterpret_cast<ipt_full_problem*>(
        open_full_csr(ctx->c, n, d_re, d_im, rowptr, cols, val_re, val_im, false));
  });
}

int ipt_apply_map_full_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                           const int64_t* rowptr, const int32_t* cols, const double* val_re,
                           const double* val_im, const double* z_re, const double* z_im,
                           double* f_re, double* f_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (ctx->c.nranks != 1) throw InvalidArgument("apply_map_full: single-device context required");
    if (!z_re) throw InvalidArgument("apply_map_full: null Z");
    const bool zc = any_nonzero(z_im, n > 0 ? n * n : 0);
    std::unique_ptr<FullProblem, void (*)(FullProblem*)> P(
        open_full_csr(ctx->c, n, d_re, d_im, rowptr, cols, val_re, val_im, zc), full_free);
    apply_one_map(*P, z_re, z_im, f_re, f_im);
  });
}

int ipt_apply_map_full(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                       const double* delta_re, const double* delta_im, const double* z_re,
                       const double* z_im, double* f_re, double* f_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (ctx->c.nranks != 1) throw InvalidArgument("apply_map_full: single-device context required");
    if (!z_re) throw InvalidArgument("apply_map_full: null Z");
    std::unique_ptr<FullProblem, void (*)(FullProblem*)> P(full_upload(ctx->c, n, d_re, d_im, delta_re, delta_im),
                                                           full_free);
    bool zc = false;
    if (z_im) for (int64_t t = 0; t < n * n && !zc; ++t) zc = z_im[t] != 0.0;
    if (zc && !full_is_complex(*P)) {
      // a complex Z on a real Delta: re-upload on the complex path
      P.reset(full_upload(ctx->c, n, d_re, d_im, delta_re, delta_im, /*force_complex=*/true));
    }
    apply_one_map(*P, z_re, z_im, f_re, f_im);
  });
}

// ------------------------------------------------------------------ tcgen05 INT8 GEMM

int ipt_i8_gemm(ipt_ctx* ctx, int64_t M, int64_t N, int64_t K, const int8_t* A, const int8_t* B, int32_t* C,
                int32_t iters, double* ms_per_gemm) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    Ctx& c = ctx->c;
    if (!A || !B) throw InvalidArgument("i8 gemm: null input");
    DevBuf dA, dB, dC;  // byte buffers carried in double-sized DevBufs
    dA.alloc(size_t(ceil_div(M * K, 8)), false);
    dB.alloc(size_t(ceil_div(N * K, 8)), false);
    dC.alloc(size_t(ceil_div(M * N * 4, 8)), false);
    IPT_CUDA(cudaMemcpyAsync(dA.get(), A, size_t(M) * K, cudaMemcpyHostToDevice, c.stream));
    IPT_CUDA(cudaMemcpyAsync(dB.get(), B, size_t(N) * K, cudaMemcpyHostToDevice, c.stream));
    auto* a8 = reinterpret_cast<const int8_t*>(dA.get());
    auto* b8 = reinterpret_cast<const int8_t*>(dB.get());
    auto* c32 = reinterpret_cast<int32_t*>(dC.get());
    i8_gemm_device(c.stream, M, N, K, a8, b8, c32);
    c.sync();
    if (iters > 0 && ms_per_gemm) {
      IPT_CUDA(cudaEventRecord(c.ev[0], c.stream));
      for (int i = 0; i < iters; ++i) i8_gemm_device(c.stream, M, N, K, a8, b8, c32);
      IPT_CUDA(cudaEventRecord(c.ev[1], c.stream));
      c.sync();
      float ms = 0.f;
      IPT_CUDA(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
      *ms_per_gemm = ms / iters;
    }
    if (C) IPT_CUDA(cudaMemcpy(C, dC.get(), size_t(M) * N * 4, cudaMemcpyDeviceToHost));
  });
}

int ipt_ozaki_dgemm(ipt_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, const double* B, double* C,
                    int32_t iters, double* ms_per_gemm) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    Ctx& c = ctx->c;
    if (M < 0 || N < 0 || K < 0) throw InvalidArgument("ozaki dgemm: negative size");
    if ((M * K > 0 && !A) || (N * K > 0 && !B) || (M * N > 0 && !C)) throw InvalidArgument("ozaki dgemm: null buffer");
    if (M == 0 || N == 0) return;
    DevBuf dA, dB, dC, part;
    dA.alloc(size_t(std::max<int64_t>(M * K, 1)), false);
    dB.alloc(size_t(std::max<int64_t>(N * K, 1)), false);
    dC.alloc(size_t(M * N), false);
    if (K > 0) {
      h2d_rows(c, dA.get(), K, A, K, M, K);
      h2d_rows(c, dB.get(), K, B, K, N, K);
    }
    ozaki_dgemm_device(c.stream, M, N, K, dA.get(), dB.get(), dC.get(), part);
    if (iters > 0 && ms_per_gemm) {
      IPT_CUDA(cudaEventRecord(c.ev[0], c.stream));
      for (int i = 0; i < iters; ++i) ozaki_dgemm_device(c.stream, M, N, K, dA.get(), dB.get(), dC.get(), part);
      IPT_CUDA(cudaEventRecord(c.ev[1], c.stream));
      c.sync();
      float ms = 0.f;
      IPT_CUDA(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
      *ms_per_gemm = ms / iters;
    }
    d2h_rows(c, C, N, dC.get(), N, M, N);
  });
}

// ------------------------------------------------------------------ dense LU

int ipt_lu_factor(ipt_ctx* ctx, int64_t n, const double* a_re, const double* a_im, ipt_lu** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (!out) throw InvalidArgument("lu_factor: null out");
    *out = reinterpret_cast<ipt_lu*>(lu_factor_device(ctx->c, n, a_re, a_im));
  });
}

int ipt_lu_from_host(ipt_ctx* ctx, int64_t n, const double* lu_re, const double* lu_im, const int64_t* perm,
                     int singular, ipt_lu** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (!out) throw InvalidArgument("lu: null out");
    *out = reinterpret_cast<ipt_lu*>(lu_from_host(ctx->c, n, lu_re, lu_im, perm, singular != 0));
  });
}

int ipt_lu_info(const ipt_lu* lu, int64_t* n, int* singular) {
  if (!lu) return IPT_ERR_INVALID;
  const LuProblem& F = *reinterpret_cast<const LuProblem*>(lu);
  if (n) *n = lu_size(F);
  if (singular) *singular = lu_singular(F) ? 1 : 0;
  return IPT_OK;
}

int ipt_lu_download(ipt_ctx* ctx, ipt_lu* lu, double* lu_re, double* lu_im, int64_t* perm) {
  return guarded([&] {
    check_ctx(ctx);
    if (!lu) throw InvalidArgument("lu: null factors");
    DeviceGuard g(ctx->c.device);
    lu_download(*reinterpret_cast<LuProblem*>(lu), lu_re, lu_im, perm);
  });
}

int ipt_lu_solve(ipt_ctx* ctx, ipt_lu* lu, int64_t nrhs, const double* b_re, const double* b_im, double* x_re,
                 double* x_im) {
  return guarded([&] {
    check_ctx(ctx);
    if (!lu) throw InvalidArgument("lu_solve: null factors");
    DeviceGuard g(ctx->c.device);
    lu_solve_device(*reinterpret_cast<LuProblem*>(lu), nrhs, b_re, b_im, x_re, x_im, false);
  });
}

int ipt_lu_solve_adjoint(ipt_ctx* ctx, ipt_lu* lu, int64_t nrhs, const double* b_re, const double* b_im,
                         double* x_re, double* x_im) {
  return guarded([&] {
    check_ctx(ctx);
    if (!lu) throw InvalidArgument("lu_solve_adjoint: null factors");
    DeviceGuard g(ctx->c.device);
    lu_solve_device(*reinterpret_cast<LuProblem*>(lu), nrhs, b_re, b_im, x_re, x_im, true);
  });
}

void ipt_lu_free(ipt_lu* lu) { lu_free(reinterpret_cast<LuProblem*>(lu)); }

int ipt_sigma_min(ipt_ctx* ctx, int64_t n, const double* z_re, const double* z_im, int32_t max_iters,
                  double tol, double* out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (n <= 0) throw InvalidArgument("smallest_singular_value_estimate: square input required");
    Ctx& c = ctx->c;
    bool cplx = false;
    if (z_im) for (int64_t t = 0; t < n * n && !cplx; ++t) cplx = z_im[t] != 0.0;
    const int64_t ld = round_up(n, 16);
    const int64_t ldz = cplx ? 2 * ld : ld;
    DevBuf Z;
    Z.alloc(size_t(round_up(n, kBN)) * ldz);
    upload_as_colmajor(c, z_re, n, n, Z.get(), ldz);
    if (cplx) upload_as_colmajor(c, z_im, n, n, Z.get() + ld, ldz);
    *out = sigma_min_device(c, n, Z.get(), cplx ? Z.get() + ld : nullptr, ldz, max_iters, tol);
  });
}

// ------------------------------------------------------------------ single pair

static SingleProblem* as_single(ipt_single_problem* p) { return reinterpret_cast<SingleProblem*>(p); }

int ipt_single_upload_dense(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                            const double* delta_re, const double* delta_im, ipt_single_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    *out = reinterpret_cast<ipt_single_problem*>(single_upload(ctx->c, n, d_re, d_im, false, delta_re,
                                                               delta_im, nullptr, nullptr, nullptr,
                                                               nullptr, true));
  });
}

int ipt_single_upload_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                          const int64_t* rowptr, const int32_t* cols, const double* val_re,
                          const double* val_im, ipt_single_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    *out = reinterpret_cast<ipt_single_problem*>(single_upload(ctx->c, n, d_re, d_im, true, nullptr,
                                                               nullptr, rowptr, cols, val_re, val_im,
                                                               false));
  });
}

int ipt_single_upload_csr_shared(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                                 const int64_t* rowptr, const int32_t* cols, const double* val_re,
                                 const double* val_im, ipt_single_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    *out = reinterpret_cast<ipt_single_problem*>(single_upload(ctx->c, n, d_re, d_im, true, nullptr,
                                                               nullptr, rowptr, cols, val_re, val_im,
                                                               true));
  });
}

int ipt_single_upload_dense_rows(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                                 const double* delta_re, const double* delta_im, int64_t row_begin,
                                 int64_t row_end, ipt_single_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (row_begin < 0) throw InvalidArgument("solve_single: bad row block");
    *out = reinterpret_cast<ipt_single_problem*>(single_upload(ctx->c, n, d_re, d_im, false, delta_re, delta_im,
                                                               nullptr, nullptr, nullptr, nullptr, true, false,
                                                               row_begin, row_end));
  });
}

int ipt_single_upload_csr_rows(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                               const int64_t* rowptr, const int32_t* cols, const double* val_re,
                               const double* val_im, int64_t row_begin, int64_t row_end,
                               ipt_single_problem** out) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (row_begin < 0) throw InvalidArgument("solve_single: bad row block");
    *out = reinterpret_cast<ipt_single_problem*>(single_upload(ctx->c, n, d_re, d_im, true, nullptr, nullptr,
                                                               rowptr, cols, val_re, val_im, false, false,
                                                               row_begin, row_end));
  });
}

int ipt_single_reset(ipt_ctx* ctx, ipt_single_problem* prob, int64_t anchor, const double* warm_re,
                     const double* warm_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    single_reset(*as_single(prob), anchor, warm_re, warm_im, 1000);
  });
}

int ipt_single_iterate(ipt_ctx* ctx, ipt_single_problem* prob, const ipt_params* params, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    single_iterate(*as_single(prob), params_or_default(params), stats);
  });
}

int ipt_single_finalize(ipt_ctx* ctx, ipt_single_problem* prob, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    single_finalize(*as_single(prob), stats);
  });
}

int ipt_single_download(ipt_ctx* ctx, ipt_single_problem* prob, double* z_re, double* z_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    single_download(*as_single(prob), z_re, z_im);
  });
}

void ipt_single_free(ipt_single_problem* prob) { single_free(as_single(prob)); }

static int single_solve_common(ipt_ctx* ctx, SingleProblem* raw, int64_t anchor, const double* warm_re,
                               const double* warm_im, const ipt_params* params, double* z_re,
                               double* z_im, ipt_stats* stats) {
  std::unique_ptr<SingleProblem, void (*)(SingleProblem*)> P(raw, single_free);
  const ipt_params prm = params_or_default(params);
  HostPhases ph("single_solve");
  single_reset(*P, anchor, prm.schedule == IPT_SCHEDULE_CONTINUATION ? nullptr : warm_re,
               prm.schedule == IPT_SCHEDULE_CONTINUATION ? nullptr : warm_im, prm.max_iterations);
  ph.mark("reset");
  single_iterate(*P, prm, stats);
  ph.mark("iterate");
  single_finalize(*P, stats);
  ph.mark("finalize");
  single_download(*P, z_re, z_im);
  ph.mark("download");
  (void)ctx;
  return IPT_OK;
}

int ipt_single_solve_dense(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                           const double* delta_re, const double* delta_im, int64_t anchor,
                           const double* warm_re, const double* warm_im, const ipt_params* params,
                           double* z_re, double* z_im, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    const ipt_params prm = params_or_default(params);
    if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
    if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
    if (anchor < 0 || anchor >= n) throw InvalidArgument("solver: anchor out of range");
    const bool wc = prm.schedule != IPT_SCHEDULE_CONTINUATION && any_nonzero(warm_im, n);
    single_solve_common(ctx, single_upload(ctx->c, n, d_re, d_im, false, delta_re, delta_im, nullptr,
                                           nullptr, nullptr, nullptr, true, wc),
                        anchor, warm_re, warm_im, params, z_re, z_im, stats);
  });
}

int ipt_single_solve_csr(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                         const int64_t* rowptr, const int32_t* cols, const double* val_re,
                         const double* val_im, int64_t anchor, const double* warm_re,
                         const double* warm_im, const ipt_params* params, double* z_re, double* z_im,
                         ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    const ipt_params prm = params_or_default(params);
    if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
    if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
    if (anchor < 0 || anchor >= n) throw InvalidArgument("solver: anchor out of range");
    const bool wc = prm.schedule != IPT_SCHEDULE_CONTINUATION && any_nonzero(warm_im, n);
    HostPhases ph("ipt_single_solve_csr");
    single_solve_common(ctx, single_upload(ctx->c, n, d_re, d_im, true, nullptr, nullptr, rowptr, cols,
                                           val_re, val_im, true, wc),
                        anchor, warm_re, warm_im, params, z_re, z_im, stats);
  });
}

static int accelerated_common(ipt_ctx* ctx, SingleProblem* raw, int64_t anchor, const ipt_params* params,
                              int32_t memory, double residual_tol, double* z, ipt_stats* stats) {
  std::unique_ptr<SingleProblem, void (*)(SingleProblem*)> P(raw, single_free);
  const ipt_params prm = params_or_default(params);
  single_reset(*P, anchor, nullptr, nullptr, prm.max_iterations);
  single_accelerated(*P, prm, memory, residual_tol, 0.0, stats);
  single_download(*P, z, nullptr);
  (void)ctx;
  return IPT_OK;
}

int ipt_single_solve_accelerated_dense(ipt_ctx* ctx, int64_t n, const double* d, const double* delta,
                                       int64_t anchor, const ipt_params* params, int32_t memory,
                                       double residual_tol, double* z, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (anchor < 0 || anchor >= n) throw InvalidArgument("solver: anchor out of range");
    accelerated_common(ctx, single_upload(ctx->c, n, d, nullptr, false, delta, nullptr, nullptr, nullptr, nullptr,
                                          nullptr, true),
                       anchor, params, memory, residual_tol, z, stats);
  });
}

int ipt_single_solve_accelerated_csr(ipt_ctx* ctx, int64_t n, const double* d, const int64_t* rowptr,
                                     const int32_t* cols, const double* vals, int64_t anchor,
                                     const ipt_params* params, int32_t memory, double residual_tol,
                                     double* z, ipt_stats* stats) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (anchor < 0 || anchor >= n) throw InvalidArgument("solver: anchor out of range");
    accelerated_common(ctx, single_upload(ctx->c, n, d, nullptr, true, nullptr, nullptr, rowptr, cols, vals,
                                          nullptr, true),
                       anchor, params, memory, residual_tol, z, stats);
  });
}

int ipt_apply_map_single_dense(ipt_ctx* ctx, int64_t n, const double* d_re, const double* d_im,
                               const double* delta_re, const double* delta_im, int64_t anchor,
                               const double* z_re, const double* z_im, double* f_re, double* f_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (anchor < 0 || anchor >= n) throw InvalidArgument("solver: anchor out of range");
    bool zc = false;
    if (z_im) for (int64_t t = 0; t < n && !zc; ++t) zc = z_im[t] != 0.0;
    std::unique_ptr<SingleProblem, void (*)(SingleProblem*)> P(
        single_upload(ctx->c, n, d_re, d_im, false, delta_re, delta_im, nullptr, nullptr, nullptr, nullptr,
                      true, /*force_complex=*/zc),
        single_free);
    single_reset(*P, anchor, z_re, z_im, 1, /*renormalize=*/false);
    ipt_params prm;
    ipt_default_params(&prm);
    prm.max_iterations = 1;
    prm.ignore_convergence = 1;
    prm.divergence_threshold = DBL_MAX;
    single_iterate(*P, prm, nullptr);
    single_download(*P, f_re, f_im);
  });
}

int ipt_full_run_maps(ipt_ctx* ctx, ipt_full_problem* prob, int32_t count, double* ms_total,
                      double* ms_dominant) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (count < 0) throw InvalidArgument("run_maps: negative count");
    full_run_maps(*reinterpret_cast<FullProblem*>(prob), count, ms_total, ms_dominant);
  });
}

int ipt_single_debug_peers(ipt_single_problem* prob, int32_t npeers) {
  if (!prob) return IPT_ERR_INVALID;
  return guarded([&] { single_debug_peers(*reinterpret_cast<SingleProblem*>(prob), npeers); });
}

int ipt_single_debug_peer_z(ipt_single_problem* prob, int32_t peer, int32_t buf, double* out) {
  if (!prob || !out) return IPT_ERR_INVALID;
  return guarded([&] { single_debug_peer_z(*reinterpret_cast<SingleProblem*>(prob), peer, buf, out); });
}

int ipt_single_run_steps(ipt_ctx* ctx, ipt_single_problem* prob, int32_t count, double* ms_total,
                         double* ms_dominant) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (count < 0) throw InvalidArgument("run_steps: negative count");
    single_run_steps(*as_single(prob), count, ms_total, ms_dominant);
  });
}

// ------------------------------------------------------------------ kernels::

}  // extern "C"

namespace {

// The left factor of kernels::matmul in the DMMA kernel's layouts, uploaded once:
//   real A    : R = A (mpad x ldk, rows zero-padded to the 128-row tile, K to 16)
//   complex A : S = [Ar; Ai] (2m rows) for a real right factor (one 2m x n GEMM), and,
//               built on the device at the first complex right factor, [Ar | -Ai] and
//               [Ai | Ar] (K = 2 ldk) for Cr = Ar Br - Ai Bi, Ci = Ai Br + Ar Bi.
struct GemmOperand {
  int64_t m = 0, k = 0, ldk = 0;
  bool cplx = false;
  DevBuf S, Acat, A2cat;
  void upload(Ctx& c, int64_t m_, int64_t k_, const double* a_re, const double* a_im) {
    m = m_;
    k = k_;
    ldk = round_up(std::max<int64_t>(k, 1), 16);
    cplx = any_nonzero(a_im, m * k);
    S.alloc(size_t(round_up(cplx ? 2 * m : m, kBM)) * ldk);
    if (k > 0) {
      h2d_rows(c, S.get(), ldk, a_re, k, m, k);  // pinned, double-buffered
      if (cplx) h2d_rows(c, S.get() + m * ldk, ldk, a_im, k, m, k);
    }
  }
  void build_cat(Ctx& c) {
    if (Acat.count) return;
    cudaStream_t s = c.stream;
    const int64_t K = 2 * ldk, mpad = round_up(m, kBM);
    Acat.alloc(size_t(mpad) * K);
    A2cat.alloc(size_t(mpad) * K);
    const double* ar = S.get();
    const double* ai = S.get() + m * ldk;
    auto put = [&](double* dst, const double* src) {
      IPT_CUDA(cudaMemcpy2DAsync(dst, K * sizeof(double), src, ldk * sizeof(double), ldk * sizeof(double), m,
                                 cudaMemcpyDeviceToDevice, s));
    };
    put(Acat.get(), ar);
    put(A2cat.get(), ai);
    put(A2cat.get() + ldk, ar);
    DevBuf neg;
    neg.alloc(size_t(m) * ldk, false);
    scale_copy(s, ai, neg.get(), size_t(m) * ldk, -1.0);
    put(Acat.get() + ldk, neg.get());
    c.sync();
  }
  // C (m x n, row-major planar) = A B, B (k x n row-major planar, b_im nullable)
  void apply(Ctx& c, int64_t n, const double* b_re, const double* b_im, double* c_re, double* c_im) {
    cudaStream_t s = c.stream;
    if (m == 0 || n == 0) return;
    const bool b_cplx = any_nonzero(b_im, k * n);
    auto up_cols = [&](double* dst, int64_t ld, const double* src) {  // k x n -> column-major
      if (k > 0) upload_as_colmajor(c, src, k, n, dst, ld);
    };
    DevBuf B, C, rm;
    rm.alloc(size_t(m) * n, false);
    auto download = [&](const double* src, int64_t ldc, double* dst) {
      transpose_to_rowmajor(s, src, ldc, m, n, rm.get(), n);
      d2h_rows(c, dst, n, rm.get(), n, m, n);
    };
    if (!cplx && !b_cplx) {  // one real GEMM
      B.alloc(size_t(round_up(n, kBN)) * ldk);
      up_cols(B.get(), ldk, b_re);
      C.alloc(size_t(n) * m, false);
      gemm_tn_store(s, m, n, ldk, S.get(), ldk, B.get(), ldk, C.get(), m);
      download(C.get(), m, c_re);
      if (c_im) std::memset(c_im, 0, sizeof(double) * m * n);
    } else if (!cplx) {  // real A: A [Br | Bi] as one m x 2n real GEMM
      B.alloc(size_t(round_up(2 * n, kBN)) * ldk);
      up_cols(B.get(), ldk, b_re);
      up_cols(B.get() + n * ldk, ldk, b_im);
      C.alloc(size_t(2 * n) * m, false);
      gemm_tn_store(s, m, 2 * n, ldk, S.get(), ldk, B.get(), ldk, C.get(), m);
      download(C.get(), m, c_re);
      if (c_im) download(C.get() + n * m, m, c_im);
    } else if (!b_cplx) {  // real B: [Ar; Ai] B as one 2m x n real GEMM
      B.alloc(size_t(round_up(n, kBN)) * ldk);
      up_cols(B.get(), ldk, b_re);
      C.alloc(size_t(n) * 2 * m, false);
      gemm_tn_store(s, 2 * m, n, ldk, S.get(), ldk, B.get(), ldk, C.get(), 2 * m);
      download(C.get(), 2 * m, c_re);
      if (c_im) download(C.get() + m, 2 * m, c_im);
    } else {  // both complex: [Ar | -Ai][Br; Bi] and [Ai | Ar][Br; Bi] (K = 2 ldk)
      build_cat(c);
      const int64_t K = 2 * ldk;
      B.alloc(size_t(round_up(n, kBN)) * K);
      up_cols(B.get(), K, b_re);
      up_cols(B.get() + ldk, K, b_im);
      C.alloc(size_t(n) * m, false);
      gemm_tn_store(s, m, n, K, Acat.get(), K, B.get(), K, C.get(), m);
      download(C.get(), m, c_re);
      if (c_im) {
        gemm_tn_store(s, m, n, K, A2cat.get(), K, B.get(), K, C.get(), m);
        download(C.get(), m, c_im);
      }
    }
  }
};

}  // namespace

struct ipt_gemm_operand {
  GemmOperand A;
  ipt_ctx* ctx = nullptr;
  int device = 0;
};

extern "C" {

int ipt_gemm(ipt_ctx* ctx, int64_t m, int64_t k, int64_t n, const double* a_re, const double* a_im,
             const double* b_re, const double* b_im, double* c_re, double* c_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (m < 0 || k < 0 || n < 0) throw InvalidArgument("matmul: negative shape");
    if (m == 0 || n == 0) return;
    GemmOperand A;
    A.upload(ctx->c, m, k, a_re, a_im);
    A.apply(ctx->c, n, b_re, b_im, c_re, c_im);
  });
}

int ipt_gemm_operand_create(ipt_ctx* ctx, int64_t m, int64_t k, const double* a_re, const double* a_im,
                            ipt_gemm_operand** out) {
  return guarded([&] {
    check_ctx(ctx);
    if (out == nullptr || m <= 0 || k < 0 || a_re == nullptr) throw InvalidArgument("gemm operand: bad arguments");
    DeviceGuard g(ctx->c.device);
    auto h = std::make_unique<ipt_gemm_operand>();
    h->A.upload(ctx->c, m, k, a_re, a_im);
    h->ctx = ctx;
    h->device = ctx->c.device;
    *out = h.release();
  });
}

int ipt_gemm_operand_apply(ipt_ctx* ctx, ipt_gemm_operand* a, int64_t n, const double* b_re, const double* b_im,
                           double* c_re, double* c_im) {
  return guarded([&] {
    check_ctx(ctx);
    if (a == nullptr || a->ctx != ctx) throw InvalidArgument("gemm operand: belongs to another context");
    if (n < 0) throw InvalidArgument("matmul: negative shape");
    DeviceGuard g(ctx->c.device);
    a->A.apply(ctx->c, n, b_re, b_im, c_re, c_im);
  });
}

void ipt_gemm_operand_free(ipt_gemm_operand* a) {
  if (!a) return;
  DeviceGuard g(a->device);
  delete a;
}

int ipt_matvec_dense(ipt_ctx* ctx, int64_t m, int64_t n, const double* a_re, const double* a_im,
                     const double* x_re, const double* x_im, double* y_re, double* y_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (m != n) {  // rectangular: one-column product
      const int rc = ipt_gemm(ctx, m, n, 1, a_re, a_im, x_re, x_im, y_re, y_im);
      if (rc != IPT_OK) throw CudaError(g_last_error);
      return;
    }
    std::vector<double> dz(size_t(std::max<int64_t>(n, 1)), 0.0);
    std::unique_ptr<SingleProblem, void (*)(SingleProblem*)> P(
        single_upload(ctx->c, n, dz.data(), nullptr, false, a_re, a_im, nullptr, nullptr, nullptr, nullptr, true),
        single_free);
    single_matvec(*P, x_re, x_im, y_re, y_im);
  });
}

int ipt_matvec_csr(ipt_ctx* ctx, int64_t m, int64_t n, const int64_t* rowptr, const int32_t* cols,
                   const double* val_re, const double* val_im, const double* x_re, const double* x_im,
                   double* y_re, double* y_im) {
  return guarded([&] {
    check_ctx(ctx);
    DeviceGuard g(ctx->c.device);
    if (m != n) throw InvalidArgument("matvec_csr: square operator required");
    std::vector<double> dz(size_t(std::max<int64_t>(n, 1)), 0.0);
    std::unique_ptr<SingleProblem, void (*)(SingleProblem*)> P(
        single_upload(ctx->c, n, dz.data(), nullptr, true, nullptr, nullptr, rowptr, cols, val_re, val_im, true),
        single_free);
    single_matvec(*P, x_re, x_im, y_re, y_im);
  });
}

struct ipt_operator {
  SingleProblem* P = nullptr;
  ipt_ctx* ctx = nullptr;  // the creating context (matvec must use it); free needs only the device
  int device = 0;
  int64_t bytes = 0;
};

int ipt_operator_create_dense(ipt_ctx* ctx, int64_t n, const double* a_re, const double* a_im,
                              ipt_operator** out) {
  return guarded([&] {
    check_ctx(ctx);
    if (out == nullptr || n <= 0 || a_re == nullptr) throw InvalidArgument("operator: bad arguments");
    if (ctx->c.nranks != 1) throw InvalidArgument("operator: single-rank context required");
    DeviceGuard g(ctx->c.device);
    std::vector<double> dz(size_t(n), 0.0);
    auto* op = new ipt_operator();
    op->P = single_upload(ctx->c, n, dz.data(), nullptr, false, a_re, a_im, nullptr, nullptr, nullptr, nullptr, true);
    single_forget_host(*op->P);
    op->ctx = ctx;
    op->device = ctx->c.device;
    op->bytes = int64_t(round_up(n, 16)) * n * (any_nonzero(a_im, n * n) ? 16 : 8);
    *out = op;
  });
}

int ipt_operator_create_csr(ipt_ctx* ctx, int64_t n, const int64_t* rowptr, const int32_t* cols,
                            const double* val_re, const double* val_im, ipt_operator** out) {
  return guarded([&] {
    check_ctx(ctx);
    if (out == nullptr || n <= 0 || rowptr == nullptr) throw InvalidArgument("operator: bad arguments");
    if (ctx->c.nranks != 1) throw InvalidArgument("operator: single-rank context required");
    DeviceGuard g(ctx->c.device);
    std::vector<double> dz(size_t(n), 0.0);
    auto* op = new ipt_operator();
    op->P = single_upload(ctx->c, n, dz.data(), nullptr, true, nullptr, nullptr, rowptr, cols, val_re, val_im, true);
    single_forget_host(*op->P);
    op->ctx = ctx;
    op->device = ctx->c.device;
    const int64_t nnz = rowptr[n] - rowptr[0];
    op->bytes = nnz * (val_im ? 20 : 12) + 8 * (n + 1);
    *out = op;
  });
}

int ipt_operator_matvec(ipt_ctx* ctx, ipt_operator* op, const double* x_re, const double* x_im, double* y_re,
                        double* y_im) {
  return guarded([&] {
    check_ctx(ctx);
    if (op == nullptr || op->ctx != ctx) throw InvalidArgument("operator: belongs to another context");
    DeviceGuard g(ctx->c.device);
    single_matvec(*op->P, x_re, x_im, y_re, y_im);
  });
}

int64_t ipt_operator_bytes(const ipt_operator* op) { return op ? op->bytes : 0; }

void ipt_operator_free(ipt_operator* op) {
  if (!op) return;
  DeviceGuard g(op->device);
  single_free(op->P);
  delete op;
}

}  // extern "C"
