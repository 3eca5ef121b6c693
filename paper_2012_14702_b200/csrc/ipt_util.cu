// Small device utilities: buffers, transposes, deterministic partial reduction.
#include <algorithm>
#include <atomic>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <condition_variable>
#include <functional>
#include <thread>
#include <unordered_map>
#include <vector>

#include "ipt_internal.cuh"

namespace iptb {

std::atomic<int64_t> g_launches{0};

double ProfMarks::now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
ProfMarks::ProfMarks(const char* n) : name(n), on(std::getenv("IPT_PROFILE") != nullptr), last(now()) {}
void ProfMarks::mark(const char* what, bool sync_device) {
  if (!on) return;
  if (sync_device) cudaDeviceSynchronize();
  const double t = now();
  char buf[96];
  std::snprintf(buf, sizeof buf, " %s %.1f", what, 1e3 * (t - last));
  line += buf;
  last = t;
}
ProfMarks::~ProfMarks() {
  if (on) std::fprintf(stderr, "[ipt] %s ms:%s\n", name, line.c_str());
}

// Device buffers come from the stream-ordered pool (cudaMallocAsync on the legacy
// stream) so the many small, short-lived buffers of the kernels:: / apply_map entry
// points do not pay cudaMalloc / cudaFree (a device-wide sync) per call. A buffer is
// freed in stream order after the calling entry point's library stream
// (set_release_stream), so a scratch buffer that goes out of scope while a kernel on
// that stream still reads it is not reused before the kernel completes (this raced
// between ranks sharing one device: the K16 closing residual read its int32 products
// after another rank's allocation had been handed the same memory).
namespace {
void configure_pool_once() {
  static std::mutex mu;
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (dev < 0 || dev >= 64 || done[dev]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    // Keep freed memory mapped for reuse: trimming the pool at every synchronisation
    // unmaps tens of GB after a large solve and the next solve pays to map it again
    // (~1 s per 17 GB measured). The context releases the cache (ipt_ctx_destroy).
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done[dev] = true;
}
}  // namespace

void release_cached_device_memory(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    cudaDeviceSynchronize();
    cudaMemPoolTrimTo(pool, 0);
  }
}

namespace {
thread_local cudaStream_t g_release_stream = nullptr;
}
void set_release_stream(cudaStream_t s) { g_release_stream = s; }

// Guard zones (IPT_GUARD=1; compute-sanitizer is not available on this pool): every pool
// buffer gets kGuardDoubles of a byte pattern before and after it; the release checks
// both zones after a device synchronisation and counts a violation (an out-of-bounds
// write by some kernel near this buffer) in ipt_guard_violations(). Off by default.
namespace {
constexpr size_t kGuardDoubles = 512;  // 4 KB each side
constexpr unsigned char kGuardByte = 0xA5;
bool guard_on() {
  static const bool on = [] {
    const char* e = std::getenv("IPT_GUARD");
    return e && e[0] == '1';
  }();
  return on;
}
std::mutex g_guard_mu;
std::unordered_map<const double*, std::pair<double*, size_t>> g_guard_bufs;  // p -> (base, doubles)
std::atomic<int64_t> g_guard_bad{0};
std::atomic<int64_t> g_guard_checked{0};

bool guard_release(double* p) {
  double* base = nullptr;
  size_t n = 0;
  {
    std::lock_guard<std::mutex> lk(g_guard_mu);
    auto it = g_guard_bufs.find(p);
    if (it == g_guard_bufs.end()) return false;
    base = it->second.first;
    n = it->second.second;
    g_guard_bufs.erase(it);
  }
  cudaDeviceSynchronize();
  std::vector<unsigned char> h(2 * kGuardDoubles * sizeof(double));
  const size_t gb = kGuardDoubles * sizeof(double);
  cudaMemcpy(h.data(), base, gb, cudaMemcpyDeviceToHost);
  cudaMemcpy(h.data() + gb, base + kGuardDoubles + n, gb, cudaMemcpyDeviceToHost);
  g_guard_checked.fetch_add(1);
  for (size_t b = 0; b < h.size(); ++b)
    if (h[b] != kGuardByte) {
      g_guard_bad.fetch_add(1);
      std::fprintf(stderr, "[ipt] guard violation: %s guard of a %zu-double buffer, byte %zu\n",
                   b < gb ? "leading" : "trailing", n, b < gb ? gb - b : b - gb);
      break;
    }
  cudaFree(base);
  return true;
}
}  // namespace

int64_t guard_violations() { return g_guard_bad.load(); }
int64_t guard_checked() { return g_guard_checked.load(); }

namespace {
__global__ void write_past_end_kernel(double* p, int64_t n) { p[n] = 1.0; }
}  // namespace

// Negative control of the guard zones: one write one element past a 100-double buffer.
int64_t guard_selftest() {
  const int64_t before = guard_violations();
  {
    DevBuf b;
    b.alloc(100);
    write_past_end_kernel<<<1, 1>>>(b.get(), 100);
    IPT_CUDA(cudaDeviceSynchronize());
  }
  return guard_violations() - before;
}

void DevBuf::alloc(size_t n, bool zero) {
  release();
  if (n == 0) n = 1;
  configure_pool_once();
  if (guard_on()) {
    double* base = nullptr;
    IPT_CUDA(cudaMalloc(&base, (n + 2 * kGuardDoubles) * sizeof(double)));
    IPT_CUDA(cudaMemset(base, kGuardByte, (n + 2 * kGuardDoubles) * sizeof(double)));
    p = base + kGuardDoubles;
    if (zero) IPT_CUDA(cudaMemset(p, 0, n * sizeof(double)));
    IPT_CUDA(cudaDeviceSynchronize());
    count = n;
    std::lock_guard<std::mutex> lk(g_guard_mu);
    g_guard_bufs[p] = {base, n};
    return;
  }
  IPT_CUDA(cudaMallocAsync(&p, n * sizeof(double), nullptr));
  count = n;
  if (zero) IPT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(double), nullptr));
  // The library stream is non-blocking w.r.t. the legacy stream: the allocation (and the
  // memset) must be complete before any copy or kernel on the library stream uses it.
  IPT_CUDA(cudaStreamSynchronize(nullptr));
}
void DevBuf::alloc_plain(size_t n) {
  release();
  if (n == 0) n = 1;
  IPT_CUDA(cudaMalloc(&p, n * sizeof(double)));
  plain = true;
  count = n;
  IPT_CUDA(cudaMemset(p, 0, n * sizeof(double)));
}
void DevBuf::release() {
  if (p && !plain && guard_on() && guard_release(p)) {
    p = nullptr;
    count = 0;
    return;
  }
  if (p) {
    if (plain) cudaFree(p);
    else cudaFreeAsync(p, g_release_stream);
  }
  p = nullptr;
  plain = false;
  count = 0;
}

// ----------------------------------------------------------- staged transfers

namespace {
constexpr size_t kStageBytes = size_t(64) << 20;  // per buffer

void ensure_staging(Ctx& c) {
  if (c.stage[0]) return;
  for (int b = 0; b < 2; ++b) {
    IPT_CUDA(cudaMallocHost(&c.stage[b], kStageBytes));
    IPT_CUDA(cudaEventCreateWithFlags(&c.stage_ev[b], cudaEventDisableTiming));
  }
  c.stage_doubles = kStageBytes / sizeof(double);
}

unsigned copy_threads() {
  const unsigned h = std::thread::hardware_concurrency();
  return std::max(1u, std::min(16u, h ? h : 8u));
}

// Persistent host workers for the staged copies (a pool instead of std::thread per
// 64 MB chunk: spawning 16 threads per chunk cost ~8 ms per GB moved).
class HostPool {
 public:
  explicit HostPool(unsigned n) {
    for (unsigned i = 1; i < n; ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  unsigned size() const { return static_cast<unsigned>(workers_.size()) + 1; }
  // f(k) for k in [0, parts), the calling thread taking part; returns when all are done.
  // One job at a time (callers serialise on run_mu_).
  void run(unsigned parts, const std::function<void(unsigned)>& f) {
    std::lock_guard<std::mutex> run_lk(run_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      job_ = &f;
      parts_ = parts;
      next_ = 0;
      done_ = 0;
      ++gen_;
    }
    cv_.notify_all();
    work();
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [this] { return done_ == parts_; });
    job_ = nullptr;
  }

 private:
  void work() {
    while (true) {
      unsigned k;
      const std::function<void(unsigned)>* f;
      {
        std::lock_guard<std::mutex> lk(mu_);
        if (job_ == nullptr || next_ >= parts_) return;
        k = next_++;
        f = job_;
      }
      (*f)(k);
      std::lock_guard<std::mutex> lk(mu_);
      if (++done_ == parts_) done_cv_.notify_all();
    }
  }
  void loop() {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || (gen_ != seen && job_ != nullptr); });
        if (stop_) return;
        seen = gen_;
      }
      work();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex mu_, run_mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(unsigned)>* job_ = nullptr;
  unsigned parts_ = 0, next_ = 0, done_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

HostPool& host_pool() {
  static HostPool pool(copy_threads());
  return pool;
}

// rows x cols doubles between two pitched host arrays, split over the host workers (by
// bytes: a contiguous block is one flat range, otherwise whole rows, or column slices of
// the rows when there are fewer rows than workers).
void host_copy_rows(double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  const unsigned t = total >= (int64_t(1) << 18) ? host_pool().size() : 1u;
  if (t <= 1) {
    for (int64_t r = 0; r < rows; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, sizeof(double) * cols);
    return;
  }
  if (dpitch == cols && spitch == cols) {
    const int64_t step = (total + t - 1) / t;
    host_pool().run(t, [&](unsigned k) {
      const int64_t a = int64_t(k) * step, b = std::min(total, a + step);
      if (a < b) std::memcpy(dst + a, src + a, sizeof(double) * (b - a));
    });
    return;
  }
  if (rows >= int64_t(t)) {
    const int64_t step = (rows + t - 1) / t;
    host_pool().run(t, [&](unsigned k) {
      const int64_t a = int64_t(k) * step, b = std::min(rows, a + step);
      for (int64_t r = a; r < b; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, sizeof(double) * cols);
    });
    return;
  }
  const int64_t step = (cols + t - 1) / t;
  host_pool().run(t, [&](unsigned k) {
    const int64_t a = int64_t(k) * step, b = std::min(cols, a + step);
    if (a < b)
      for (int64_t r = 0; r < rows; ++r) std::memcpy(dst + r * dpitch + a, src + r * spitch + a, sizeof(double) * (b - a));
  });
}
// Large host destinations (a fresh n x n result array) are first-touched here in
// parallel: transparent huge pages requested for the range, then every page touched
// by all copy threads at once, so the staged copies below do not take ~2 M
// serialised 4 KB page faults.
std::mutex g_prefault_mu;
std::vector<std::pair<const void*, size_t>> g_prefaulted;  // ranges already first-touched

void prefault_host_destination(double* dst, size_t bytes) {
  if (bytes < (size_t(256) << 20)) return;
  const uintptr_t huge = uintptr_t(2) << 20;
  const uintptr_t b0 = (reinterpret_cast<uintptr_t>(dst) + huge - 1) & ~(huge - 1);
  const uintptr_t b1 = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~(huge - 1);
  if (b1 > b0) madvise(reinterpret_cast<void*>(b0), b1 - b0, MADV_HUGEPAGE);
  const unsigned t = copy_threads();
  const size_t page = 4096;
  const uintptr_t p0 = (reinterpret_cast<uintptr_t>(dst) + page - 1) & ~(page - 1);
  const uintptr_t p1 = (reinterpret_cast<uintptr_t>(dst) + bytes) & ~(page - 1);
  if (p1 <= p0) return;
  const size_t span = ((p1 - p0) / t + huge - 1) & ~(huge - 1);
  // one store per 4 KB page (with THP, one fault per 2 MB); measured faster than
  // MADV_POPULATE_WRITE, which the kernel serialises
  host_pool().run(t, [&](unsigned k) {
    const uintptr_t a = p0 + k * span, b = std::min<uintptr_t>(p1, a + span);
    for (uintptr_t q = a; q < b; q += page) *reinterpret_cast<volatile char*>(q) = 0;
  });
}

}  // namespace

// A result destination can be first-touched on a host thread while the device iterates;
// d2h_rows then skips its own prefault for exactly that range.
void prefault_host_async_part(double* dst, size_t bytes) {
  prefault_host_destination(dst, bytes);
  std::lock_guard<std::mutex> lk(g_prefault_mu);
  g_prefaulted.emplace_back(dst, bytes);
}

bool take_prefaulted(const void* p, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_prefault_mu);
  for (auto it = g_prefaulted.begin(); it != g_prefaulted.end(); ++it)
    if (it->first == p && it->second == bytes) {
      g_prefaulted.erase(it);
      return true;
    }
  return false;
}

void release_staging(Ctx& c) {
  for (int b = 0; b < 2; ++b) {
    if (c.stage[b]) cudaFreeHost(c.stage[b]);
    if (c.stage_ev[b]) cudaEventDestroy(c.stage_ev[b]);
    c.stage[b] = nullptr;
    c.stage_ev[b] = nullptr;
  }
  c.stage_doubles = 0;
}

void h2d_rows(Ctx& c, double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t rows,
              int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  cudaStream_t st = stream ? stream : c.stream;
  ensure_staging(c);
  const int64_t per = std::max<int64_t>(1, static_cast<int64_t>(c.stage_doubles) / cols);
  if (per < 1 || cols > static_cast<int64_t>(c.stage_doubles)) {  // a row larger than a buffer
    IPT_CUDA(cudaMemcpy2DAsync(dst, dpitch * sizeof(double), src, spitch * sizeof(double), cols * sizeof(double),
                               rows, cudaMemcpyHostToDevice, st));
    IPT_CUDA(cudaStreamSynchronize(st));
    return;
  }
  int b = 0;
  bool used[2] = {false, false};
  const bool prof = std::getenv("IPT_PROFILE") != nullptr;
  double t_wait = 0.0, t_copy = 0.0;
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_start = now();
  // a transfer that fits one staging buffer still goes in >= 4 chunks of >= 1 MB, so the
  // host copy of chunk k+1 overlaps the DMA of chunk k
  const int64_t min_rows = std::max<int64_t>(1, (int64_t(1) << 17) / cols);
  const int64_t step = std::max(min_rows, std::min(per, (rows + 3) / 4));
  for (int64_t r0 = 0; r0 < rows; r0 += step, b ^= 1) {
    const int64_t nr = std::min(step, rows - r0);
    double t0 = now();
    if (used[b]) IPT_CUDA(cudaEventSynchronize(c.stage_ev[b]));  // DMA of this buffer done
    double t1 = now();
    host_copy_rows(c.stage[b], cols, src + r0 * spitch, spitch, nr, cols);
    t_wait += t1 - t0;
    t_copy += now() - t1;
    IPT_CUDA(cudaMemcpy2DAsync(dst + r0 * dpitch, dpitch * sizeof(double), c.stage[b], cols * sizeof(double),
                               cols * sizeof(double), nr, cudaMemcpyHostToDevice, st));
    IPT_CUDA(cudaEventRecord(c.stage_ev[b], st));
    used[b] = true;
  }
  IPT_CUDA(cudaStreamSynchronize(st));
  if (prof && rows * cols >= (int64_t(1) << 24))
    std::fprintf(stderr, "[ipt] h2d_rows %.2f GB: %.1f ms (host copy %.1f, DMA wait %.1f, %u threads)\n",
                 8e-9 * double(rows) * double(cols), 1e3 * (now() - t_start), 1e3 * t_copy, 1e3 * t_wait,
                 copy_threads());
}

// A flat pageable host buffer to the device through the same pinned, double-buffered,
// multi-threaded staging as h2d_rows (8 MB rows; the sub-8-byte tail by a plain copy).
void h2d_bytes(Ctx& c, void* dst, const void* src, size_t bytes) {
  constexpr int64_t kRow = int64_t(1) << 20;  // doubles per staged row
  const int64_t nd = static_cast<int64_t>(bytes / sizeof(double));
  const int64_t rows = nd / kRow;
  auto* d8 = static_cast<double*>(dst);
  const auto* s8 = static_cast<const double*>(src);
  if (rows > 0) h2d_rows(c, d8, kRow, s8, kRow, rows, kRow);
  const int64_t done = rows * kRow;
  if (nd > done) h2d_rows(c, d8 + done, nd - done, s8 + done, nd - done, 1, nd - done);
  const size_t tail = bytes - sizeof(double) * size_t(nd);
  if (tail) {
    IPT_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(dst) + bytes - tail, reinterpret_cast<const char*>(src) + bytes - tail,
                             tail, cudaMemcpyHostToDevice, c.stream));
    IPT_CUDA(cudaStreamSynchronize(c.stream));
  }
}

void d2h_rows(Ctx& c, double* dst, int64_t dpitch, const double* src, int64_t spitch, int64_t rows,
              int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  cudaStream_t st = stream ? stream : c.stream;
  ensure_staging(c);
  const int64_t per_max = static_cast<int64_t>(c.stage_doubles) / cols;
  if (per_max < 1) {
    IPT_CUDA(cudaMemcpy2DAsync(dst, dpitch * sizeof(double), src, spitch * sizeof(double), cols * sizeof(double),
                               rows, cudaMemcpyDeviceToHost, st));
    IPT_CUDA(cudaStreamSynchronize(st));
    return;
  }
  // DMA chunk k+1 into one buffer while the host drains chunk k from the other (a
  // transfer that fits one buffer still goes in >= 4 chunks of >= 1 MB to overlap them).
  const int64_t per = std::max(std::max<int64_t>(1, (int64_t(1) << 17) / cols), std::min(per_max, (rows + 3) / 4));
  const int64_t nchunks = (rows + per - 1) / per;
  auto issue = [&](int64_t k) {
    const int64_t r0 = k * per, nr = std::min(per, rows - r0);
    const int b = static_cast<int>(k & 1);
    IPT_CUDA(cudaMemcpy2DAsync(c.stage[b], cols * sizeof(double), src + r0 * spitch, spitch * sizeof(double),
                               cols * sizeof(double), nr, cudaMemcpyDeviceToHost, st));
    IPT_CUDA(cudaEventRecord(c.stage_ev[b], st));
  };
  const bool prof = std::getenv("IPT_PROFILE") != nullptr;
  double t_wait = 0.0, t_copy = 0.0;
  auto now = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_start = now();
  issue(0);  // the first DMA runs while the destination is prefaulted
  if (dpitch == cols && !take_prefaulted(dst, sizeof(double) * size_t(rows) * size_t(cols)))
    prefault_host_destination(dst, sizeof(double) * size_t(rows) * size_t(cols));
  const double t_fault = now() - t_start;
  for (int64_t k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) issue(k + 1);
    const int b = static_cast<int>(k & 1);
    const double t0 = now();
    IPT_CUDA(cudaEventSynchronize(c.stage_ev[b]));
    const double t1 = now();
    const int64_t r0 = k * per, nr = std::min(per, rows - r0);
    host_copy_rows(dst + r0 * dpitch, dpitch, c.stage[b], cols, nr, cols);
    t_wait += t1 - t0;
    t_copy += now() - t1;
  }
  IPT_CUDA(cudaStreamSynchronize(st));
  if (prof && rows * cols >= (int64_t(1) << 24))
    std::fprintf(stderr, "[ipt] d2h_rows %.2f GB: %.1f ms (prefault %.1f, host copy %.1f, DMA wait %.1f, %u threads)\n",
                 8e-9 * double(rows) * double(cols), 1e3 * (now() - t_start), 1e3 * t_fault, 1e3 * t_copy,
                 1e3 * t_wait, copy_threads());
}

// Interleaved complex host rows (the C++ carrier, std::complex<double>) to planar device
// rows: the host workers de-interleave each chunk into the pinned staging buffer (real
// plane in its first half, imaginary plane in the second) while checking the imaginary
// parts; the imaginary plane of a chunk is sent only when it holds a nonzero (dim is
// zeroed by the caller). *any_im reports whether any was sent.
void h2d_rows_split(Ctx& c, double* dre, double* dim, int64_t dpitch, const double* src_c, int64_t rows,
                    int64_t cols, bool* any_im) {
  *any_im = false;
  if (rows <= 0 || cols <= 0) return;
  cudaStream_t st = c.stream;
  ensure_staging(c);
  const int64_t half = static_cast<int64_t>(c.stage_doubles) / 2;
  const int64_t per = half / cols;
  if (per < 1) throw InvalidArgument("h2d_rows_split: row longer than the staging buffer");
  int b = 0;
  bool used[2] = {false, false};
  std::atomic<bool> chunk_im{false};
  for (int64_t r0 = 0; r0 < rows; r0 += per, b ^= 1) {
    const int64_t nr = std::min(per, rows - r0);
    if (used[b]) IPT_CUDA(cudaEventSynchronize(c.stage_ev[b]));
    double* re = c.stage[b];
    double* im = c.stage[b] + half;
    const double* s0 = src_c + 2 * r0 * cols;
    const int64_t total = nr * cols;
    chunk_im.store(false, std::memory_order_relaxed);
    const unsigned t = total >= (int64_t(1) << 16) ? host_pool().size() : 1u;
    const int64_t step = (total + t - 1) / t;
    auto work = [&](unsigned k) {
      const int64_t a = int64_t(k) * step, e = std::min(total, a + step);
      bool nz = false;
      for (int64_t q = a; q < e; ++q) {
        re[q] = s0[2 * q];
        im[q] = s0[2 * q + 1];
        nz = nz || s0[2 * q + 1] != 0.0;
      }
      if (nz) chunk_im.store(true, std::memory_order_relaxed);
    };
    if (t <= 1) work(0);
    else host_pool().run(t, work);
    IPT_CUDA(cudaMemcpy2DAsync(dre + r0 * dpitch, dpitch * sizeof(double), re, cols * sizeof(double),
                               cols * sizeof(double), nr, cudaMemcpyHostToDevice, st));
    if (chunk_im.load()) {
      *any_im = true;
      IPT_CUDA(cudaMemcpy2DAsync(dim + r0 * dpitch, dpitch * sizeof(double), im, cols * sizeof(double),
                                 cols * sizeof(double), nr, cudaMemcpyHostToDevice, st));
    }
    IPT_CUDA(cudaEventRecord(c.stage_ev[b], st));
    used[b] = true;
  }
  IPT_CUDA(cudaStreamSynchronize(st));
}

// Planar device rows to interleaved complex host rows (sim == nullptr: imaginary parts 0),
// the host workers interleaving out of the pinned staging buffer while the next chunk's
// DMA runs.
void d2h_rows_merge(Ctx& c, double* dst_c, int64_t dpitch, const double* sre, const double* sim, int64_t spitch,
                    int64_t rows, int64_t cols, cudaStream_t stream) {
  if (rows <= 0 || cols <= 0) return;
  cudaStream_t st = stream ? stream : c.stream;
  ensure_staging(c);
  const int64_t half = static_cast<int64_t>(c.stage_doubles) / 2;
  const int64_t per = half / cols;
  if (per < 1) throw InvalidArgument("d2h_rows_merge: row longer than the staging buffer");
  const int64_t nchunks = (rows + per - 1) / per;
  auto issue = [&](int64_t k) {
    const int64_t r0 = k * per, nr = std::min(per, rows - r0);
    const int b = static_cast<int>(k & 1);
    IPT_CUDA(cudaMemcpy2DAsync(c.stage[b], cols * sizeof(double), sre + r0 * spitch, spitch * sizeof(double),
                               cols * sizeof(double), nr, cudaMemcpyDeviceToHost, st));
    if (sim)
      IPT_CUDA(cudaMemcpy2DAsync(c.stage[b] + half, cols * sizeof(double), sim + r0 * spitch,
                                 spitch * sizeof(double), cols * sizeof(double), nr, cudaMemcpyDeviceToHost, st));
    IPT_CUDA(cudaEventRecord(c.stage_ev[b], st));
  };
  issue(0);
  for (int64_t k = 0; k < nchunks; ++k) {
    if (k + 1 < nchunks) issue(k + 1);
    const int b = static_cast<int>(k & 1);
    IPT_CUDA(cudaEventSynchronize(c.stage_ev[b]));
    const int64_t r0 = k * per, nr = std::min(per, rows - r0);
    const double* re = c.stage[b];
    const double* im = c.stage[b] + half;
    const int64_t total = nr * cols;
    const unsigned t = total >= (int64_t(1) << 16) ? host_pool().size() : 1u;
    const int64_t step = (total + t - 1) / t;
    auto work = [&](unsigned kk) {
      const int64_t a = int64_t(kk) * step, e = std::min(total, a + step);
      if (dpitch == cols) {  // whole rows: one flat range
        double* d0 = dst_c + 2 * r0 * cols;
        for (int64_t q = a; q < e; ++q) {
          d0[2 * q] = re[q];
          d0[2 * q + 1] = sim ? im[q] : 0.0;
        }
        return;
      }
      for (int64_t q = a; q < e;) {  // a column block: row segments
        const int64_t row = q / cols, col = q % cols, len = std::min(e - q, cols - col);
        double* d = dst_c + 2 * ((r0 + row) * dpitch + col);
        for (int64_t t = 0; t < len; ++t) {
          d[2 * t] = re[q + t];
          d[2 * t + 1] = sim ? im[q + t] : 0.0;
        }
        q += len;
      }
    };
    if (t <= 1) work(0);
    else host_pool().run(t, work);
  }
  IPT_CUDA(cudaStreamSynchronize(st));
}

// 32x32 tiles through shared memory; src column-major (element (r, c) at c*ld_src + r),
// dst row-major (element (r, c) at r*ld_dst + c).
__global__ void transpose_kernel(const double* __restrict__ src, int64_t ld_src, int64_t rows,
                                 int64_t cols, double* __restrict__ dst, int64_t ld_dst,
                                 double sign) {
  __shared__ double tile[32][33];
  const int64_t r0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[c * ld_src + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) dst[r * ld_dst + c] = sign * tile[threadIdx.x][k];
  }
}

void transpose_to_rowmajor(cudaStream_t s, const double* src, int64_t ld_src, int64_t rows,
                           int64_t cols, double* dst, int64_t ld_dst, double sign) {
  if (rows == 0 || cols == 0) return;
  dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(cols, 32)));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(src, ld_src, rows, cols, dst, ld_dst, sign);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void fill_zero(cudaStream_t s, double* p, size_t count) {
  IPT_CUDA(cudaMemsetAsync(p, 0, count * sizeof(double), s));
}

__global__ void scale_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, size_t n,
                                  double f) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = f * src[i];
}
void scale_copy(cudaStream_t s, const double* src, double* dst, size_t count, double factor) {
  if (count == 0) return;
  const unsigned grid = static_cast<unsigned>(std::min<size_t>(ceil_div(count, 256), 148 * 16));
  scale_copy_kernel<<<grid, 256, 0, s>>>(src, dst, count, factor);
  IPT_LAUNCH_CHECK();
  count_launch();
}

// Sum the per-CTA partials in a fixed order (thread t takes t, t+512, ...; then
// the fixed block tree), so the reduced scalars are run-to-run identical.
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int64_t count,
                                       double* __restrict__ out4, const LoopState* state) {
  if (state != nullptr && state->done) return;
  __shared__ double red[16][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    v[0] += partials[4 * i + 0];
    v[1] += partials[4 * i + 1];
    v[2] += partials[4 * i + 2];
    v[3] = nan_max(v[3], partials[4 * i + 3]);
  }
  block_reduce4<16>(v, red);
  if (threadIdx.x == 0) {
    out4[0] = v[0];
    out4[1] = v[1];
    out4[2] = v[2];
    out4[3] = v[3];
  }
}

void reduce_partials(cudaStream_t s, const double* partials, int64_t count, double* out4,
                     const LoopState* state) {
  reduce_partials_kernel<<<1, 512, 0, s>>>(partials, count, out4, state);
  IPT_LAUNCH_CHECK();
  count_launch();
}

}  // namespace iptb
