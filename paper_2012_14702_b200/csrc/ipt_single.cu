// Single-eigenpair IPT on the device: solve_single / solve_single_continuation /
// apply_map_single (proj/src/solver.cpp:49-154) and kernels::matvec
// (proj/src/kernels.cpp:112-140).
//
// One iteration = K7/K8 + K9 fused:
//   anchor pre-pass : w_a = Delta[a, :] . z         (one warp, same summation order as below)
//   map kernel      : w_i = Delta[i, :] . z (dense GEMV, 16-byte streaming loads, or CSR
//                     SpMV, 16 lanes per row) and, in registers,
//                     fz_i = scale * (g_i * (z_i * w_a - w_i)), fz_a = 1, g_i = 1/(d_i - d_a)
//                     (single_step.hpp:11-17) plus the partial sums of |z-fz|^2, |z|^2, |fz|^2
//   decide          : fixed-order reduction, rel_step (single_step.hpp:19-26), divergence
//                     then convergence (solver.cpp:72-80), continuation schedule (:146-152).
// With a communicator the rows are sharded in equal chunks, every rank keeps row a, and
// the new iterate is all-gathered in place (one NCCL all-gather + one all-reduce / step).
//
// HBM layout: dense Delta row-major, ld = round_up(n,16) (rows of this rank only);
// CSR int64 row offsets (rebased to the shard), int32 columns, fp64 values;
// z ping-pong vectors of length nranks*chunk, replicated.
#include <algorithm>
#include <cmath>
#include <climits>
#include <cstdlib>
#include <complex>
#include <cstring>
#include <memory>

#include "ipt_internal.cuh"

namespace iptb {

constexpr int kMaxPeers = 7;  // one 8-GPU node
enum PeerKind : int { kPeerNone = 0, kPeerIpc = 1, kPeerOwned = 2, kPeerBorrowed = 3 };

struct SingleProblem {
  Ctx* ctx = nullptr;
  int64_t n = 0;
  bool csr = false, cplx = false;
  int64_t chunk = 0, r0 = 0, r1 = 0;  // rows of this rank
  // dense
  DevBuf A, Ai;
  int64_t lda = 0;
  // csr
  std::unique_ptr<int64_t, void (*)(void*)> rowptr{nullptr, [](void* p) { cudaFree(p); }};
  std::unique_ptr<int32_t, void (*)(void*)> cols{nullptr, [](void* p) { cudaFree(p); }};
  DevBuf vals, valsi;
  // balanced CSR variants: first row group of every warp of the map grid (nwarps + 1)
  std::unique_ptr<int32_t, void (*)(void*)> wgroups{nullptr, [](void* p) { cudaFree(p); }};
  bool spmv_bal = false;  // the map runs the balanced group ranges (wgroups)
  // anchor row copy (dense: lda doubles; csr: its nonzeros)
  DevBuf arow, arowi;
  std::unique_ptr<int32_t, void (*)(void*)> acols{nullptr, [](void* p) { cudaFree(p); }};
  int64_t annz = 0;
  int anchor_phase = 0;  // grouped CSR kernels: lane phase of the anchor row in its row group
  int64_t anchor = -1;
  // host copies needed to (re)build the anchor row for a new anchor
  const int64_t* h_rowptr = nullptr;  // the caller's row offsets (or h_rowptr_copy)
  std::vector<int64_t> h_rowptr_copy;
  int64_t nnz_total = 0;
  const int32_t* h_cols = nullptr;
  const double *h_vals = nullptr, *h_valsi = nullptr, *h_dense = nullptr, *h_densei = nullptr;
  std::vector<int32_t> h_cols_copy;
  std::vector<double> h_vals_copy, h_valsi_copy;
  DevBuf dre, dim;
  DevBuf z[2], zi[2];
  DevBuf w, wi;              // complex path / matvec scratch
  DevBuf zc;                 // complex CSR path: the iterate interleaved (re, im) for 16-byte gathers
  bool cspmv_simple = false; // IPT_CSPMV_SIMPLE at upload: the thread-per-row complex CSR kernel
  DevBuf wa;                 // anchor value (re, im)
  DevBuf partials;
  int64_t npart = 0;
  DevBuf sums;
  LoopState* state = nullptr;
  DevBuf trace;
  int trace_cap = 0;
  int enq = 0;
  // Fused all-gather over peer memory (real maps with a communicator): the map kernel
  // stores its rows of the new iterate straight into every peer's z buffer (CUDA IPC
  // over NVLink) instead of an NCCL all-gather after it; z[b] are then cudaMalloc'd
  // (exportable). peer_z[b][q]: peer q's z[b].
  bool p2p = false;
  int npeers = 0;
  double* peer_z[2][kMaxPeers] = {};
  // peer_z opened by cudaIpcOpenMemHandle (NCCL ranks), owned stand-ins (single-rank
  // test hook), or borrowed from ranks of the same process (local communicator)
  int peer_kind = 0;
  // fused step tail: arrival counter of the map kernel's CTAs; w_a of z[enq & 1] already
  // formed by the previous step's tail (else the next step launches the anchor kernel)
  unsigned* tail_counter = nullptr;  // inside `sums`
  bool wa_fresh = false;
  ~SingleProblem() {
    if (state) cudaFree(state);
    for (int b = 0; b < 2; ++b)
      for (int q = 0; q < npeers; ++q)
        if (peer_z[b][q]) {
          if (peer_kind == kPeerIpc) cudaIpcCloseMemHandle(peer_z[b][q]);
          else if (peer_kind == kPeerOwned) cudaFree(peer_z[b][q]);
        }
  }
};

namespace {

constexpr int kGemvRows = 4;        // rows per warp (dense)
constexpr int kGemvWarps = 8;
constexpr int kRowsPerBlock = kGemvRows * kGemvWarps;
// CSR variants. Row kernels (lanes per row, entries in flight per lane), measured at
// config 5 (N = 2^21, 64 nnz/row, profiles/r01_spmv_variants.txt): {8,4} 0.674 ms,
// {16,4} 0.689, {16,6} 0.753, {32,2} 0.832, {8,8} 0.905. Warp-contiguous row groups
// (spmv_group_kernel): 4 rows x 4 in flight 0.644 ms with L2 cache hints, 0.632 ms
// without (variant 9); with the next group's row offsets loaded while the current group
// streams 0.627 ms (variant 16; round 2, with the fused step tail); the four xor trees
// folded into one and 32-bit relative positions 0.613 ms (variant 20); that with the index /
// value loads software-pipelined 0.601 ms (variant 24, spmv_pipe_kernel); only the indices
// a chunk ahead, the values loaded beside the gathers, 3 entries per lane 0.583 ms
// (variant 30, the default: 64 registers, no spill; 4 per lane spills or, with the stop
// sums parked in shared memory, fits and runs 0.596 ms). All give the same bits. The memory
// ceiling of the same traffic is 0.517 ms (profiles/r01_gather_probe.txt): one L1 ->
// crossbar request per clock per SM.
// IPT_SPMV_VARIANT selects another.
// Variants 5-7: warp-contiguous row groups (spmv_group_kernel), lanes = 0 marks them,
// u = entries in flight per lane, rows = rows per warp.
struct SpmvVariant {
  int lanes, u, rows, minb;
};
constexpr SpmvVariant kSpmvVariants[] = {{16, 4, 0, 5}, {8, 8, 0, 5}, {32, 2, 0, 5}, {8, 4, 0, 5}, {16, 6, 0, 5},
                                         {0, 4, 4, 4},  {0, 2, 8, 4}, {0, 2, 4, 5}, {0, 4, 4, 3},
                                         {0, 4, 4, 4},  {0, 4, 16, 3}, {0, 8, 4, 3},  {0, 4, 2, 4},
                                         {0, 8, 2, 4},  {0, 8, 4, 4},  {0, 4, 8, 4},
                                         {0, 4, 4, 4},  {0, 4, 4, 3},  {0, 2, 4, 5},   // 16-18: + offset prefetch
                                         {0, 4, 4, 4},   // 19: 16 with nnz-balanced contiguous group ranges per warp
                                         {0, 4, 4, 4},  {0, 4, 4, 5},  {0, 8, 4, 4},   // 20-22: 16 with folded row sums
                                         {0, 4, 4, 4},  {0, 2, 4, 4},  {0, 2, 4, 5},  {0, 4, 4, 3},
                                         {0, 2, 4, 6},  {0, 3, 4, 4},   // 23-28: 20 with software-pipelined loads
                                         {0, 4, 4, 4},  {0, 3, 4, 4},  {0, 2, 4, 4},  {0, 2, 4, 5}};  // 29-32: only the indices run ahead
constexpr int kNumSpmvVariants = sizeof(kSpmvVariants) / sizeof(kSpmvVariants[0]);
constexpr int kSpmvDefault = 30;  // warp-contiguous groups of 4 rows, folded row sums, indices one chunk ahead, 3 entries per lane in flight
inline int spmv_variant() {
  static const int v = [] {
    const char* e = std::getenv("IPT_SPMV_VARIANT");
    const int k = e ? std::atoi(e) : kSpmvDefault;
    // 21-23, 25-29, 32: measured (register spills, profiles/r02_spmv_fold_pipe.txt) and dropped
    const bool dropped = (k >= 21 && k <= 23) || (k >= 25 && k <= 29) || k == 32;
    return (k >= 0 && k < kNumSpmvVariants && !dropped) ? k : kSpmvDefault;
  }();
  return v;
}
inline bool spmv_grouped() { return kSpmvVariants[spmv_variant()].lanes == 0; }
inline int spmv_rows_per_block() {
  const SpmvVariant& v = kSpmvVariants[spmv_variant()];
  return v.lanes ? 256 / v.lanes : 8 * v.rows;
}

constexpr int kSpmvMinBlocks = 5;       // 48 registers (no spills): 5 CTAs (40 warps) per SM

enum MapMode : int { kMvStore = 0, kMvMap = 1, kMvFinal = 2, kMvAccel = 3 };

__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Row dot products of R consecutive rows against z (length K2 double2, zero padded),
// lane-strided with two accumulators per row; the order per row does not depend on R.
template <int R>
__device__ __forceinline__ void rows_dot(const double* __restrict__ A, int64_t lda, int nrows,
                                         const double* __restrict__ z, int64_t K2, double out[R]) {
  const int lane = threadIdx.x & 31;
  double ax[R], ay[R];
#pragma unroll
  for (int r = 0; r < R; ++r) ax[r] = ay[r] = 0.0;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  int64_t k = lane;
  for (; k + 96 < K2; k += 128) {
    double2 zz[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) zz[u] = z2[k + 32 * u];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nrows) {
        const double2* a2 = reinterpret_cast<const double2*>(A + r * lda);
        double2 av[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) av[u] = ld_stream(a2 + k + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ax[r] = __fma_rn(av[u].x, zz[u].x, ax[r]);
          ay[r] = __fma_rn(av[u].y, zz[u].y, ay[r]);
        }
      }
    }
  }
  for (; k < K2; k += 32) {
    const double2 zz = z2[k];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < nrows) {
        const double2 av = ld_stream(reinterpret_cast<const double2*>(A + r * lda) + k);
        ax[r] = __fma_rn(av.x, zz.x, ax[r]);
        ay[r] = __fma_rn(av.y, zz.y, ay[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double s = ax[r] + ay[r];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    out[r] = s;
  }
}

// L2 policies: the matrix streams through once (evict_first); the iterate z is the
// 16.8 MB gather target that must stay resident in the 126 MB L2 (evict_last).
__device__ __forceinline__ uint64_t policy_stream() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_keep() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_stream_f64(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ld_keep_f64(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}

// One CSR row over a group of LANES lanes. Lane sl takes entries beg+sl,
// beg+sl+LANES, ... in ascending order (fixed per-lane order + xor tree: deterministic);
// U entries per lane are in flight at once (all index/value loads issue before the
// dependent gathers).
template <int LANES, int U>
__device__ __forceinline__ double csr_row_dot(const int32_t* __restrict__ cols,
                                              const double* __restrict__ vals, int64_t beg,
                                              int64_t end, const double* __restrict__ z, int sl,
                                              uint64_t pol_stream, uint64_t pol_keep) {
  double s = 0.0;
  for (int64_t p0 = beg + sl; p0 < end; p0 += U * LANES) {
    int32_t c[U];
    double v[U], zz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + u * LANES;
      c[u] = p < end ? ld_stream_i32(cols + p, pol_stream) : 0;
      v[u] = p < end ? ld_stream_f64(vals + p, pol_stream) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) zz[u] = (p0 + u * LANES < end) ? ld_keep_f64(z + c[u], pol_keep) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (p0 + u * LANES < end) s = __fma_rn(v[u], zz[u], s);
  }
#pragma unroll
  for (int off = LANES / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return s;
}

// R consecutive CSR rows per warp, streamed as ONE contiguous entry range: lane l takes
// entries beg+l, beg+l+32, ... (fully coalesced index/value loads, one misaligned
// sector per instruction at most) and adds each product to the accumulator of the row
// it falls in; each row's 32 lane sums are then combined by the xor tree. A row's sum
// is fixed by the lane phase (rowptr[row] - rowptr[group start]) mod 32, which the
// anchor kernel reproduces (anchor_csr_phase_kernel), so w_a is the same number.
__device__ __forceinline__ int32_t ld_nc_i32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_nc_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// Row offsets of the group starting at local row lr0: lane k <= R holds rowptr[lr0 + k]
// (clamped at the end of the rows).
template <int R>
__device__ __forceinline__ long long group_offsets(const int64_t* __restrict__ rowptr, int64_t lr0, int64_t rows,
                                                   int lane) {
  return lane <= R ? rowptr[lr0 + lane < rows ? lr0 + lane : rows] : 0;
}

template <int R, int U, bool POL = true>
__device__ __forceinline__ void group_row_sums_at(long long mine, const int32_t* __restrict__ cols,
                                                  const double* __restrict__ vals, const double* __restrict__ z,
                                                  int lane, uint64_t pol_stream, uint64_t pol_keep, double (&s)[R]);

template <int R, int U, bool POL = true>
__device__ __forceinline__ void group_row_sums(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                                               const double* __restrict__ vals, const double* __restrict__ z,
                                               int64_t lr0, int64_t rows, int lane, uint64_t pol_stream,
                                               uint64_t pol_keep, double (&s)[R]) {
  group_row_sums_at<R, U, POL>(group_offsets<R>(rowptr, lr0, rows, lane), cols, vals, z, lane, pol_stream, pol_keep,
                               s);
}

template <int R, int U, bool POL>
__device__ __forceinline__ void group_row_sums_at(long long mine, const int32_t* __restrict__ cols,
                                                  const double* __restrict__ vals, const double* __restrict__ z,
                                                  int lane, uint64_t pol_stream, uint64_t pol_keep, double (&s)[R]) {
  int64_t rb[R + 1];
#pragma unroll
  for (int k = 0; k <= R; ++k) rb[k] = __shfl_sync(0xffffffffu, mine, k);
#pragma unroll
  for (int k = 0; k < R; ++k) s[k] = 0.0;
  const int64_t end = rb[R];
  for (int64_t p0 = rb[0] + lane; p0 < end; p0 += 32 * U) {
    int32_t c[U];
    double v[U], zz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + 32 * u;
      if (POL) {
        c[u] = p < end ? ld_stream_i32(cols + p, pol_stream) : 0;
        v[u] = p < end ? ld_stream_f64(vals + p, pol_stream) : 0.0;
      } else {
        c[u] = p < end ? ld_nc_i32(cols + p) : 0;
        v[u] = p < end ? ld_nc_f64(vals + p) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      zz[u] = (p0 + 32 * u < end) ? (POL ? ld_keep_f64(z + c[u], pol_keep) : __ldg(z + c[u])) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t p = p0 + 32 * u;
      if (p < end) {
        int r = 0;
#pragma unroll
        for (int k = 1; k < R; ++k) r += p >= rb[k];
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k == r) s[k] = __fma_rn(v[u], zz[u], s[k]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s[k] += __shfl_xor_sync(0xffffffffu, s[k], off);
}

// Four per-lane partial sums (rows 0-3 of a group) -> row k's total on lane k, by one
// transposed xor tree: after level 16 a lane keeps two rows, after level 8 one (row
// 2 bit4 + bit3 of the lane), levels 4 / 2 / 1 as usual, one shuffle brings row k to lane
// k. Each level adds the two numbers the full per-row xor tree adds on that lane, so the
// totals are bit for bit those of four separate trees (7 double shuffles instead of 20).
__device__ __forceinline__ double fold_rows4(double s0, double s1, double s2, double s3, int lane) {
  const bool b16 = lane & 16, b8 = lane & 8;
  double k0 = b16 ? s2 : s0, k1 = b16 ? s3 : s1;
  k0 += __shfl_xor_sync(0xffffffffu, b16 ? s0 : s2, 16);
  k1 += __shfl_xor_sync(0xffffffffu, b16 ? s1 : s3, 16);
  double k = b8 ? k1 : k0;
  k += __shfl_xor_sync(0xffffffffu, b8 ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
  return __shfl_sync(0xffffffffu, k, (lane & 3) * 8);
}

// group_row_sums_at for R = 4 with the same sums at lower instruction cost (round 2):
//  * entry positions relative to the group start in 32 bits (one 64-bit base broadcast +
//    four 32-bit offsets: 6 SHFL instead of 10; 32-bit row selection);
//  * the four xor trees folded into one transposed tree: after level 16 a lane keeps two
//    rows, after level 8 one row (row 2 bit4 + bit3 of the lane), levels 4/2/1 as before,
//    and one shuffle returns row k to lane k: 7 double shuffles instead of 20. Every
//    level adds the same two numbers the full xor tree adds on that lane, so each row sum
//    is bit for bit group_row_sums_at's.
// Returns this lane's row sum (row k on lane k < 4).
template <int U>
__device__ __forceinline__ double group_row_sums4_folded(long long mine, const int32_t* __restrict__ cols,
                                                         const double* __restrict__ vals,
                                                         const double* __restrict__ z, int lane) {
  const long long base = __shfl_sync(0xffffffffu, mine, 0);
  const int rel = static_cast<int>(mine - base);
  const int r1 = __shfl_sync(0xffffffffu, rel, 1), r2 = __shfl_sync(0xffffffffu, rel, 2),
            r3 = __shfl_sync(0xffffffffu, rel, 3), end = __shfl_sync(0xffffffffu, rel, 4);
  const int32_t* __restrict__ gc = cols + base;
  const double* __restrict__ gv = vals + base;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  for (int q0 = lane; q0 < end; q0 += 32 * U) {
    int32_t c[U];
    double v[U], zz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + 32 * u;
      c[u] = q < end ? ld_nc_i32(gc + q) : 0;
      v[u] = q < end ? ld_nc_f64(gv + q) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) zz[u] = (q0 + 32 * u < end) ? __ldg(z + c[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = q0 + 32 * u;
      if (q < end) {
        if (q < r2) {
          if (q < r1) s0 = __fma_rn(v[u], zz[u], s0);
          else s1 = __fma_rn(v[u], zz[u], s1);
        } else {
          if (q < r3) s2 = __fma_rn(v[u], zz[u], s2);
          else s3 = __fma_rn(v[u], zz[u], s3);
        }
      }
    }
  }
  return fold_rows4(s0, s1, s2, s3, lane);
}

struct MapArgs {
  const double* d;     // global diagonal
  const double* z;     // current iterate (global indexing)
  double* fz;          // next iterate (global indexing) / matvec output
  const double* wa;    // anchor value
  int64_t anchor;
  int64_t row0;        // global index of local row 0
  int64_t rows;        // local rows
  const LoopState* state;
  int schedule;
  double snap;
  double* partials;
  double* peer[kMaxPeers];  // kMvMap: the same rows of the new iterate in every peer's z
  int npeers;
  const int32_t* wgroups;   // balanced CSR variants: first row group of each warp (else null)
  // Fused step tail (kMvMap; tail_mode 0: none). The last CTA to finish sums the per-CTA
  // partials in reduce_partials_kernel's order into tail_sums; mode 2 (one rank) then also
  // applies the stop decision (decide_single_dev) and forms w_a of the new iterate for the
  // next step (the anchor kernels' arithmetic), so a step is ONE launch. Mode 1 (several
  // ranks) stops after the sums: the all-reduce and decide_anchor_kernel follow.
  int tail_mode;
  unsigned* tail_counter;  // zero between launches (reset by the last CTA)
  LoopState* tail_state;
  double* tail_sums;
  int tail_k, tail_max_iter, tail_schedule, tail_ignore;
  double tail_tol, tail_div, tail_alpha, tail_snap;
  double* tail_trace;
  // anchor row of the next w_a: CSR (columns, values, nnz, lane phase) or dense (row, lda)
  const int32_t* a_cols;
  const double* a_vals;
  int64_t a_nnz;
  int a_phase;
  int64_t a_lda;
};

// Remote stores of the fused all-gather must be visible system-wide before the
// collective that orders the next step (reduce_and_allreduce) starts.
__device__ __forceinline__ void peer_fence(const MapArgs& a) {
  if (a.npeers > 0) __threadfence_system();
}

// Per-row epilogue shared by dense and CSR kernels. Accumulates into v.
template <int MODE>
__device__ __forceinline__ void row_epilogue_vals(const MapArgs& a, int64_t i, double zi, double di, double w,
                                                  double scale, double lam, double v[4]);
template <int MODE>
__device__ __forceinline__ void row_epilogue(const MapArgs& a, int64_t i, double w, double scale,
                                             double lam, double v[4]) {
  row_epilogue_vals<MODE>(a, i, a.z[i], MODE == kMvStore ? 0.0 : a.d[i], w, scale, lam, v);
}
// The same epilogue with z_i and d_i already loaded (the pipelined CSR kernel loads them
// while the row's entries stream).
template <int MODE>
__device__ __forceinline__ void row_epilogue_vals(const MapArgs& a, int64_t i, double zi, double di, double w,
                                                  double scale, double lam, double v[4]) {
  if (MODE == kMvStore) {
    a.fz[i] = w;
  } else if (MODE == kMvMap) {
    double f;
    if (i == a.anchor) {
      f = 1.0;
    } else {
      const double g = __ddiv_rn(1.0, __dsub_rn(di, a.d[a.anchor]));
      f = __dmul_rn(scale, __dmul_rn(g, __dsub_rn(__dmul_rn(zi, *a.wa), w)));
    }
    a.fz[i] = f;
    for (int q = 0; q < a.npeers; ++q) a.peer[q][i] = f;  // fused all-gather (NVLink stores)
    const double df = __dsub_rn(zi, f);
    v[0] = __fma_rn(df, df, v[0]);
    v[1] = __fma_rn(zi, zi, v[1]);
    v[2] = __fma_rn(f, f, v[2]);
    v[3] = nan_max(v[3], fabs(df));
  } else if (MODE == kMvFinal) {  // residual |d z + w - lam z|^2 and |z|^2 (solver.cpp:86-91)
    const double r = __dsub_rn(__dadd_rn(__dmul_rn(di, zi), w), __dmul_rn(lam, zi));
    v[0] = __fma_rn(r, r, v[0]);
    v[1] = __fma_rn(zi, zi, v[1]);
  } else {  // kMvAccel: true residual AND the plain image f(z) (anderson.cpp:204-223)
    const double r = __dsub_rn(__dadd_rn(__dmul_rn(di, zi), w), __dmul_rn(lam, zi));
    double f;
    if (i == a.anchor) {
      f = 1.0;
    } else {
      const double g = __ddiv_rn(1.0, __dsub_rn(di, a.d[a.anchor]));
      f = __dmul_rn(g, __dsub_rn(__dmul_rn(zi, *a.wa), w));
    }
    a.fz[i] = f;
    const double df = __dsub_rn(f, zi);
    v[0] = __fma_rn(r, r, v[0]);
    v[1] = __fma_rn(zi, zi, v[1]);
    v[2] = __fma_rn(df, df, v[2]);
    v[3] = nan_max(v[3], fabs(df));
  }
}

__device__ __forceinline__ double schedule_scale(const MapArgs& a) {
  if (a.schedule == IPT_SCHEDULE_PLAIN || a.state == nullptr) return 1.0;
  const double ak = a.state->scale_ak;
  return ak <= a.snap ? 1.0 : 1.0 - ak;
}

// The reference's per-iteration tests (solver.cpp:69-80): divergence first (from the
// NaN-propagating |fz|^2), then convergence (gated by the continuation schedule,
// solver.cpp:146-152), then the iteration cap.
__device__ __forceinline__ void decide_single_dev(LoopState* st, double diff2, double base2, double new2, double mx,
                                                  int k, double tol, int max_iter, double div_thr, int schedule,
                                                  double alpha, double snap, int ignore_conv, double* trace) {
  const double step = sqrt(diff2) / sqrt(base2);
  st->iterations = k + 1;
  st->final_step = step;
  st->final_max_abs = mx;
  if (trace) trace[k] = step;
  const double ak = st->scale_ak;
  const bool gate = schedule == IPT_SCHEDULE_PLAIN || ak <= snap;
  const double zn = sqrt(new2);
  if (!isfinite(zn) || zn > div_thr) {
    st->status = kDiverged;
    st->done = 1;
  } else if (!ignore_conv && gate && step <= tol) {
    st->status = kConverged;
    st->done = 1;
  } else if (k + 1 >= max_iter) {
    st->status = kMaxIterations;
    st->done = 1;
  }
  if (schedule == IPT_SCHEDULE_CONTINUATION) st->scale_ak = ak * alpha;
}

// w_a = Delta[a, :] . z by one warp, bit for bit the anchor kernels' sums (CSR: entry k on
// lane (phase + k) mod 32, ascending per lane, xor tree; dense: rows_dot<1>). z is read
// through L2 (other CTAs of this launch wrote it).
__device__ __forceinline__ void anchor_value_warp(const MapArgs& a, const double* __restrict__ z) {
  const int lane = threadIdx.x & 31;
  double sacc = 0.0;
  if (a.a_cols != nullptr) {
    for (int64_t k = (lane - a.a_phase + 32) & 31; k < a.a_nnz; k += 32)
      sacc = __fma_rn(a.a_vals[k], __ldcg(z + a.a_cols[k]), sacc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
  } else {
    // rows_dot<1> with the z loads through L2
    const double2* a2 = reinterpret_cast<const double2*>(a.a_vals);
    const double2* z2 = reinterpret_cast<const double2*>(z);
    const int64_t K2 = a.a_lda / 2;
    double ax = 0.0, ay = 0.0;
    int64_t k = lane;
    for (; k + 96 < K2; k += 128) {
      double2 zz[4], av[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) zz[u] = __ldcg(z2 + k + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = ld_stream(a2 + k + 32 * u);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ax = __fma_rn(av[u].x, zz[u].x, ax);
        ay = __fma_rn(av[u].y, zz[u].y, ay);
      }
    }
    for (; k < K2; k += 32) {
      const double2 zz = __ldcg(z2 + k);
      const double2 av = ld_stream(a2 + k);
      ax = __fma_rn(av.x, zz.x, ax);
      ay = __fma_rn(av.y, zz.y, ay);
    }
    sacc = ax + ay;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, off);
  }
  if (lane == 0) *const_cast<double*>(a.wa) = sacc;
}

// Fused step tail, called by every thread of every CTA after its partials are written
// (blockDim.x == 256). See MapArgs::tail_mode.
__device__ __forceinline__ void step_tail(const MapArgs& a) {
  __shared__ int s_last;
  __shared__ double s_red[16][4];
  __threadfence();  // this thread's fz / peer / partial stores before the arrival count
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.tail_counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // reduce_partials_kernel's order: 512 virtual threads (t and t + 256 here), each summing
  // partials t, t + 512, ...; xor tree per virtual warp; virtual warps 0..15 in order.
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  double lo[4] = {0.0, 0.0, 0.0, 0.0}, hi[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t count = gridDim.x;
  for (int64_t i = t; i < count; i += 512) {
    lo[0] += __ldcg(a.partials + 4 * i + 0);
    lo[1] += __ldcg(a.partials + 4 * i + 1);
    lo[2] += __ldcg(a.partials + 4 * i + 2);
    lo[3] = nan_max(lo[3], __ldcg(a.partials + 4 * i + 3));
  }
  for (int64_t i = t + 256; i < count; i += 512) {
    hi[0] += __ldcg(a.partials + 4 * i + 0);
    hi[1] += __ldcg(a.partials + 4 * i + 1);
    hi[2] += __ldcg(a.partials + 4 * i + 2);
    hi[3] = nan_max(hi[3], __ldcg(a.partials + 4 * i + 3));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      lo[q] += __shfl_xor_sync(0xffffffffu, lo[q], off);
      hi[q] += __shfl_xor_sync(0xffffffffu, hi[q], off);
    }
    lo[3] = nan_max(lo[3], __shfl_xor_sync(0xffffffffu, lo[3], off));
    hi[3] = nan_max(hi[3], __shfl_xor_sync(0xffffffffu, hi[3], off));
  }
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      s_red[warp][q] = lo[q];
      s_red[warp + 8][q] = hi[q];
    }
  }
  __syncthreads();
  if (t == 0) {
    double r0 = s_red[0][0], r1 = s_red[0][1], r2 = s_red[0][2], r3 = s_red[0][3];
#pragma unroll
    for (int w = 1; w < 16; ++w) {
      r0 += s_red[w][0];
      r1 += s_red[w][1];
      r2 += s_red[w][2];
      r3 = nan_max(r3, s_red[w][3]);
    }
    a.tail_sums[0] = r0;
    a.tail_sums[1] = r1;
    a.tail_sums[2] = r2;
    a.tail_sums[3] = r3;
    if (a.tail_mode == 2)
      decide_single_dev(a.tail_state, r0, r1, r2, r3, a.tail_k, a.tail_tol, a.tail_max_iter, a.tail_div,
                        a.tail_schedule, a.tail_alpha, a.tail_snap, a.tail_ignore, a.tail_trace);
    *a.tail_counter = 0u;
  }
  if (a.tail_mode != 2) return;
  __syncthreads();
  if (warp == 0 && !a.tail_state->done) anchor_value_warp(a, a.fz);
}

template <int MODE>
__global__ void __launch_bounds__(kGemvWarps * 32) gemv_map_kernel(const double* __restrict__ A,
                                                                   int64_t lda, MapArgs a) {
  if (a.state != nullptr && a.state->done) return;
  __shared__ double red[kGemvWarps][4];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t lr0 = int64_t(blockIdx.x) * kRowsPerBlock + warp * kGemvRows;
  const int64_t left = a.rows - lr0;
  const int nrows = left <= 0 ? 0 : (left >= kGemvRows ? kGemvRows : static_cast<int>(left));
  double w[kGemvRows];
  if (nrows > 0) rows_dot<kGemvRows>(A + lr0 * lda, lda, nrows, a.z, lda / 2, w);
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const double scale = MODE == kMvMap ? schedule_scale(a) : 1.0;
  const double lam = (MODE == kMvFinal || MODE == kMvAccel) ? a.d[a.anchor] + *a.wa : 0.0;
#pragma unroll
  for (int r = 0; r < kGemvRows; ++r)
    if (lane == r && r < nrows) row_epilogue<MODE>(a, a.row0 + lr0 + r, w[r], scale, lam, v);
  if (MODE == kMvStore) return;
  if (MODE == kMvMap) peer_fence(a);
  block_reduce4<kGemvWarps>(v, red);
  if (threadIdx.x == 0) {
    double* o = a.partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
  if (MODE == kMvMap && a.tail_mode != 0) step_tail(a);
}

template <int MODE, int LANES, int U>
__global__ void __launch_bounds__(256, kSpmvMinBlocks) spmv_map_kernel(const int64_t* __restrict__ rowptr,
                                                       const int32_t* __restrict__ cols,
                                                       const double* __restrict__ vals, MapArgs a) {
  if (a.state != nullptr && a.state->done) return;
  __shared__ double red[8][4];
  constexpr int kRows = 256 / LANES;
  const int sl = threadIdx.x % LANES;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const double scale = MODE == kMvMap ? schedule_scale(a) : 1.0;
  const double lam = (MODE == kMvFinal || MODE == kMvAccel) ? a.d[a.anchor] + *a.wa : 0.0;
  const uint64_t pol_s = policy_stream(), pol_k = policy_keep();
  // Persistent fixed grid: block b owns row groups b, b + grid, ... (a fixed map, so the
  // per-block partial sums and their reduction are run-to-run identical).
  const int64_t groups = ceil_div(a.rows, kRows);
  for (int64_t grp = blockIdx.x; grp < groups; grp += gridDim.x) {
    const int64_t lr = grp * kRows + threadIdx.x / LANES;
    // all lanes of a row group take part in the shuffle even past the end
    const bool valid = lr < a.rows;
    const int64_t beg = valid ? rowptr[lr] : 0, end = valid ? rowptr[lr + 1] : 0;
    const double w = csr_row_dot<LANES, U>(cols, vals, beg, end, a.z, sl, pol_s, pol_k);
    if (valid && sl == 0) row_epilogue<MODE>(a, a.row0 + lr, w, scale, lam, v);
  }
  if (MODE == kMvStore) return;
  if (MODE == kMvMap) peer_fence(a);
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = a.partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
}

template <int MODE, int R, int U, int MINB, bool POL = true, bool PF = false, bool BAL = false, bool FOLD = false>
__global__ void __launch_bounds__(256, MINB) spmv_group_kernel(const int64_t* __restrict__ rowptr,
                                                                         const int32_t* __restrict__ cols,
                                                                         const double* __restrict__ vals, MapArgs a) {
  if (a.state != nullptr && a.state->done) return;
  __shared__ double red[8][4];
  const int lane = threadIdx.x & 31;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const double scale = MODE == kMvMap ? schedule_scale(a) : 1.0;
  const double lam = (MODE == kMvFinal || MODE == kMvAccel) ? a.d[a.anchor] + *a.wa : 0.0;
  const uint64_t pol_s = policy_stream(), pol_k = policy_keep();
  // Persistent fixed grid: warp w of block b owns row groups (b*8 + w) + k*(grid*8), or
  // (BAL) the contiguous group range [wgroups[w], wgroups[w+1]) cut at equal nonzero counts.
  // The groups themselves (R consecutive rows from a multiple of R) and so every row's sum
  // are the same either way; only which warp -- and CTA partial -- takes them changes.
  const int64_t groups = ceil_div(a.rows, int64_t(R));
  const int64_t wglob = blockIdx.x * int64_t(8) + (threadIdx.x >> 5);
  const int64_t g_begin = BAL ? a.wgroups[wglob] : wglob;
  const int64_t g_end = BAL ? a.wgroups[wglob + 1] : groups;
  const int64_t g_step = BAL ? 1 : int64_t(gridDim.x) * 8;
  // PF: the next group's row offsets load while this group streams (one dependent
  // load off the critical path per group)
  long long next_off = PF && g_begin < g_end ? group_offsets<R>(rowptr, g_begin * R, a.rows, lane) : 0;
  for (int64_t grp = g_begin; grp < g_end; grp += g_step) {
    const int64_t lr0 = grp * R;
    double sum[R];
    if (FOLD) {  // PF, R = 4, plain nc loads: the folded tree leaves row k's sum on lane k
      static_assert(!FOLD || (R == 4 && PF && !POL), "folded sums: R = 4, offset prefetch, plain loads");
      const long long off = next_off;
      if (grp + g_step < g_end) next_off = group_offsets<R>(rowptr, (grp + g_step) * R, a.rows, lane);
      const double w = group_row_sums4_folded<U>(off, cols, vals, a.z, lane);
      if (lane < R && lr0 + lane < a.rows) row_epilogue<MODE>(a, a.row0 + lr0 + lane, w, scale, lam, v);
      continue;
    }
    if (PF) {
      const long long off = next_off;
      if (grp + g_step < g_end) next_off = group_offsets<R>(rowptr, (grp + g_step) * R, a.rows, lane);
      group_row_sums_at<R, U, POL>(off, cols, vals, a.z, lane, pol_s, pol_k, sum);
    } else {
      group_row_sums<R, U, POL>(rowptr, cols, vals, a.z, lr0, a.rows, lane, pol_s, pol_k, sum);
    }
    if (lane < R && lr0 + lane < a.rows) {
      double w = sum[0];
#pragma unroll
      for (int k = 1; k < R; ++k)
        if (lane == k) w = sum[k];
      row_epilogue<MODE>(a, a.row0 + lr0 + lane, w, scale, lam, v);
    }
  }
  if (MODE == kMvStore) return;
  if (MODE == kMvMap) peer_fence(a);
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = a.partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
  if (MODE == kMvMap && a.tail_mode != 0) step_tail(a);
}

// spmv_group_kernel<MODE, 4, U, MINB, plain loads, offset prefetch, folded sums> with the
// loads software-pipelined (round 2): the K8 map is bound by load latency, not by a
// throughput (ncu: issue slots 36 % busy, long-scoreboard stalls, the L1 -> crossbar request
// path 80 % busy), because a warp alternates between waiting for a chunk's index / value
// loads and waiting for its z gathers. Here the next chunk's indices and values (the next
// group's first chunk after a group's last, its offsets known two groups ahead) are
// requested before the current chunk's gathers are consumed, and the rows' d_i, z_i of the
// epilogue load at the group's start. XL (the default): only the indices run a chunk ahead
// and the values load beside the gathers, which frees the registers for a third entry per
// lane at 4 CTAs per SM. Same groups, same lanes, same order of operations: every row sum,
// iterate and stop sum is bit for bit spmv_group_kernel's.
__device__ __forceinline__ double ld_nc_gather_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <int MODE, int U, int MINB, bool XL = false, bool BAL = false>
__global__ void __launch_bounds__(256, MINB) spmv_pipe_kernel(const int64_t* __restrict__ rowptr,
                                                              const int32_t* __restrict__ cols,
                                                              const double* __restrict__ vals, MapArgs a) {
  if (a.state != nullptr && a.state->done) return;
  constexpr int R = 4;
  __shared__ double red[8][4];
  const int lane = threadIdx.x & 31;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const double scale = MODE == kMvMap ? schedule_scale(a) : 1.0;
  const double lam = (MODE == kMvFinal || MODE == kMvAccel) ? a.d[a.anchor] + *a.wa : 0.0;
  // round-robin over the grid's warps, or (BAL) this warp's contiguous nonzero-balanced
  // range of groups, as in spmv_group_kernel
  // (group indices fit 32 bits: rows < 2^31 for int32 columns)
  const int wglob = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int g_begin = BAL ? a.wgroups[wglob] : wglob;
  const int groups = BAL ? a.wgroups[wglob + 1] : static_cast<int>(ceil_div(a.rows, int64_t(R)));
  const int g_step = BAL ? 1 : static_cast<int>(gridDim.x) * 8;
  // offsets of this group and the next one in registers, the one after that in flight
  long long off0 = g_begin < groups ? group_offsets<R>(rowptr, int64_t(g_begin) * R, a.rows, lane) : 0;
  long long off1 =
      g_begin + g_step < groups ? group_offsets<R>(rowptr, int64_t(g_begin + g_step) * R, a.rows, lane) : 0;
  int32_t c[U];
  double x[U];
  {  // first chunk of the first group
    const long long base = __shfl_sync(0xffffffffu, off0, 0);
    const int end = static_cast<int>(__shfl_sync(0xffffffffu, off0, R) - base);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int q = lane + 32 * u;
      c[u] = q < end ? ld_nc_i32(cols + base + q) : 0;
      if (!XL) x[u] = q < end ? ld_nc_f64(vals + base + q) : 0.0;
    }
  }
  for (int grp = g_begin; grp < groups; grp += g_step) {
    const int64_t lr0 = int64_t(grp) * R;
    const long long off2 =
        grp + 2 * g_step < groups ? group_offsets<R>(rowptr, int64_t(grp + 2 * g_step) * R, a.rows, lane) : 0;
    const bool mine = lane < R && lr0 + lane < a.rows;
    const int64_t gi = a.row0 + lr0 + lane;
    const double zi = (mine && MODE != kMvStore) ? a.z[gi] : 0.0;  // store mode: a plain matvec, z may be shorter
    const double di = (mine && MODE != kMvStore) ? a.d[gi] : 0.0;
    const long long base = __shfl_sync(0xffffffffu, off0, 0);
    const int rel = static_cast<int>(off0 - base);
    const int r1 = __shfl_sync(0xffffffffu, rel, 1), r2 = __shfl_sync(0xffffffffu, rel, 2),
              r3 = __shfl_sync(0xffffffffu, rel, 3), end = __shfl_sync(0xffffffffu, rel, 4);
    const bool more = grp + g_step < groups;
    const long long nbase = __shfl_sync(0xffffffffu, off1, 0);
    const int nend = more ? static_cast<int>(__shfl_sync(0xffffffffu, off1, R) - nbase) : 0;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int qc = 0;
    do {  // a group without entries still takes one (empty) pass: its chunk registers are consumed
      double zz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) zz[u] = (qc + lane + 32 * u < end) ? ld_nc_gather_f64(a.z + c[u]) : 0.0;
      if (XL) {  // XL: only the indices run a chunk ahead; the values load beside the gathers
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = (qc + lane + 32 * u < end) ? ld_nc_f64(vals + base + qc + lane + 32 * u) : 0.0;
      }
      int32_t nc[U];
      double nx[U];
      const bool last = qc + 32 * U >= end;
      const long long pb = last ? nbase : base;
      const int pq = last ? lane : qc + 32 * U + lane, pe = last ? nend : end;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = pq + 32 * u;
        nc[u] = q < pe ? ld_nc_i32(cols + pb + q) : 0;
        if (!XL) nx[u] = q < pe ? ld_nc_f64(vals + pb + q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = qc + lane + 32 * u;
        if (q < end) {
          if (q < r2) {
            if (q < r1) s0 = __fma_rn(x[u], zz[u], s0);
            else s1 = __fma_rn(x[u], zz[u], s1);
          } else {
            if (q < r3) s2 = __fma_rn(x[u], zz[u], s2);
            else s3 = __fma_rn(x[u], zz[u], s3);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        c[u] = nc[u];
        if (!XL) x[u] = nx[u];
      }
      qc += 32 * U;
    } while (qc < end);
    const double w = fold_rows4(s0, s1, s2, s3, lane);
    if (mine) row_epilogue_vals<MODE>(a, gi, zi, di, w, scale, lam, v);
    off0 = off1;
    off1 = off2;
  }
  if (MODE == kMvStore) return;
  if (MODE == kMvMap) peer_fence(a);
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = a.partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
  if (MODE == kMvMap && a.tail_mode != 0) step_tail(a);
}

// The anchor row's sum exactly as spmv_group_kernel forms it: entry k of the row on
// lane (phase + k) mod 32, ascending per lane, then the xor tree.
__global__ void anchor_csr_phase_kernel(const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                        int64_t nnz, int phase, const double* __restrict__ z, double* wa,
                                        const LoopState* st) {
  if (st != nullptr && st->done) return;
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int64_t k = (lane - phase + 32) & 31; k < nnz; k += 32) s = __fma_rn(vals[k], z[cols[k]], s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) wa[0] = s;
}

// w_a with exactly the per-row arithmetic of the map kernels.
__global__ void anchor_dense_kernel(const double* __restrict__ arow, int64_t lda,
                                    const double* __restrict__ z, double* wa, const LoopState* st) {
  if (st != nullptr && st->done) return;
  double w[1];
  rows_dot<1>(arow, lda, 1, z, lda / 2, w);
  if (threadIdx.x == 0) wa[0] = w[0];
}
template <int LANES, int U>
__global__ void anchor_csr_kernel(const int32_t* __restrict__ cols, const double* __restrict__ vals,
                                  int64_t nnz, const double* __restrict__ z, double* wa,
                                  const LoopState* st) {
  if (st != nullptr && st->done) return;
  const double w = csr_row_dot<LANES, U>(cols, vals, 0, nnz, z, threadIdx.x % LANES, policy_stream(), policy_keep());
  if (threadIdx.x == 0) wa[0] = w;
}

__global__ void decide_single_kernel(LoopState* st, const double* __restrict__ sums, int k, double tol,
                                     int max_iter, double div_thr, int schedule, double alpha,
                                     double snap, int ignore_conv, double* trace) {
  if (st->done) return;
  decide_single_dev(st, sums[0], sums[1], sums[2], sums[3], k, tol, max_iter, div_thr, schedule, alpha, snap,
                    ignore_conv, trace);
}

// Several ranks: after the all-reduce of the stop sums, the decision and (if the loop goes
// on) w_a of the new iterate, which every rank's fused all-gather has completed by now.
__global__ void decide_anchor_kernel(LoopState* st, const double* __restrict__ sums, int k, double tol,
                                     int max_iter, double div_thr, int schedule, double alpha, double snap,
                                     int ignore_conv, double* trace, MapArgs a) {
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    s_go = 0;
    if (!st->done) {
      decide_single_dev(st, sums[0], sums[1], sums[2], sums[3], k, tol, max_iter, div_thr, schedule, alpha, snap,
                        ignore_conv, trace);
      s_go = !st->done;
    }
  }
  __syncthreads();
  if (s_go) anchor_value_warp(a, a.fz);
}

// ---- complex correctness path: generic complex matvec then an elementwise map ----
__global__ void cmatvec_dense_kernel(const double* __restrict__ Ar, const double* __restrict__ Ai,
                                     int64_t lda, int64_t rows, int64_t ncols,
                                     const double* __restrict__ xr, const double* __restrict__ xi,
                                     double* yr, double* yi, int64_t row0) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  double sr = 0.0, si = 0.0;
  for (int64_t j = lane; j < ncols; j += 32) {
    const double ar = Ar[r * lda + j], ai = Ai ? Ai[r * lda + j] : 0.0;
    sr += ar * xr[j] - ai * xi[j];
    si += ar * xi[j] + ai * xr[j];
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, off);
    si += __shfl_xor_sync(0xffffffffu, si, off);
  }
  if (lane == 0) {
    yr[row0 + r] = sr;
    yi[row0 + r] = si;
  }
}
__global__ void cmatvec_csr_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ cols,
                                   const double* __restrict__ vr, const double* __restrict__ vi,
                                   int64_t rows, const double* __restrict__ xr,
                                   const double* __restrict__ xi, double* yr, double* yi, int64_t row0) {
  const int64_t r = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= rows) return;
  double sr = 0.0, si = 0.0;
  for (int64_t p = rowptr[r]; p < rowptr[r + 1]; ++p) {
    const double ar = vr[p], ai = vi ? vi[p] : 0.0;
    const int32_t c = cols[p];
    sr += ar * xr[c] - ai * xi[c];
    si += ar * xi[c] + ai * xr[c];
  }
  yr[row0 + r] = sr;
  yi[row0 + r] = si;
}



// Complex CSR matvec, w = Delta z over the local rows, as the real map streams it: a warp
// takes R consecutive rows as ONE contiguous entry range (coalesced column / value loads),
// gathers z from an interleaved copy (one 16-byte load, one L2 sector, per entry instead of
// two) and keeps per-row (re, im) accumulators, combined per row by the xor tree.
__global__ void interleave_kernel(const double* __restrict__ re, const double* __restrict__ im, int64_t n,
                                  double2* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    out[i] = make_double2(re[i], im[i]);
}

template <int R, int U, bool VI>
__global__ void __launch_bounds__(256) cspmv_group_kernel(const int64_t* __restrict__ rowptr,
                                                          const int32_t* __restrict__ cols,
                                                          const double* __restrict__ vr,
                                                          const double* __restrict__ vi,
                                                          const double2* __restrict__ zc, int64_t rows,
                                                          double* __restrict__ wr, double* __restrict__ wi,
                                                          int64_t row0) {
  const int lane = threadIdx.x & 31;
  const int64_t groups = ceil_div(rows, int64_t(R));
  const int64_t nwarps = int64_t(gridDim.x) * 8;
  for (int64_t grp = blockIdx.x * int64_t(8) + (threadIdx.x >> 5); grp < groups; grp += nwarps) {
    const int64_t lr0 = grp * R;
    const long long mine = group_offsets<R>(rowptr, lr0, rows, lane);
    int64_t rb[R + 1];
#pragma unroll
    for (int k = 0; k <= R; ++k) rb[k] = __shfl_sync(0xffffffffu, mine, k);
    double sr[R], si[R];
#pragma unroll
    for (int k = 0; k < R; ++k) sr[k] = si[k] = 0.0;
    const int64_t end = rb[R];
    for (int64_t p0 = rb[0] + lane; p0 < end; p0 += 32 * U) {
      int32_t c[U];
      double a[U], b[U];
      double2 zz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = p0 + 32 * u;
        c[u] = p < end ? ld_nc_i32(cols + p) : 0;
        a[u] = p < end ? ld_nc_f64(vr + p) : 0.0;
        b[u] = (VI && p < end) ? ld_nc_f64(vi + p) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) zz[u] = p0 + 32 * u < end ? __ldg(zc + c[u]) : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t p = p0 + 32 * u;
        if (p < end) {
          int r = 0;
#pragma unroll
          for (int k = 1; k < R; ++k) r += p >= rb[k];
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k == r) {
              // (a + ib)(x + iy): re += a x - b y, im += a y + b x
              sr[k] = __fma_rn(a[u], zz[u].x, sr[k]);
              si[k] = __fma_rn(a[u], zz[u].y, si[k]);
              if (VI) {
                sr[k] = __fma_rn(-b[u], zz[u].y, sr[k]);
                si[k] = __fma_rn(b[u], zz[u].x, si[k]);
              }
            }
        }
      }
    }
    static_assert(R == 4, "fold_rows4");
    const double xr = fold_rows4(sr[0], sr[1], sr[2], sr[3], lane);
    const double xi = fold_rows4(si[0], si[1], si[2], si[3], lane);
    if (lane < R && lr0 + lane < rows) {
      wr[row0 + lr0 + lane] = xr;
      wi[row0 + lr0 + lane] = xi;
    }
  }
}

// cspmv_group_kernel<4, ., VI> with the real map's pipelining (spmv_pipe_kernel, XL): the
// next chunk's indices are requested before the current chunk's gathers are consumed, the
// values load beside the gathers, offsets run two groups ahead. Same groups, lanes and
// order of operations: the same sums bit for bit.
template <int U, bool VI>
__global__ void __launch_bounds__(256, VI ? 3 : 4) cspmv_pipe_kernel(const int64_t* __restrict__ rowptr,
                                                            const int32_t* __restrict__ cols,
                                                            const double* __restrict__ vr,
                                                            const double* __restrict__ vi,
                                                            const double2* __restrict__ zc, int64_t rows,
                                                            double* __restrict__ wr, double* __restrict__ wi,
                                                            int64_t row0) {
  constexpr int R = 4;
  const int lane = threadIdx.x & 31;
  const int groups = static_cast<int>(ceil_div(rows, int64_t(R)));
  const int g_begin = blockIdx.x * 8 + (threadIdx.x >> 5), g_step = static_cast<int>(gridDim.x) * 8;
  long long off0 = g_begin < groups ? group_offsets<R>(rowptr, int64_t(g_begin) * R, rows, lane) : 0;
  long long off1 = g_begin + g_step < groups ? group_offsets<R>(rowptr, int64_t(g_begin + g_step) * R, rows, lane) : 0;
  int32_t c[U];
  {
    const long long base = __shfl_sync(0xffffffffu, off0, 0);
    const int end = static_cast<int>(__shfl_sync(0xffffffffu, off0, R) - base);
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = lane + 32 * u < end ? ld_nc_i32(cols + base + lane + 32 * u) : 0;
  }
  for (int grp = g_begin; grp < groups; grp += g_step) {
    const int64_t lr0 = int64_t(grp) * R;
    const long long off2 =
        grp + 2 * g_step < groups ? group_offsets<R>(rowptr, int64_t(grp + 2 * g_step) * R, rows, lane) : 0;
    const long long base = __shfl_sync(0xffffffffu, off0, 0);
    const int rel = static_cast<int>(off0 - base);
    const int r1 = __shfl_sync(0xffffffffu, rel, 1), r2 = __shfl_sync(0xffffffffu, rel, 2),
              r3 = __shfl_sync(0xffffffffu, rel, 3), end = __shfl_sync(0xffffffffu, rel, 4);
    const bool more = grp + g_step < groups;
    const long long nbase = __shfl_sync(0xffffffffu, off1, 0);
    const int nend = more ? static_cast<int>(__shfl_sync(0xffffffffu, off1, R) - nbase) : 0;
    double sr[R] = {0.0, 0.0, 0.0, 0.0}, si[R] = {0.0, 0.0, 0.0, 0.0};
    int qc = 0;
    do {
      double2 zz[U];
      double a[U], b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = qc + lane + 32 * u;
        zz[u] = q < end ? __ldg(zc + c[u]) : make_double2(0.0, 0.0);
        a[u] = q < end ? ld_nc_f64(vr + base + q) : 0.0;
        b[u] = (VI && q < end) ? ld_nc_f64(vi + base + q) : 0.0;
      }
      const bool last = qc + 32 * U >= end;
      const long long pb = last ? nbase : base;
      const int pq = last ? lane : qc + 32 * U + lane, pe = last ? nend : end;
      int32_t nc[U];
#pragma unroll
      for (int u = 0; u < U; ++u) nc[u] = pq + 32 * u < pe ? ld_nc_i32(cols + pb + pq + 32 * u) : 0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int q = qc + lane + 32 * u;
        if (q < end) {
          const int r = (q >= r1) + (q >= r2) + (q >= r3);
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k == r) {
              // (a + ib)(x + iy): re += a x - b y, im += a y + b x
              sr[k] = __fma_rn(a[u], zz[u].x, sr[k]);
              si[k] = __fma_rn(a[u], zz[u].y, si[k]);
              if (VI) {
                sr[k] = __fma_rn(-b[u], zz[u].y, sr[k]);
                si[k] = __fma_rn(b[u], zz[u].x, si[k]);
              }
            }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = nc[u];
      qc += 32 * U;
    } while (qc < end);
    const double xr = fold_rows4(sr[0], sr[1], sr[2], sr[3], lane);
    const double xi = fold_rows4(si[0], si[1], si[2], si[3], lane);
    if (lane < R && lr0 + lane < rows) {
      wr[row0 + lr0 + lane] = xr;
      wi[row0 + lr0 + lane] = xi;
    }
    off0 = off1;
    off1 = off2;
  }
}

// mode 1: map ; mode 2: final residual. Fixed grid => deterministic partials.
__global__ void cmap_kernel(int mode, const double* __restrict__ zr, const double* __restrict__ zi,
                            const double* __restrict__ wr, const double* __restrict__ wi,
                            const double* __restrict__ dr, const double* __restrict__ di,
                            int64_t anchor, int64_t row0, int64_t rows, double* fr, double* fi,
                            const LoopState* st, int schedule, double snap, double* partials) {
  if (st != nullptr && st->done && mode == 1) return;
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  double scale = 1.0;
  if (mode == 1 && schedule == IPT_SCHEDULE_CONTINUATION && st) {
    const double ak = st->scale_ak;
    scale = ak <= snap ? 1.0 : 1.0 - ak;
  }
  const cd wa{wr[anchor], wi[anchor]};
  const cd da{dr[anchor], di[anchor]};
  const cd lam{da.re + wa.re, da.im + wa.im};
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < rows; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = row0 + e;
    const cd z{zr[i], zi[i]}, w{wr[i], wi[i]}, d{dr[i], di[i]};
    if (mode == 1) {
      cd f;
      if (i == anchor) {
        f = {1.0, 0.0};
      } else {
        const cd g = cdiv(cd{1.0, 0.0}, csub(d, da));
        const cd t = cmul(g, csub(cmul(z, wa), w));
        f = {scale * t.re, scale * t.im};
      }
      fr[i] = f.re;
      fi[i] = f.im;
      const cd df = csub(z, f);
      v[0] += df.re * df.re + df.im * df.im;
      v[1] += z.re * z.re + z.im * z.im;
      v[2] += f.re * f.re + f.im * f.im;
      v[3] = nan_max(v[3], hypot(df.re, df.im));
    } else {
      const cd dz = cmul(d, z), lz = cmul(lam, z);
      const cd r{dz.re + w.re - lz.re, dz.im + w.im - lz.im};
      v[0] += r.re * r.re + r.im * r.im;
      v[1] += z.re * z.re + z.im * z.im;
    }
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
}
constexpr int kCmapBlocks = 296;

template <int MODE>
void launch_spmv(unsigned grid, cudaStream_t s, const int64_t* rowptr, const int32_t* cols, const double* vals,
                 const MapArgs& a) {
  if (a.wgroups != nullptr) {  // balanced group ranges (decided per problem at upload)
    if (spmv_variant() == 19)
      spmv_group_kernel<MODE, 4, 4, 4, false, true, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a);
    else
      spmv_pipe_kernel<MODE, 3, 4, true, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a);
    return;
  }
  switch (spmv_variant()) {
#define IPT_SPMV(K, L, UU) \
  case K: spmv_map_kernel<MODE, L, UU><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
#define IPT_SPMVG(K, R, UU, MB) \
  case K: spmv_group_kernel<MODE, R, UU, MB><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    IPT_SPMV(0, 16, 4) IPT_SPMV(1, 8, 8) IPT_SPMV(2, 32, 2) IPT_SPMV(3, 8, 4) IPT_SPMV(4, 16, 6)
    IPT_SPMVG(5, 4, 4, 4) IPT_SPMVG(6, 8, 2, 4) IPT_SPMVG(7, 4, 2, 5) IPT_SPMVG(8, 4, 4, 3)
    case 9: spmv_group_kernel<MODE, 4, 4, 4, false><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    IPT_SPMVG(10, 16, 4, 3) IPT_SPMVG(11, 4, 8, 3)
    case 12: spmv_group_kernel<MODE, 2, 4, 4, false><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 13: spmv_group_kernel<MODE, 2, 8, 4, false><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 14: spmv_group_kernel<MODE, 4, 8, 4, false><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 15: spmv_group_kernel<MODE, 8, 4, 4, false><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 16: spmv_group_kernel<MODE, 4, 4, 4, false, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 17: spmv_group_kernel<MODE, 4, 4, 3, false, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 18: spmv_group_kernel<MODE, 4, 2, 5, false, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 19: spmv_group_kernel<MODE, 4, 4, 4, false, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 20: spmv_group_kernel<MODE, 4, 4, 4, false, true, false, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 24: spmv_pipe_kernel<MODE, 2, 4><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 30: spmv_pipe_kernel<MODE, 3, 4, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    case 31: spmv_pipe_kernel<MODE, 2, 4, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
    default: spmv_pipe_kernel<MODE, 3, 4, true><<<grid, 256, 0, s>>>(rowptr, cols, vals, a); break;
#undef IPT_SPMV
#undef IPT_SPMVG
  }
}

int64_t map_blocks(const SingleProblem& P) {
  if (P.cplx) return kCmapBlocks;
  const int64_t rows = P.r1 - P.r0;
  const int64_t spmv_grid = int64_t(kNumSMs) * kSpmvVariants[spmv_variant()].minb;
  return P.csr ? std::min<int64_t>(spmv_grid, ceil_div(rows, spmv_rows_per_block())) : ceil_div(rows, kRowsPerBlock);
}

MapArgs map_args(SingleProblem& P, int src) {
  MapArgs a{};
  a.d = P.dre.get();
  a.z = P.z[src].get();
  a.fz = P.z[src ^ 1].get();
  if (P.p2p && !P.cplx) {
    a.npeers = P.npeers;
    for (int q = 0; q < P.npeers; ++q) a.peer[q] = P.peer_z[src ^ 1][q];
  }
  a.wa = P.wa.get();
  a.wgroups = P.wgroups.get();
  a.anchor = P.anchor;
  a.row0 = P.r0;
  a.rows = P.r1 - P.r0;
  a.state = P.state;
  a.partials = P.partials.get();
  return a;
}

void enqueue_anchor(SingleProblem& P, int src, const LoopState* st) {
  cudaStream_t s = P.ctx->stream;
  if (P.csr) {
    switch (spmv_variant()) {
#define IPT_ANCHOR(K, L, UU)                                                                                   \
  case K:                                                                                                      \
    anchor_csr_kernel<L, UU><<<1, 32, 0, s>>>(P.acols.get(), P.arow.get(), P.annz, P.z[src].get(), P.wa.get(), st); \
    break;
      IPT_ANCHOR(0, 16, 4) IPT_ANCHOR(1, 8, 8) IPT_ANCHOR(2, 32, 2) IPT_ANCHOR(3, 8, 4) IPT_ANCHOR(4, 16, 6)
#undef IPT_ANCHOR
      default:
        anchor_csr_phase_kernel<<<1, 32, 0, s>>>(P.acols.get(), P.arow.get(), P.annz, P.anchor_phase,
                                                 P.z[src].get(), P.wa.get(), st);
        break;
    }
  } else {
    anchor_dense_kernel<<<1, 32, 0, s>>>(P.arow.get(), P.lda, P.z[src].get(), P.wa.get(), st);
  }
  IPT_LAUNCH_CHECK();
  count_launch();
}

// Complex path: w = Delta z (local rows) into P.w / P.wi (global indexing).
void enqueue_cmatvec(SingleProblem& P, int src) {
  cudaStream_t s = P.ctx->stream;
  const int64_t rows = P.r1 - P.r0;
  if (rows <= 0) return;
  if (P.csr && !P.cspmv_simple) {
    const int64_t vlen = P.n;  // the replicated iterate (global indexing)
    // (a real Delta meets a complex vector here too: kernels::matvec with complex x)
    if (P.zc.count < 2 * size_t(vlen)) P.zc.alloc(2 * size_t(std::max<int64_t>(vlen, 1)), false);
    interleave_kernel<<<static_cast<unsigned>(std::min<int64_t>(ceil_div(vlen, 256), 1184)), 256, 0, s>>>(
        P.z[src].get(), P.zi[src].get(), vlen, reinterpret_cast<double2*>(P.zc.get()));
    IPT_LAUNCH_CHECK();
    count_launch();
    // IPT_CSPMV=0: the group kernel; 2 / 3: the pipelined kernel, entries per lane in flight.
    // Complex Hermitian config-5 pattern, step with its elementwise map: 0.968 / 0.758 /
    // 0.716 ms (the thread-per-row kernel of round 1: 2.37 ms). Same sums bit for bit.
    static const int ckind = [] {
      const char* e = std::getenv("IPT_CSPMV");
      return e ? std::atoi(e) : 3;
    }();
    const double2* zc = reinterpret_cast<const double2*>(P.zc.get());
    // resident CTAs per SM: 4, or 3 for the pipelined kernel with complex values (70-78 registers)
    const int per_sm = (ckind != 0 && P.valsi.count) ? 3 : 4;
    const unsigned grid =
        static_cast<unsigned>(std::min<int64_t>(int64_t(kNumSMs) * per_sm, ceil_div(rows, int64_t(32))));
#define IPT_CSPMV_ARGS P.rowptr.get(), P.cols.get(), P.vals.get()
    if (P.valsi.count) {
      if (ckind == 0)
        cspmv_group_kernel<4, 4, true><<<grid, 256, 0, s>>>(IPT_CSPMV_ARGS, P.valsi.get(), zc, rows, P.w.get(),
                                                           P.wi.get(), P.r0);
      else if (ckind == 3)
        cspmv_pipe_kernel<3, true><<<grid, 256, 0, s>>>(IPT_CSPMV_ARGS, P.valsi.get(), zc, rows, P.w.get(),
                                                        P.wi.get(), P.r0);
      else
        cspmv_pipe_kernel<2, true><<<grid, 256, 0, s>>>(IPT_CSPMV_ARGS, P.valsi.get(), zc, rows, P.w.get(),
                                                        P.wi.get(), P.r0);
    } else {
      if (ckind == 0)
        cspmv_group_kernel<4, 4, false><<<grid, 256, 0, s>>>(IPT_CSPMV_ARGS, nullptr, zc, rows, P.w.get(),
                                                            P.wi.get(), P.r0);
      else if (ckind == 3)
        cspmv_pipe_kernel<3, false><<<grid, 256, 0, s>>>(IPT_CSPMV_ARGS, nullptr, zc, rows, P.w.get(),
                                                         P.wi.get(), P.r0);
      else
        cspmv_pipe_kernel<2, false><<<grid, 256, 0, s>>>(IPT_CSPMV_ARGS, nullptr, zc, rows, P.w.get(),
                                                         P.wi.get(), P.r0);
    }
#undef IPT_CSPMV_ARGS
  } else if (P.csr) {
    cmatvec_csr_kernel<<<static_cast<unsigned>(ceil_div(rows, 256)), 256, 0, s>>>(
        P.rowptr.get(), P.cols.get(), P.vals.get(), P.valsi.count ? P.valsi.get() : nullptr, rows,
        P.z[src].get(), P.zi[src].get(), P.w.get(), P.wi.get(), P.r0);
  } else {
    cmatvec_dense_kernel<<<static_cast<unsigned>(ceil_div(rows, 8)), 256, 0, s>>>(
        P.A.get(), P.Ai.count ? P.Ai.get() : nullptr, P.lda, rows, P.n, P.z[src].get(),
        P.zi[src].get(), P.w.get(), P.wi.get(), P.r0);
  }
  IPT_LAUNCH_CHECK();
  count_launch();
}

void allgather_z(SingleProblem& P, int buf) {
  Ctx& c = *P.ctx;
  if (c.nranks <= 1) return;
  c.comm->all_gather(P.z[buf].get(), P.chunk, CommType::F64, c.stream);
  if (P.cplx) c.comm->all_gather(P.zi[buf].get(), P.chunk, CommType::F64, c.stream);
}
void allgather_w(SingleProblem& P) {
  Ctx& c = *P.ctx;
  if (c.nranks <= 1) return;
  c.comm->all_gather(P.w.get(), P.chunk, CommType::F64, c.stream);
  c.comm->all_gather(P.wi.get(), P.chunk, CommType::F64, c.stream);
}

void reduce_and_allreduce(SingleProblem& P, const LoopState* st, bool with_max) {
  Ctx& c = *P.ctx;
  reduce_partials(c.stream, P.partials.get(), map_blocks(P), P.sums.get(), st);
  if (c.nranks > 1) {
    c.comm->all_reduce(P.sums.get(), 3, CommType::F64, CommOp::Sum, c.stream);
    if (with_max) c.comm->all_reduce(P.sums.get() + 3, 1, CommType::F64, CommOp::Max, c.stream);
  }
}

// The step's reduction / decision / next anchor value fused into the map kernel (one launch
// per step on one rank, map + decide_anchor_kernel with several): dense GEMV and the
// grouped CSR kernels (whose anchor sum the tail reproduces). IPT_SINGLE_FUSED=0: the
// separate anchor / reduction / decision launches.
bool fused_step(const SingleProblem& P) {
  static const bool on = [] {
    const char* e = std::getenv("IPT_SINGLE_FUSED");
    return !(e && e[0] == '0');
  }();
  return on && !P.cplx && (!P.csr || spmv_grouped());
}

void set_anchor_args(const SingleProblem& P, MapArgs& a) {
  if (P.csr) {
    a.a_cols = P.acols.get();
    a.a_vals = P.arow.get();
    a.a_nnz = P.annz;
    a.a_phase = P.anchor_phase;
  } else {
    a.a_cols = nullptr;
    a.a_vals = P.arow.get();
    a.a_lda = P.lda;
  }
}

void set_tail_args(SingleProblem& P, MapArgs& a, int mode, int k, const ipt_params& prm) {
  a.tail_mode = mode;
  a.tail_counter = P.tail_counter;
  a.tail_state = P.state;
  a.tail_sums = P.sums.get();
  a.tail_k = k;
  a.tail_max_iter = prm.max_iterations;
  a.tail_schedule = prm.schedule;
  a.tail_ignore = prm.ignore_convergence;
  a.tail_tol = prm.tolerance;
  a.tail_div = prm.divergence_threshold;
  a.tail_alpha = prm.shrink_alpha;
  a.tail_snap = 0.25 * prm.tolerance;
  a.tail_trace = prm.record_trace ? P.trace.get() : nullptr;
  set_anchor_args(P, a);
}

template <int MODE>
void enqueue_real_map(SingleProblem& P, int src, const ipt_params* prm, double* fz_out = nullptr,
                      int tail_mode = 0, int k = 0) {
  cudaStream_t s = P.ctx->stream;
  MapArgs a = map_args(P, src);
  if (tail_mode) set_tail_args(P, a, tail_mode, k, *prm);
  // a rank without rows still runs one CTA when the tail writes its (zero) stop sums
  const unsigned min_grid = tail_mode ? 1u : 0u;
  if (MODE == kMvFinal || MODE == kMvAccel) a.state = nullptr;
  if (fz_out) {
    a.fz = fz_out;
    a.npeers = 0;  // not the next iterate: no fused all-gather
  }
  if (prm) {
    a.schedule = prm->schedule;
    a.snap = 0.25 * prm->tolerance;
  }
  const unsigned grid = std::max(static_cast<unsigned>(map_blocks(P)), min_grid);
  if (grid == 0) return;
  if (P.csr)
    launch_spmv<MODE>(grid, s, P.rowptr.get(), P.cols.get(), P.vals.get(), a);
  else
    gemv_map_kernel<MODE><<<grid, kGemvWarps * 32, 0, s>>>(P.A.get(), P.lda, a);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void enqueue_iteration(SingleProblem& P, int k, const ipt_params& prm, cudaEvent_t ev_a = nullptr,
                       cudaEvent_t ev_b = nullptr) {
  Ctx& c = *P.ctx;
  const int src = k & 1;
  LoopState* st = P.state;
  if (fused_step(P)) {
    // w_a of z[src]: formed by the previous step's tail, else by the anchor kernel
    if (!P.wa_fresh) enqueue_anchor(P, src, st);
    if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, c.stream));
    enqueue_real_map<kMvMap>(P, src, &prm, nullptr, c.nranks > 1 ? 1 : 2, k);
    if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, c.stream));
    P.wa_fresh = true;
    if (c.nranks > 1) {
      if (!P.p2p) allgather_z(P, src ^ 1);
      c.comm->all_reduce(P.sums.get(), 3, CommType::F64, CommOp::Sum, c.stream);
      c.comm->all_reduce(P.sums.get() + 3, 1, CommType::F64, CommOp::Max, c.stream);
      MapArgs a = map_args(P, src);
      set_anchor_args(P, a);
      decide_anchor_kernel<<<1, 32, 0, c.stream>>>(
          st, P.sums.get(), k, prm.tolerance, prm.max_iterations, prm.divergence_threshold, prm.schedule,
          prm.shrink_alpha, 0.25 * prm.tolerance, prm.ignore_convergence,
          prm.record_trace ? P.trace.get() : nullptr, a);
      IPT_LAUNCH_CHECK();
      count_launch();
    }
    return;
  }
  if (!P.cplx) {
    enqueue_anchor(P, src, st);
    if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, c.stream));
    enqueue_real_map<kMvMap>(P, src, &prm);
    if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, c.stream));
  } else {
    enqueue_cmatvec(P, src);
    allgather_w(P);
    cmap_kernel<<<kCmapBlocks, 256, 0, c.stream>>>(
        1, P.z[src].get(), P.zi[src].get(), P.w.get(), P.wi.get(), P.dre.get(), P.dim.get(),
        P.anchor, P.r0, P.r1 - P.r0, P.z[src ^ 1].get(), P.zi[src ^ 1].get(), st, prm.schedule,
        0.25 * prm.tolerance, P.partials.get());
    IPT_LAUNCH_CHECK();
    count_launch();
  }
  // Real maps with peer buffers stored their rows into every rank's z in the map kernel
  // (fused all-gather); the all-reduce of the stop sums right after orders those stores
  // before any rank's next step.
  if (!(P.p2p && !P.cplx)) allgather_z(P, src ^ 1);
  reduce_and_allreduce(P, st, true);
  decide_single_kernel<<<1, 1, 0, c.stream>>>(
      st, P.sums.get(), k, prm.tolerance, prm.max_iterations, prm.divergence_threshold, prm.schedule,
      prm.shrink_alpha, 0.25 * prm.tolerance, prm.ignore_convergence,
      prm.record_trace ? P.trace.get() : nullptr);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void upload_anchor_row(SingleProblem& P) {
  cudaStream_t s = P.ctx->stream;
  const int64_t a = P.anchor;
  if (!P.csr) {
    P.arow.alloc(P.lda);
    IPT_CUDA(cudaMemcpyAsync(P.arow.get(), P.h_dense + a * P.n, sizeof(double) * P.n, cudaMemcpyHostToDevice, s));
  } else {
    const int64_t b = P.h_rowptr[a], e = P.h_rowptr[a + 1];
    P.annz = e - b;
    if (spmv_grouped()) {  // row group of the anchor on its owner rank (equal row chunks)
      const int64_t R = kSpmvVariants[spmv_variant()].rows;
      const int64_t r0o = (a / P.chunk) * P.chunk;
      const int64_t gstart = r0o + R * ((a - r0o) / R);
      P.anchor_phase = static_cast<int>((b - P.h_rowptr[gstart]) & 31);
    }
    P.arow.alloc(std::max<int64_t>(P.annz, 1));
    int32_t* ac = nullptr;
    IPT_CUDA(cudaMalloc(&ac, sizeof(int32_t) * std::max<int64_t>(P.annz, 1)));
    P.acols.reset(ac);
    if (P.annz) {
      IPT_CUDA(cudaMemcpyAsync(P.arow.get(), P.h_vals + b, sizeof(double) * P.annz, cudaMemcpyHostToDevice, s));
      IPT_CUDA(cudaMemcpyAsync(ac, P.h_cols + b, sizeof(int32_t) * P.annz, cudaMemcpyHostToDevice, s));
    }
  }
  P.ctx->sync();
}

// Fused all-gather setup: both z buffers become cudaMalloc'd and are exchanged over the
// library communicator (NCCL: CUDA IPC handles, every rank maps its peers' buffers; local
// ranks: the pointers themselves). The outcome is agreed by all ranks, so if any rank
// cannot map a peer all of them keep the collective all-gather. IPT_P2P=0 keeps it too.
void setup_peer_gather(SingleProblem& P, int64_t zlen) {
  Ctx& c = *P.ctx;
  const int g = c.nranks;
  if (g <= 1 || P.cplx || g - 1 > kMaxPeers) return;
  const char* e = std::getenv("IPT_P2P");
  if (e && e[0] == '0') return;
  // cudaMalloc'd: exportable by CUDA IPC (NCCL ranks) and peer-accessible without pool
  // access grants (local ranks on several devices)
  for (int b = 0; b < 2; ++b) P.z[b].alloc_plain(zlen);
  void* mine[2] = {P.z[0].get(), P.z[1].get()};
  void* peers[2][8] = {};
  bool ipc = false;
  const bool all_ok = c.comm->map_peers(mine, 2, peers, &ipc);
  if (!all_ok) return;
  for (int b = 0; b < 2; ++b)
    for (int q = 0; q < g - 1; ++q) P.peer_z[b][q] = static_cast<double*>(peers[b][q]);
  P.npeers = g - 1;
  P.peer_kind = ipc ? kPeerIpc : kPeerBorrowed;
  P.p2p = true;
}

}  // namespace

void single_forget_host(SingleProblem& P) {
  P.h_rowptr = nullptr;
  P.h_dense = P.h_densei = nullptr;
  P.h_cols = nullptr;
  P.h_vals = P.h_valsi = nullptr;
}

// Tests on one GPU: npeers local buffer pairs stand in for the peers' z (the map kernel
// stores its rows into them exactly as into IPC-mapped peer memory).
void single_debug_peers(SingleProblem& P, int npeers) {
  if (npeers < 0 || npeers > kMaxPeers || P.cplx || P.ctx->nranks != 1)
    throw InvalidArgument("debug peers: 0..7 peers on a real single-rank problem");
  for (int b = 0; b < 2; ++b)
    for (int q = 0; q < npeers; ++q) {
      IPT_CUDA(cudaMalloc(&P.peer_z[b][q], sizeof(double) * P.z[b].count));
      IPT_CUDA(cudaMemset(P.peer_z[b][q], 0, sizeof(double) * P.z[b].count));
    }
  P.npeers = npeers;
  P.peer_kind = kPeerOwned;
  P.p2p = npeers > 0;
}

void single_debug_peer_z(SingleProblem& P, int peer, int buf, double* out) {
  if (peer < 0 || peer >= P.npeers || buf < 0 || buf > 1) throw InvalidArgument("debug peers: bad index");
  IPT_CUDA(cudaMemcpy(out, P.peer_z[buf][peer], sizeof(double) * P.n, cudaMemcpyDeviceToHost));
}



// ------------------------------------------------------------ C++ entry points

SingleProblem* single_upload(Ctx& c, int64_t n, const double* d_re, const double* d_im, bool csr,
                             const double* dense_re, const double* dense_im, const int64_t* rowptr,
                             const int32_t* cols, const double* val_re, const double* val_im,
                             bool keep_host_anchor_source, bool force_complex, int64_t row_begin,
                             int64_t row_end) {
  NvtxRange nvtx_("ipt:single_upload");
  if (n <= 0) throw InvalidArgument("solve_single: empty problem");
  auto P = std::make_unique<SingleProblem>();
  P->ctx = &c;
  P->n = n;
  P->csr = csr;
  bool any_im = false;
  if (d_im) for (int64_t i = 0; i < n && !any_im; ++i) any_im = d_im[i] != 0.0;
  if (!csr && dense_im) for (int64_t t = 0; t < n * n && !any_im; ++t) any_im = dense_im[t] != 0.0;
  if (csr && val_im) for (int64_t t = 0; t < rowptr[n] && !any_im; ++t) any_im = val_im[t] != 0.0;
  P->cplx = any_im || force_complex;
  P->chunk = ceil_div(n, c.nranks);
  P->r0 = std::min<int64_t>(n, c.rank * P->chunk);
  P->r1 = std::min<int64_t>(n, (c.rank + 1) * P->chunk);
  if (row_begin >= 0) {  // explicit row block on a single-rank context (the unit a rank maps)
    if (c.nranks != 1) throw InvalidArgument("solve_single: explicit row blocks need a single-rank context");
    if (!(row_begin < row_end && row_end <= n)) throw InvalidArgument("solve_single: bad row block");
    P->r0 = row_begin;
    P->r1 = row_end;
  }
  const int64_t rows = P->r1 - P->r0;
  const int64_t vlen = P->chunk * c.nranks;
  cudaStream_t s = c.stream;
  ProfMarks pm("single_upload");
  if (!csr) {
    P->lda = round_up(n, 16);
    P->A.alloc(size_t(std::max<int64_t>(rows, 1)) * P->lda);
    if (rows) h2d_rows(c, P->A.get(), P->lda, dense_re + P->r0 * n, n, rows, n);  // pinned, double-buffered
    if (P->cplx && dense_im) {
      P->Ai.alloc(size_t(std::max<int64_t>(rows, 1)) * P->lda);
      if (rows)
        IPT_CUDA(cudaMemcpy2DAsync(P->Ai.get(), P->lda * sizeof(double), dense_im + P->r0 * n,
                                   n * sizeof(double), n * sizeof(double), rows, cudaMemcpyHostToDevice, s));
    }
    P->h_dense = dense_re;
    P->h_densei = dense_im;
  } else {
    const int64_t b = rowptr[P->r0], e = rowptr[P->r1];
    const int64_t nnz = e - b;
    // one pass: monotonicity check of all offsets and this rank's rebased offsets
    std::vector<int64_t> rp(rows + 1);
    for (int64_t i = 0; i < n; ++i) {
      if (rowptr[i + 1] < rowptr[i]) throw InvalidArgument("csr: row offsets must be non-decreasing");
      if (i >= P->r0 && i <= P->r1) rp[i - P->r0] = rowptr[i] - b;
    }
    rp[rows] = e - b;
    int64_t* drp = nullptr;
    IPT_CUDA(cudaMalloc(&drp, sizeof(int64_t) * (rows + 1)));
    P->rowptr.reset(drp);
    h2d_bytes(c, drp, rp.data(), sizeof(int64_t) * (rows + 1));
    const int vdef = spmv_variant();
    if ((vdef == kSpmvDefault || vdef == 19) && !P->cplx) {
      // Balanced group ranges: warp w of the map grid takes groups [gs[w], gs[w+1]),
      // cut where the running cost (nonzeros + kRowCost per row) crosses w / nwarps of the
      // total -- a few very long rows no longer pile onto one warp of the round-robin.
      // Taken when the round-robin's busiest warp would carry more than kImbalance x the
      // mean cost (tools/probes/skew_probe.py: 0.2 % of rows with 8000 entries, imbalance
      // 2.14: 0.957 -> 0.690 ms; lognormal row lengths, 1.27: 0.556 -> 0.515 ms; heavy rows
      // clustered in blocks, 1.27: 0.583 -> 0.650 ms, slower; config 5, 1.01: the
      // round-robin's interleaved streams are ~1 % faster). IPT_SPMV_VARIANT=19: always
      // balanced, IPT_SPMV_BALANCE=0: never.
      static const int64_t kRowCost = [] {  // a row's offsets and epilogue, in entry-equivalents
        const char* e = std::getenv("IPT_SPMV_ROWCOST");
        return e ? std::max<int64_t>(0, std::atoll(e)) : int64_t(16);
      }();
      constexpr double kImbalance = 1.5;
      const int R = kSpmvVariants[vdef].rows;
      const int64_t groups = ceil_div(rows, int64_t(R));
      const int64_t nw = std::max<int64_t>(map_blocks(*P), 1) * 8;
      auto cost = [&](int64_t g) {
        const int64_t r = std::min<int64_t>(g * R, rows);
        return rp[r] + kRowCost * r;
      };
      const int64_t total = cost(groups);
      bool balance = vdef == 19;
      if (!balance && groups > 0) {
        static const bool allowed = [] {
          const char* e = std::getenv("IPT_SPMV_BALANCE");
          return !(e && e[0] == '0');
        }();
        if (allowed) {
          std::vector<int64_t> rr(nw, 0);
          for (int64_t g = 0; g < groups; ++g) rr[g % nw] += cost(g + 1) - cost(g);
          const int64_t mx = *std::max_element(rr.begin(), rr.end());
          const double imb = double(mx) * double(nw) / double(std::max<int64_t>(total, 1));
          balance = imb > kImbalance;
          if (std::getenv("IPT_PROFILE"))
            std::fprintf(stderr, "[ipt] csr map: round-robin imbalance %.3f -> %s group ranges\n", imb,
                         balance ? "balanced" : "round-robin");
        }
      }
      // the round-robin kernel keeps entry positions relative to the group start in 32 bits
      for (int64_t g = 0; g < groups && !balance; ++g)
        balance = rp[std::min<int64_t>((g + 1) * R, rows)] - rp[g * R] > int64_t(INT32_MAX) - 4096;
      P->spmv_bal = balance;
    }
    if (P->spmv_bal) {
      static const int64_t kRowCost = [] {
        const char* e = std::getenv("IPT_SPMV_ROWCOST");
        return e ? std::max<int64_t>(0, std::atoll(e)) : int64_t(16);
      }();
      const int R = kSpmvVariants[spmv_variant()].rows;
      const int64_t groups = ceil_div(rows, int64_t(R));
      const int64_t nw = std::max<int64_t>(map_blocks(*P), 1) * 8;
      auto cost = [&](int64_t g) {
        const int64_t r = std::min<int64_t>(g * R, rows);
        return rp[r] + kRowCost * r;
      };
      const int64_t total = cost(groups);
      std::vector<int32_t> gs(nw + 1);
      int64_t g = 0;
      for (int64_t w = 0; w < nw; ++w) {
        const int64_t target = static_cast<int64_t>((static_cast<__int128>(total) * w) / nw);
        while (g < groups && cost(g) < target) ++g;
        gs[w] = static_cast<int32_t>(g);
      }
      gs[nw] = static_cast<int32_t>(groups);
      int32_t* dgs = nullptr;
      IPT_CUDA(cudaMalloc(&dgs, sizeof(int32_t) * (nw + 1)));
      P->wgroups.reset(dgs);
      h2d_bytes(c, dgs, gs.data(), sizeof(int32_t) * (nw + 1));
    }
    int32_t* dc = nullptr;
    IPT_CUDA(cudaMalloc(&dc, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
    P->cols.reset(dc);
    P->vals.alloc(std::max<int64_t>(nnz, 1), false);
    pm.mark("rowptr");
    if (nnz) {  // pinned staging: ~4x the pageable copy rate for the 1.6 GB of config 5
      h2d_bytes(c, dc, cols + b, sizeof(int32_t) * nnz);
      h2d_bytes(c, P->vals.get(), val_re + b, sizeof(double) * nnz);
    }
    pm.mark("h2d");
    if (P->cplx && val_im) {
      P->valsi.alloc(std::max<int64_t>(nnz, 1), false);
      if (nnz) IPT_CUDA(cudaMemcpyAsync(P->valsi.get(), val_im + b, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
    }
    P->nnz_total = rowptr[n] - rowptr[0];
    if (keep_host_anchor_source) {
      P->h_rowptr = rowptr;
    } else {
      P->h_rowptr_copy.assign(rowptr, rowptr + n + 1);
      P->h_rowptr = P->h_rowptr_copy.data();
    }
    if (keep_host_anchor_source) {
      P->h_cols = cols;
      P->h_vals = val_re;
      P->h_valsi = val_im;
    } else {
      P->h_cols_copy.assign(cols, cols + rowptr[n]);
      P->h_vals_copy.assign(val_re, val_re + rowptr[n]);
      P->h_cols = P->h_cols_copy.data();
      P->h_vals = P->h_vals_copy.data();
    }
  }
  P->dre.alloc(n);
  P->dim.alloc(n);
  h2d_bytes(c, P->dre.get(), d_re, sizeof(double) * n);
  if (d_im) h2d_bytes(c, P->dim.get(), d_im, sizeof(double) * n);
  // z vectors padded to a multiple of 2 for the 16-byte GEMV loads (pad stays zero)
  const int64_t zlen = round_up(std::max(vlen, P->lda), 16);
  for (int b2 = 0; b2 < 2; ++b2) {
    P->z[b2].alloc(zlen);
    P->zi[b2].alloc(zlen);
  }
  pm.mark("host_copies");
  setup_peer_gather(*P, zlen);
  P->w.alloc(zlen);
  P->wi.alloc(zlen);
  if (P->csr && P->cplx) P->zc.alloc(2 * size_t(std::max<int64_t>(n, 1)), false);
  P->cspmv_simple = std::getenv("IPT_CSPMV_SIMPLE") != nullptr;
  P->wa.alloc(2);
  P->npart = std::max<int64_t>(map_blocks(*P), 1);
  P->partials.alloc(size_t(P->npart) * 4);
  // 4 stop sums, a barrier token (single_reset) and the fused tail's arrival counter (a
  // zeroed 8-byte slot: the counter is an unsigned in it)
  P->sums.alloc(6);
  P->tail_counter = reinterpret_cast<unsigned*>(P->sums.get() + 5);
  IPT_CUDA(cudaMalloc(&P->state, sizeof(LoopState)));
  pm.mark("allocs");
  c.sync();
  return P.release();
}

void single_free(SingleProblem* P) { delete P; }

// Warm start: renormalised to z[anchor] = 1 (solver.cpp:39-43), uploaded.
static void single_reset_warm(SingleProblem& P, int64_t anchor, const double* warm_re, const double* warm_im,
                       bool renormalize) {
  cudaStream_t s = P.ctx->stream;
  const int64_t n = P.n;
  std::vector<double> zr(n, 0.0), zi(n, 0.0);
  if (!renormalize) {
    for (int64_t j = 0; j < n; ++j) {
      zr[j] = warm_re[j];
      zi[j] = warm_im ? warm_im[j] : 0.0;
    }
  } else {
    const double ar = warm_re[anchor], ai = warm_im ? warm_im[anchor] : 0.0;
    if (ar == 0.0 && ai == 0.0) throw InvalidArgument("solver: warm start has zero anchor coordinate");
    if (!P.cplx && (warm_im == nullptr || ai == 0.0)) {
      for (int64_t j = 0; j < n; ++j) zr[j] = warm_re[j] / ar;
      if (warm_im) for (int64_t j = 0; j < n; ++j) zi[j] = warm_im[j] / ar;
    } else {
      const double den = ar * ar + ai * ai;  // (x + iy) / (ar + i ai)
      for (int64_t j = 0; j < n; ++j) {
        const double x = warm_re[j], y = warm_im ? warm_im[j] : 0.0;
        const std::complex<double> q = std::complex<double>(x, y) / std::complex<double>(ar, ai);
        zr[j] = q.real();
        zi[j] = q.imag();
        (void)den;
      }
    }
    zr[anchor] = 1.0;
    zi[anchor] = 0.0;
    bool im_nonzero = false;
    for (int64_t j = 0; j < n && !im_nonzero; ++j) im_nonzero = zi[j] != 0.0;
    if (im_nonzero && !P.cplx) throw InvalidArgument("solver: complex warm start on a real problem");
  }
  fill_zero(s, P.z[0].get(), P.z[0].count);
  fill_zero(s, P.z[1].get(), P.z[1].count);
  fill_zero(s, P.zi[0].get(), P.zi[0].count);
  fill_zero(s, P.zi[1].get(), P.zi[1].count);
  IPT_CUDA(cudaMemcpyAsync(P.z[0].get(), zr.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  IPT_CUDA(cudaMemcpyAsync(P.zi[0].get(), zi.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  P.ctx->sync();  // (zr / zi are about to go out of scope)
}

static void finish_reset(SingleProblem& P, int max_iter_hint) {
  Ctx& c = *P.ctx;
  cudaStream_t s = c.stream;
  if (P.trace_cap < max_iter_hint) {
    P.trace.alloc(max_iter_hint);
    P.trace_cap = max_iter_hint;
  }
  P.enq = 0;
  P.wa_fresh = false;
  // Fused all-gather: peers store rows of step 0 into this rank's z[1] (zeroed above) and,
  // across solves, into buffers this rank may still be reading (a previous finalize). A
  // stream-ordered all-reduce here orders every rank's reset (and everything before it)
  // before any rank's first map.
  if (P.p2p && c.nranks > 1) c.comm->all_reduce(P.sums.get() + 4, 1, CommType::F64, CommOp::Sum, s);
  c.sync();
}

void single_reset(SingleProblem& P, int64_t anchor, const double* warm_re, const double* warm_im,
                  int max_iter_hint, bool renormalize) {
  NvtxRange nvtx_("ipt:single_reset");
  Ctx& c = *P.ctx;
  cudaStream_t s = c.stream;
  if (anchor < 0 || anchor >= P.n) throw InvalidArgument("solver: anchor out of range");
  if (anchor != P.anchor) {
    P.anchor = anchor;
    if (!P.cplx) upload_anchor_row(P);
  }
  if (warm_re == nullptr) {  // e_anchor, set on the device (no host vector of n doubles)
    fill_zero(s, P.z[0].get(), P.z[0].count);
    fill_zero(s, P.z[1].get(), P.z[1].count);
    fill_zero(s, P.zi[0].get(), P.zi[0].count);
    fill_zero(s, P.zi[1].get(), P.zi[1].count);
    const double one = 1.0;
    IPT_CUDA(cudaMemcpyAsync(P.z[0].get() + anchor, &one, sizeof(double), cudaMemcpyHostToDevice, s));
  } else {
    single_reset_warm(P, anchor, warm_re, warm_im, renormalize);
  }
  LoopState init{};
  init.status = kMaxIterations;
  init.scale_ak = 1.0;
  IPT_CUDA(cudaMemcpyAsync(P.state, &init, sizeof(LoopState), cudaMemcpyHostToDevice, s));
  finish_reset(P, max_iter_hint);
}

void single_iterate(SingleProblem& P, const ipt_params& prm, ipt_stats* stats) {
  NvtxRange nvtx_("ipt:single_iterate");
  Ctx& c = *P.ctx;
  if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
  if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
  if (!(prm.divergence_threshold > 1.0)) throw InvalidArgument("config: divergence_threshold must exceed 1");
  if (prm.schedule == IPT_SCHEDULE_CONTINUATION && !(prm.shrink_alpha >= 0.0 && prm.shrink_alpha < 1.0))
    throw InvalidArgument("continuation: shrink factor must lie in [0, 1)");
  if (P.anchor < 0) throw InvalidArgument("single: reset() must set an anchor first");
  if (prm.record_trace && P.trace_cap < prm.max_iterations) {
    P.trace.alloc(prm.max_iterations);
    P.trace_cap = prm.max_iterations;
  }
  // Iterations are enqueued in batches between host checks; iterations past the
  // decision exit at their first instruction (LoopState::done).
  const int64_t bytes_per_it = P.csr ? P.nnz_total * 12 : P.n * P.n * 8;
  const int batch = bytes_per_it >= (int64_t(1) << 31) ? 2 : 32;
  IPT_CUDA(cudaEventRecord(c.ev[0], c.stream));
  while (P.enq < prm.max_iterations) {
    for (int b = 0; b < batch && P.enq < prm.max_iterations; ++b) enqueue_iteration(P, P.enq++, prm);
    IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (c.h_state->done) break;
  }
  IPT_CUDA(cudaEventRecord(c.ev[1], c.stream));
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  if (stats) {
    float ms = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
    const LoopState& h = *c.h_state;
    stats->iterations = h.iterations;
    stats->status = h.status;
    stats->final_step = h.final_step;
    stats->final_max_abs = h.final_max_abs;
    stats->product_count = h.iterations;
    stats->ms_loop = ms;
    if (prm.record_trace && stats->trace && h.iterations > 0)
      IPT_CUDA(cudaMemcpy(stats->trace, P.trace.get(), sizeof(double) * h.iterations, cudaMemcpyDeviceToHost));
  }
}

// Post-loop product, eigenvalue lambda = d_a + (Delta z)_a and residual (solver.cpp:83-91).
void single_finalize(SingleProblem& P, ipt_stats* stats) {
  NvtxRange nvtx_("ipt:single_finalize");
  Ctx& c = *P.ctx;
  P.wa_fresh = false;
  cudaStream_t s = c.stream;
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
  c.sync();
  const int cur = c.h_state->iterations & 1;
  IPT_CUDA(cudaEventRecord(c.ev[0], s));
  double wa[2] = {0.0, 0.0};
  if (!P.cplx) {
    enqueue_anchor(P, cur, nullptr);
    enqueue_real_map<kMvFinal>(P, cur, nullptr);
    IPT_CUDA(cudaMemcpyAsync(wa, P.wa.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  } else {
    enqueue_cmatvec(P, cur);
    allgather_w(P);
    cmap_kernel<<<kCmapBlocks, 256, 0, s>>>(2, P.z[cur].get(), P.zi[cur].get(), P.w.get(), P.wi.get(),
                                            P.dre.get(), P.dim.get(), P.anchor, P.r0, P.r1 - P.r0,
                                            nullptr, nullptr, nullptr, 0, 0.0, P.partials.get());
    IPT_LAUNCH_CHECK();
    count_launch();
    IPT_CUDA(cudaMemcpyAsync(wa, P.w.get() + P.anchor, sizeof(double), cudaMemcpyDeviceToHost, s));
    IPT_CUDA(cudaMemcpyAsync(wa + 1, P.wi.get() + P.anchor, sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  reduce_and_allreduce(P, nullptr, false);
  double h4[4];
  IPT_CUDA(cudaMemcpyAsync(h4, P.sums.get(), sizeof(h4), cudaMemcpyDeviceToHost, s));
  IPT_CUDA(cudaEventRecord(c.ev[1], s));
  c.sync();
  if (stats) {
    float ms = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms, c.ev[0], c.ev[1]));
    std::vector<double> dr(1), di(1);
    IPT_CUDA(cudaMemcpy(dr.data(), P.dre.get() + P.anchor, sizeof(double), cudaMemcpyDeviceToHost));
    IPT_CUDA(cudaMemcpy(di.data(), P.dim.get() + P.anchor, sizeof(double), cudaMemcpyDeviceToHost));
    stats->eigenvalue_re = dr[0] + wa[0];
    stats->eigenvalue_im = P.cplx ? di[0] + wa[1] : 0.0;
    stats->residual = std::sqrt(h4[0]) / std::sqrt(h4[1]);
    stats->product_count = c.h_state->iterations + 1;
    stats->ms_final = ms;
  }
}

void single_download(SingleProblem& P, double* z_re, double* z_im) {
  NvtxRange nvtx_("ipt:single_download");
  Ctx& c = *P.ctx;
  const int cur = c.h_state->iterations & 1;
  if (z_re) IPT_CUDA(cudaMemcpy(z_re, P.z[cur].get(), sizeof(double) * P.n, cudaMemcpyDeviceToHost));
  if (z_im) {
    if (P.cplx) IPT_CUDA(cudaMemcpy(z_im, P.zi[cur].get(), sizeof(double) * P.n, cudaMemcpyDeviceToHost));
    else std::memset(z_im, 0, sizeof(double) * P.n);
  }
}

// Bench / profiling: exactly `count` further iterations (convergence ignored), timed on the
// library stream: the whole sequence and the fused GEMV/SpMV map kernel alone.
void single_run_steps(SingleProblem& P, int count, double* ms_total, double* ms_map) {
  Ctx& c = *P.ctx;
  P.wa_fresh = false;
  ipt_params prm;
  ipt_default_params(&prm);
  prm.max_iterations = 0x7fffffff;
  prm.ignore_convergence = 1;
  prm.divergence_threshold = 1.0e300;
  LoopState init{};
  init.status = kMaxIterations;
  init.scale_ak = 1.0;
  IPT_CUDA(cudaMemcpyAsync(P.state, &init, sizeof(LoopState), cudaMemcpyHostToDevice, c.stream));
  std::vector<cudaEvent_t> ev(2 * size_t(count) + 2);
  for (auto& e : ev) IPT_CUDA(cudaEventCreate(&e));
  c.sync();
  IPT_CUDA(cudaEventRecord(ev[0], c.stream));
  for (int i = 0; i < count; ++i) enqueue_iteration(P, P.enq++, prm, ev[2 + 2 * i], ev[3 + 2 * i]);
  IPT_CUDA(cudaEventRecord(ev[1], c.stream));
  c.sync();
  float ms = 0.f;
  IPT_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  *ms_total = ms;
  double m = 0.0;
  for (int i = 0; i < count && !P.cplx; ++i) {
    IPT_CUDA(cudaEventElapsedTime(&ms, ev[2 + 2 * i], ev[3 + 2 * i]));
    m += ms;
  }
  *ms_map = m;
  for (auto& e : ev) cudaEventDestroy(e);
}

// kernels::matvec on device-resident data: y = Delta x (one pass, no epilogue).
void single_matvec(SingleProblem& P, const double* x_re, const double* x_im, double* y_re, double* y_im) {
  NvtxRange nvtx_("ipt:single_matvec");
  Ctx& c = *P.ctx;
  P.wa_fresh = false;
  cudaStream_t s = c.stream;
  const int64_t n = P.n;
  IPT_CUDA(cudaMemcpyAsync(P.z[0].get(), x_re, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (x_im) IPT_CUDA(cudaMemcpyAsync(P.zi[0].get(), x_im, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  else fill_zero(s, P.zi[0].get(), n);
  if (!P.cplx && (x_im == nullptr)) {
    MapArgs a = map_args(P, 0);
    a.state = nullptr;
    a.fz = P.w.get();
    const unsigned grid = static_cast<unsigned>(map_blocks(P));
    if (grid) {
      if (P.csr) launch_spmv<kMvStore>(grid, s, P.rowptr.get(), P.cols.get(), P.vals.get(), a);
      else gemv_map_kernel<kMvStore><<<grid, kGemvWarps * 32, 0, s>>>(P.A.get(), P.lda, a);
      IPT_LAUNCH_CHECK();
      count_launch();
    }
    fill_zero(s, P.wi.get(), n);
  } else {
    enqueue_cmatvec(P, 0);
  }
  if (c.nranks > 1) allgather_w(P);
  IPT_CUDA(cudaMemcpyAsync(y_re, P.w.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  if (y_im) IPT_CUDA(cudaMemcpyAsync(y_im, P.wi.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
  c.sync();
}


// ======================================================================================
// Anderson-accelerated single pair (solve_single_accelerated, proj/src/anderson.cpp:15-247),
// real inputs, one device. Per pass: the fused kMvAccel map kernel gives the true residual
// |Dz + w - lambda z| (the stop test, anderson.cpp:204-215) and the plain image f(z) in
// one sweep of Delta; the memory-m mixing (anderson.cpp:95-178) runs on device vectors:
// difference columns, modified Gram-Schmidt with one reorthogonalisation pass, the
// affine recombination of the stored images and the anchor re-pin. Every inner product is
// a fixed-order reduction; the h x h triangular / Tikhonov solves run on the host.
// ======================================================================================
namespace {

constexpr int kVecBlocks = 296;

__global__ void vdot_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                            double* __restrict__ partials) {
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    v[0] = __fma_rn(a[i], b[i], v[0]);
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = 0.0; o[2] = 0.0; o[3] = 0.0;
  }
}
// y -= c[0] * x   (MGS projection, anderson.cpp:32)
__global__ void vaxpy_kernel(double* __restrict__ y, const double* __restrict__ x, int64_t n, const double* c) {
  const double cc = *c;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = __fma_rn(-cc, x[i], y[i]);
}
// q = v / sqrt(nn[0])   (anderson.cpp:38-39)
__global__ void vnormalize_kernel(double* __restrict__ q, const double* __restrict__ v, int64_t n, const double* nn) {
  const double vn = sqrt(*nn);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    q[i] = v[i] / vn;
}
__global__ void vsub_kernel(double* __restrict__ d, const double* __restrict__ a, const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    d[i] = __dsub_rn(a[i], b[i]);
}
struct ImgList {
  const double* img[17];
  double w[17];
  int count;
};
// next = sum_j w_j img_j, accumulated in j order from 0 (anderson.cpp:154-159)
__global__ void vcombine_kernel(double* __restrict__ next, const ImgList L, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < L.count; ++j) s = __fma_rn(L.w[j], L.img[j][i], s);
    next[i] = s;
  }
}
// re-pin the chart coordinate (anderson.cpp:162-167): divide by next[a] unless it is 0 or 1
__global__ void vrepin_kernel(double* __restrict__ next, int64_t n, int64_t anchor, const double* za_p) {
  const double za = *za_p;
  const bool div = za != 0.0 && za != 1.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if (i == anchor) next[i] = 1.0;
    else if (div) next[i] = next[i] / za;
  }
}
__global__ void copy_scalar_kernel(double* dst, const double* src) { *dst = *src; }

struct AccelWork {
  SingleProblem& P;
  int64_t n;
  cudaStream_t s;
  DevBuf part, scal;
  int next_slot = 0;
  explicit AccelWork(SingleProblem& p) : P(p), n(p.n), s(p.ctx->stream) {
    part.alloc(size_t(kVecBlocks) * 4);
    scal.alloc(4 * 1024);
  }
  double* slot() {  // a fresh 4-double device scalar slot (reset each iteration)
    if (next_slot >= 1024) throw InvalidArgument("anderson: scalar pool exhausted");
    return scal.get() + 4 * (next_slot++);
  }
  double* dot(const double* a, const double* b) {
    double* out = slot();
    vdot_kernel<<<kVecBlocks, 256, 0, s>>>(a, b, n, part.get());
    reduce_partials(s, part.get(), kVecBlocks, out, nullptr);
    count_launch();
    return out;
  }
  void axpy(double* y, const double* x, const double* c) {
    vaxpy_kernel<<<kVecBlocks, 256, 0, s>>>(y, x, n, c);
    count_launch();
  }
  void normalize(double* q, const double* v, const double* nn) {
    vnormalize_kernel<<<kVecBlocks, 256, 0, s>>>(q, v, n, nn);
    count_launch();
  }
  void sub(double* d, const double* a, const double* b) {
    vsub_kernel<<<kVecBlocks, 256, 0, s>>>(d, a, b, n);
    count_launch();
  }
  void copy(double* d, const double* a) { IPT_CUDA(cudaMemcpyAsync(d, a, sizeof(double) * n, cudaMemcpyDeviceToDevice, s)); }
};

// Host replica of lu_factor / lu_solve for the tiny Tikhonov system (lu.cpp:10-69).
bool small_lu_solve(std::vector<double> a, int h, std::vector<double> b, std::vector<double>& x) {
  std::vector<int> perm(h);
  for (int i = 0; i < h; ++i) perm[i] = i;
  double scale = 0.0;
  for (double v : a) scale = std::max(scale, std::fabs(v));
  const double tiny = scale * 2.220446049250313e-16 * h;
  for (int k = 0; k < h; ++k) {
    int piv = k;
    double best = std::fabs(a[k * h + k]);
    for (int i = k + 1; i < h; ++i)
      if (std::fabs(a[i * h + k]) > best) best = std::fabs(a[i * h + k]), piv = i;
    if (best <= tiny) return false;
    if (piv != k) {
      for (int j = 0; j < h; ++j) std::swap(a[k * h + j], a[piv * h + j]);
      std::swap(perm[k], perm[piv]);
    }
    for (int i = k + 1; i < h; ++i) {
      const double m = a[i * h + k] / a[k * h + k];
      a[i * h + k] = m;
      if (m != 0.0)
        for (int j = k + 1; j < h; ++j) a[i * h + j] -= m * a[k * h + j];
    }
  }
  x.assign(h, 0.0);
  for (int i = 0; i < h; ++i) x[i] = b[perm[i]];
  for (int i = 1; i < h; ++i)
    for (int j = 0; j < i; ++j) x[i] -= a[i * h + j] * x[j];
  for (int i = h - 1; i >= 0; --i) {
    for (int j = i + 1; j < h; ++j) x[i] -= a[i * h + j] * x[j];
    x[i] /= a[i * h + i];
  }
  for (double v : x)
    if (!std::isfinite(v)) return false;
  return true;
}

}  // namespace

void single_accelerated(SingleProblem& P, const ipt_params& prm, int memory, double residual_tol,
                        double regularization, ipt_stats* stats) {
  NvtxRange nvtx_("ipt:single_accelerated");
  Ctx& c = *P.ctx;
  P.wa_fresh = false;
  if (P.cplx) throw InvalidArgument("solve_single_accelerated (device): real inputs only");
  if (c.nranks != 1) throw InvalidArgument("solve_single_accelerated (device): single GPU only");
  if (memory < 0 || memory > 16) throw InvalidArgument("anderson: memory must lie in [0, 16]");
  if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
  if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
  const int64_t n = P.n;
  AccelWork W(P);
  cudaStream_t s = W.s;
  // work vectors (length of the padded iterate so the GEMV's 16-byte loads stay in bounds)
  const size_t vlen = P.z[0].count;
  DevBuf fzb, gcur, vtmp, nxt;
  fzb.alloc(vlen);
  gcur.alloc(vlen);
  vtmp.alloc(vlen);
  nxt.alloc(vlen);
  std::vector<DevBuf> Hg(memory + 1), Hf(memory + 1), Q(std::max(memory, 1)), Cc(std::max(memory, 1));
  for (auto& b : Hg) b.alloc(vlen);
  for (auto& b : Hf) b.alloc(vlen);
  for (auto& b : Q) b.alloc(vlen);
  for (auto& b : Cc) b.alloc(vlen);
  std::vector<int> hist;  // slot indices into Hg/Hf, oldest first
  std::vector<int> free_slots;
  for (int k = memory; k >= 0; --k) free_slots.push_back(k);
  double prev_res = -1.0;
  int streak = 0;
  std::vector<double> trace;
  int cur = 0;  // z lives in P.z[cur]
  int iterations = 0, status = kMaxIterations;
  long matvecs = 0;
  double final_step = 0.0, lam = 0.0, resid = 0.0;
  bool finished = false;
  std::vector<double> h4(4);
  auto fetch = [&](const double* dptr, double* out, int count) {
    IPT_CUDA(cudaMemcpyAsync(out, dptr, sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  };
  for (int k = 0; k < prm.max_iterations; ++k) {
    W.next_slot = 0;
    enqueue_anchor(P, cur, nullptr);
    enqueue_real_map<kMvAccel>(P, cur, &prm, fzb.get());
    reduce_partials(s, P.partials.get(), map_blocks(P), P.sums.get(), nullptr);
    double wa = 0.0;
    fetch(P.sums.get(), h4.data(), 4);
    fetch(P.wa.get(), &wa, 1);
    c.sync();
    ++matvecs;
    iterations = k + 1;
    const double da = [&] {
      double v = 0.0;
      IPT_CUDA(cudaMemcpy(&v, P.dre.get() + P.anchor, sizeof(double), cudaMemcpyDeviceToHost));
      return v;
    }();
    const double lambda = da + wa;
    const double rnorm = std::sqrt(h4[0]), znorm = std::sqrt(h4[1]);
    if (rnorm <= residual_tol) {
      lam = lambda;
      resid = rnorm / znorm;
      status = kConverged;
      finished = true;
      break;
    }
    const double step = std::sqrt(h4[2]) / std::sqrt(h4[1]);  // rel_step(z, fz)
    const double res = std::sqrt(h4[2]);                       // |f(z) - z|
    // restart after three consecutive worsening residuals (anderson.cpp:99-112)
    if (prev_res >= 0.0 && res > prev_res) {
      if (++streak >= 3) {
        for (int sl : hist) free_slots.push_back(sl);
        hist.clear();
        streak = 0;
      }
    } else {
      streak = 0;
    }
    prev_res = res;
    double* z = P.z[cur].get();
    W.sub(gcur.get(), fzb.get(), z);  // g = f(z) - z
    const int h = static_cast<int>(hist.size());
    double* znew = nullptr;
    if (memory == 0 || h == 0) {
      znew = fzb.get();
    } else {
      // difference columns C_j = g_{j+1} - g_j over the history extended by the current g
      for (int j = 0; j < h; ++j) W.sub(Cc[j].get(), j + 1 < h ? Hg[hist[j + 1]].get() : gcur.get(), Hg[hist[j]].get());
      double* fro_parts[17];
      for (int j = 0; j < h; ++j) fro_parts[j] = W.dot(Cc[j].get(), Cc[j].get());
      // MGS with reorthogonalisation (anderson.cpp:26-40)
      std::vector<std::vector<double*>> rc(h, std::vector<double*>(h * 2, nullptr));
      std::vector<double*> vn2(h);
      for (int j = 0; j < h; ++j) {
        W.copy(vtmp.get(), Cc[j].get());
        for (int pass = 0; pass < 2; ++pass)
          for (int i = 0; i < j; ++i) {
            double* cc = W.dot(Q[i].get(), vtmp.get());
            rc[j][pass * h + i] = cc;
            W.axpy(vtmp.get(), Q[i].get(), cc);
          }
        vn2[j] = W.dot(vtmp.get(), vtmp.get());
        W.normalize(Q[j].get(), vtmp.get(), vn2[j]);
      }
      std::vector<double*> bq(h);
      for (int i = 0; i < h; ++i) bq[i] = W.dot(Q[i].get(), gcur.get());
      std::vector<double> S(4 * 1024);
      fetch(W.scal.get(), S.data(), 4 * W.next_slot);
      c.sync();
      auto val = [&](double* d) { return S[static_cast<size_t>(d - W.scal.get())]; };
      double fro = 0.0;
      for (int j = 0; j < h; ++j) fro += val(fro_parts[j]);
      fro = std::sqrt(fro);
      const double rank_tol = 1e-13 * fro;
      std::vector<double> R(h * h, 0.0), b(h), gamma;
      bool ok = true;
      for (int j = 0; j < h && ok; ++j) {
        for (int pass = 0; pass < 2; ++pass)
          for (int i = 0; i < j; ++i) R[i * h + j] += val(rc[j][pass * h + i]);
        const double vn = std::sqrt(val(vn2[j]));
        if (!(vn > rank_tol)) ok = false;
        R[j * h + j] = vn;
      }
      if (ok) {
        for (int i = 0; i < h; ++i) b[i] = val(bq[i]);
        gamma.assign(h, 0.0);
        for (int ii = h - 1; ii >= 0; --ii) {
          double sacc = b[ii];
          for (int j = ii + 1; j < h; ++j) sacc -= R[ii * h + j] * gamma[j];
          gamma[ii] = sacc / R[ii * h + ii];
        }
      } else {  // Tikhonov-regularised normal equations (anderson.cpp:55-79)
        W.next_slot = 0;
        std::vector<double*> gram(h * h), gb(h);
        for (int i = 0; i < h; ++i) {
          for (int j = 0; j < h; ++j) gram[i * h + j] = W.dot(Cc[i].get(), Cc[j].get());
          gb[i] = W.dot(Cc[i].get(), gcur.get());
        }
        fetch(W.scal.get(), S.data(), 4 * W.next_slot);
        c.sync();
        std::vector<double> A(h * h), bb(h);
        double sc = 0.0;
        for (int i = 0; i < h; ++i) {
          for (int j = 0; j < h; ++j) A[i * h + j] = val(gram[i * h + j]);
          sc = std::max(sc, std::fabs(A[i * h + i]));
          bb[i] = val(gb[i]);
        }
        const double lambda_reg = (regularization > 0.0 ? regularization : 1e-12) * sc;
        for (int i = 0; i < h; ++i) A[i * h + i] += lambda_reg;
        ok = small_lu_solve(A, h, bb, gamma);
      }
      if (!ok) {
        znew = fzb.get();
      } else {
        ImgList L{};
        L.count = h + 1;
        L.w[0] = gamma[0];
        for (int j = 1; j < h; ++j) L.w[j] = gamma[j] - gamma[j - 1];
        L.w[h] = 1.0 - gamma[h - 1];
        for (int j = 0; j < h; ++j) L.img[j] = Hf[hist[j]].get();
        L.img[h] = fzb.get();
        vcombine_kernel<<<kVecBlocks, 256, 0, s>>>(nxt.get(), L, n);
        double* za = W.slot();
        copy_scalar_kernel<<<1, 1, 0, s>>>(za, nxt.get() + P.anchor);
        vrepin_kernel<<<kVecBlocks, 256, 0, s>>>(nxt.get(), n, P.anchor, za);
        count_launch(3);
        znew = nxt.get();
      }
    }
    // push (g, f(z)) and drop the oldest beyond the memory (anderson.cpp:169-175)
    if (memory > 0) {
      const int slot = free_slots.back();
      free_slots.pop_back();
      W.copy(Hg[slot].get(), gcur.get());
      W.copy(Hf[slot].get(), fzb.get());
      hist.push_back(slot);
      while (static_cast<int>(hist.size()) > memory) {
        free_slots.push_back(hist.front());
        hist.erase(hist.begin());
      }
    }
    W.copy(P.z[cur ^ 1].get(), znew);
    cur ^= 1;
    final_step = step;
    if (prm.record_trace) trace.push_back(step);
    double* zz = W.dot(P.z[cur].get(), P.z[cur].get());
    double zn2 = 0.0;
    fetch(zz, &zn2, 1);
    c.sync();
    const double zn = std::sqrt(zn2);
    if (!std::isfinite(zn) || zn > prm.divergence_threshold) {
      status = kDiverged;
      break;
    }
  }
  if (!finished) {  // closing product (anderson.cpp:238-245)
    enqueue_anchor(P, cur, nullptr);
    enqueue_real_map<kMvFinal>(P, cur, nullptr);
    reduce_partials(s, P.partials.get(), map_blocks(P), P.sums.get(), nullptr);
    double wa = 0.0, da = 0.0;
    fetch(P.sums.get(), h4.data(), 4);
    fetch(P.wa.get(), &wa, 1);
    c.sync();
    IPT_CUDA(cudaMemcpy(&da, P.dre.get() + P.anchor, sizeof(double), cudaMemcpyDeviceToHost));
    ++matvecs;
    lam = da + wa;
    resid = std::sqrt(h4[0]) / std::sqrt(h4[1]);
  }
  // expose the result where single_download reads it (P.z[iterations & 1])
  LoopState st{};
  st.iterations = iterations;
  st.status = status;
  st.done = 1;
  st.final_step = final_step;
  if (cur != (iterations & 1)) {
    IPT_CUDA(cudaMemcpyAsync(P.z[iterations & 1].get(), P.z[cur].get(), sizeof(double) * n,
                             cudaMemcpyDeviceToDevice, s));
  }
  IPT_CUDA(cudaMemcpyAsync(P.state, &st, sizeof(LoopState), cudaMemcpyHostToDevice, s));
  *c.h_state = st;
  c.sync();
  if (stats) {
    stats->iterations = iterations;
    stats->status = status;
    stats->final_step = final_step;
    stats->residual = resid;
    stats->eigenvalue_re = lam;
    stats->eigenvalue_im = 0.0;
    stats->product_count = matvecs;
    if (prm.record_trace && stats->trace)
      std::memcpy(stats->trace, trace.data(), sizeof(double) * trace.size());
  }
}
}  // namespace iptb
