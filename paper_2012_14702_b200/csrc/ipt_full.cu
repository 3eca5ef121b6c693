// Full-spectrum IPT on the device: solve_full / apply_map_full
// (proj/src/solver.cpp:156-273), column-sharded over a NCCL communicator.
//
// HBM layout (per rank):
//   Delta : rows_pad x ld, row-major, zero-padded (ld = round_up(n,16), rows_pad = round_up(n,128)).
//           Complex inputs keep A1 = Dr, A2 = Di, A3 = Dr + Di (rows_pad x ld each) so
//           that W = Delta Z is three real DMMA GEMMs (3M): T1 = Dr Zr, T2 = Di Zi, and
//           T3 = A3 (Zr + Zi) whose epilogue forms W and applies the complex map.
//   Z[2]  : ping-pong column blocks, column-major, ldz = ld (real) or 2ld ([re; im] per column),
//           cols_pad = round_up(ncols,128) columns; this rank owns global columns [col0, col0+ncols).
//   d     : n, replicated; wd / lam : per local column.
//   Sparse real Delta (CSR, f2): int64 row offsets, int32 columns, fp64 values; Z[2]
//           hold the local columns ROW-major during the loop (see FullProblem).
// Per iteration: K2 diag pre-pass (wd_j = (Delta Z)_jj), K1 DMMA GEMM with the fused map
// epilogue writing F(Z) into the other Z buffer and per-CTA partial sums, a fixed-order
// reduction, [NCCL all-reduce of 3 sums + 1 max], and a single-thread decide kernel
// that applies the reference's divergence-then-convergence tests (solver.cpp:236-249).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <utility>
#include <vector>

#include "dmma_gemm.cuh"
#include "ipt_internal.cuh"
#include "ozaki.cuh"

namespace iptb {

struct FullProblem {
  Ctx* ctx = nullptr;
  int64_t n = 0, ld = 0, rows_pad = 0;
  int64_t col0 = 0, ncols = 0, cols_pad = 0;
  bool cplx = false;
  DevBuf A1, A2, A3;        // real: A1 = Delta; complex: Dr, Di, Dr + Di
  int64_t lda = 0;  // = K of the GEMM
  DevBuf dre, dim;
  DevBuf Z[2];
  int64_t ldz = 0;
  DevBuf T1, T2, S;         // complex only: Dr Zr, Di Zi, Zr + Zi (cols_pad x ld)
  DevBuf wd, wdi, lam, lami;
  DevBuf partials;
  DevBuf sums;
  LoopState* state = nullptr;
  DevBuf trace, trace_max;
  int trace_cap = 0;
  int enq = 0;              // maps enqueued since reset
  DevBuf gathered;          // rank 0 with nranks > 1: full Z (n columns, ldz)
  bool local_output = false;  // IPT_OUTPUT_LOCAL_COLUMNS: each rank downloads its own columns
  bool finalized = false;
  // Sparse real Delta (CSR, f2): during the loop Z[2] hold the local columns ROW-major
  // (n rows x cols_pad, ldr = cols_pad), the layout a CSR x dense product gathers
  // contiguously; finalize/download convert the last iterate to column-major once.
  bool sparse = false;
  std::unique_ptr<int64_t, void (*)(void*)> rowptr{nullptr, [](void* p) { cudaFree(p); }};
  std::unique_ptr<int32_t, void (*)(void*)> cidx{nullptr, [](void* p) { cudaFree(p); }};
  DevBuf vals;
  int64_t nnz = 0, ldr = 0;
  const double* zcm = nullptr;  // sparse: column-major copy of the final iterate
  bool delta_finite = false;    // real dense Delta has no Inf/NaN (identity-start shortcut allowed)
  bool start_identity = false;  // Z[0] is the identity (no warm start)
  const double* z_after_loop = nullptr;  // current iterate when full_iterate returned
  double* rm_ptr[2] = {nullptr, nullptr};  // row-major copies of Z (in the free ping-pong buffer) for an overlapped download
  // Ozaki scheme II product (IPT_PRODUCT_OZAKI): Delta's residues (built once), the current
  // Z's residues, the product residues
  int product = IPT_PRODUCT_DMMA;
  OzakiOperand oz_delta, oz_z;
  DevBuf oz_R;
  OzakiOperand oz_delta_i, oz_delta_s;  // complex 3M: Di and Dr + Di
  bool oz_finite = false;                // Delta has no Inf / NaN (the Ozaki product is exact)
  bool oz_delta_ready = false;
  DevBuf oz_dt;     // Delta transposed (the split-off diagonal term reads Delta_ij by column)
  DevBuf oz_mods;   // device int: moduli the current product needs
  bool oz_split = true;
  // K16 closing residual from the last map + an INT8 correction (ipt_closing.cu)
  ClosingWork closing;
  bool closing_on = false;
  ~FullProblem() {
    if (state) cudaFree(state);
  }
};

// ----------------------------------------------------------------- kernels

__global__ void identity_columns_kernel(double* Z, int64_t ldz, int64_t ncols, int64_t col0) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < ncols) Z[j * ldz + col0 + j] = 1.0;
}

// K2: wd_j = sum_k A[col0+j, k] Z[k, j] over the zero-padded K; one warp per column,
// 16-byte loads, fixed per-lane order + xor tree (deterministic). Optionally
// lam_j = d_{col0+j} + wd_j (the eigenvalue formula of solver.cpp:256).
__global__ void diag_dot_kernel(const double* __restrict__ A, int64_t lda,
                                const double* __restrict__ Z, int64_t ldz, int64_t K,
                                int64_t ncols, int64_t col0, double* __restrict__ wd,
                                const double* __restrict__ d, double* __restrict__ lam,
                                const LoopState* state) {
  if (state != nullptr && state->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= ncols) return;
  const double2* a = reinterpret_cast<const double2*>(A + (col0 + j) * lda);
  const double2* z = reinterpret_cast<const double2*>(Z + j * ldz);
  const int64_t K2 = K / 2;
  double sx = 0.0, sy = 0.0;
  int64_t k = lane;
  for (; k + 96 < K2; k += 128) {
    const double2 a0 = __ldg(a + k), a1 = __ldg(a + k + 32), a2 = __ldg(a + k + 64), a3 = __ldg(a + k + 96);
    const double2 z0 = z[k], z1 = z[k + 32], z2 = z[k + 64], z3 = z[k + 96];
    sx = __fma_rn(a0.x, z0.x, sx); sy = __fma_rn(a0.y, z0.y, sy);
    sx = __fma_rn(a1.x, z1.x, sx); sy = __fma_rn(a1.y, z1.y, sy);
    sx = __fma_rn(a2.x, z2.x, sx); sy = __fma_rn(a2.y, z2.y, sy);
    sx = __fma_rn(a3.x, z3.x, sx); sy = __fma_rn(a3.y, z3.y, sy);
  }
  for (; k < K2; k += 32) {
    const double2 a0 = __ldg(a + k);
    const double2 z0 = z[k];
    sx = __fma_rn(a0.x, z0.x, sx); sy = __fma_rn(a0.y, z0.y, sy);
  }
  double s = sx + sy;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) {
    wd[j] = s;
    if (lam != nullptr) lam[j] = d[col0 + j] + s;
  }
}

// The reference's stop logic, one thread (solver.cpp:236-249 + BASELINE max-abs rule).
__global__ void decide_full_kernel(LoopState* st, const double* __restrict__ sums, int k,
                                   double tol, int max_iter, double div_thr, int rule,
                                   int ignore_conv, double* trace, double* trace_max) {
  if (st->done) return;
  const double diff2 = sums[0], cur2 = sums[1], new2 = sums[2], mx = sums[3];
  const double step = sqrt(diff2) / sqrt(cur2);
  st->iterations = k + 1;
  st->final_step = step;
  st->final_max_abs = mx;
  st->sums[0] = diff2;
  st->sums[1] = cur2;
  st->sums[2] = new2;
  st->sums[3] = mx;
  if (trace) trace[k] = step;
  if (trace_max) trace_max[k] = mx;
  const double zn = sqrt(new2);
  if (!isfinite(zn) || zn > div_thr) {
    st->status = kDiverged;
    st->done = 1;
  } else if (!ignore_conv && (rule == kStopMaxAbs ? (mx < tol) : (step <= tol))) {
    st->status = kConverged;
    st->done = 1;
  } else if (k + 1 >= max_iter) {
    st->status = kMaxIterations;
    st->done = 1;
  }
}

// ---- complex full spectrum (a16/f3): K2 pre-pass and operand preparation of the 3M product ----

constexpr int kEpiBlocks = 1184;  // cap of the persistent sparse-map grid (8 CTAs x 148 SMs)

// K2 (complex): wd_j = sum_k Delta[jg, k] Z[k, j] with Delta = Dr + i Di and Z = Zr + i Zi
// (planes ld apart in a column of Z); warp per column, fixed lane order + xor tree.
__global__ void complex_diag_kernel(const double* __restrict__ Dr, const double* __restrict__ Di, int64_t lda,
                                    const double* __restrict__ Z, int64_t ldz, int64_t ld, int64_t n,
                                    int64_t ncols, int64_t col0, double* __restrict__ wdr,
                                    double* __restrict__ wdi, const LoopState* state) {
  if (state != nullptr && state->done) return;
  const int lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  if (j >= ncols) return;
  const double* ar = Dr + (col0 + j) * lda;
  const double* ai = Di + (col0 + j) * lda;
  const double* zr = Z + j * ldz;
  const double* zi = zr + ld;
  double sr = 0.0, si = 0.0;
  for (int64_t k = lane; k < n; k += 32) {
    const double a = __ldg(ar + k), b = __ldg(ai + k), x = zr[k], y = zi[k];
    sr = __fma_rn(a, x, sr);
    sr = __fma_rn(-b, y, sr);
    si = __fma_rn(a, y, si);
    si = __fma_rn(b, x, si);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    sr += __shfl_xor_sync(0xffffffffu, sr, off);
    si += __shfl_xor_sync(0xffffffffu, si, off);
  }
  if (lane == 0) {
    wdr[j] = sr;
    wdi[j] = si;
  }
}

// S[:, j] = Zr[:, j] + Zi[:, j] over the padded ld rows (the B operand of the T3 GEMM).
__global__ void plane_sum_kernel(const double* __restrict__ Z, int64_t ldz, int64_t ld, int64_t ncols,
                                 double* __restrict__ S, const LoopState* state) {
  if (state != nullptr && state->done) return;
  const int64_t total = ld * ncols;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < total; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / ld, i = e - j * ld;
    S[j * ld + i] = Z[j * ldz + i] + Z[j * ldz + ld + i];
  }
}

__global__ void add_planes_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ c,
                                  int64_t count) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x)
    c[e] = a[e] + b[e];
}

__global__ void complex_lambda_kernel(const double* wdr, const double* wdi, const double* dr,
                                      const double* di, int64_t ncols, int64_t col0, double* lr,
                                      double* li) {
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j < ncols) {
    lr[j] = dr[col0 + j] + wdr[j];
    li[j] = di[col0 + j] + wdi[j];
  }
}

// Warm start renormalisation (solver.cpp:190-201): Z[:, j] /= Z[j, j]; Z[j, j] = 1.
__global__ void renormalize_columns_kernel(double* Z, int64_t ldz, int64_t ld, int64_t n,
                                           int64_t ncols, int64_t col0, int cplx) {
  const int64_t j = blockIdx.x;
  if (j >= ncols) return;
  double* zr = Z + j * ldz;
  const int64_t jg = col0 + j;
  const cd zjj{zr[jg], cplx ? zr[ld + jg] : 0.0};
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    if (i == jg) continue;
    if (cplx) {
      const cd q = cdiv(cd{zr[i], zr[ld + i]}, zjj);
      zr[i] = q.re;
      zr[ld + i] = q.im;
    } else {
      zr[i] = __ddiv_rn(zr[i], zjj.re);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    zr[jg] = 1.0;
    if (cplx) zr[ld + jg] = 0.0;
  }
}

// ---- sparse Delta (f2): CSR x row-major Z with the map epilogue fused ----
// matmul_sparse_parallel (proj/src/kernels.cpp:88-108) accumulates W_ij over the CSR
// entries of row i in storage order; every kernel below keeps that order with one
// rounding per term (fma), so W_jj of the diagonal pre-pass and W_ij of the product
// are the same numbers.

struct SpmmArgs {
  const int64_t* rowptr;
  const int32_t* cols;
  const double* vals;
  const double* Z;  // row-major, ldr
  int64_t ldr;
  double* F;        // row-major, ldr (map mode)
  const double* d;
  const double* wd;   // map: (Delta Z)_jj per local column
  const double* lam;  // resid: lambda_j per local column
  int64_t n, ncols, col0;
  double* partials;
  const LoopState* state;
};

// K2 (sparse): wd_j = sum_p vals[p] Z[cols[p], j] over row col0+j, one thread per column.
__global__ void sparse_diag_kernel(SpmmArgs a, double* __restrict__ wd, double* __restrict__ lam) {
  if (a.state != nullptr && a.state->done) return;
  const int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (j >= a.ncols) return;
  const int64_t jg = a.col0 + j;
  double s = 0.0;
  for (int64_t p = a.rowptr[jg]; p < a.rowptr[jg + 1]; ++p)
    s = __fma_rn(__ldg(a.vals + p), a.Z[int64_t(__ldg(a.cols + p)) * a.ldr + j], s);
  wd[j] = s;
  if (lam != nullptr) lam[j] = a.d[jg] + s;
}

// K1 (sparse): one warp per (row i, chunk of 32*VEC columns); lane l owns columns
// chunk*32*VEC + l*VEC .. +VEC. The row's CSR entries are loaded 32 at a time and
// broadcast by shuffle; each entry gathers VEC contiguous doubles of Z row k
// (a full 32-byte sector per lane at VEC = 4). Work items run chunk-major, so the
// warps in flight share one column chunk of Z (n x 1 KB) in L2. The persistent grid
// is fixed (spmm_grid()), so the per-CTA partials and their reduction are deterministic.
// MODE 0: map (F and the 4 partial sums), 1: residual sum; U entries in flight per lane.
template <int MODE, int VEC, int MINB, int U>
__global__ void __launch_bounds__(256, MINB) spmm_full_kernel(SpmmArgs a) {
  if (a.state != nullptr && a.state->done) return;
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const int lane = threadIdx.x & 31;
  constexpr int CW = 32 * VEC;
  const int64_t nch = (a.ncols + CW - 1) / CW;
  const int64_t items = nch * a.n;
  const int64_t step = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t it = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); it < items; it += step) {
    const int64_t ch = it / a.n, i = it - ch * a.n;
    const int64_t j0 = ch * CW + lane * VEC;
    const double* zc = a.Z + j0;
    double acc[VEC];
#pragma unroll
    for (int t = 0; t < VEC; ++t) acc[t] = 0.0;
    const int64_t rb = a.rowptr[i], re = a.rowptr[i + 1];
    for (int64_t base = rb; base < re; base += 32) {
      const int cnt = static_cast<int>(re - base < 32 ? re - base : 32);
      int kc = 0;
      double kv = 0.0;
      if (lane < cnt) {
        kc = __ldg(a.cols + base + lane);
        kv = __ldg(a.vals + base + lane);
      }
      int q = 0;
      for (; q + U <= cnt; q += U) {
        double2 z[U][VEC / 2];
        double vv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t k = __shfl_sync(0xffffffffu, kc, q + u);
          vv[u] = __shfl_sync(0xffffffffu, kv, q + u);
          const double2* src = reinterpret_cast<const double2*>(zc + k * a.ldr);
#pragma unroll
          for (int h = 0; h < VEC / 2; ++h) z[u][h] = __ldg(src + h);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int h = 0; h < VEC / 2; ++h) {
            acc[2 * h] = __fma_rn(vv[u], z[u][h].x, acc[2 * h]);
            acc[2 * h + 1] = __fma_rn(vv[u], z[u][h].y, acc[2 * h + 1]);
          }
      }
      for (; q < cnt; ++q) {
        const int64_t k = __shfl_sync(0xffffffffu, kc, q);
        const double vq = __shfl_sync(0xffffffffu, kv, q);
        const double2* src = reinterpret_cast<const double2*>(zc + k * a.ldr);
#pragma unroll
        for (int h = 0; h < VEC / 2; ++h) {
          const double2 z = __ldg(src + h);
          acc[2 * h] = __fma_rn(vq, z.x, acc[2 * h]);
          acc[2 * h + 1] = __fma_rn(vq, z.y, acc[2 * h + 1]);
        }
      }
    }
    // epilogue: the dense K1 formulas (dmma_gemm.cuh), row-major addressing
    const double di = a.d[i];
    const double* zrow = zc + i * a.ldr;
    double zi[VEC];
#pragma unroll
    for (int h = 0; h < VEC / 2; ++h) {
      const double2 z = *reinterpret_cast<const double2*>(zrow + 2 * h);
      zi[2 * h] = z.x;
      zi[2 * h + 1] = z.y;
    }
#pragma unroll
    for (int t = 0; t < VEC; ++t) {
      const int64_t j = j0 + t;
      if (j >= a.ncols) continue;
      const double z = zi[t], w = acc[t];
      if (MODE == 0) {
        const int64_t jg = a.col0 + j;
        const double f = (i == jg) ? 1.0 : __ddiv_rn(__dsub_rn(__dmul_rn(z, a.wd[j]), w), __dsub_rn(di, a.d[jg]));
        a.F[i * a.ldr + j] = f;
        const double df = __dsub_rn(f, z);
        v[0] = __fma_rn(df, df, v[0]);
        v[1] = __fma_rn(z, z, v[1]);
        v[2] = __fma_rn(f, f, v[2]);
        v[3] = nan_max(v[3], fabs(df));
      } else {
        const double r = __dsub_rn(__dadd_rn(__dmul_rn(di, z), w), __dmul_rn(z, a.lam[j]));
        v[0] = __fma_rn(r, r, v[0]);
      }
    }
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = a.partials + size_t(blockIdx.x) * 4;
    o[0] = v[0]; o[1] = v[1]; o[2] = v[2]; o[3] = v[3];
  }
}

// F(I) without the product (dense real Delta, identity start): W = Delta I is Delta
// itself, bit for bit (every other term of the GEMM sum is an exact zero), so the
// first map is evaluated by loading W_ij = Delta[i, col0 + j] into the accumulator
// fragments of the same CTA tile / warp / lane layout as K1 and running K1's own
// epilogue: F, the identity reset and the per-CTA partial sums are identical to
// the GEMM path's. Only used when Delta is all-finite (an Inf would make the GEMM's
// zero terms NaN).
__global__ void __launch_bounds__(kGemmThreads) map_identity_kernel(const GemmParams p) {
  if (p.state != nullptr && p.state->done) return;
  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  const int64_t m0 = int64_t(tm) * kBM, n0 = int64_t(tn) * kBN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  double acc[4][4][4];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t i = m0 + wm * 64 + mi * 16 + g + ((r >> 1) << 3);
        const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + (r & 1);
        acc[mi][ni][r] = (i < p.n_rows && j < p.n_cols) ? __ldg(p.A + i * p.lda + p.col0 + j) : 0.0;
      }
  __shared__ double red[kConsumerWarps][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  gemm_epilogue<kGemmMap>(p, acc, m0, n0, warp, lane, v);
  block_reduce4<kConsumerWarps>(v, red);
  if (threadIdx.x == 0) {
    double* out = p.partials + size_t(blockIdx.x) * 4;
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
    out[3] = v[3];
  }
}

__global__ void count_nonfinite_kernel(const double* __restrict__ A, int64_t count, int* out) {
  int bad = 0;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += int64_t(gridDim.x) * blockDim.x)
    bad |= !isfinite(A[e]);
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0 && bad) atomicOr(out, 1);
}

// --------------------------------------------------------------- host side

namespace {

// Tuned variants of K10 (IPT_SPMM_VARIANT selects one; profiles/r01_spmm_variants.txt).
struct SpmmVariant {
  void (*map)(SpmmArgs);
  void (*resid)(SpmmArgs);
  const char* name;
};
const SpmmVariant kSpmmVariants[] = {
    {spmm_full_kernel<0, 4, 2, 4>, spmm_full_kernel<1, 4, 2, 4>, "vec4 minb2 u4"},
    {spmm_full_kernel<0, 4, 3, 4>, spmm_full_kernel<1, 4, 3, 4>, "vec4 minb3 u4"},
    {spmm_full_kernel<0, 4, 4, 4>, spmm_full_kernel<1, 4, 4, 4>, "vec4 minb4 u4"},
    {spmm_full_kernel<0, 2, 4, 4>, spmm_full_kernel<1, 2, 4, 4>, "vec2 minb4 u4"},
    {spmm_full_kernel<0, 4, 2, 8>, spmm_full_kernel<1, 4, 2, 8>, "vec4 minb2 u8"},
    {spmm_full_kernel<0, 4, 3, 8>, spmm_full_kernel<1, 4, 3, 8>, "vec4 minb3 u8"},
    {spmm_full_kernel<0, 2, 6, 8>, spmm_full_kernel<1, 2, 6, 8>, "vec2 minb6 u8"},
};
constexpr int kSpmmDefault = 0;

const SpmmVariant& spmm_variant() {
  static const int v = [] {
    const char* e = std::getenv("IPT_SPMM_VARIANT");
    const int k = e ? std::atoi(e) : kSpmmDefault;
    const int nv = static_cast<int>(sizeof(kSpmmVariants) / sizeof(kSpmmVariants[0]));
    return (k >= 0 && k < nv) ? k : kSpmmDefault;
  }();
  return kSpmmVariants[v];
}

// IPT_IDENTITY_SHORTCUT=0 runs the first map from I through the GEMM as well.
bool identity_shortcut_enabled() {
  const char* e = std::getenv("IPT_IDENTITY_SHORTCUT");
  return !(e && std::strcmp(e, "0") == 0);
}

SpmmArgs spmm_args(FullProblem& P, const double* Zs, double* Fd, const LoopState* st) {
  SpmmArgs a{};
  a.rowptr = P.rowptr.get();
  a.cols = P.cidx.get();
  a.vals = P.vals.get();
  a.Z = Zs;
  a.ldr = P.ldr;
  a.F = Fd;
  a.d = P.dre.get();
  a.wd = P.wd.get();
  a.lam = P.lam.get();
  a.n = P.n;
  a.ncols = P.ncols;
  a.col0 = P.col0;
  a.partials = P.partials.get();
  a.state = st;
  return a;
}

void launch_sparse_diag(FullProblem& P, const double* Zs, double* lam, const LoopState* st) {
  const unsigned grid = static_cast<unsigned>(ceil_div(P.ncols, 256));
  if (grid == 0) return;
  sparse_diag_kernel<<<grid, 256, 0, P.ctx->stream>>>(spmm_args(P, Zs, nullptr, st), P.wd.get(), lam);
  IPT_LAUNCH_CHECK();
  count_launch();
}

// Persistent grid: every resident CTA of the map kernel, once (a fixed number on a
// given device, so the partial-sum order is fixed); both modes use it.
int spmm_grid() {
  static const int g = [] {
    int dev = 0, sms = 0, per_sm = 0;
    IPT_CUDA(cudaGetDevice(&dev));
    IPT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    IPT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmm_variant().map, 256, 0));
    return std::max(1, std::min(kEpiBlocks, sms * std::max(per_sm, 1)));
  }();
  return g;
}

void launch_spmm(FullProblem& P, int mode, const double* Zs, double* Fd, const LoopState* st) {
  const SpmmArgs a = spmm_args(P, Zs, Fd, st);
  cudaStream_t s = P.ctx->stream;
  const unsigned grid = static_cast<unsigned>(spmm_grid());
  const SpmmVariant& v = spmm_variant();
  (mode == 0 ? v.map : v.resid)<<<grid, 256, 0, s>>>(a);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void launch_diag(FullProblem& P, const double* A, const double* Zsrc, double* out, double* lam,
                 const double* dvec, const LoopState* st) {
  const int warps = 8;
  const unsigned grid = static_cast<unsigned>(ceil_div(P.ncols, warps));
  if (grid == 0) return;
  diag_dot_kernel<<<grid, warps * 32, 0, P.ctx->stream>>>(A, P.lda, Zsrc, P.ldz, P.lda, P.ncols,
                                                           P.col0, out, dvec, lam, st);
  IPT_LAUNCH_CHECK();
  count_launch();
}

GemmParams gemm_params(FullProblem& P, const double* A, const double* Bz, double* C, int64_t ldc) {
  GemmParams g{};
  g.K = P.lda;
  g.A = A;
  g.lda = P.lda;
  g.B = Bz;
  g.ldb = P.ldz;
  g.C = C;
  g.ldc = ldc;
  g.tiles_m = static_cast<int>(ceil_div(P.n, kBM));
  g.tiles_n = static_cast<int>(ceil_div(P.ncols, kBN));
  g.d = P.dre.get();
  g.wd = P.wd.get();
  g.lam = P.lam.get();
  g.col0 = P.col0;
  g.row0 = 0;
  g.n_rows = P.n;
  g.n_cols = P.ncols;
  g.partials = P.partials.get();
  g.state = P.state;
  return g;
}

int64_t num_partials(const FullProblem& P) {
  if (P.sparse) return spmm_grid();
  return static_cast<int64_t>(gemm_tiles(P.n, P.ncols));
}

// Complex 3M product for the current Z (zs): wd (K2), S = Zr + Zi, T1 = Dr Zr, T2 = Di Zi,
// then the T3 GEMM with the complex epilogue `mode` (map into zd, or the residual).
bool use_ozaki(const FullProblem& P);

// Complex 3M with each real product by Ozaki scheme II: T1 = Dr Zr and T2 = Di Zi are
// reconstructed into P.T1 / P.T2, then T3 = (Dr + Di)(Zr + Zi) is reconstructed with the
// complex map (mode 3) or closing residual (mode 4) epilogue, the same formulas as the
// kGemmMapC / kGemmResidC GEMM epilogues. Each product takes the moduli its operand's
// column 1-norms require (no diagonal split: 14 on the IPT iterates).
void ozaki_apply_complex(FullProblem& P, const double* zs, double* zd, int mode, const LoopState* st,
                         cudaEvent_t ev_a, cudaEvent_t ev_b) {
  cudaStream_t s = P.ctx->stream;
  const int64_t kpad = round_up(P.n, kOzakiKPad);
  const int64_t arows = round_up(P.n, 512);
  if (!P.oz_delta_ready) {
    P.oz_delta.build(s, P.A1.get(), P.lda, P.n, P.n, arows, kpad);
    P.oz_delta_i.build(s, P.A2.get(), P.lda, P.n, P.n, arows, kpad);
    P.oz_delta_s.build(s, P.A3.get(), P.lda, P.n, P.n, arows, kpad);
    P.oz_mods.alloc(2, false);
    P.oz_delta_ready = true;
  }
  int* mods = reinterpret_cast<int*>(P.oz_mods.get());
  int64_t plane = 0;
  if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, s));
  const OzakiOperand* ops[2] = {&P.oz_delta, &P.oz_delta_i};
  const double* xs[2] = {zs, zs + P.ld};
  double* outs[2] = {P.T1.get(), P.T2.get()};
  for (int t = 0; t < 2; ++t) {
    P.oz_z.build(s, xs[t], P.ldz, P.ncols, P.n, P.cols_pad, kpad, -1, mods + t);
    ozaki_products(s, P.oz_z, *ops[t], P.cols_pad, arows, P.oz_R, plane, mods + t);
    OzakiMapArgs a{};
    a.R = reinterpret_cast<const int8_t*>(P.oz_R.get());
    a.plane = plane;
    a.ldr = arows;
    a.eA = ops[t]->exps();
    a.eB = P.oz_z.exps();
    a.F = outs[t];
    a.ldz = P.ld;
    a.n = P.n;
    a.ncols = P.ncols;
    a.col0 = P.col0;
    a.mode = 2;
    a.partials = P.partials.get();
    a.state = st;
    a.moduli = mods + t;
    ozaki_reconstruct(s, a);
  }
  P.oz_z.build(s, P.S.get(), P.ld, P.ncols, P.n, P.cols_pad, kpad, -1, mods + 2);
  ozaki_products(s, P.oz_z, P.oz_delta_s, P.cols_pad, arows, P.oz_R, plane, mods + 2);
  if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, s));
  OzakiMapArgs a{};
  a.R = reinterpret_cast<const int8_t*>(P.oz_R.get());
  a.plane = plane;
  a.ldr = arows;
  a.eA = P.oz_delta_s.exps();
  a.eB = P.oz_z.exps();
  a.Z = zs;
  a.Zi = zs + P.ld;
  a.ldz = P.ldz;
  a.T1 = P.T1.get();
  a.T2 = P.T2.get();
  a.ldt = P.ld;
  a.d = P.dre.get();
  a.di = P.dim.get();
  a.wd = P.wd.get();
  a.wdi = P.wdi.get();
  a.lam = P.lam.get();
  a.lami = P.lami.get();
  a.F = zd;
  a.Fi = zd ? zd + P.ld : nullptr;
  a.n = P.n;
  a.ncols = P.ncols;
  a.col0 = P.col0;
  a.mode = mode == kGemmMapC ? 3 : 4;
  a.partials = P.partials.get();
  a.state = st;
  a.moduli = mods + 2;
  ozaki_reconstruct(s, a);
}

void launch_complex_products(FullProblem& P, const double* zs, double* zd, int mode, const LoopState* st,
                             cudaEvent_t ev_a, cudaEvent_t ev_b) {
  Ctx& c = *P.ctx;
  const unsigned gd = static_cast<unsigned>(ceil_div(P.ncols, 8));
  if (gd == 0) return;
  complex_diag_kernel<<<gd, 256, 0, c.stream>>>(P.A1.get(), P.A2.get(), P.lda, zs, P.ldz, P.ld, P.n, P.ncols,
                                                P.col0, P.wd.get(), P.wdi.get(), st);
  plane_sum_kernel<<<1184, 256, 0, c.stream>>>(zs, P.ldz, P.ld, P.ncols, P.S.get(), st);
  IPT_LAUNCH_CHECK();
  count_launch(2);
  if (mode == kGemmResidC) {
    complex_lambda_kernel<<<static_cast<unsigned>(ceil_div(P.ncols, 256)), 256, 0, c.stream>>>(
        P.wd.get(), P.wdi.get(), P.dre.get(), P.dim.get(), P.ncols, P.col0, P.lam.get(), P.lami.get());
    IPT_LAUNCH_CHECK();
    count_launch();
  }
  if (use_ozaki(P)) {
    ozaki_apply_complex(P, zs, zd, mode, st, ev_a, ev_b);
    return;
  }
  if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, c.stream));
  GemmParams g1 = gemm_params(P, P.A1.get(), zs, P.T1.get(), P.ld);
  g1.state = st;
  launch_gemm(kGemmStore, g1, c.stream);
  GemmParams g2 = gemm_params(P, P.A2.get(), zs + P.ld, P.T2.get(), P.ld);
  g2.state = st;
  launch_gemm(kGemmStore, g2, c.stream);
  GemmParams g3 = gemm_params(P, P.A3.get(), P.S.get(), zd, P.ldz);
  g3.ldb = P.ld;
  g3.state = st;
  g3.T1 = P.T1.get();
  g3.T2 = P.T2.get();
  g3.ldt = P.ld;
  g3.zre = zs;
  g3.zim = zs + P.ld;
  g3.ldzz = P.ldz;
  g3.wdi = P.wdi.get();
  g3.di = P.dim.get();
  g3.lami = P.lami.get();
  g3.Cim = zd ? zd + P.ld : nullptr;
  launch_gemm(mode, g3, c.stream);
  if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, c.stream));
}

void allreduce_sums(FullProblem& P, bool with_max) {
  Ctx& c = *P.ctx;
  if (c.nranks <= 1) return;
  c.comm->all_reduce(P.sums.get(), 3, CommType::F64, CommOp::Sum, c.stream);
  if (with_max) c.comm->all_reduce(P.sums.get() + 3, 1, CommType::F64, CommOp::Max, c.stream);
}

bool use_ozaki(const FullProblem& P) {
  return P.product == IPT_PRODUCT_OZAKI && !P.sparse && P.oz_finite && P.n <= kOzakiMaxK && P.ncols > 0;
}

int64_t map_partials(const FullProblem& P) { return use_ozaki(P) ? kOzakiGrid : num_partials(P); }

// W = Delta Z by Ozaki scheme II, then the map (mode 0) or the closing residual (mode 1).
// ev_a / ev_b (optional) bracket the 16 INT8 GEMMs alone (the roofline kernel).
void ozaki_apply(FullProblem& P, const double* zs, double* zd, int mode, const LoopState* st,
                 cudaEvent_t ev_a = nullptr, cudaEvent_t ev_b = nullptr) {
  cudaStream_t s = P.ctx->stream;
  const int64_t kpad = round_up(P.n, kOzakiKPad);
  const int64_t arows = round_up(P.n, 512);  // the 256 x 512 pair tile of the INT8 GEMM
  if (!P.oz_delta_ready) {
    P.oz_delta.build(s, P.A1.get(), P.lda, P.n, P.n, arows, kpad);
    if (P.oz_split) {
      P.oz_dt.alloc(P.n * P.lda, false);
      ozaki_transpose(s, P.A1.get(), P.lda, P.n, P.oz_dt.get(), P.lda);
      P.oz_mods.alloc(1, false);
    }
    P.oz_delta_ready = true;
  }
  // Z'_jj is split off (Z_jj = 1 in every iterate), so the product needs only as many
  // moduli as the off-diagonal column norms require (ozaki.cuh)
  int* mods = P.oz_split ? reinterpret_cast<int*>(P.oz_mods.get()) : nullptr;
  P.oz_z.build(s, zs, P.ldz, P.ncols, P.n, P.cols_pad, kpad, P.oz_split ? P.col0 : -1, mods);
  int64_t plane = 0;
  if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, s));
  ozaki_products(s, P.oz_z, P.oz_delta, P.cols_pad, arows, P.oz_R, plane, mods);
  if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, s));
  OzakiMapArgs a{};
  a.R = reinterpret_cast<const int8_t*>(P.oz_R.get());
  a.plane = plane;
  a.ldr = arows;
  a.eA = P.oz_delta.exps();
  a.eB = P.oz_z.exps();
  a.Z = zs;
  a.ldz = P.ldz;
  if (P.oz_split) {
    a.dZ = P.oz_z.diag.get();
    a.DT = P.oz_dt.get();
    a.lddt = P.lda;
    a.moduli = mods;
  }
  a.F = zd;
  a.d = P.dre.get();
  a.wd = P.wd.get();
  a.lam = P.lam.get();
  a.n = P.n;
  a.ncols = P.ncols;
  a.col0 = P.col0;
  a.mode = mode;
  a.partials = P.partials.get();
  a.state = st;
  ozaki_reconstruct(s, a);
}

// Enqueue map application number k (reads Z[k&1], writes Z[(k+1)&1]).
void enqueue_map(FullProblem& P, int k, const ipt_params& prm, cudaEvent_t ev_a = nullptr,
                 cudaEvent_t ev_b = nullptr) {
  Ctx& c = *P.ctx;
  const double* zs = P.Z[k & 1].get();
  double* zd = P.Z[(k + 1) & 1].get();
  LoopState* st = P.state;
  if (P.sparse) {
    launch_sparse_diag(P, zs, nullptr, st);
    if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, c.stream));
    launch_spmm(P, 0, zs, zd, st);
    if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, c.stream));
  } else if (!P.cplx) {
    launch_diag(P, P.A1.get(), zs, P.wd.get(), nullptr, nullptr, st);
    GemmParams g = gemm_params(P, P.A1.get(), zs, zd, P.ldz);
    int64_t nparts = num_partials(P);
    if (k == 0 && P.start_identity && P.delta_finite && identity_shortcut_enabled()) {
      const unsigned tiles = static_cast<unsigned>(gemm_tiles(P.n, P.ncols));
      if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, c.stream));
      if (tiles) {  // (a rank may own no column when g > n)
        map_identity_kernel<<<tiles, kGemmThreads, 0, c.stream>>>(g);
        IPT_LAUNCH_CHECK();
        count_launch();
      }
      if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, c.stream));
    } else if (use_ozaki(P)) {
      ozaki_apply(P, zs, zd, 0, st, ev_a, ev_b);  // events around the INT8 GEMMs only
      nparts = kOzakiGrid;
    } else {
      if (ev_a) IPT_CUDA(cudaEventRecord(ev_a, c.stream));
      launch_gemm(kGemmMap, g, c.stream);
      if (ev_b) IPT_CUDA(cudaEventRecord(ev_b, c.stream));
    }
    reduce_partials(c.stream, P.partials.get(), nparts, P.sums.get(), st);
    allreduce_sums(P, true);
    decide_full_kernel<<<1, 1, 0, c.stream>>>(
        st, P.sums.get(), k, prm.tolerance, prm.max_iterations, prm.divergence_threshold,
        prm.stop_rule, prm.ignore_convergence, prm.record_trace ? P.trace.get() : nullptr,
        prm.record_trace ? P.trace_max.get() : nullptr);
    IPT_LAUNCH_CHECK();
    count_launch();
    return;
  } else {
    launch_complex_products(P, zs, zd, kGemmMapC, st, ev_a, ev_b);
  }
  reduce_partials(c.stream, P.partials.get(), map_partials(P), P.sums.get(), st);
  allreduce_sums(P, true);
  decide_full_kernel<<<1, 1, 0, c.stream>>>(
      st, P.sums.get(), k, prm.tolerance, prm.max_iterations, prm.divergence_threshold,
      prm.stop_rule, prm.ignore_convergence, prm.record_trace ? P.trace.get() : nullptr,
      prm.record_trace ? P.trace_max.get() : nullptr);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void upload_rowmajor(cudaStream_t s, double* dst, int64_t dpitch, const double* src, int64_t rows,
                     int64_t cols, int64_t spitch) {
  if (rows == 0 || cols == 0) return;
  IPT_CUDA(cudaMemcpy2DAsync(dst, dpitch * sizeof(double), src, spitch * sizeof(double),
                             cols * sizeof(double), rows, cudaMemcpyHostToDevice, s));
}

}  // namespace

// ------------------------------------------------------------ C++ entry points

// This rank's column block: the communicator's shard, or an explicit [begin, end)
// on a single-rank context (a column block is an independent sub-problem of the map).
static void column_block(const Ctx& c, int64_t n, int64_t begin, int64_t end, int64_t& col0, int64_t& ncols) {
  if (begin < 0) {
    int64_t c1 = 0;
    c.shard(n, col0, c1);
    ncols = c1 - col0;
    return;
  }
  if (c.nranks != 1) throw InvalidArgument("solve_full: explicit column blocks need a single-rank context");
  if (!(begin < end && end <= n)) throw InvalidArgument("solve_full: bad column block");
  col0 = begin;
  ncols = end - begin;
}

FullProblem* full_upload(Ctx& c, int64_t n, const double* d_re, const double* d_im,
                         const double* delta_re, const double* delta_im, bool force_complex,
                         int64_t col_begin, int64_t col_end, const double* delta_c) {
  NvtxRange nvtx_("ipt:full_upload");
  if (n <= 0) throw InvalidArgument("solve_full: empty problem");
  if (!d_re || !(delta_re || delta_c)) throw InvalidArgument("solve_full: null input");
  auto P = std::make_unique<FullProblem>();
  P->ctx = &c;
  P->n = n;
  {
    const char* e = std::getenv("IPT_OZAKI_SPLIT");  // 0: all 16 moduli, no diagonal split
    P->oz_split = !(e && e[0] == '0');
  }
  P->ld = round_up(n, 16);
  P->rows_pad = round_up(n, kBM);
  column_block(c, n, col_begin, col_end, P->col0, P->ncols);
  P->cols_pad = round_up(std::max<int64_t>(P->ncols, 1), kBN);
  bool any_im = false;
  if (d_im) for (int64_t i = 0; i < n && !any_im; ++i) any_im = d_im[i] != 0.0;
  if (delta_im && !delta_c) for (int64_t t = 0; t < n * n && !any_im; ++t) any_im = delta_im[t] != 0.0;
  P->cplx = any_im || force_complex;
  P->lda = P->ld;                          // K of every real GEMM
  cudaStream_t s = c.stream;

  ProfMarks pm("full_upload");
  if (delta_c) {
    // Interleaved complex Delta (the C++ carrier): de-interleaved in the staging pass; the
    // imaginary plane crosses PCIe only where it is nonzero, and decides the path. With a
    // communicator each rank sends its slice of rows and the planes are all-gathered.
    const int64_t up_chunk = c.nranks > 1 ? ceil_div(P->rows_pad, int64_t(c.nranks)) : P->rows_pad;
    const size_t cap = size_t(std::max(P->rows_pad, up_chunk * c.nranks)) * P->lda;
    P->A1.alloc(cap);
    P->A2.alloc(cap);
    const int64_t r0 = std::min<int64_t>(n, c.rank * up_chunk), r1 = std::min<int64_t>(n, (c.rank + 1) * up_chunk);
    bool im_sent = false;
    if (r1 > r0)
      h2d_rows_split(c, P->A1.get() + r0 * P->lda, P->A2.get() + r0 * P->lda, P->lda, delta_c + 2 * r0 * n,
                     r1 - r0, n, &im_sent);
    int flag = (im_sent || P->cplx) ? 1 : 0;
    if (c.nranks > 1) {
      DevBuf f;
      f.alloc(1);
      int* df = reinterpret_cast<int*>(f.get());
      IPT_CUDA(cudaMemcpyAsync(df, &flag, sizeof(int), cudaMemcpyHostToDevice, s));
      c.comm->all_reduce(df, 1, CommType::I32, CommOp::Max, s);
      IPT_CUDA(cudaMemcpyAsync(&flag, df, sizeof(int), cudaMemcpyDeviceToHost, s));
      c.sync();
      c.comm->all_gather(P->A1.get(), size_t(up_chunk * P->lda), CommType::F64, s);
      if (flag) c.comm->all_gather(P->A2.get(), size_t(up_chunk * P->lda), CommType::F64, s);
    }
    P->cplx = flag != 0;
    if (!P->cplx) {
      P->A2.release();
    } else {
      P->A3.alloc(cap, false);
      add_planes_kernel<<<1184, 256, 0, s>>>(P->A1.get(), P->A2.get(), P->A3.get(), int64_t(P->rows_pad) * P->lda);
      IPT_LAUNCH_CHECK();
      count_launch();
    }
    pm.mark("h2d_split");
  }
  P->ldz = P->cplx ? 2 * P->ld : P->ld;    // Z columns: [re] or [re; im]
  // With a communicator every rank passes the same Delta (replicated); each uploads only
  // its 1/g slice of rows over PCIe and an in-place NCCL all-gather over NVLink assembles
  // the whole matrix on every GPU (g x less host traffic than g full uploads).
  const bool sharded_upload = c.nranks > 1 && !P->cplx;
  const int64_t up_chunk = ceil_div(P->rows_pad, int64_t(c.nranks));
  if (!delta_c) {
    P->A1.alloc(size_t(sharded_upload ? std::max(P->rows_pad, up_chunk * c.nranks) : P->rows_pad) * P->lda);
    pm.mark("alloc_delta");
  }
  if (delta_c) {
    // (uploaded above)
  } else if (sharded_upload) {
    const int64_t r0 = std::min<int64_t>(n, c.rank * up_chunk), r1 = std::min<int64_t>(n, (c.rank + 1) * up_chunk);
    if (r1 > r0) h2d_rows(c, P->A1.get() + r0 * P->lda, P->lda, delta_re + r0 * n, n, r1 - r0, n);
    c.comm->all_gather(P->A1.get(), size_t(up_chunk * P->lda), CommType::F64, s);
    pm.mark("h2d+allgather");
  } else if (!P->cplx) {
    h2d_rows(c, P->A1.get(), P->lda, delta_re, n, n, n);  // pinned, double-buffered
    pm.mark("h2d");
  } else {
    // A1 = Dr, A2 = Di, A3 = Dr + Di (zero padded): the operands of the 3M product
    h2d_rows(c, P->A1.get(), P->lda, delta_re, n, n, n);
    P->A2.alloc(size_t(P->rows_pad) * P->lda);
    if (delta_im) h2d_rows(c, P->A2.get(), P->lda, delta_im, n, n, n);
    P->A3.alloc(size_t(P->rows_pad) * P->lda, false);
    const int64_t cnt = P->rows_pad * P->lda;
    add_planes_kernel<<<1184, 256, 0, s>>>(P->A1.get(), P->A2.get(), P->A3.get(), cnt);
    IPT_LAUNCH_CHECK();
    count_launch();
    pm.mark("h2d");
  }
  P->dre.alloc(n);
  P->dim.alloc(n);
  IPT_CUDA(cudaMemcpyAsync(P->dre.get(), d_re, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  if (d_im) IPT_CUDA(cudaMemcpyAsync(P->dim.get(), d_im, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  for (auto& z : P->Z) z.alloc(size_t(P->cols_pad) * P->ldz);
  pm.mark("alloc_z");
  if (P->cplx) {
    P->T1.alloc(size_t(P->cols_pad) * P->ld);
    P->T2.alloc(size_t(P->cols_pad) * P->ld);
    P->S.alloc(size_t(P->cols_pad) * P->ld);
  }
  P->wd.alloc(P->cols_pad);
  P->wdi.alloc(P->cols_pad);
  P->lam.alloc(P->cols_pad);
  P->lami.alloc(P->cols_pad);
  P->partials.alloc(size_t(std::max<int64_t>(num_partials(*P), kOzakiGrid)) * 4);
  P->sums.alloc(4);
  IPT_CUDA(cudaMalloc(&P->state, sizeof(LoopState)));
  {
    int* flag = nullptr;
    IPT_CUDA(cudaMalloc(&flag, sizeof(int)));
    IPT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), s));
    count_nonfinite_kernel<<<1184, 256, 0, s>>>(P->A1.get(), int64_t(P->rows_pad) * P->lda, flag);
    if (P->cplx) count_nonfinite_kernel<<<1184, 256, 0, s>>>(P->A2.get(), int64_t(P->rows_pad) * P->lda, flag);
    IPT_LAUNCH_CHECK();
    count_launch(P->cplx ? 2 : 1);
    int h = 1;
    IPT_CUDA(cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    c.sync();
    cudaFree(flag);
    P->delta_finite = !P->cplx && h == 0;  // (the real identity-start shortcut)
    P->oz_finite = h == 0;
    pm.mark("finite_check");
  }
  c.sync();
  return P.release();
}

// Real CSR Delta (rowptr[n+1] with any base, cols in [0, n)): the sparse map path.
FullProblem* full_upload_csr(Ctx& c, int64_t n, const double* d, const int64_t* rowptr,
                             const int32_t* cols, const double* vals, int64_t col_begin, int64_t col_end) {
  NvtxRange nvtx_("ipt:full_upload_csr");
  if (n <= 0) throw InvalidArgument("solve_full: empty problem");
  if (!d || !rowptr) throw InvalidArgument("solve_full: null input");
  const int64_t b = rowptr[0], nnz = rowptr[n] - rowptr[0];
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) throw InvalidArgument("csr: row offsets must be non-decreasing");
  if (nnz > 0 && (!cols || !vals)) throw InvalidArgument("solve_full: null input");
  for (int64_t p = 0; p < nnz; ++p)
    if (cols[b + p] < 0 || cols[b + p] >= n) throw InvalidArgument("csr: column index out of bounds");
  auto P = std::make_unique<FullProblem>();
  P->ctx = &c;
  P->n = n;
  P->ld = round_up(n, 16);
  P->rows_pad = round_up(n, kBM);
  column_block(c, n, col_begin, col_end, P->col0, P->ncols);
  P->cols_pad = round_up(std::max<int64_t>(P->ncols, 1), kBN);
  P->cplx = false;
  P->sparse = true;
  P->lda = P->ld;
  P->ldz = P->ld;
  P->ldr = P->cols_pad;
  P->nnz = nnz;
  cudaStream_t s = c.stream;
  std::vector<int64_t> rp(n + 1);
  for (int64_t i = 0; i <= n; ++i) rp[i] = rowptr[i] - b;
  int64_t* drp = nullptr;
  IPT_CUDA(cudaMalloc(&drp, sizeof(int64_t) * (n + 1)));
  P->rowptr.reset(drp);
  IPT_CUDA(cudaMemcpyAsync(drp, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s));
  int32_t* dc = nullptr;
  IPT_CUDA(cudaMalloc(&dc, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  P->cidx.reset(dc);
  P->vals.alloc(std::max<int64_t>(nnz, 1), false);
  if (nnz) {
    IPT_CUDA(cudaMemcpyAsync(dc, cols + b, sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, s));
    IPT_CUDA(cudaMemcpyAsync(P->vals.get(), vals + b, sizeof(double) * nnz, cudaMemcpyHostToDevice, s));
  }
  P->dre.alloc(n);
  P->dim.alloc(n);
  IPT_CUDA(cudaMemcpyAsync(P->dre.get(), d, sizeof(double) * n, cudaMemcpyHostToDevice, s));
  // n rows x cols_pad (row-major) fits in cols_pad x ldz (ldz >= n)
  for (auto& z : P->Z) z.alloc(size_t(P->cols_pad) * P->ldz);
  P->wd.alloc(P->cols_pad);
  P->wdi.alloc(P->cols_pad);
  P->lam.alloc(P->cols_pad);
  P->lami.alloc(P->cols_pad);
  P->partials.alloc(size_t(kEpiBlocks) * 4);
  P->sums.alloc(4);
  IPT_CUDA(cudaMalloc(&P->state, sizeof(LoopState)));
  c.sync();
  return P.release();
}

bool full_is_sparse(const FullProblem& P) { return P.sparse; }

void full_free(FullProblem* P) { delete P; }

void full_reset(FullProblem& P, const double* warm_re, const double* warm_im, int max_iter_hint,
                bool renormalize) {
  NvtxRange nvtx_("ipt:full_reset");
  Ctx& c = *P.ctx;
  cudaStream_t s = c.stream;
  const int64_t n = P.n;
  fill_zero(s, P.Z[0].get(), P.Z[0].count);
  P.start_identity = (warm_re == nullptr);
  P.z_after_loop = nullptr;
  if (warm_re == nullptr) {
    const unsigned grid = static_cast<unsigned>(ceil_div(P.ncols, 256));
    if (grid) {
      identity_columns_kernel<<<grid, 256, 0, s>>>(P.Z[0].get(), P.ldz, P.ncols, P.col0);
      IPT_LAUNCH_CHECK();
      count_launch();
    }
  } else if (P.ncols > 0) {
    // Host row-major n x n -> this rank's column-major block: upload the row-major rows of
    // the column slice, then transpose on the device.
    for (int64_t j = 0; j < P.ncols && renormalize; ++j) {
      const int64_t jg = P.col0 + j;
      const bool zero = warm_re[jg * n + jg] == 0.0 && (warm_im == nullptr || warm_im[jg * n + jg] == 0.0);
      if (zero) throw InvalidArgument("solve_full: warm start has zero diagonal entry");
    }
    if (!P.cplx && warm_im)
      for (int64_t t = 0; t < n * n; ++t)
        if (warm_im[t] != 0.0)
          throw InvalidArgument("solve_full: complex warm start on a real problem (open it complex)");
    DevBuf rm;
    rm.alloc(size_t(n) * std::max<int64_t>(P.ncols, 1), false);
    for (int part = 0; part < (warm_im && P.cplx ? 2 : 1); ++part) {
      const double* src = part == 0 ? warm_re : warm_im;
      // rm: n rows x ncols, row-major (ld = ncols)
      upload_rowmajor(s, rm.get(), P.ncols, src + P.col0, n, P.ncols, n);
      // row-major (n x ncols) is column-major (ncols x n): transpose into Z (column-major n x ncols)
      transpose_to_rowmajor(s, rm.get(), P.ncols, P.ncols, n, P.Z[0].get() + (part ? P.ld : 0), P.ldz);
    }
    if (renormalize && P.ncols > 0) {
      renormalize_columns_kernel<<<static_cast<unsigned>(P.ncols), 256, 0, s>>>(
          P.Z[0].get(), P.ldz, P.ld, n, P.ncols, P.col0, P.cplx ? 1 : 0);
      IPT_LAUNCH_CHECK();
      count_launch();
    }
    c.sync();
  }
  if (P.sparse) {
    // column-major start -> the row-major loop layout (Z[1] becomes Z[0])
    fill_zero(s, P.Z[1].get(), P.Z[1].count);
    transpose_to_rowmajor(s, P.Z[0].get(), P.ldz, n, P.ncols, P.Z[1].get(), P.ldr);
    std::swap(P.Z[0].p, P.Z[1].p);
    fill_zero(s, P.Z[1].get(), P.Z[1].count);
    P.zcm = nullptr;
  }
  LoopState init{};
  init.status = kMaxIterations;
  init.scale_ak = 1.0;
  IPT_CUDA(cudaMemcpyAsync(P.state, &init, sizeof(LoopState), cudaMemcpyHostToDevice, s));
  if (P.trace_cap < max_iter_hint) {
    P.trace.alloc(max_iter_hint);
    P.trace_max.alloc(max_iter_hint);
    P.trace_cap = max_iter_hint;
  }
  P.enq = 0;
  P.finalized = false;
  P.gathered.release();
  P.closing_on = false;
}

// The Ozaki product needs residue planes of Delta, Z and the products (16 bytes per
// element each) and Delta transposed: when they do not fit next to what the solve holds,
// W = Delta Z stays on the DMMA path (FP64 either way).
int effective_product(const FullProblem& P, int product) {
  if (product != IPT_PRODUCT_OZAKI || P.oz_delta_ready) return product;
  const int64_t kpad = round_up(P.n, kOzakiKPad), arows = round_up(P.n, 512);
  const double ndelta = P.cplx ? 3.0 : 1.0;
  const double need = double(kOzakiMods) * (ndelta * double(arows) * kpad + double(P.cols_pad) * kpad +
                                            double(P.cols_pad) * arows) +
                      (P.oz_split && !P.cplx ? 8.0 * double(P.n) * double(P.lda) : 0.0) + double(1 << 30);
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) {
    cudaGetLastError();
    return product;
  }
  return need <= double(free_b) ? product : IPT_PRODUCT_DMMA;
}

void full_set_product(FullProblem& P, int product) { P.product = effective_product(P, product); }

int full_ozaki_moduli(FullProblem& P) {
  if (!use_ozaki(P)) return 0;
  if (!P.cplx && !P.oz_split) return kOzakiMods;
  int m[3] = {0, 0, 0};
  IPT_CUDA(cudaMemcpyAsync(m, P.oz_mods.get(), sizeof(int) * (P.cplx ? 3 : 1), cudaMemcpyDeviceToHost,
                           P.ctx->stream));
  IPT_CUDA(cudaStreamSynchronize(P.ctx->stream));
  return std::max(m[0], std::max(m[1], m[2]));  // complex: the largest of T1, T2, T3
}

void full_iterate(FullProblem& P, const ipt_params& prm, ipt_stats* stats) {
  NvtxRange nvtx_("ipt:full_iterate");
  Ctx& c = *P.ctx;
  P.product = effective_product(P, prm.product);
  if (!(prm.tolerance > 0.0)) throw InvalidArgument("config: tolerance must be positive");
  if (prm.max_iterations <= 0) throw InvalidArgument("config: max_iterations must be positive");
  if (!(prm.divergence_threshold > 1.0)) throw InvalidArgument("config: divergence_threshold must exceed 1");
  if (prm.record_trace && P.trace_cap < prm.max_iterations) {
    P.trace.alloc(prm.max_iterations);
    P.trace_max.alloc(prm.max_iterations);
    P.trace_cap = prm.max_iterations;
  }
  // Large problems: one host check per iteration is free next to a >=10 ms GEMM.
  // Small problems: enqueue several iterations per check; the done flag makes the
  // surplus launches exit immediately.
  // The batch must be the same on every rank (each map carries collectives): size it from
  // the global shard width, not this rank's column count.
  const int64_t work = c.nranks > 1 ? P.n * ceil_div(P.n, int64_t(c.nranks)) : P.n * P.ncols;
  const int batch = work >= (int64_t(2048) * 2048) ? 1 : 16;
  IPT_CUDA(cudaEventRecord(c.ev[0], c.stream));
  while (P.enq < prm.max_iterations) {
    for (int b = 0; b < batch && P.enq < prm.max_iterations; ++b) enqueue_map(P, P.enq++, prm);
    IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (c.h_state->done) break;
  }
  IPT_CUDA(cudaEventRecord(c.ev[1], c.stream));
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  P.z_after_loop = P.Z[c.h_state->iterations & 1].get();
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
    if (prm.record_trace && h.iterations > 0) {
      if (stats->trace)
        IPT_CUDA(cudaMemcpy(stats->trace, P.trace.get(), sizeof(double) * h.iterations, cudaMemcpyDeviceToHost));
      if (stats->trace_max_abs)
        IPT_CUDA(cudaMemcpy(stats->trace_max_abs, P.trace_max.get(), sizeof(double) * h.iterations,
                            cudaMemcpyDeviceToHost));
    }
  }
}

// Current iterate after the loop: map k wrote Z[(k+1)&1], so after `it` maps it is Z[it & 1].
static const double* current_z(FullProblem& P) {
  return P.Z[P.ctx->h_state->iterations & 1].get();
}

// Sparse path: the column-major form of the current (row-major) iterate, built once
// in the other ping-pong buffer. Dense path: the current iterate itself.
static const double* final_colmajor_z(FullProblem& P) {
  if (!P.sparse) return current_z(P);
  if (P.zcm == nullptr) {
    const int cur = P.ctx->h_state->iterations & 1;
    double* dst = P.Z[cur ^ 1].get();
    cudaStream_t s = P.ctx->stream;
    fill_zero(s, dst, P.Z[cur ^ 1].count);
    // row-major n x ncols (ldr) == column-major ncols x n -> column-major n x ncols (ldz)
    transpose_to_rowmajor(s, P.Z[cur].get(), P.ldr, P.ncols, P.n, dst, P.ldz);
    P.zcm = dst;
  }
  return P.zcm;
}

// K16 (ipt_closing.cu): after a converged loop with a small last step the closing residual
// needs no second FP64 product -- the last map's product plus an INT8 tensor-core correction
// Delta (Z_new - Z_old) give it. Its inputs are taken here, while Z_old (the other ping-pong
// buffer) is still intact: callers that stage a download in that buffer call this first.
// IPT_CLOSING=exact keeps the full closing product.
void full_prepare_closing(FullProblem& P) {
  Ctx& c = *P.ctx;
  if (P.closing_on || P.sparse || P.cplx || !P.delta_finite) return;
  const char* e = std::getenv("IPT_CLOSING");
  if (e && std::strcmp(e, "exact") == 0) return;
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, c.stream));
  c.sync();
  const LoopState& h = *c.h_state;
  if (h.iterations < 1 || h.status != kConverged || !(h.final_step <= 1e-6) || P.n < 512 || P.n > (int64_t(1) << 17))
    return;
  cudaStream_t s = c.stream;
  ProfMarks pm("closing_prepare");
  if (!P.closing.delta_ready) P.closing.delta_digits(s, P.A1.get(), P.lda, P.n);
  pm.mark("delta_digits", true);
  const int cur = h.iterations & 1;
  P.closing.step_digits(s, P.Z[cur].get(), P.Z[cur ^ 1].get(), P.ldz, P.ncols, P.wd.get());
  pm.mark("step_digits", true);
  P.closing_on = true;
}

// Closing product: Lambda and |MZ - Z Lambda|_F (solver.cpp:252-270), then the
// eigenvector gather to rank 0 and sigma_min (solver.cpp:271) on rank 0.
void full_finalize(FullProblem& P, const ipt_params& prm, ipt_stats* stats) {
  NvtxRange nvtx_("ipt:full_finalize");
  Ctx& c = *P.ctx;
  cudaStream_t s = c.stream;
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
  c.sync();
  const double* z = current_z(P);
  full_prepare_closing(P);
  IPT_CUDA(cudaEventRecord(c.ev[0], s));
  int64_t nparts = map_partials(P);
  if (P.closing_on) {
    launch_diag(P, P.A1.get(), z, P.wd.get(), P.lam.get(), P.dre.get(), nullptr);  // wd_new, Lambda
    P.closing.residual(s, z, P.ldz, P.col0, P.wd.get(), P.partials.get());
    nparts = closing_partials();
    P.closing_on = false;
  } else if (P.sparse) {
    launch_sparse_diag(P, z, P.lam.get(), nullptr);
    launch_spmm(P, 1, z, nullptr, nullptr);
  } else if (!P.cplx && use_ozaki(P)) {
    launch_diag(P, P.A1.get(), z, P.wd.get(), P.lam.get(), P.dre.get(), nullptr);
    ozaki_apply(P, z, nullptr, 1, nullptr);
  } else if (!P.cplx) {
    launch_diag(P, P.A1.get(), z, P.wd.get(), P.lam.get(), P.dre.get(), nullptr);
    GemmParams g = gemm_params(P, P.A1.get(), z, nullptr, 0);
    g.state = nullptr;
    launch_gemm(kGemmResid, g, s);
  } else {
    launch_complex_products(P, z, nullptr, kGemmResidC, nullptr, nullptr, nullptr);
  }
  reduce_partials(s, P.partials.get(), nparts, P.sums.get(), nullptr);
  allreduce_sums(P, false);
  double h4[4];
  IPT_CUDA(cudaMemcpyAsync(h4, P.sums.get(), sizeof(h4), cudaMemcpyDeviceToHost, s));
  IPT_CUDA(cudaEventRecord(c.ev[1], s));
  c.sync();
  float ms_final = 0.f;
  IPT_CUDA(cudaEventElapsedTime(&ms_final, c.ev[0], c.ev[1]));
  z = final_colmajor_z(P);

  // Gather the column shards on rank 0 (one final eigenvector gather), unless every rank
  // writes its own columns to the host (IPT_OUTPUT_LOCAL_COLUMNS).
  P.local_output = c.nranks > 1 && prm.output_mode == IPT_OUTPUT_LOCAL_COLUMNS;
  bool gathered = false;  // (every rank takes part in the gather exactly once)
  auto gather_z = [&] {
    if (gathered) return;
    gathered = true;
    if (c.rank == 0) P.gathered.alloc(size_t(round_up(P.n, kBN)) * P.ldz);
    std::vector<size_t> counts(c.nranks), displs(c.nranks);
    for (int r = 0; r < c.nranks; ++r) {
      const int64_t r0 = P.n * r / c.nranks, r1 = P.n * (r + 1) / c.nranks;
      counts[r] = size_t(r1 - r0) * P.ldz;
      displs[r] = size_t(r0) * P.ldz;
    }
    c.comm->gather(z, size_t(P.ncols) * P.ldz, P.gathered.get(), counts.data(), displs.data(), CommType::F64, 0, s);
    c.sync();
  };
  if (c.nranks > 1 && !P.local_output) gather_z();

  double sig = 0.0;
  float ms_sigma = 0.f;
  if (prm.want_sigma_min && (c.nranks > 1 || P.ncols == P.n)) {
    IPT_CUDA(cudaEventRecord(c.ev[2], s));
    if (c.nranks > 1) {
      // on the shards: y = Z p all-reduced per CG step, no gather of Z
      bool ok = false;
      sig = sigma_min_sharded(c, P.n, P.col0, P.ncols, z, P.cplx ? z + P.ld : nullptr, P.ldz, 50, 1e-4, &ok);
      if (!ok) {  // CG missed: the factor path on rank 0 over the gathered Z, shared by a sum
        gather_z();
        DevBuf one;
        one.alloc(1);
        if (c.rank == 0) {
          sig = sigma_min_device(c, P.n, P.gathered.get(), P.cplx ? P.gathered.get() + P.ld : nullptr, P.ldz, 50,
                                 1e-4);
          IPT_CUDA(cudaMemcpyAsync(one.get(), &sig, sizeof(double), cudaMemcpyHostToDevice, s));
        }
        c.comm->all_reduce(one.get(), 1, CommType::F64, CommOp::Sum, s);
        IPT_CUDA(cudaMemcpyAsync(&sig, one.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
      }
    } else {
      sig = sigma_min_device(c, P.n, z, P.cplx ? z + P.ld : nullptr, P.ldz, 50, 1e-4);
    }
    IPT_CUDA(cudaEventRecord(c.ev[3], s));
    c.sync();
    IPT_CUDA(cudaEventElapsedTime(&ms_sigma, c.ev[2], c.ev[3]));
  }
  P.finalized = true;
  if (stats) {
    stats->residual = std::sqrt(h4[0]);
    stats->min_singular_value_estimate = sig;
    stats->product_count = c.h_state->iterations + 1;
    stats->ms_final = ms_final;
    stats->ms_sigma = ms_sigma;
  }
}

// Single-rank column block [col0, col0 + ncols): Z block (n x ncols, row-major planar)
// and its eigenvalues.
void full_download_block(FullProblem& P, double* z_re, double* z_im, double* lam_re, double* lam_im) {
  NvtxRange nvtx_("ipt:full_download_block");
  Ctx& c = *P.ctx;
  if (c.nranks != 1) throw InvalidArgument("download: column blocks are single-rank");
  cudaStream_t s = c.stream;
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
  c.sync();
  const int64_t n = P.n, nc = P.ncols;
  std::vector<double> lr(nc), li(nc);
  IPT_CUDA(cudaMemcpyAsync(lr.data(), P.lam.get(), sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
  IPT_CUDA(cudaMemcpyAsync(li.data(), P.lami.get(), sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
  c.sync();
  if (lam_re) std::memcpy(lam_re, lr.data(), sizeof(double) * nc);
  if (lam_im) {
    if (P.cplx) std::memcpy(lam_im, li.data(), sizeof(double) * nc);
    else std::memset(lam_im, 0, sizeof(double) * nc);
  }
  const double* zsrc = final_colmajor_z(P);
  DevBuf rm;
  rm.alloc(size_t(n) * nc, false);
  for (int part = 0; part < 2; ++part) {
    double* dst = part == 0 ? z_re : z_im;
    if (dst == nullptr) continue;
    if (part == 1 && !P.cplx) {
      std::memset(dst, 0, sizeof(double) * n * nc);
      continue;
    }
    transpose_to_rowmajor(s, zsrc + (part ? P.ld : 0), P.ldz, n, nc, rm.get(), nc);
    d2h_rows(c, dst, nc, rm.get(), nc, n, nc);
  }
}

// Eigenvalues of every rank's columns on rank 0 (lam computed in finalize).
static void gather_eigenvalues(FullProblem& P, std::vector<double>& lr, std::vector<double>& li) {
  Ctx& c = *P.ctx;
  cudaStream_t s = c.stream;
  const int64_t n = P.n;
  lr.assign(n, 0.0);
  li.assign(n, 0.0);
  if (c.nranks > 1) {
    DevBuf all_r, all_i;
    all_r.alloc(n);
    all_i.alloc(n);
    std::vector<size_t> counts(c.nranks), displs(c.nranks);
    for (int r = 0; r < c.nranks; ++r) {
      const int64_t r0 = n * r / c.nranks, r1 = n * (r + 1) / c.nranks;
      counts[r] = size_t(r1 - r0);
      displs[r] = size_t(r0);
    }
    c.comm->gather(P.lam.get(), size_t(P.ncols), all_r.get(), counts.data(), displs.data(), CommType::F64, 0, s);
    c.comm->gather(P.lami.get(), size_t(P.ncols), all_i.get(), counts.data(), displs.data(), CommType::F64, 0, s);
    if (c.rank == 0) {
      IPT_CUDA(cudaMemcpyAsync(lr.data(), all_r.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      IPT_CUDA(cudaMemcpyAsync(li.data(), all_i.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    }
    c.sync();
  } else {
    IPT_CUDA(cudaMemcpyAsync(lr.data(), P.lam.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    IPT_CUDA(cudaMemcpyAsync(li.data(), P.lami.get(), sizeof(double) * n, cudaMemcpyDeviceToHost, s));
    c.sync();
  }
}

// Z (row-major planar) and eigenvalues to the host; rank 0 receives everything.
void full_download(FullProblem& P, double* z_re, double* z_im, double* lam_re, double* lam_im) {
  NvtxRange nvtx_("ipt:full_download");
  Ctx& c = *P.ctx;
  if (c.nranks == 1 && P.ncols != P.n) throw InvalidArgument("download: column block problem (use the block download)");
  cudaStream_t s = c.stream;
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
  c.sync();
  const int64_t n = P.n;
  if (P.local_output) {  // this rank's columns into the full-size outputs
    const int64_t c0 = P.col0, nc = P.ncols;
    std::vector<double> lr(nc), li(nc);
    IPT_CUDA(cudaMemcpyAsync(lr.data(), P.lam.get(), sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    IPT_CUDA(cudaMemcpyAsync(li.data(), P.lami.get(), sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    c.sync();
    if (lam_re) std::memcpy(lam_re + c0, lr.data(), sizeof(double) * nc);
    if (lam_im) for (int64_t j = 0; j < nc; ++j) lam_im[c0 + j] = P.cplx ? li[j] : 0.0;
    const double* zsrc = final_colmajor_z(P);
    DevBuf rm;
    rm.alloc(size_t(n) * std::max<int64_t>(nc, 1), false);
    for (int part = 0; part < 2; ++part) {
      double* dst = part == 0 ? z_re : z_im;
      if (dst == nullptr || nc == 0) continue;
      if (part == 1 && !P.cplx) {
        for (int64_t i = 0; i < n; ++i) std::memset(dst + i * n + c0, 0, sizeof(double) * nc);
        continue;
      }
      transpose_to_rowmajor(s, zsrc + (part ? P.ld : 0), P.ldz, n, nc, rm.get(), nc);
      d2h_rows(c, dst + c0, n, rm.get(), nc, n, nc);
    }
    return;
  }
  std::vector<double> lr, li;
  gather_eigenvalues(P, lr, li);
  if (c.rank != 0) return;
  if (lam_re) std::memcpy(lam_re, lr.data(), sizeof(double) * n);
  if (lam_im) {
    if (P.cplx) std::memcpy(lam_im, li.data(), sizeof(double) * n);
    else std::memset(lam_im, 0, sizeof(double) * n);
  }
  const double* zsrc = c.nranks > 1 ? P.gathered.get() : final_colmajor_z(P);
  if (zsrc == nullptr) throw InvalidArgument("download: finalize must run before download");
  DevBuf rm;
  rm.alloc(size_t(n) * n, false);
  for (int part = 0; part < 2; ++part) {
    double* dst = part == 0 ? z_re : z_im;
    if (dst == nullptr) continue;
    if (part == 1 && !P.cplx) {
      std::memset(dst, 0, sizeof(double) * n * n);
      continue;
    }
    transpose_to_rowmajor(s, zsrc + (part ? P.ld : 0), P.ldz, n, n, rm.get(), n);
    d2h_rows(c, dst, n, rm.get(), n, n, n);  // pinned, double-buffered
  }
}

bool full_is_complex(const FullProblem& P) { return P.cplx; }

bool full_can_download_early(const FullProblem& P) { return P.ctx->nranks == 1 && !P.sparse && P.ncols == P.n; }
int64_t full_n(const FullProblem& P) { return P.n; }

// Main thread, before full_finalize: transpose the final Z into row-major staging
// buffers on ctx.stream (a few ms; a kernel on a second stream would starve behind
// the closing-product GEMM, which holds every SM). full_download_z then only needs
// the copy engines, so it overlaps the closing product and sigma_min.
void full_prepare_download(FullProblem& P, bool want_re, bool want_im) {
  Ctx& c = *P.ctx;
  const int64_t n = P.n;
  const double* zsrc = P.z_after_loop;
  if (zsrc == nullptr) throw InvalidArgument("download: iterate must run first");
  // The row-major copies go into the other ping-pong buffer (the previous iterate, no
  // longer read; cols_pad x ldz >= n^2 per part, both parts for complex) -- no extra
  // 8.6 GB allocation at N = 32768.
  double* other = zsrc == P.Z[0].get() ? P.Z[1].get() : P.Z[0].get();
  for (int part = 0; part < 2; ++part) {
    P.rm_ptr[part] = nullptr;
    if (!(part == 0 ? want_re : want_im) || (part == 1 && !P.cplx)) continue;
    P.rm_ptr[part] = other + size_t(part) * size_t(n) * size_t(n);
    transpose_to_rowmajor(c.stream, zsrc + (part ? P.ld : 0), P.ldz, n, n, P.rm_ptr[part], n);
  }
  c.sync();
}

void full_download_z(FullProblem& P, double* z_re, double* z_im) {
  NvtxRange nvtx_("ipt:full_download_z");
  Ctx& c = *P.ctx;
  const int64_t n = P.n;
  for (int part = 0; part < 2; ++part) {
    double* dst = part == 0 ? z_re : z_im;
    if (dst == nullptr) continue;
    if (part == 1 && !P.cplx) {
      std::memset(dst, 0, sizeof(double) * n * n);
      continue;
    }
    if (P.rm_ptr[part] == nullptr) throw InvalidArgument("download: prepare must run first");
    d2h_rows(c, dst, n, P.rm_ptr[part], n, n, n, c.stream2);
  }
  IPT_CUDA(cudaStreamSynchronize(c.stream2));
}

// The same downloads into interleaved complex host arrays (the C++ carrier's layout).
void full_download_interleaved(FullProblem& P, double* z_c, double* lam_c) {
  NvtxRange nvtx_("ipt:full_download");
  Ctx& c = *P.ctx;
  if (c.nranks == 1 && P.ncols != P.n) throw InvalidArgument("download: column block problem (use the block download)");
  cudaStream_t s = c.stream;
  IPT_CUDA(cudaMemcpyAsync(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
  c.sync();
  const int64_t n = P.n;
  if (P.local_output) {  // this rank's columns into the full-size outputs
    const int64_t c0 = P.col0, nc = P.ncols;
    std::vector<double> lr(nc), li(nc);
    IPT_CUDA(cudaMemcpyAsync(lr.data(), P.lam.get(), sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    IPT_CUDA(cudaMemcpyAsync(li.data(), P.lami.get(), sizeof(double) * nc, cudaMemcpyDeviceToHost, s));
    c.sync();
    if (lam_c)
      for (int64_t j = 0; j < nc; ++j) {
        lam_c[2 * (c0 + j)] = lr[j];
        lam_c[2 * (c0 + j) + 1] = P.cplx ? li[j] : 0.0;
      }
    if (z_c == nullptr || nc == 0) return;
    const double* zsrc = final_colmajor_z(P);
    DevBuf rre, rim;
    rre.alloc(size_t(n) * nc, false);
    transpose_to_rowmajor(s, zsrc, P.ldz, n, nc, rre.get(), nc);
    if (P.cplx) {
      rim.alloc(size_t(n) * nc, false);
      transpose_to_rowmajor(s, zsrc + P.ld, P.ldz, n, nc, rim.get(), nc);
    }
    d2h_rows_merge(c, z_c + 2 * c0, n, rre.get(), P.cplx ? rim.get() : nullptr, nc, n, nc);
    return;
  }
  std::vector<double> lr, li;
  gather_eigenvalues(P, lr, li);
  if (c.rank != 0) return;
  if (lam_c)
    for (int64_t j = 0; j < n; ++j) {
      lam_c[2 * j] = lr[j];
      lam_c[2 * j + 1] = P.cplx ? li[j] : 0.0;
    }
  if (z_c == nullptr) return;
  const double* zsrc = c.nranks > 1 ? P.gathered.get() : final_colmajor_z(P);
  if (zsrc == nullptr) throw InvalidArgument("download: finalize must run before download");
  DevBuf rre, rim;
  rre.alloc(size_t(n) * n, false);
  transpose_to_rowmajor(s, zsrc, P.ldz, n, n, rre.get(), n);
  if (P.cplx) {
    rim.alloc(size_t(n) * n, false);
    transpose_to_rowmajor(s, zsrc + P.ld, P.ldz, n, n, rim.get(), n);
  }
  d2h_rows_merge(c, z_c, n, rre.get(), P.cplx ? rim.get() : nullptr, n, n, n);
}

// Early (overlapped) download after full_prepare_download(P, true, P.cplx), on stream2.
void full_download_z_interleaved(FullProblem& P, double* z_c) {
  NvtxRange nvtx_("ipt:full_download_z");
  Ctx& c = *P.ctx;
  if (P.rm_ptr[0] == nullptr || (P.cplx && P.rm_ptr[1] == nullptr))
    throw InvalidArgument("download: prepare must run first");
  d2h_rows_merge(c, z_c, P.n, P.rm_ptr[0], P.cplx ? P.rm_ptr[1] : nullptr, P.n, P.n, P.n, c.stream2);
  IPT_CUDA(cudaStreamSynchronize(c.stream2));
}

void full_release_download(FullProblem& P) {
  P.rm_ptr[0] = P.rm_ptr[1] = nullptr;
}

// Bench / profiling: exactly `count` further map applications (convergence ignored),
// timed with CUDA events on the library stream: the whole sequence and the K1 GEMM
// launches alone (the dominant kernel of the roofline; with the Ozaki product, its 16
// INT8 GEMM launches).
void full_run_maps(FullProblem& P, int count, double* ms_total, double* ms_gemm) {
  Ctx& c = *P.ctx;
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
  for (int i = 0; i < count; ++i) enqueue_map(P, P.enq++, prm, ev[2 + 2 * i], ev[3 + 2 * i]);
  IPT_CUDA(cudaEventRecord(ev[1], c.stream));
  c.sync();
  float ms = 0.f;
  IPT_CUDA(cudaEventElapsedTime(&ms, ev[0], ev[1]));
  *ms_total = ms;
  double g = 0.0;
  for (int i = 0; i < count; ++i) {
    IPT_CUDA(cudaEventElapsedTime(&ms, ev[2 + 2 * i], ev[3 + 2 * i]));
    g += ms;
  }
  *ms_gemm = g;
  for (auto& e : ev) cudaEventDestroy(e);
  IPT_CUDA(cudaMemcpy(c.h_state, P.state, sizeof(LoopState), cudaMemcpyDeviceToHost));
}

void full_local_columns(const FullProblem& P, int64_t* c0, int64_t* c1) {
  *c0 = P.col0;
  *c1 = P.col0 + P.ncols;
}

}  // namespace iptb
