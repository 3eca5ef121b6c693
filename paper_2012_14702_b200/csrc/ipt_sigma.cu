// K6: smallest_singular_value_estimate (proj/src/solver.cpp:275-297) on the device.
//
// The reference forms H = Z^H Z, factors it with a serial partial-pivot LU
// (lu.cpp:10-51) and runs <= 50 steps of inverse power iteration from the
// fixed start vector deterministic_unit(n) (solver.cpp:95-109), stopping when
// |u_k| changes by <= tol relative; the estimate is 1/sqrt(|u|).
//
// Here, first: the same iteration with each solve H u = v done matrix-free by
// conjugate gradients on Z^T Z (two GEMV passes over Z in HBM per CG step; the
// converged IPT basis Z = I + small makes H so well conditioned that CG reaches
// |r| <= 1e-15 |v| in a handful of steps). If any solve misses that within 64
// steps, the factorisation path runs instead:
// H = Z^T Z through the DMMA GEMM, a blocked right-looking Cholesky
// (H is symmetric positive definite for a full-rank Z; the reference's
// "singular" outcome is reproduced by the same pivot threshold
// max|H| * eps * n), and the same inverse power iteration with two blocked
// triangular solves per step. The iterates match the reference's to rounding,
// so the stopping step and the estimate agree. Complex Z uses the real
// embedding [[Zr, -Zi], [Zi, Zr]], on which the iteration from [v; 0] is the
// complex iteration from v written in real coordinates.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <vector>

#include "dmma_gemm.cuh"
#include "ipt_internal.cuh"

namespace iptb {

namespace {

constexpr int NB = 128;          // Cholesky / triangular block
constexpr int LDS = NB + 1;      // padded smem row

// Factor the b x b diagonal block at (kb, kb) of column-major H in place (lower).
__global__ void __launch_bounds__(512) potrf_block_kernel(double* H, int64_t ldh, int64_t kb, int b,
                                                          double tiny, int* singular) {
  extern __shared__ double S[];  // [NB][LDS], S[r*LDS + c] = H(kb+r, kb+c)
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int c = e / b, r = e % b;
    S[r * LDS + c] = (r >= c) ? H[(kb + c) * ldh + kb + r] : 0.0;
  }
  __syncthreads();
  __shared__ int bad;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int c = 0; c < b; ++c) {
    if (tid == 0) {
      const double v = S[c * LDS + c];
      if (!(v > tiny)) {
        bad = 1;
        S[c * LDS + c] = 1.0;
      } else {
        S[c * LDS + c] = sqrt(v);
      }
    }
    __syncthreads();
    const double piv = S[c * LDS + c];
    for (int r = c + 1 + tid; r < b; r += blockDim.x) S[r * LDS + c] = S[r * LDS + c] / piv;
    __syncthreads();
    // trailing lower update: rows r > c, cols q in (c, r]
    const int m = b - c - 1;
    for (int e = tid; e < m * m; e += blockDim.x) {
      const int r = c + 1 + e / m, q = c + 1 + e % m;
      if (q <= r) S[r * LDS + q] = __fma_rn(-S[r * LDS + c], S[q * LDS + c], S[r * LDS + q]);
    }
    __syncthreads();
  }
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int c = e / b, r = e % b;
    if (r >= c) H[(kb + c) * ldh + kb + r] = S[r * LDS + c];
  }
  if (tid == 0 && bad) atomicExch(singular, 1);
}

// L21 = H21 L11^{-T}: rows [kb+b, kb+b+rem), 32 rows per CTA staged through smem,
// 4 rows per warp, x distributed over lanes (x[p] on lane p%32, slot p/32).
// Writes L21 back into H (column-major) and into the row-major panel P (ld NB,
// zero-padded to NB columns) used as both operands of the trailing update.
__global__ void __launch_bounds__(256) trsm_panel_kernel(double* H, int64_t ldh, int64_t kb, int b,
                                                         int64_t rem, double* P, int64_t ldp) {
  extern __shared__ double sm[];
  double* L = sm;                 // [NB][LDS] lower factor of the diagonal block
  double* R = sm + NB * LDS;      // [32][LDS] rows of H21
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t i0 = int64_t(blockIdx.x) * 32;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int c = e / b, r = e % b;
    L[r * LDS + c] = (r >= c) ? H[(kb + c) * ldh + kb + r] : 0.0;
  }
  for (int e = tid; e < 32 * b; e += blockDim.x) {
    const int p = e / 32, r = e % 32;
    const int64_t i = i0 + r;
    R[r * LDS + p] = (i < rem) ? H[(kb + p) * ldh + kb + b + i] : 0.0;
  }
  __syncthreads();
  for (int rr = 0; rr < 4; ++rr) {
    const int r = warp * 4 + rr;
    double x[NB / 32];
#pragma unroll
    for (int s = 0; s < NB / 32; ++s) {
      const int p = s * 32 + lane;
      x[s] = p < b ? R[r * LDS + p] : 0.0;
    }
    // solve x L11^T = h  <=>  L11 x^T = h^T (forward substitution, column oriented)
    for (int p = 0; p < b; ++p) {
      const int owner = p & 31, slot = p >> 5;
      double xp = 0.0;
#pragma unroll
      for (int s = 0; s < NB / 32; ++s)
        if (s == slot) xp = x[s];
      xp = __shfl_sync(0xffffffffu, xp, owner);
      xp = xp / L[p * LDS + p];
#pragma unroll
      for (int s = 0; s < NB / 32; ++s) {
        const int q = s * 32 + lane;
        if (q == p) x[s] = xp;
        else if (q > p && q < b) x[s] = __fma_rn(-L[q * LDS + p], xp, x[s]);
      }
    }
#pragma unroll
    for (int s = 0; s < NB / 32; ++s) R[r * LDS + s * 32 + lane] = (s * 32 + lane < b) ? x[s] : 0.0;
  }
  __syncthreads();
  for (int e = tid; e < 32 * NB; e += blockDim.x) {
    const int r = e / NB, p = e % NB;
    const int64_t i = i0 + r;
    if (i < rem) P[i * ldp + p] = p < b ? R[r * LDS + p] : 0.0;
  }
  for (int e = tid; e < 32 * b; e += blockDim.x) {
    const int p = e / 32, r = e % 32;
    const int64_t i = i0 + r;
    if (i < rem) H[(kb + p) * ldh + kb + b + i] = R[r * LDS + p];
  }
}

__global__ void absmax_kernel(const double* __restrict__ H, int64_t ldh, int64_t m, double* out) {
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < m * m;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t c = e / m, r = e % m;
    if (r >= c) v[3] = nan_max(v[3], fabs(H[c * ldh + r]));  // symmetric: lower triangle only
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) out[blockIdx.x * 4 + 3] = v[3], out[blockIdx.x * 4 + 0] = 0.0,
                        out[blockIdx.x * 4 + 1] = 0.0, out[blockIdx.x * 4 + 2] = 0.0;
}

// Triangular solve pieces on a vector x (in place), L lower in column-major H.
// diag: x_b <- L_bb^{-1} x_b (forward) or L_bb^{-T} x_b (backward); one CTA.
__global__ void tri_diag_kernel(const double* __restrict__ H, int64_t ldh, int64_t kb, int b,
                                double* x, int transpose) {
  extern __shared__ double L[];  // [NB][LDS]
  __shared__ double xs[NB];
  const int tid = threadIdx.x;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int c = e / b, r = e % b;
    L[r * LDS + c] = (r >= c) ? H[(kb + c) * ldh + kb + r] : 0.0;
  }
  for (int p = tid; p < b; p += blockDim.x) xs[p] = x[kb + p];
  __syncthreads();
  if (!transpose) {
    for (int p = 0; p < b; ++p) {
      if (tid == 0) xs[p] = xs[p] / L[p * LDS + p];
      __syncthreads();
      const double xp = xs[p];
      for (int q = p + 1 + tid; q < b; q += blockDim.x) xs[q] = __fma_rn(-L[q * LDS + p], xp, xs[q]);
      __syncthreads();
    }
  } else {
    for (int p = b - 1; p >= 0; --p) {
      if (tid == 0) xs[p] = xs[p] / L[p * LDS + p];
      __syncthreads();
      const double xp = xs[p];
      for (int q = tid; q < p; q += blockDim.x) xs[q] = __fma_rn(-L[p * LDS + q], xp, xs[q]);
      __syncthreads();
    }
  }
  for (int p = tid; p < b; p += blockDim.x) x[kb + p] = xs[p];
}

// Forward update: x[r] -= sum_p L[r, kb+p] x[kb+p] for r in [kb+b, m); thread per row.
__global__ void tri_fwd_update_kernel(const double* __restrict__ H, int64_t ldh, int64_t kb, int b,
                                      int64_t m, double* x) {
  __shared__ double xb[NB];
  for (int p = threadIdx.x; p < b; p += blockDim.x) xb[p] = x[kb + p];
  __syncthreads();
  const int64_t r = kb + b + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (r >= m) return;
  double s = 0.0;
  for (int p = 0; p < b; ++p) s = __fma_rn(H[(kb + p) * ldh + r], xb[p], s);
  x[r] -= s;
}

// Backward update: x[r] -= sum_p L[kb+p, r] x[kb+p] for r in [0, kb); warp per row.
__global__ void tri_bwd_update_kernel(const double* __restrict__ H, int64_t ldh, int64_t kb, int b,
                                      double* x) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= kb) return;
  double s = 0.0;
  for (int p = lane; p < b; p += 32) s = __fma_rn(H[r * ldh + kb + p], x[kb + p], s);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) x[r] -= s;
}

// |u|_2 into out[0] (squared when `squared`: column shards all-reduce it first).
__global__ void norm2_kernel(const double* __restrict__ u, int64_t m, double* out, int squared) {
  __shared__ double red[32][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) v[0] = __fma_rn(u[i], u[i], v[0]);
  block_reduce4<32>(v, red);
  if (threadIdx.x == 0) out[0] = squared ? v[0] : sqrt(v[0]);
}

__global__ void normalize_kernel(const double* __restrict__ u, double* __restrict__ v, int64_t m,
                                 const double* un, int squared) {
  const double s = squared ? sqrt(*un) : *un;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    v[i] = u[i] / s;
}

__global__ void embed_complex_kernel(const double* __restrict__ zr, const double* __restrict__ zi,
                                     int64_t ldz, int64_t n, double* __restrict__ E, int64_t lde) {
  // E = [[Zr, -Zi], [Zi, Zr]] (2n x 2n), column-major
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / n, i = e % n;
    const double a = zr[j * ldz + i], b = zi[j * ldz + i];
    E[j * lde + i] = a;
    E[j * lde + n + i] = b;
    E[(n + j) * lde + i] = -b;
    E[(n + j) * lde + n + i] = a;
  }
}

// A column block of the embedding: E = [[Zr, -Zi], [Zi, Zr]] restricted to this rank's
// columns j and n + j, stored as 2 ncols local columns (2n rows each).
__global__ void embed_complex_cols_kernel(const double* __restrict__ zr, const double* __restrict__ zi,
                                          int64_t ldz, int64_t n, int64_t ncols, double* __restrict__ E,
                                          int64_t lde) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n * ncols;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = e / n, i = e % n;
    const double a = zr[j * ldz + i], b = zi[j * ldz + i];
    E[j * lde + i] = a;
    E[j * lde + n + i] = b;
    E[(ncols + j) * lde + i] = -b;
    E[(ncols + j) * lde + n + i] = a;
  }
}

// ---------------------------------------------------------------------------
// Matrix-free inverse iteration: u = (Z^T Z)^{-1} v by conjugate gradients with
// Z resident in HBM (two GEMV passes over Z per CG step, no SYRK, no factor).
// Used when CG reaches |r| <= 1e-15 |b| within kCgMaxIters steps, which it does in
// a handful of steps for the well-conditioned bases IPT converges to (Z = I + small);
// otherwise the Cholesky path below runs. Every reduction is fixed-order.

constexpr int kCgMaxIters = 64;
constexpr int kCgBatch = 8;
constexpr int kZpRows = 512;       // rows per CTA of the Z p pass (2 per thread)
constexpr int kZpCols = 1024;      // columns per CTA of the Z p pass
constexpr int kVecBlocks = 296;    // fixed grid of the vector kernels
constexpr double kCgRelTol = 1e-15;

struct CgState {
  double rr, bb, alpha, beta;
  int done, iters;
};

// ypart[c][i] = sum_{j in chunk c} Z[i, j] p_j (column-major Z, rows x cols, 2 rows per
// thread). One rank: rows == cols (square Z); column shards: cols = the local columns.
__global__ void __launch_bounds__(256) cg_zp_kernel(const double* __restrict__ Z, int64_t ld, int64_t rows,
                                                    int64_t cols, const double* __restrict__ p,
                                                    double* __restrict__ ypart, const CgState* st) {
  if (st->done) return;
  const int64_t i = int64_t(blockIdx.x) * kZpRows + 2 * threadIdx.x;
  const int64_t j0 = int64_t(blockIdx.y) * kZpCols;
  const int64_t j1 = j0 + kZpCols < cols ? j0 + kZpCols : cols;
  if (i >= rows) return;
  double a0 = 0.0, a1 = 0.0;
  const double* zc = Z + i;
  int64_t j = j0;
  for (; j + 4 <= j1; j += 4) {
    const double2 z0 = *reinterpret_cast<const double2*>(zc + j * ld);
    const double2 z1 = *reinterpret_cast<const double2*>(zc + (j + 1) * ld);
    const double2 z2 = *reinterpret_cast<const double2*>(zc + (j + 2) * ld);
    const double2 z3 = *reinterpret_cast<const double2*>(zc + (j + 3) * ld);
    const double p0 = __ldg(p + j), p1 = __ldg(p + j + 1), p2 = __ldg(p + j + 2), p3 = __ldg(p + j + 3);
    a0 = __fma_rn(z0.x, p0, a0); a1 = __fma_rn(z0.y, p0, a1);
    a0 = __fma_rn(z1.x, p1, a0); a1 = __fma_rn(z1.y, p1, a1);
    a0 = __fma_rn(z2.x, p2, a0); a1 = __fma_rn(z2.y, p2, a1);
    a0 = __fma_rn(z3.x, p3, a0); a1 = __fma_rn(z3.y, p3, a1);
  }
  for (; j < j1; ++j) {
    const double2 z0 = *reinterpret_cast<const double2*>(zc + j * ld);
    const double pj = __ldg(p + j);
    a0 = __fma_rn(z0.x, pj, a0);
    a1 = __fma_rn(z0.y, pj, a1);
  }
  double* out = ypart + int64_t(blockIdx.y) * (rows + 2) + i;
  out[0] = a0;
  if (i + 1 < rows) out[1] = a1;
}

__global__ void cg_yreduce_kernel(const double* __restrict__ ypart, int64_t rows, int nchunks,
                                  double* __restrict__ y, const CgState* st) {
  if (st->done) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < rows; i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += ypart[int64_t(c) * (rows + 2) + i];
    y[i] = s;
  }
}

// q_j = Z[:, j] . y (warp per column, y zero beyond m) and per-CTA partials of p . q.
__global__ void __launch_bounds__(256) cg_ztq_kernel(const double* __restrict__ Z, int64_t ld, int64_t rows,
                                                     int64_t cols, const double* __restrict__ y,
                                                     const double* __restrict__ p, double* __restrict__ q,
                                                     double* __restrict__ partials, const CgState* st) {
  if (st->done) return;
  __shared__ double red[8][4];
  const int lane = threadIdx.x & 31;
  const int64_t j = blockIdx.x * int64_t(8) + (threadIdx.x >> 5);
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  if (j < cols) {
    const double2* zc = reinterpret_cast<const double2*>(Z + j * ld);
    const double2* yy = reinterpret_cast<const double2*>(y);
    const int64_t K2 = (rows + 1) / 2;
    double sx = 0.0, sy = 0.0;
    int64_t k = lane;
    for (; k + 96 < K2; k += 128) {
      const double2 a0 = zc[k], a1 = zc[k + 32], a2 = zc[k + 64], a3 = zc[k + 96];
      const double2 b0 = yy[k], b1 = yy[k + 32], b2 = yy[k + 64], b3 = yy[k + 96];
      sx = __fma_rn(a0.x, b0.x, sx); sy = __fma_rn(a0.y, b0.y, sy);
      sx = __fma_rn(a1.x, b1.x, sx); sy = __fma_rn(a1.y, b1.y, sy);
      sx = __fma_rn(a2.x, b2.x, sx); sy = __fma_rn(a2.y, b2.y, sy);
      sx = __fma_rn(a3.x, b3.x, sx); sy = __fma_rn(a3.y, b3.y, sy);
    }
    for (; k < K2; k += 32) {
      const double2 a0 = zc[k], b0 = yy[k];
      sx = __fma_rn(a0.x, b0.x, sx); sy = __fma_rn(a0.y, b0.y, sy);
    }
    double s = sx + sy;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) q[j] = s;
    v[0] = lane == 0 ? p[j] * s : 0.0;
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x * 4] = v[0];
}

// one thread block: fixed-order sum of `count` strided partials
__device__ double cg_sum_partials(const double* __restrict__ partials, int64_t count) {
  __shared__ double red[16][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) v[0] += partials[4 * i];
  block_reduce4<16>(v, red);
  return v[0];  // valid in thread 0
}

// Column shards: the fixed-order local sum goes to out[0]; the all-reduce of it across
// ranks is the `global` operand of the kernels below (nullptr: one rank, the partials).
__global__ void cg_local_sum_kernel(const double* __restrict__ partials, int64_t count, double* out,
                                    const CgState* st) {
  if (st != nullptr && st->done) return;
  const double s = cg_sum_partials(partials, count);
  if (threadIdx.x == 0) out[0] = s;
}

__global__ void cg_alpha_kernel(const double* __restrict__ partials, int64_t count, CgState* st,
                                const double* global) {
  if (st->done) return;
  const double pq = global ? *global : cg_sum_partials(partials, count);
  if (threadIdx.x == 0) st->alpha = st->rr / pq;
}

// x += alpha p, r -= alpha q, partials of r . r
__global__ void cg_update_kernel(int64_t m, const double* __restrict__ p, const double* __restrict__ q,
                                 double* __restrict__ x, double* __restrict__ r, double* __restrict__ partials,
                                 const CgState* st) {
  if (st->done) return;
  __shared__ double red[8][4];
  const double a = st->alpha;
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    x[i] = __fma_rn(a, p[i], x[i]);
    const double ri = __fma_rn(-a, q[i], r[i]);
    r[i] = ri;
    v[0] = __fma_rn(ri, ri, v[0]);
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x * 4] = v[0];
}

__global__ void cg_beta_kernel(const double* __restrict__ partials, int64_t count, CgState* st,
                               const double* global) {
  if (st->done) return;
  const double rr = global ? *global : cg_sum_partials(partials, count);
  if (threadIdx.x == 0) {
    st->beta = rr / st->rr;
    st->rr = rr;
    st->iters += 1;
    if (!(rr > kCgRelTol * kCgRelTol * st->bb)) st->done = 1;  // also stops on NaN
  }
}

__global__ void cg_p_kernel(int64_t m, const double* __restrict__ r, double* __restrict__ p, const CgState* st) {
  if (st->done) return;
  const double b = st->beta;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = __fma_rn(b, p[i], r[i]);
}

// x = 0, r = p = b, partials of b . b
__global__ void cg_init_kernel(int64_t m, const double* __restrict__ b, double* __restrict__ x,
                               double* __restrict__ r, double* __restrict__ p, double* __restrict__ partials) {
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < m; i += int64_t(gridDim.x) * blockDim.x) {
    const double bi = b[i];
    x[i] = 0.0;
    r[i] = bi;
    p[i] = bi;
    v[0] = __fma_rn(bi, bi, v[0]);
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) partials[blockIdx.x * 4] = v[0];
}

__global__ void cg_start_kernel(const double* __restrict__ partials, int64_t count, CgState* st,
                                const double* global) {
  const double bb = global ? *global : cg_sum_partials(partials, count);
  if (threadIdx.x == 0) {
    st->rr = bb;
    st->bb = bb;
    st->alpha = st->beta = 0.0;
    st->iters = 0;
    st->done = (bb > 0.0) ? 0 : 1;
  }
}

// Host replica of deterministic_unit (solver.cpp:95-109).
std::vector<double> deterministic_unit(int64_t n) {
  std::vector<double> v(n);
  uint64_t x = 0x243f6a8885a308d3ull;
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    z ^= z >> 31;
    v[i] = 0.5 + static_cast<double>(z >> 40) / static_cast<double>(1 << 24);
  }
  for (int64_t i = 0; i < n; ++i) s += v[i] * v[i];
  const double nv = std::sqrt(s);
  for (auto& e : v) e /= nv;
  return v;
}

// The reference's inverse power iteration (solver.cpp:283-296) with the solves done
// by CG on Z^T Z. Returns false (caller factors instead) if any inner solve misses
// the tolerance within kCgMaxIters steps. Z is rows x cols; v0 is the start vector's
// entries for these columns. With `comm` the columns are this rank's shard: y = Z p is
// all-reduced over the ranks and every dot product is a local fixed-order sum followed
// by an all-reduce, so all ranks take the same decisions (one rank: comm == nullptr,
// rows == cols, the partials are summed directly).
bool sigma_min_cg(Ctx& c, int64_t rows, int64_t cols, const std::vector<double>& v0, const double* Z, int64_t ld,
                  int max_iters, double tol, Comm* comm, double* estimate, int* outer_steps, int* cg_steps) {
  cudaStream_t s = c.stream;
  const bool prof = std::getenv("IPT_PROFILE") != nullptr;
  auto wall = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  double t_mark = wall();
  const int nchunks = static_cast<int>(std::max<int64_t>(1, ceil_div(cols, kZpCols)));
  const int64_t clen = cols + 2, rlen = rows + 2;
  DevBuf x, r, p, q, y, ypart, v, un, parts, glob;
  x.alloc(clen);
  r.alloc(clen);
  p.alloc(clen);
  q.alloc(clen);
  v.alloc(clen);
  y.alloc(rlen);
  un.alloc(1);
  glob.alloc(4);
  ypart.alloc(size_t(nchunks) * rlen, false);
  const int64_t ztq_blocks = std::max<int64_t>(1, ceil_div(cols, 8));
  parts.alloc(size_t(std::max<int64_t>(ztq_blocks, kVecBlocks)) * 4);
  CgState* st = nullptr;
  IPT_CUDA(cudaMalloc(&st, sizeof(CgState)));
  std::unique_ptr<CgState, void (*)(CgState*)> st_guard(st, [](CgState* pp) { cudaFree(pp); });
  CgState* h_st = reinterpret_cast<CgState*>(c.h_aux);  // pinned scratch
  static_assert(sizeof(CgState) <= 256, "pinned scratch too small");
  if (cols > 0) IPT_CUDA(cudaMemcpyAsync(v.get(), v0.data(), sizeof(double) * cols, cudaMemcpyHostToDevice, s));
  if (prof) {
    c.sync();
    std::fprintf(stderr, "[ipt]   cg setup %.1f ms\n", 1e3 * (wall() - t_mark));
    t_mark = wall();
  }
  const int sq = comm ? 1 : 0;
  // all-reduced sum of the local partials into glob[slot] (column shards only)
  auto global_sum = [&](int64_t count, int slot, const CgState* gate) -> const double* {
    if (!comm) return nullptr;
    cg_local_sum_kernel<<<1, 512, 0, s>>>(parts.get(), count, glob.get() + slot, gate);
    count_launch();
    comm->all_reduce(glob.get() + slot, 1, CommType::F64, CommOp::Sum, s);
    return glob.get() + slot;
  };
  const dim3 zp_grid(static_cast<unsigned>(std::max<int64_t>(1, ceil_div(rows, kZpRows))), static_cast<unsigned>(nchunks));
  double rho = 0.0;
  int steps = 0, total_cg = 0;
  for (int it = 0; it < max_iters; ++it) {
    steps = it + 1;
    cg_init_kernel<<<kVecBlocks, 256, 0, s>>>(cols, v.get(), x.get(), r.get(), p.get(), parts.get());
    count_launch();
    cg_start_kernel<<<1, 512, 0, s>>>(parts.get(), kVecBlocks, st, global_sum(kVecBlocks, 0, nullptr));
    count_launch();
    int done = 0;
    for (int k = 0; k < kCgMaxIters && !done; k += kCgBatch) {
      for (int b = 0; b < kCgBatch; ++b) {
        cg_zp_kernel<<<zp_grid, 256, 0, s>>>(Z, ld, rows, cols, p.get(), ypart.get(), st);
        cg_yreduce_kernel<<<kVecBlocks, 256, 0, s>>>(ypart.get(), rows, nchunks, y.get(), st);
        count_launch(2);
        if (comm) comm->all_reduce(y.get(), size_t(rows), CommType::F64, CommOp::Sum, s);
        cg_ztq_kernel<<<static_cast<unsigned>(ztq_blocks), 256, 0, s>>>(Z, ld, rows, cols, y.get(), p.get(), q.get(),
                                                                        parts.get(), st);
        count_launch();
        cg_alpha_kernel<<<1, 512, 0, s>>>(parts.get(), ztq_blocks, st, global_sum(ztq_blocks, 1, st));
        cg_update_kernel<<<kVecBlocks, 256, 0, s>>>(cols, p.get(), q.get(), x.get(), r.get(), parts.get(), st);
        count_launch(2);
        cg_beta_kernel<<<1, 512, 0, s>>>(parts.get(), kVecBlocks, st, global_sum(kVecBlocks, 2, st));
        cg_p_kernel<<<kVecBlocks, 256, 0, s>>>(cols, r.get(), p.get(), st);
        count_launch(2);
      }
      IPT_LAUNCH_CHECK();
      IPT_CUDA(cudaMemcpyAsync(h_st, st, sizeof(CgState), cudaMemcpyDeviceToHost, s));
      c.sync();
      done = h_st->done;
      if (prof) {
        std::fprintf(stderr, "[ipt]   cg batch %.1f ms (done %d, iters %d)\n", 1e3 * (wall() - t_mark), done, h_st->iters);
        t_mark = wall();
      }
    }
    total_cg += h_st->iters;
    if (!done || !(h_st->rr <= kCgRelTol * kCgRelTol * h_st->bb)) return false;
    norm2_kernel<<<1, 1024, 0, s>>>(x.get(), cols, un.get(), sq);
    count_launch();
    if (comm) comm->all_reduce(un.get(), 1, CommType::F64, CommOp::Sum, s);
    normalize_kernel<<<kVecBlocks, 256, 0, s>>>(x.get(), v.get(), cols, un.get(), sq);
    count_launch();
    IPT_LAUNCH_CHECK();
    double h_un = 0.0;
    IPT_CUDA(cudaMemcpyAsync(&h_un, un.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    c.sync();
    if (comm) h_un = std::sqrt(h_un);
    if (!std::isfinite(h_un) || h_un == 0.0) return false;
    if (it > 0 && std::fabs(h_un - rho) <= tol * h_un) {
      rho = h_un;
      break;
    }
    rho = h_un;
  }
  *estimate = 1.0 / std::sqrt(rho);
  *outer_steps = steps;
  *cg_steps = total_cg;
  return true;
}

}  // namespace

double sigma_min_device(Ctx& c, int64_t n, const double* zr, const double* zi, int64_t ldz,
                        int max_iters, double tol) {
  NvtxRange nvtx_("ipt:sigma_min");
  cudaStream_t s = c.stream;
  const bool cplx = zi != nullptr;
  const int64_t m = cplx ? 2 * n : n;
  const double* Z = zr;
  int64_t ld = ldz;
  DevBuf E;
  if (cplx) {
    ld = round_up(m, 16);
    E.alloc(size_t(round_up(m, kBN)) * ld);
    embed_complex_kernel<<<1184, 256, 0, s>>>(zr, zi, ldz, n, E.get(), ld);
    IPT_LAUNCH_CHECK();
    count_launch();
    Z = E.get();
  }
  const bool prof = std::getenv("IPT_PROFILE") != nullptr;
  auto wall = [] { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  {
    // IPT_SIGMA=factor skips the matrix-free attempt (tests compare the two paths)
    const char* mode = std::getenv("IPT_SIGMA");
    if (!(mode && std::strcmp(mode, "factor") == 0)) {
      const double t0 = wall();
      double est = 0.0;
      int outer = 0, inner = 0;
      std::vector<double> v0 = deterministic_unit(n);  // complex: the iteration from [v; 0]
      v0.resize(m, 0.0);
      const bool ok = sigma_min_cg(c, m, m, v0, Z, ld, max_iters, tol, nullptr, &est, &outer, &inner);
      if (prof)
        std::fprintf(stderr, "[ipt] sigma_min n=%lld: matrix-free CG %s, %.1f ms (%d outer steps, %d CG steps)\n",
                     static_cast<long long>(m), ok ? "converged" : "fell back", 1e3 * (wall() - t0), outer, inner);
      if (ok) return est;
    }
  }
  const int64_t ldh = round_up(m, 16);
  DevBuf H;
  H.alloc(size_t(ldh) * m, false);
  {  // H = Z^T Z, lower tiles only (the Cholesky below reads the lower triangle): SYRK
    GemmParams g{};
    g.K = ld;
    g.A = Z;
    g.lda = ld;
    g.B = Z;
    g.ldb = ld;
    g.C = H.get();
    g.ldc = ldh;
    g.tiles_m = static_cast<int>(ceil_div(m, kBM));
    g.tiles_n = g.tiles_m;
    g.lower_only = 1;
    g.n_rows = m;
    g.n_cols = m;
    launch_gemm(kGemmStore, g, s);
  }

  DevBuf scratch;
  scratch.alloc(1184 * 4 + 8);
  absmax_kernel<<<1184, 256, 0, s>>>(H.get(), ldh, m, scratch.get());
  IPT_LAUNCH_CHECK();
  count_launch();
  reduce_partials(s, scratch.get(), 1184, scratch.get() + 1184 * 4, nullptr);
  double hmax4[4];
  IPT_CUDA(cudaMemcpyAsync(hmax4, scratch.get() + 1184 * 4, sizeof(hmax4), cudaMemcpyDeviceToHost, s));
  c.sync();
  const double tiny = hmax4[3] * 2.220446049250313e-16 * static_cast<double>(m);
  const double t_syrk = wall();

  int* d_sing = nullptr;
  IPT_CUDA(cudaMalloc(&d_sing, sizeof(int)));
  IPT_CUDA(cudaMemsetAsync(d_sing, 0, sizeof(int), s));
  // Two-level right-looking Cholesky: outer panels of kW = 512 columns, factored in
  // NB = 128 sub-blocks (potrf + trsm + an intra-panel update with K = 128); the
  // trailing matrix then takes ONE K = 512 DMMA update per outer panel, so the
  // read-modify-write of each trailing tile is amortised over 4x more k-steps.
  constexpr int64_t kW = 4 * NB;
  DevBuf Pb;  // L21 of the current outer panel, row-major, row i = matrix row kb + i
  Pb.alloc((size_t(round_up(m, kBM)) + kW) * kW);
  static PerDeviceOnce attr;
  attr.run([] {
    IPT_CUDA(cudaFuncSetAttribute(potrf_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(NB * LDS * sizeof(double))));
    IPT_CUDA(cudaFuncSetAttribute(trsm_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int((NB + 32) * LDS * sizeof(double))));
    IPT_CUDA(cudaFuncSetAttribute(tri_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(NB * LDS * sizeof(double))));
  });
  auto sub_update = [&](const double* panel, int64_t k, int64_t r0, int64_t rows, int64_t cols) {
    // H[r0.., r0..r0+cols) -= panel[r0..] panel[r0..r0+cols)^T, lower tiles of the block
    if (rows <= 0 || cols <= 0) return;
    GemmParams g{};
    g.K = k;
    g.A = panel;
    g.lda = kW;
    g.B = panel;
    g.ldb = kW;
    g.C = H.get() + r0 * ldh + r0;
    g.ldc = ldh;
    g.tiles_m = static_cast<int>(ceil_div(rows, kBM));
    g.tiles_n = static_cast<int>(ceil_div(cols, kBN));
    g.n_rows = rows;
    g.n_cols = cols;
    launch_gemm(kGemmSub, g, s);
  };
  for (int64_t kb = 0; kb < m; kb += kW) {
    const int64_t wcols = std::min<int64_t>(kW, m - kb);
    for (int64_t jb = 0; jb < wcols; jb += NB) {
      const int64_t c0 = kb + jb;
      const int b = static_cast<int>(std::min<int64_t>(NB, m - c0));
      potrf_block_kernel<<<1, 512, NB * LDS * sizeof(double), s>>>(H.get(), ldh, c0, b, tiny, d_sing);
      IPT_LAUNCH_CHECK();
      count_launch();
      const int64_t rem = m - c0 - b;
      if (rem <= 0) break;
      // L21 of this sub-block -> H and the panel (rows c0+b.., columns jb..jb+b of the panel)
      double* pblk = Pb.get() + (jb + b) * kW + jb;
      trsm_panel_kernel<<<static_cast<unsigned>(ceil_div(rem, 32)), 256, (NB + 32) * LDS * sizeof(double), s>>>(
          H.get(), ldh, c0, b, rem, pblk, kW);
      IPT_LAUNCH_CHECK();
      count_launch();
      // intra-panel update of the panel's remaining columns (K = b)
      const int64_t cols_left = wcols - jb - b;
      if (cols_left > 0) sub_update(pblk, NB, c0 + b, rem, cols_left);
    }
    // trailing update with the whole panel (K = 512, zero-padded when narrower)
    const int64_t r0 = kb + wcols;
    if (r0 < m) sub_update(Pb.get() + wcols * kW, kW, r0, m - r0, m - r0);
  }
  int sing = 0;
  IPT_CUDA(cudaMemcpyAsync(&sing, d_sing, sizeof(int), cudaMemcpyDeviceToHost, s));
  c.sync();
  cudaFree(d_sing);
  const double t_chol = wall();
  if (sing) return 0.0;

  // inverse power iteration (solver.cpp:283-296)
  std::vector<double> v0 = deterministic_unit(n);
  DevBuf v, u, un;
  v.alloc(m);
  u.alloc(m);
  un.alloc(1);
  IPT_CUDA(cudaMemcpyAsync(v.get(), v0.data(), sizeof(double) * n, cudaMemcpyHostToDevice, s));
  double rho = 0.0;
  int iters_done = 0;
  for (int it = 0; it < max_iters; ++it) {
    iters_done = it + 1;
    IPT_CUDA(cudaMemcpyAsync(u.get(), v.get(), sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
    for (int64_t kb = 0; kb < m; kb += NB) {  // L y = v
      const int b = static_cast<int>(std::min<int64_t>(NB, m - kb));
      tri_diag_kernel<<<1, 256, NB * LDS * sizeof(double), s>>>(H.get(), ldh, kb, b, u.get(), 0);
      count_launch();
      const int64_t rem = m - kb - b;
      if (rem > 0) {
        tri_fwd_update_kernel<<<static_cast<unsigned>(ceil_div(rem, 256)), 256, 0, s>>>(H.get(), ldh, kb, b, m, u.get());
        count_launch();
      }
    }
    const int64_t last = (m - 1) / NB * NB;
    for (int64_t kb = last; kb >= 0; kb -= NB) {  // L^T u = y
      const int b = static_cast<int>(std::min<int64_t>(NB, m - kb));
      tri_diag_kernel<<<1, 256, NB * LDS * sizeof(double), s>>>(H.get(), ldh, kb, b, u.get(), 1);
      count_launch();
      if (kb > 0) {
        tri_bwd_update_kernel<<<static_cast<unsigned>(ceil_div(kb, 8)), 256, 0, s>>>(H.get(), ldh, kb, b, u.get());
        count_launch();
      }
    }
    IPT_LAUNCH_CHECK();
    norm2_kernel<<<1, 1024, 0, s>>>(u.get(), m, un.get(), 0);
    normalize_kernel<<<296, 256, 0, s>>>(u.get(), v.get(), m, un.get(), 0);
    count_launch(2);
    IPT_LAUNCH_CHECK();
    double h_un = 0.0;
    IPT_CUDA(cudaMemcpyAsync(&h_un, un.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    c.sync();
    if (!std::isfinite(h_un) || h_un == 0.0) return 0.0;
    if (it > 0 && std::fabs(h_un - rho) <= tol * h_un) {
      rho = h_un;
      break;
    }
    rho = h_un;
  }
  if (prof)
    std::fprintf(stderr, "[ipt] sigma_min n=%lld: cholesky %.1f ms, inverse iteration %.1f ms (%d steps)\n",
                 static_cast<long long>(m), 1e3 * (t_chol - t_syrk), 1e3 * (wall() - t_chol), iters_done);
  return 1.0 / std::sqrt(rho);
}

// Column shards (rank's columns [col0, col0 + ncols) of the n x n Z, column-major, ldz):
// the same inverse iteration by CG with y = Z p all-reduced, so Z is never gathered.
// *ok == false: CG missed its tolerance (the caller gathers Z for the factor path).
double sigma_min_sharded(Ctx& c, int64_t n, int64_t col0, int64_t ncols, const double* zr, const double* zi,
                         int64_t ldz, int max_iters, double tol, bool* ok) {
  NvtxRange nvtx_("ipt:sigma_min_sharded");
  cudaStream_t s = c.stream;
  const bool cplx = zi != nullptr;
  const std::vector<double> unit = deterministic_unit(n);
  std::vector<double> v0(size_t(cplx ? 2 : 1) * ncols, 0.0);  // complex: [v; 0] restricted to columns j, n + j
  for (int64_t j = 0; j < ncols; ++j) v0[j] = unit[col0 + j];
  const double* Z = zr;
  int64_t ld = ldz, rows = n, cols = ncols;
  DevBuf E;
  if (cplx) {
    rows = 2 * n;
    cols = 2 * ncols;
    ld = round_up(rows, 16);
    E.alloc(size_t(std::max<int64_t>(cols, 1)) * ld);
    embed_complex_cols_kernel<<<1184, 256, 0, s>>>(zr, zi, ldz, n, ncols, E.get(), ld);
    IPT_LAUNCH_CHECK();
    count_launch();
    Z = E.get();
  }
  double est = 0.0;
  int outer = 0, inner = 0;
  *ok = sigma_min_cg(c, rows, cols, v0, Z, ld, max_iters, tol, c.comm.get(), &est, &outer, &inner);
  if (std::getenv("IPT_PROFILE"))
    std::fprintf(stderr, "[ipt] sigma_min (column shards) n=%lld: CG %s (%d outer steps, %d CG steps)\n",
                 static_cast<long long>(rows), *ok ? "converged" : "missed", outer, inner);
  return est;
}

}  // namespace iptb
