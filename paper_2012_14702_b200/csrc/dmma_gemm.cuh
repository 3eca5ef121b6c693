// K1: FP64 tensor-core (DMMA) TN GEMM for sm_100a with the IPT map epilogue.
//
// C[i, j] = sum_k A[i, k] * B[k, j]
//   A : M x K row-major (K contiguous)      -> Delta, rows of the operator
//   B : K x Ncols column-major (K contiguous)-> Z, the current eigenbasis block
// Both operands are K-major, which is the `.row.col` form of
// mma.sync.aligned.m16n8k4.row.col.f64 (8x8x4 DMMA in SASS). tcgen05 has no
// f64 kind, so on B200 the FP64 tensor path is the warp-level DMMA; measured
// peak 37.1 TFLOP/s (profiles/r01_fp64_probe.txt).
//
// Epilogue modes (fused, no W = Delta Z round trip through HBM):
//   kGemmStore : C = W (col-major)                                   [plain product]
//   kGemmMap   : F_ij = (i == j_glob) ? 1 : (Z_ij * wd_j - W_ij) / (d_i - d_jglob)
//                stored to C; per-CTA partials {sum (F-Z)^2, sum Z^2, sum F^2, max|F-Z|}
//                -> proj/src/solver.cpp:212-229 (F at :220)
//   kGemmResid : partial sum |d_i Z_ij + W_ij - Z_ij lam_j|^2, nothing stored
//                -> proj/src/solver.cpp:258-267
//   kGemmSub   : C -= W (blocked Cholesky trailing update, lower tiles only)
//
// Tiling: CTA 128x128, BK = 16 doubles, 4-stage cp.async pipeline into a
// 128-byte-XOR-swizzled shared layout (conflict-free fragment reads), 8 warps
// each owning a 64x32 accumulator tile (64 doubles / thread). All operands are
// zero-padded by the caller to whole tiles, so the main loop has no bounds
// checks; only the epilogue is predicated on the true (n_rows, n_cols).
#pragma once

#include "ipt_common.cuh"

namespace iptb {

enum GemmMode : int { kGemmStore = 0, kGemmMap = 1, kGemmResid = 2, kGemmSub = 3 };

constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kBK = 16;
constexpr int kStages = 4;
constexpr int kGemmThreads = 256;
constexpr int kGroupM = 8;  // tile-row group for L2-friendly rasterisation
constexpr int kStageDoubles = (kBM + kBN) * kBK;
constexpr size_t kGemmSmemBytes = size_t(kStages) * kStageDoubles * sizeof(double);

struct GemmParams {
  int64_t K;                // loop length, multiple of kBK, operands zero-padded to it
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int tiles_m, tiles_n;
  // IPT epilogue inputs
  const double* d;          // diagonal of M, global row/column index
  const double* wd;         // (Delta Z)_jj per local column
  const double* lam;        // eigenvalues per local column (resid mode)
  int64_t col0;             // global column index of local column 0
  int64_t row0;             // global row index of local row 0 (sub-blocks)
  int64_t n_rows, n_cols;   // true extents of C
  double* partials;         // [tiles_m * tiles_n][4]
  const LoopState* state;   // nullable; CTA exits if state->done
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Element (r, k) of a 16-double-wide shared tile row. A fragment read covers rows
// g = 0..7 x k0..k0+3 (one 32-byte unit pair per row); XORing the unit index with
// 2*(r&3) sends the four rows of each half-warp phase to four distinct unit pairs,
// i.e. all 32 banks once per phase (conflict-free LDS.64).
__device__ __forceinline__ int swz(int r, int k) { return r * kBK + ((((k >> 1) ^ ((r & 3) << 1)) << 1) | (k & 1)); }

// Grouped rasterisation: kGroupM tile-rows at a time, column-major inside the group,
// so the ~148 co-resident CTAs share a few Delta row panels and Z column panels in L2.
__device__ __forceinline__ void tile_coords(int lin, int tiles_m, int tiles_n, int& tm, int& tn) {
  const int per_group = kGroupM * tiles_n;
  const int group = lin / per_group;
  const int first_m = group * kGroupM;
  const int gsize = min(tiles_m - first_m, kGroupM);
  const int in = lin - group * per_group;
  tm = first_m + in % gsize;
  tn = in / gsize;
}

template <int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1) dmma_gemm_kernel(const GemmParams p) {
  if (p.state != nullptr && p.state->done) return;
  extern __shared__ __align__(128) double smem[];

  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  if (MODE == kGemmSub && tn > tm) return;  // strictly-upper tiles of a symmetric update
  const int64_t m0 = int64_t(tm) * kBM, n0 = int64_t(tn) * kBN;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, 64 x 32 each

  const double* __restrict__ Ag = p.A + m0 * p.lda;
  const double* __restrict__ Bg = p.B + n0 * p.ldb;
  const int KT = static_cast<int>(p.K / kBK);

  auto load_stage = [&](int s, int kt) {
    double* as = smem + s * kStageDoubles;
    double* bs = as + kBM * kBK;
    const int64_t k0 = int64_t(kt) * kBK;
#pragma unroll
    for (int i = 0; i < (kBM * kBK / 2) / kGemmThreads; ++i) {
      const int c = tid + i * kGemmThreads;
      const int row = c >> 3, u = c & 7;
      cp_async16(as + row * kBK + ((u ^ ((row & 3) << 1)) << 1), Ag + row * p.lda + k0 + u * 2);
    }
#pragma unroll
    for (int i = 0; i < (kBN * kBK / 2) / kGemmThreads; ++i) {
      const int c = tid + i * kGemmThreads;
      const int col = c >> 3, u = c & 7;
      cp_async16(bs + col * kBK + ((u ^ ((col & 3) << 1)) << 1), Bg + col * p.ldb + k0 + u * 2);
    }
  };

  double acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < KT) load_stage(s, s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nk = kt + kStages - 1;
      if (nk < KT) load_stage(nk % kStages, nk);
      cp_async_commit();
    }
    const double* as = smem + (kt % kStages) * kStageDoubles;
    const double* bs = as + kBM * kBK;
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const int k = kk * 4 + t;
      double af[4][2], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = wm * 64 + mi * 16 + g;
        af[mi][0] = as[swz(r, k)];
        af[mi][1] = as[swz(r + 8, k)];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = bs[swz(wn * 32 + ni * 8 + g, k)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_16x8x4(acc[mi][ni], af[mi][0], af[mi][1], bf[ni]);
    }
  }
  cp_async_wait<0>();

  // ------------------------------ epilogue ------------------------------
  if (MODE == kGemmStore || MODE == kGemmSub) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t i = m0 + wm * 64 + mi * 16 + g + ((r >> 1) << 3);
          const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + (r & 1);
          if (i < p.n_rows && j < p.n_cols) {
            double* cp = p.C + j * p.ldc + i;
            if (MODE == kGemmStore) *cp = acc[mi][ni][r];
            else *cp = __dsub_rn(*cp, acc[mi][ni][r]);
          }
        }
    return;
  }

  __shared__ double red[kGemmThreads / 32][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int ni = 0; ni < 4; ++ni)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + e;
      if (j >= p.n_cols) continue;
      const int64_t jg = p.col0 + j;
      const double dj = p.d[jg];
      const double wj = MODE == kGemmMap ? p.wd[j] : p.lam[j];
      const double* zcol = p.B + j * p.ldb;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int64_t i = m0 + wm * 64 + mi * 16 + g + h * 8;
          if (i >= p.n_rows) continue;
          const int64_t ig = p.row0 + i;
          const double w = acc[mi][ni][h * 2 + e];
          const double z = zcol[i];
          if (MODE == kGemmMap) {
            // (z * wd - w) / (d_i - d_j): each operation rounded on its own, as
            // the reference's complex arithmetic does for zero imaginary parts.
            const double f = (ig == jg) ? 1.0
                                        : __ddiv_rn(__dsub_rn(__dmul_rn(z, wj), w), __dsub_rn(p.d[ig], dj));
            p.C[j * p.ldc + i] = f;
            const double df = __dsub_rn(f, z);
            v[0] = __fma_rn(df, df, v[0]);
            v[1] = __fma_rn(z, z, v[1]);
            v[2] = __fma_rn(f, f, v[2]);
            v[3] = nan_max(v[3], fabs(df));
          } else {  // kGemmResid
            const double r = __dsub_rn(__dadd_rn(__dmul_rn(p.d[ig], z), w), __dmul_rn(z, wj));
            v[0] = __fma_rn(r, r, v[0]);
          }
        }
    }
  block_reduce4<kGemmThreads / 32>(v, red);
  if (threadIdx.x == 0) {
    double* out = p.partials + size_t(blockIdx.x) * 4;
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
    out[3] = v[3];
  }
}

}  // namespace iptb
