// K1: FP64 tensor-core (DMMA) TN GEMM for sm_100a with the IPT map epilogue.
//
// C[i, j] = sum_k A[i, k] * B[k, j]
//   A : M x K row-major (K contiguous)       -> Delta, rows of the operator
//   B : K x Ncols column-major (K contiguous) -> Z, the current eigenbasis block
// Both operands are K-major, which is the `.row.col` form of
// mma.sync.aligned.m16n8k4.row.col.f64 (SASS DMMA.8x8x4). tcgen05 has no f64
// kind, so on B200 the FP64 tensor path is the warp-level DMMA; measured issue
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
//   kGemmMapC / kGemmResidC : complex Delta Z by three real GEMMs (3M): T1 = Dr Zr and
//                T2 = Di Zi stored, this launch computes T3 = (Dr + Di)(Zr + Zi) and forms
//                W = (T1 - T2) + i (T3 - T1 - T2) in the epilogue, then the complex map
//                (F stored to C / Cim) or the complex residual, with the same partials.
//
// Main loop (dmma_tma_kernel): CTA tile 128x128, BK = 16 doubles, a 6-stage
// TMA pipeline (cp.async.bulk.tensor with 128-byte swizzle, full/empty mbarriers;
// thread 0 issues the loads one stage behind the consumers, so no separate
// producer warp competes for the 255-register budget) feeding 8 warps, each owning a 64x32
// accumulator tile (64 doubles / thread). Within a k-tile, mma slot t of step kk
// takes k = 8*(t>>1) + 2*kk + (t&1): with the TMA 128B swizzle (16-byte unit u of
// row r stored at u ^ (r&7)) every LDS.64 fragment phase then hits all 32 banks
// once. The k order inside a tile is a permutation, so A and B agree and the sum
// is unchanged. All operands are zero-padded by the caller to whole tiles, so the
// main loop has no bounds checks; only the epilogue is predicated.
#pragma once

#include <cuda.h>

#include "ipt_common.cuh"

namespace iptb {

enum GemmMode : int {
  kGemmStore = 0,
  kGemmMap = 1,
  kGemmResid = 2,
  kGemmSub = 3,
  kGemmMapC = 4,
  kGemmResidC = 5,
  kGemmSubC = 6,   // complex C -= W with W from T1, T2 and this launch's T3 (3M), C / Cim planes
  kGemmSubAll = 7  // C -= W on every tile (general, not a symmetric lower update)
};

constexpr int kBM = 128;
constexpr int kBN = 128;
constexpr int kBK = 16;
constexpr int kStages = 6;
constexpr int kConsumerWarps = 8;
constexpr int kGemmThreads = kConsumerWarps * 32;  // thread 0 doubles as the TMA producer
constexpr int kGroupM = 8;  // tile-row group for L2-friendly rasterisation
constexpr int kTileDoubles = kBM * kBK;                   // one operand tile = 16 KB
constexpr int kStageBytes = 2 * kTileDoubles * 8;         // A + B
constexpr size_t kGemmSmemBytes = size_t(kStages) * kStageBytes + 1024 /*align*/ + 2 * kStages * 8;

struct GemmParams {
  int64_t K;                // loop length, multiple of kBK, operands zero-padded to it
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  int tiles_m, tiles_n;
  int lower_only;           // symmetric result: compute only tiles with tile_n <= tile_m
  // IPT epilogue inputs
  const double* d;          // diagonal of M, global row/column index
  const double* wd;         // (Delta Z)_jj per local column
  const double* lam;        // eigenvalues per local column (resid mode)
  int64_t col0;             // global column index of local column 0
  int64_t row0;             // global row index of local row 0 (sub-blocks)
  int64_t n_rows, n_cols;   // true extents of C
  double* partials;         // [tiles_m * tiles_n][4]
  const LoopState* state;   // nullable; CTA exits if state->done
  // complex epilogues (kGemmMapC / kGemmResidC)
  const double* T1;         // Dr Zr, column-major (ldt)
  const double* T2;         // Di Zi
  int64_t ldt;
  const double* zre;        // current Z planes, column-major (ldzz)
  const double* zim;
  int64_t ldzz;
  const double* wdi;        // imaginary parts of wd, d, lam
  const double* di;
  const double* lami;
  double* Cim;              // imaginary plane of F (map), ldc
};

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ void dmma_16x8x4(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 "
      "{%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

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

// Element (r, k) of a TMA SWIZZLE_128B tile with 16-double (128-byte) rows.
__device__ __forceinline__ int swz128(int r, int k) { return r * kBK + ((((k >> 1) ^ (r & 7)) << 1) | (k & 1)); }

// ------------------------------------------------------------------ epilogue

template <int MODE>
__device__ __forceinline__ void gemm_epilogue(const GemmParams& p, double (&acc)[4][4][4], int64_t m0,
                                              int64_t n0, int warp, int lane, double v[4]) {
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;
  if (MODE == kGemmStore || MODE == kGemmSub || MODE == kGemmSubAll) {
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
            else *cp = __dsub_rn(*cp, acc[mi][ni][r]);  // kGemmSub, kGemmSubAll
          }
        }
    return;
  }
  if (MODE == kGemmSubC) {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t i = m0 + wm * 64 + mi * 16 + g + ((r >> 1) << 3);
          const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + (r & 1);
          if (i < p.n_rows && j < p.n_cols) {
            const double t1 = p.T1[j * p.ldt + i], t2 = p.T2[j * p.ldt + i];
            p.C[j * p.ldc + i] -= t1 - t2;
            p.Cim[j * p.ldc + i] -= acc[mi][ni][r] - t1 - t2;
          }
        }
    return;
  }
  if (MODE == kGemmMapC || MODE == kGemmResidC) {
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + e;
        if (j >= p.n_cols) continue;
        const int64_t jg = p.col0 + j;
        const cd dj{p.d[jg], p.di[jg]};
        const cd wj = MODE == kGemmMapC ? cd{p.wd[j], p.wdi[j]} : cd{p.lam[j], p.lami[j]};
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int64_t i = m0 + wm * 64 + mi * 16 + g + h * 8;
            if (i >= p.n_rows) continue;
            const int64_t ig = p.row0 + i;
            const double t1 = p.T1[j * p.ldt + i], t2 = p.T2[j * p.ldt + i];
            const cd w{t1 - t2, acc[mi][ni][h * 2 + e] - t1 - t2};
            const cd z{p.zre[j * p.ldzz + i], p.zim[j * p.ldzz + i]};
            const cd di{p.d[ig], p.di[ig]};
            if (MODE == kGemmMapC) {
              const cd f = (ig == jg) ? cd{1.0, 0.0} : cdiv(csub(cmul(z, wj), w), csub(di, dj));
              p.C[j * p.ldc + i] = f.re;
              p.Cim[j * p.ldc + i] = f.im;
              const cd df = csub(f, z);
              v[0] += df.re * df.re + df.im * df.im;
              v[1] += z.re * z.re + z.im * z.im;
              v[2] += f.re * f.re + f.im * f.im;
              v[3] = nan_max(v[3], hypot(df.re, df.im));
            } else {
              const cd r = csub(cadd(cmul(di, z), w), cmul(z, wj));
              v[0] += r.re * r.re + r.im * r.im;
            }
          }
      }
    return;
  }
  // Real map / residual. The thread's 8 rows' d_i load once, and each column's 8 entries of
  // Z load together, one column ahead of the column being computed and stored (round 2:
  // with the load of every Z_ij behind the store of the previous F_ij, which the compiler
  // may not reorder -- C could alias B -- the 64 elements of a thread were 64 dependent
  // memory round trips, ~50 us per 128 x 128 tile). The arithmetic per element is unchanged.
  double di[4][2];
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t i = m0 + wm * 64 + mi * 16 + g + h * 8;
      di[mi][h] = i < p.n_rows ? p.d[p.row0 + i] : 0.0;
    }
  double zb[2][4][2];
  auto load_col = [&](int c, double (&z)[4][2]) {
    const int64_t j = n0 + wn * 32 + (c >> 1) * 8 + 2 * t + (c & 1);
    const double* zcol = p.B + j * p.ldb;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = m0 + wm * 64 + mi * 16 + g + h * 8;
        z[mi][h] = (j < p.n_cols && i < p.n_rows) ? zcol[i] : 0.0;
      }
  };
  load_col(0, zb[0]);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int ni = c >> 1, e = c & 1;
    if (c + 1 < 8) load_col(c + 1, zb[(c + 1) & 1]);
    const int64_t j = n0 + wn * 32 + ni * 8 + 2 * t + e;
    if (j >= p.n_cols) continue;
    const int64_t jg = p.col0 + j;
    const double dj = p.d[jg];
    const double wj = MODE == kGemmMap ? p.wd[j] : p.lam[j];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t i = m0 + wm * 64 + mi * 16 + g + h * 8;
        if (i >= p.n_rows) continue;
        const int64_t ig = p.row0 + i;
        const double w = acc[mi][ni][h * 2 + e];
        const double z = zb[c & 1][mi][h];
        if (MODE == kGemmMap) {
          // (z * wd - w) / (d_i - d_j): each operation rounded on its own, as
          // the reference's complex arithmetic does for zero imaginary parts.
          const double f = (ig == jg) ? 1.0 : __ddiv_rn(__dsub_rn(__dmul_rn(z, wj), w), __dsub_rn(di[mi][h], dj));
          p.C[j * p.ldc + i] = f;
          const double df = __dsub_rn(f, z);
          v[0] = __fma_rn(df, df, v[0]);
          v[1] = __fma_rn(z, z, v[1]);
          v[2] = __fma_rn(f, f, v[2]);
          v[3] = nan_max(v[3], fabs(df));
        } else {  // kGemmResid
          const double r = __dsub_rn(__dadd_rn(__dmul_rn(di[mi][h], z), w), __dmul_rn(z, wj));
          v[0] = __fma_rn(r, r, v[0]);
        }
      }
  }
}

// ------------------------------------------------------------------ TMA pipeline kernel

template <int MODE>
__global__ void __launch_bounds__(kGemmThreads, 1)
    dmma_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  if (p.state != nullptr && p.state->done) return;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the 128B swizzle atoms
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  double* tiles = reinterpret_cast<double*>(base);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + size_t(kStages) * kStageBytes);
  uint64_t* empty = full + kStages;

  int tm, tn;
  tile_coords(blockIdx.x, p.tiles_m, p.tiles_n, tm, tn);
  if ((MODE == kGemmSub || p.lower_only) && tn > tm) return;  // strictly-upper tiles of a symmetric result
  const int64_t m0 = int64_t(tm) * kBM, n0 = int64_t(tn) * kBN;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KT = static_cast<int>(p.K / kBK);
  const bool producer = threadIdx.x == 0;  // one elected thread issues every TMA

  auto issue = [&](int kt) {
    const int s = kt % kStages;
    double* as = tiles + size_t(s) * 2 * kTileDoubles;
    mbar_expect_tx(&full[s], kStageBytes);
    tma_load_2d(as, &tmA, &full[s], kt * kBK, static_cast<int>(m0));
    tma_load_2d(as + kTileDoubles, &tmB, &full[s], kt * kBK, static_cast<int>(n0));
  };

  if (producer) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmB) : "memory");
    for (int kt = 0; kt < kStages - 1 && kt < KT; ++kt) issue(kt);  // fill S-1 stages
  }
  __syncthreads();

  __shared__ double red[kConsumerWarps][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps, 64 x 32 each
  double acc[4][4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.0;

  // 32-bit shared addresses: every fragment row r of this thread has r & 7 == g, so the
  // swizzled column offset of step kk is shared by all its A and B loads, and the
  // rows differ by compile-time immediates (LDS [R + imm]).
  const uint32_t tiles_u32 = smem_u32(tiles);
  const uint32_t a_row = static_cast<uint32_t>((wm * 64 + g) * kBK * 8);
  const uint32_t b_row = static_cast<uint32_t>(kTileDoubles * 8 + (wn * 32 + g) * kBK * 8);
  uint32_t xo[kBK / 4];
#pragma unroll
  for (int kk = 0; kk < kBK / 4; ++kk) {
    const int k = 8 * (t >> 1) + (t & 1) + 2 * kk;
    xo[kk] = static_cast<uint32_t>(((((k >> 1) ^ g) << 1) | (k & 1)) * 8);
  }
  auto load_frags = [&](uint32_t stage_base, int kk, double (&af)[4][2], double (&bf)[4]) {
    const uint32_t a = stage_base + a_row + xo[kk];
    const uint32_t b = stage_base + b_row + xo[kk];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      af[mi][0] = lds_f64(a + mi * 16 * kBK * 8);
      af[mi][1] = lds_f64(a + (mi * 16 + 8) * kBK * 8);
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) bf[ni] = lds_f64(b + ni * 8 * kBK * 8);
  };

  // Fragments are double-buffered one step ahead (the next k-tile's first step is
  // loaded while the last step of this one is still in the DMMA pipe).
  double af[2][4][2], bf[2][4];
  if (KT > 0) {
    mbar_wait(&full[0], 0);
    load_frags(tiles_u32, 0, af[0], bf[0]);
  }
  for (int kt = 0; kt < KT; ++kt) {
    // Refill the stage consumed at kt-1 with k-tile kt+S-1 once all 8 warps released it.
    if (producer) {
      const int nk = kt + kStages - 1;
      if (nk < KT) {
        if (kt >= 1) mbar_wait(&empty[(kt - 1) % kStages], ((kt - 1) / kStages) & 1);
        issue(nk);
      }
    }
    const int s = kt % kStages;
    const uint32_t sb = tiles_u32 + static_cast<uint32_t>(s * kStageBytes);
#pragma unroll
    for (int kk = 0; kk < kBK / 4; ++kk) {
      const int cur = kk & 1, nxt = cur ^ 1;
      if (kk + 1 < kBK / 4) {
        load_frags(sb, kk + 1, af[nxt], bf[nxt]);
      } else if (kt + 1 < KT) {
        const int s1 = (kt + 1) % kStages;
        mbar_wait(&full[s1], ((kt + 1) / kStages) & 1);
        load_frags(tiles_u32 + static_cast<uint32_t>(s1 * kStageBytes), 0, af[nxt], bf[nxt]);
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_16x8x4(acc[mi][ni], af[cur][mi][0], af[cur][mi][1], bf[cur][ni]);
    }
    // all reads of stage s have landed in registers (the DMMAs above consumed them)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  gemm_epilogue<MODE>(p, acc, m0, n0, warp, lane, v);
  if (MODE == kGemmStore || MODE == kGemmSub || MODE == kGemmSubC || MODE == kGemmSubAll) return;
  block_reduce4<kConsumerWarps>(v, red);
  if (threadIdx.x == 0) {
    double* out = p.partials + size_t(blockIdx.x) * 4;
    out[0] = v[0];
    out[1] = v[1];
    out[2] = v[2];
    out[3] = v[3];
  }
}

}  // namespace iptb
