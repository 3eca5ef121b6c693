// K16: the closing residual |MZ - Z Lambda|_F (solver.cpp:252-270) of a converged real
// dense full-spectrum solve WITHOUT a second FP64 product.
//
// The reference forms W = Delta Z once more after the loop. Here the last map already
// holds that product for the previous iterate: F(Z_old) = Z_new with
//   Z_new_ij = (Z_old_ij wd_j - W_old_ij) / (d_i - d_j),  W_old = Delta Z_old,
// so, with D = Z_new - Z_old (the last step) and W_new = W_old + Delta D, the residual
//   r_ij = d_i Z_new_ij + W_new_ij - Z_new_ij lambda_j,   lambda_j = d_j + wd_new_j,
// is, exactly in real arithmetic and for i != j,
//   r_ij = Z_new_ij (wd_old_j - wd_new_j) - D_ij wd_old_j + (Delta D)_ij
// and r_jj = wd_old_j + (Delta D)_jj - wd_new_j. The rounding of the last map's division
// that this drops is ~|W| 2^-53 per entry, the noise level of the reference's own
// residual. D of a converged loop is ~step |Z| small, so Delta D is needed to a few
// significant digits only: rows of Delta and columns of D are scaled by powers of two to
// 13-bit integers, split into int8 digits q = 128 hi + lo, and
//   Delta' D' = 2^14 (hi.hi) + 2^7 (hi.lo + lo.hi)   (lo.lo, < 2^-13 relative, dropped)
// runs as two exact int32 products on the tcgen05 INT8 tensor cores (K and 2K long). The
// error of the correction, <= 2^-13 (max_k|Delta_ik| |D_.j|_1 + max_k|D_kj| |Delta_i.|_1),
// is ~1e-4 of a term that is itself ~step of |W|.
//
// Cost at N = 32768: two INT8 products of 1 and 2 GEMM-equivalents plus three HBM passes,
// ~0.08 s, instead of the 1.95 s FP64 DMMA product.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "i8gemm.cuh"

namespace iptb {

namespace {

constexpr int kClosingBlocks = 1184;  // fixed residual grid (deterministic partials)

struct StoreI32Pitched {
  int32_t* C;
  int64_t ldc;
  __device__ bool skip() const { return false; }
  __device__ void operator()(int row, int col0, const uint32_t (&v)[32]) const {
    int4* p = reinterpret_cast<int4*>(C + int64_t(row) * ldc + col0);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      p[q] = make_int4(int(v[4 * q]), int(v[4 * q + 1]), int(v[4 * q + 2]), int(v[4 * q + 3]));
  }
};

// One vector (a row of Delta, or a column of Z_new - Z_old) per block: its max |x| sets
// the power of two e that brings it into [2^12, 2^13); q = rint(x 2^e) is split into int8
// digits lo = ((q + 64) & 127) - 64, hi = (q - lo) / 128, stored as [first | second]
// halves of a 2 kpad row (hi_first: [hi | lo], else [lo | hi]); exps[v] = e (0 for a zero
// vector, 0x7fffffff for a non-finite one).
__global__ void __launch_bounds__(256) digits_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                                     int64_t ld, int64_t len, int8_t* __restrict__ out, int64_t kpad,
                                                     int hi_first, int* __restrict__ exps) {
  __shared__ double red[8];
  __shared__ int s_e;
  const int64_t v = blockIdx.x;
  const double* av = a + v * ld;
  const double* bv = b ? b + v * ld : nullptr;
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
    const double x = bv ? av[k] - bv[k] : av[k];
    mx = nan_max(mx, fabs(x));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mx = nan_max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = red[0];
    for (int w = 1; w < 8; ++w) m = nan_max(m, red[w]);
    s_e = !isfinite(m) ? 0x7fffffff : (m == 0.0 ? 0 : 12 - ilogb(m));
    exps[v] = s_e;
  }
  __syncthreads();
  const int e = s_e;
  int8_t* row = out + v * 2 * kpad;
  int8_t* first = row;
  int8_t* second = row + kpad;
  for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
    int q = 0;
    if (e != 0x7fffffff) {
      const double x = bv ? av[k] - bv[k] : av[k];
      q = static_cast<int>(rint(ldexp(x, e)));  // |q| <= 2^13
    }
    const int lo = ((q + 64) & 127) - 64;
    const int hi = (q - lo) / 128;
    first[k] = static_cast<int8_t>(hi_first ? hi : lo);
    second[k] = static_cast<int8_t>(hi_first ? lo : hi);
  }
}

// r_ij of the header comment over the local columns, fixed grid, per-CTA partial
// {sum r^2, 0, 0, 0}.
__global__ void __launch_bounds__(256) closing_residual_kernel(
    const double* __restrict__ Z, int64_t ldz, int64_t n, int64_t ncols, int64_t col0,
    const int8_t* __restrict__ zdig, int64_t kpad, const int* __restrict__ ez, const int* __restrict__ ea,
    const int32_t* __restrict__ c1, const int32_t* __restrict__ c2, int64_t ldc, const double* __restrict__ wd_old,
    const double* __restrict__ wd_new, double* __restrict__ partials) {
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  // CTA b takes columns b, b + grid, ...; its threads stride down each column
  for (int64_t j = blockIdx.x; j < ncols; j += gridDim.x) {
    const int64_t jg = col0 + j;
    const int sj = ez[j];
    const double wo = wd_old[j], wn = wd_new[j];
    const int8_t* dj = zdig + j * 2 * kpad;  // [hi | lo]
    const int32_t* c1j = c1 + j * ldc;
    const int32_t* c2j = c2 + j * ldc;
    const double* zj = Z + j * ldz;
    // four rows per thread in flight (the pass is HBM-latency bound otherwise); the sum
    // order per thread stays i = t, t + 256, ... as in the one-row loop
    constexpr int kU = 4;
    for (int64_t i0 = threadIdx.x; i0 < n; i0 += int64_t(kU) * blockDim.x) {
      int32_t a1[kU], a2[kU], si[kU];
      int8_t dh[kU], dl[kU];
      double z[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + int64_t(u) * blockDim.x;
        const bool in = i < n;
        a1[u] = in ? c1j[i] : 0;
        a2[u] = in ? c2j[i] : 0;
        si[u] = in ? ea[i] : 0;
        dh[u] = in ? dj[i] : int8_t(0);
        dl[u] = in ? dj[kpad + i] : int8_t(0);
        z[u] = in ? zj[i] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + int64_t(u) * blockDim.x;
        if (i >= n) break;
        if (sj == 0x7fffffff || si[u] == 0x7fffffff) {  // (non-finite input: the caller keeps the exact path)
          v[0] = NAN;
          continue;
        }
        // (Delta D)_ij = (2^14 c1 + 2^7 c2) 2^-(si + sj)
        const double corr = ldexp(fma(128.0, double(a1[u]), double(a2[u])), 7 - (si[u] + sj));
        double r;
        if (i == jg) {
          r = (wo + corr) - wn;
        } else {
          const double dij = ldexp(fma(128.0, double(dh[u]), double(dl[u])), -sj);
          r = fma(z[u], wo - wn, fma(-dij, wo, corr));
        }
        v[0] = fma(r, r, v[0]);
      }
    }
  }
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = partials + size_t(blockIdx.x) * 4;
    o[0] = v[0];
    o[1] = 0.0;
    o[2] = 0.0;
    o[3] = 0.0;
  }
}

}  // namespace

int64_t closing_partials() { return kClosingBlocks; }

void ClosingWork::delta_digits(cudaStream_t s, const double* A, int64_t lda, int64_t n_) {
  n = n_;
  kpad = round_up(n, kI8BK);
  arows = round_up(n, 512);
  adig.alloc(ceil_div(arows * 2 * kpad, 8));  // zero: padded rows / K give zero products
  aexp.alloc(ceil_div(arows, 2));
  digits_kernel<<<static_cast<unsigned>(n), 256, 0, s>>>(A, nullptr, lda, n, reinterpret_cast<int8_t*>(adig.get()),
                                                         kpad, /*hi_first=*/0, reinterpret_cast<int*>(aexp.get()));
  IPT_LAUNCH_CHECK();
  count_launch();
  delta_ready = true;
}

void ClosingWork::step_digits(cudaStream_t s, const double* znew, const double* zold, int64_t ldz, int64_t ncols_,
                              const double* wd_old_src) {
  ncols = ncols_;
  mpad = round_up(std::max<int64_t>(ncols, 1), 256);
  zdig.alloc(ceil_div(mpad * 2 * kpad, 8));
  zexp.alloc(ceil_div(mpad, 2));
  wd_old.alloc(std::max<int64_t>(ncols, 1), false);
  if (ncols > 0) {
    digits_kernel<<<static_cast<unsigned>(ncols), 256, 0, s>>>(znew, zold, ldz, n,
                                                                reinterpret_cast<int8_t*>(zdig.get()), kpad,
                                                                /*hi_first=*/1, reinterpret_cast<int*>(zexp.get()));
    IPT_LAUNCH_CHECK();
    count_launch();
    IPT_CUDA(cudaMemcpyAsync(wd_old.get(), wd_old_src, sizeof(double) * ncols, cudaMemcpyDeviceToDevice, s));
  }
  step_ready = true;
}

void ClosingWork::residual(cudaStream_t s, const double* znew, int64_t ldz, int64_t col0, const double* wd_new,
                           double* partials) {
  if (!delta_ready || !step_ready) throw InvalidArgument("closing residual: digits missing");
  const int8_t* za = reinterpret_cast<const int8_t*>(zdig.get());
  const int8_t* da = reinterpret_cast<const int8_t*>(adig.get());
  DevBuf c1, c2;
  if (ncols > 0) {
    c1.alloc(ceil_div(mpad * arows, 2), false);
    c2.alloc(ceil_div(mpad * arows, 2), false);
    int32_t* p1 = reinterpret_cast<int32_t*>(c1.get());
    int32_t* p2 = reinterpret_cast<int32_t*>(c2.get());
    const bool prof = std::getenv("IPT_PROFILE") != nullptr;
    cudaEvent_t ev[4] = {};
    if (prof)
      for (auto& e : ev) IPT_CUDA(cudaEventCreate(&e));
    if (prof) IPT_CUDA(cudaEventRecord(ev[0], s));
    // c1 = Dhi . Ahi (A digits stored [lo | hi]: hi at +kpad), c2 = [Dhi | Dlo] . [Alo | Ahi]
    launch_i8gemm(s, mpad, arows, kpad, za, 2 * kpad, da + kpad, 2 * kpad, StoreI32Pitched{p1, arows});
    if (prof) IPT_CUDA(cudaEventRecord(ev[1], s));
    launch_i8gemm(s, mpad, arows, 2 * kpad, za, 2 * kpad, da, 2 * kpad, StoreI32Pitched{p2, arows});
    if (prof) IPT_CUDA(cudaEventRecord(ev[2], s));
    closing_residual_kernel<<<kClosingBlocks, 256, 0, s>>>(
        znew, ldz, n, ncols, col0, za, kpad, reinterpret_cast<const int*>(zexp.get()),
        reinterpret_cast<const int*>(aexp.get()), p1, p2, arows, wd_old.get(), wd_new, partials);
    if (prof) {
      IPT_CUDA(cudaEventRecord(ev[3], s));
      IPT_CUDA(cudaEventSynchronize(ev[3]));
      float t[3];
      for (int k = 0; k < 3; ++k) IPT_CUDA(cudaEventElapsedTime(&t[k], ev[k], ev[k + 1]));
      std::fprintf(stderr, "[ipt] closing K16: c1 %.2f ms, c2 %.2f ms, residual %.2f ms\n", t[0], t[1], t[2]);
      for (auto& e : ev) cudaEventDestroy(e);
    }
  } else {
    closing_residual_kernel<<<kClosingBlocks, 256, 0, s>>>(znew, ldz, n, 0, col0, za, kpad, nullptr, nullptr, nullptr,
                                                          nullptr, arows, nullptr, nullptr, partials);
  }
  IPT_LAUNCH_CHECK();
  count_launch();
  step_ready = false;
}

}  // namespace iptb
