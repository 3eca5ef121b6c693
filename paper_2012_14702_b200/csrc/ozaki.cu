// FP64-accurate W = A . B on the 5th-gen tensor cores: Ozaki scheme II (exact integer
// products modulo 16 pairwise-coprime moduli on the tcgen05 INT8 datapath, Chinese
// remainder reconstruction), restated here for the IPT full-spectrum map.
//
//  1. Scale: row i of A by 2^eA[i], column j of B by 2^eB[j], with the row / column
//     maximum landing in [2^52, 2^53); round to integers A', B' (|.| < 2^53, exact for
//     every entry within a binade of its row maximum, absolute error <= 2^-54 of the
//     row maximum otherwise -- within FP64 GEMM rounding, whose bound is K u |A||B|).
//  2. Residues: A' mod m_l and B' mod m_l in the symmetric range (int8), l = 1..16.
//     A = Delta is fixed for a solve: its residues are made once.
//  3. Products: P_l = A'_l . B'_l^T per modulus on tcgen05 (kind::i8, exact int32,
//     |sum| < K 2^14), reduced mod m_l in the GEMM epilogue and stored as int8.
//  4. Reconstruction: the exact integer P = A' . B'^T (|P| <= K 2^106 < M / 2,
//     M = prod m_l ~ 2^125.4 for K <= 2^17) from its 16 residues by Garner's
//     mixed-radix algorithm with balanced digits, evaluated exactly in 128-bit integers
//     and rounded once to FP64; W_ij = P_ij 2^(-eA[i] - eB[j]).
//  5. The IPT map (or the closing residual) is applied in the same pass (the K1
//     epilogue formulas), with the per-CTA partial sums of a fixed grid.
// Everything is integer-exact up to the single rounding of P and of the scaling, so the
// result is deterministic and as accurate as an FP64 GEMM; non-finite inputs are routed
// to the DMMA path by the caller.
#include <cmath>
#include <cstdint>
#include <type_traits>
#include <vector>

#include "i8gemm.cuh"
#include "ozaki.cuh"

namespace iptb {

namespace {

constexpr int kMods = kOzakiMods;

// Moduli and Garner tables as compile-time constants (every loop over l is unrolled, so
// each "% m" below is a division by a literal: multiply-shift, no integer divide).
// c[l][t] = (m_0 ... m_{t-1}) mod m_l for t < l; inv[l] = (m_0 ... m_{l-1})^-1 mod m_l.
struct Garner {
  int m[kMods];
  int c[kMods][kMods];
  int inv[kMods];
};

constexpr Garner make_garner() {
  Garner g{};
  constexpr int mods[kMods] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};
  for (int l = 0; l < kMods; ++l) g.m[l] = mods[l];
  for (int l = 0; l < kMods; ++l) {
    long long prod = 1;
    for (int t = 0; t < kMods; ++t) g.c[l][t] = 0;
    for (int t = 0; t < l; ++t) {
      g.c[l][t] = static_cast<int>(prod);
      prod = (prod * mods[t]) % mods[l];
    }
    int inv = 1;
    for (int x = 1; x < mods[l]; ++x)
      if ((prod * x) % mods[l] == 1) {
        inv = x;
        break;
      }
    g.inv[l] = inv;
  }
  return g;
}

constexpr Garner kG = make_garner();

template <int L>
__device__ __forceinline__ int sym_mod_c(int x) {
  constexpr int m = kG.m[L];
  int r = x % m;
  if (r < -(m >> 1)) r += m;
  if (r >= (m - (m >> 1))) r -= m;  // even m: [-m/2, m/2); odd m: [-(m-1)/2, (m-1)/2]
  return r;
}

__device__ __forceinline__ int sym_mod(int x, int m) {
  int r = x % m;
  if (r < -(m >> 1)) r += m;
  if (r >= (m - (m >> 1))) r -= m;
  return r;
}

// compile-time loops over the moduli
template <int L, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (L < N) {
    f(std::integral_constant<int, L>{});
    static_for<L + 1, N>(f);
  }
}

// Row (or column) exponent: max |x| * 2^e in [2^52, 2^53); flag non-finite rows.
__global__ void exponent_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t len,
                                int* __restrict__ e) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  double mx = 0.0;
  for (int64_t k = lane; k < len; k += 32) mx = nan_max(mx, fabs(X[r * ldx + k]));
  for (int off = 16; off > 0; off >>= 1) mx = nan_max(mx, __shfl_xor_sync(0xffffffffu, mx, off));
  if (lane == 0) {
    if (!isfinite(mx)) e[r] = kOzakiNonFinite;
    else if (mx == 0.0) e[r] = 0;
    else e[r] = 52 - ilogb(mx);
  }
}

// out[l][r][k] = sym(rint(x_rk 2^e_r) mod m_l) for all 16 moduli; zero padding for k >= len.
__global__ void residues_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t len,
                                const int* __restrict__ e, int8_t* __restrict__ out, int64_t ldo, int64_t plane) {
  const int64_t total = rows * ldo;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / ldo, k = t - r * ldo;
    double y = 0.0;
    const int er = e[r];
    if (k < len && er != kOzakiNonFinite) y = rint(ldexp(X[r * ldx + k], er));
    static_for<0, kMods>([&](auto L) {
      constexpr int l = decltype(L)::value;
      constexpr int m = kG.m[l];
      constexpr double minv = 1.0 / m;
      const double q = rint(y * minv);
      const int v = static_cast<int>(fma(-q, double(m), y));  // exact: |y - q m| < 2 m
      out[l * plane + t] = static_cast<int8_t>(sym_mod_c<l>(v));
    });
  }
}

// GEMM epilogue: int32 product chunk -> symmetric residue mod m (int8), 32 bytes per row chunk.
struct ModStore {
  int8_t* out;
  int64_t ld;
  int m;
  double minv;
  __device__ void operator()(int row, int col0, const uint32_t (&v)[32]) const {
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t packed = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int x = static_cast<int>(v[4 * q + b]);
        const int qq = __double2int_rn(double(x) * minv);
        const int r = sym_mod(x - qq * m, m);
        packed |= (uint32_t(uint8_t(int8_t(r)))) << (8 * b);
      }
      w[q] = packed;
    }
    int4* p = reinterpret_cast<int4*>(out + int64_t(row) * ld + col0);
    p[0] = make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
    p[1] = make_int4(int(w[4]), int(w[5]), int(w[6]), int(w[7]));
  }
};

// Reconstruct W_ij from the residues (R[l][j][i], j = column of B / Z, i = row of A) and
// apply the IPT map (mode 0) or the closing residual (mode 1) with the K1 formulas.
__global__ void __launch_bounds__(256) reconstruct_map_kernel(OzakiMapArgs a) {
  if (a.state != nullptr && a.state->done) return;
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  const int64_t total = a.n * a.ncols;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = t / a.n, i = t - j * a.n;
    const int ea = a.eA[i], eb = a.eB[j];
    double w;
    if (ea == kOzakiNonFinite || eb == kOzakiNonFinite) {
      w = __longlong_as_double(0x7ff8000000000000LL);  // NaN, as the FP64 product would give
    } else {
      int dig[kMods];
      const int8_t* rp = a.R + j * a.ldr + i;
      static_for<0, kMods>([&](auto L) {
        constexpr int l = decltype(L)::value;
        const int r = rp[l * a.plane];
        int s = 0;
        static_for<0, l>([&](auto U) {
          constexpr int u = decltype(U)::value;
          constexpr int cu = kG.c[l][u];
          s += dig[u] * cu;
        });
        constexpr int inv = kG.inv[l];
        dig[l] = sym_mod_c<l>(sym_mod_c<l>(r - s) * inv);
      });
      __int128 p = dig[kMods - 1];
      static_for<0, kMods - 1>([&](auto L) {  // Horner from the top digit, exact in 128 bits
        constexpr int l = kMods - 2 - decltype(L)::value;
        constexpr int m = kG.m[l];
        p = p * m + dig[l];
      });
      const bool neg = p < 0;
      const unsigned __int128 mag = neg ? (unsigned __int128)(-p) : (unsigned __int128)p;
      const double hi = double(uint64_t(mag >> 64)) * 18446744073709551616.0;
      const double mg = hi + double(uint64_t(mag));
      w = ldexp(neg ? -mg : mg, -(ea + eb));
    }
    const double z = a.Z[j * a.ldz + i];
    const int64_t jg = a.col0 + j;
    const double di = a.d[i];
    if (a.mode == 0) {
      const double f = (i == jg) ? 1.0 : __ddiv_rn(__dsub_rn(__dmul_rn(z, a.wd[j]), w), __dsub_rn(di, a.d[jg]));
      a.F[j * a.ldz + i] = f;
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
  block_reduce4<8>(v, red);
  if (threadIdx.x == 0) {
    double* o = a.partials + size_t(blockIdx.x) * 4;
    o[0] = v[0];
    o[1] = v[1];
    o[2] = v[2];
    o[3] = v[3];
  }
}

}  // namespace

void OzakiOperand::build(cudaStream_t s, const double* X, int64_t ldx, int64_t rows_, int64_t len_, int64_t rows_pad,
                         int64_t kpad_) {
  rows = rows_;
  len = len_;
  kpad = kpad_;
  plane = rows_pad * kpad;
  if (res.count * 8 < size_t(kMods) * plane) res.alloc(ceil_div(int64_t(kMods) * plane, 8));  // zeroed padding rows
  if (e.count < size_t(rows_pad)) e.alloc(rows_pad);
  int* ep = reinterpret_cast<int*>(e.get());
  exponent_kernel<<<static_cast<unsigned>(ceil_div(rows, 8)), 256, 0, s>>>(X, ldx, rows, len, ep);
  residues_kernel<<<2368, 256, 0, s>>>(X, ldx, rows, len, ep, reinterpret_cast<int8_t*>(res.get()), kpad, plane);
  IPT_LAUNCH_CHECK();
  count_launch(2);
}

// R[l] = (Bop . Aop^T) mod m_l for all moduli: rows of the product = rows of Bop (the Z
// columns), columns = rows of Aop (the Delta rows).
void ozaki_products(cudaStream_t s, const OzakiOperand& Zop, const OzakiOperand& Aop, int64_t zrows_pad,
                    int64_t arows_pad, DevBuf& R, int64_t& plane) {
  plane = zrows_pad * arows_pad;
  if (R.count * 8 < size_t(kMods) * plane) R.alloc(ceil_div(int64_t(kMods) * plane, 8), false);
  for (int l = 0; l < kMods; ++l) {
    const int m = kG.m[l];  // host read of the constexpr table
    ModStore epi{reinterpret_cast<int8_t*>(R.get()) + l * plane, arows_pad, m, 1.0 / m};
    launch_i8gemm(s, zrows_pad, arows_pad, Zop.kpad, reinterpret_cast<const int8_t*>(Zop.res.get()) + l * Zop.plane,
                  Zop.kpad, reinterpret_cast<const int8_t*>(Aop.res.get()) + l * Aop.plane, Aop.kpad, epi);
  }
}

void ozaki_reconstruct(cudaStream_t s, const OzakiMapArgs& a) {
  reconstruct_map_kernel<<<kOzakiGrid, 256, 0, s>>>(a);
  IPT_LAUNCH_CHECK();
  count_launch();
}

}  // namespace iptb
