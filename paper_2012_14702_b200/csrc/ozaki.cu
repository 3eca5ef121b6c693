// FP64-accurate W = A . B on the 5th-gen tensor cores: Ozaki scheme II (exact integer
// products modulo 16 pairwise-coprime moduli on the tcgen05 INT8 datapath, Chinese
// remainder reconstruction), restated here for the IPT full-spectrum map.
//
//  1. Scale: row i of A by 2^eA[i], column j of B by 2^eB[j], with the row / column
//     maximum landing in [2^52, 2^53); round to integers A', B' (|.| < 2^53, exact for
//     every entry within a binade of its row maximum, absolute error <= 2^-53 of the
//     row maximum otherwise: a product error <= 2^-53 (max|a_i.| |b_.j|_1 + max|b_.j|
//     |a_i.|_1), the order of the FP64 GEMM's normwise bound).
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
// result is deterministic with FP64-GEMM-order accuracy (step 1); non-finite inputs are routed
// to the DMMA path by the caller.
#include <algorithm>
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

// |x| < m (a remainder after a rounded quotient) -> the symmetric range of m
__device__ __forceinline__ int sym_fix_rt(int x, int m) {
  const int lo = -(m >> 1), hi = m - (m >> 1) - 1;
  x = x > hi ? x - m : x;
  return x < lo ? x + m : x;
}

// compile-time loops over the moduli
template <int L, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (L < N) {
    f(std::integral_constant<int, L>{});
    static_for<L + 1, N>(f);
  }
}

// log2(m_0 ... m_{L-1}) rounded down, L = 1 .. 16 (tests/test_ozaki_math.py checks them)
__constant__ double kLog2M[kMods] = {8.0,       15.994353, 23.977347, 31.94889,  39.897257,  47.810147,
                                     55.711013, 63.5752,   71.414403, 79.240952, 87.041852,  94.803403,
                                     102.524502, 110.161127, 117.783179, 125.375636};

// Row (or column) exponent: max |x| * 2^e in [2^52, 2^53); flag non-finite rows.
// With a moduli counter the kernel also bounds the row's integer 1-norm (off the diagonal
// for split operands, diag0 >= 0) and raises *moduli to the count that keeps
// |A' X'| < 2^53 |X'|_1 below M / 2.
__global__ void exponent_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows, int64_t len,
                                int* __restrict__ e, int64_t diag0, int* __restrict__ moduli) {
  const int lane = threadIdx.x & 31;
  const int64_t r = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t kd = diag0 >= 0 ? diag0 + r : -1;
  double mx = 0.0, off = 0.0;
  for (int64_t k = lane; k < len; k += 32) {
    const double a = fabs(X[r * ldx + k]);
    mx = nan_max(mx, a);
    off += k == kd ? 0.0 : a;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = nan_max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    off += __shfl_xor_sync(0xffffffffu, off, o);
  }
  if (lane == 0) {
    int er;
    if (!isfinite(mx)) er = kOzakiNonFinite;
    else if (mx == 0.0) er = 0;
    else er = 52 - ilogb(mx);
    e[r] = er;
    if (moduli != nullptr && er != kOzakiNonFinite) {
      // |Y'|_1 <= 2^e sum |x| (1 + K u) + K / 2 (rounding to integers); 2^-40 covers the
      // floating-point sum for K < 2^17
      const double bound = ldexp(off * (1.0 + 0x1p-40), er) + double(len);
      const double need = 54.0 + log2(bound) + 1e-3;
      int L = kOzakiMinMods;
      while (L < kMods && kLog2M[L - 1] < need) ++L;
      atomicMax(moduli, L);
    }
  }
}

// Symmetric remainder for a quotient estimate already applied: one correction step each way.
template <int L, class T>
__device__ __forceinline__ T sym_fix(T t) {
  constexpr int m = kG.m[L];
  constexpr T fm = T(m), lo = -T(m >> 1), hi = T(m - (m >> 1) - 1);
  t = t > hi ? t - fm : t;
  return t < lo ? t + fm : t;
}

// Rounding and conversion of integer-valued floats by the 1.5 * 2^p shifter: plain adds on
// the FMA pipes instead of FRND / F2I on the conversion pipe. Exact for |x| < 2^22 (FP32)
// and |x| < 2^51 (FP64); ties to even like rint.
__device__ __forceinline__ float rint_small(float x) { return __fsub_rn(__fadd_rn(x, 12582912.0f), 12582912.0f); }
__device__ __forceinline__ int int_small(float x) { return __float_as_int(__fadd_rn(x, 12582912.0f)) - 0x4B400000; }
__device__ __forceinline__ float float_small(int x) { return __fsub_rn(__int_as_float(0x4B400000 + x), 12582912.0f); }
__device__ __forceinline__ double rint_small(double x) {
  return __dsub_rn(__dadd_rn(x, 6755399441055744.0), 6755399441055744.0);
}
__device__ __forceinline__ int int_small(double x) { return __double2loint(__dadd_rn(x, 6755399441055744.0)); }

// x * 2^k: a multiplication by an exact power of two is correctly rounded, so it equals
// ldexp whenever 2^k is a normal double.
__device__ __forceinline__ double scale2(double x, int k) {
  if (k >= -1022 && k <= 1023) return x * __longlong_as_double(static_cast<long long>(k + 1023) << 52);
  return ldexp(x, k);
}

// out[l][r][k] = sym(rint(x_rk 2^e_r) mod m_l) for all 16 moduli; zero padding for k >= len.
// Eight consecutive k per thread (one 8-byte store per modulus plane).
// Split operands (diag0 >= 0): the entry at k = diag0 + r goes to diag[r] instead.
__global__ void __launch_bounds__(256) residues_kernel(const double* __restrict__ X, int64_t ldx, int64_t rows,
                                                       int64_t len, const int* __restrict__ e,
                                                       int8_t* __restrict__ out, int64_t ldo, int64_t plane,
                                                       int64_t diag0, double* __restrict__ diag,
                                                       const int* __restrict__ moduli) {
  const int nm = moduli != nullptr ? *moduli : kMods;  // planes past it are never read
  const int64_t per_row = ldo >> 3;
  const int64_t total = rows * per_row;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / per_row, k0 = (t - r * per_row) << 3;
    const int er = e[r];
    double y[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t k = k0 + q;
      y[q] = (k < len && er != kOzakiNonFinite) ? rint(scale2(X[r * ldx + k], er)) : 0.0;
      if (diag0 >= 0 && k == diag0 + r) {
        diag[r] = y[q];
        y[q] = 0.0;
      }
    }
    int8_t* dst = out + r * ldo + k0;
    static_for<0, kMods>([&](auto L) {
      constexpr int l = decltype(L)::value;
      constexpr double m = kG.m[l], minv = 1.0 / kG.m[l];
      if (l >= nm) return;
      uint32_t w[2] = {0u, 0u};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        // |y / m| < 2^46; |y - rint(y/m) m| <= m/2 + 1 and the fma is exact, so one symmetric
        // fix suffices
        const int v = sym_fix<l>(int_small(fma(-rint_small(y[q] * minv), m, y[q])));
        w[q >> 2] |= uint32_t(uint8_t(int8_t(v))) << (8 * (q & 3));
      }
      *reinterpret_cast<uint2*>(dst + l * plane) = make_uint2(w[0], w[1]);
    });
  }
}

// Division by a modulus m <= 256 without conversions: for 0 <= u < 2^31,
// floor(u / m) = umulhi(u, magic) >> 7 with magic = floor(2^39 / m) + 1 (< 2^32): the
// excess u (magic - 2^39 / m) / 2^39 < 2^31 / 2^39 = 1/256 <= 1/m cannot carry the
// quotient past the next integer. Integer pipes only (no I2F / F2I).
struct ModMagic {
  uint32_t m, magic, bias;  // bias = m floor(2^30 / m): a multiple of m, u = x + bias
};

inline ModMagic mod_magic(int m) {
  ModMagic r;
  r.m = static_cast<uint32_t>(m);
  r.magic = static_cast<uint32_t>((uint64_t(1) << 39) / uint64_t(m) + 1);
  r.bias = static_cast<uint32_t>(m) * ((uint32_t(1) << 30) / static_cast<uint32_t>(m));
  return r;
}

// x mod m in the symmetric range [-(m >> 1), m - (m >> 1) - 1], for |x| <= 2^30 - 256
__device__ __forceinline__ int sym_mod_magic(int x, const ModMagic& mm) {
  const uint32_t u = static_cast<uint32_t>(x) + mm.bias;  // in [0, 2^31)
  const uint32_t q = __umulhi(u, mm.magic) >> 7;
  const int r = static_cast<int>(u - q * mm.m);  // [0, m)
  return r > static_cast<int>(mm.m - (mm.m >> 1) - 1) ? r - static_cast<int>(mm.m) : r;
}

// GEMM epilogue: int32 product chunk -> symmetric residue mod m (int8), 32 bytes per row chunk.
// |x| <= K 2^14 <= 2^30 - 2^14 for K <= kOzakiMaxK.
struct ModStore {
  int8_t* out;
  int64_t ld;
  ModMagic mm;
  const int* moduli;  // device count of moduli in use (nullptr: all)
  int l;
  __device__ bool skip() const { return moduli != nullptr && *moduli <= l; }
  __device__ void operator()(int row, int col0, const uint32_t (&v)[32]) const {
    uint32_t w[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t packed = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int r = sym_mod_magic(static_cast<int>(v[4 * q + b]), mm);
        packed |= (uint32_t(uint8_t(int8_t(r)))) << (8 * b);
      }
      w[q] = packed;
    }
    int4* p = reinterpret_cast<int4*>(out + int64_t(row) * ld + col0);
    p[0] = make_int4(int(w[0]), int(w[1]), int(w[2]), int(w[3]));
    p[1] = make_int4(int(w[4]), int(w[5]), int(w[6]), int(w[7]));
  }
};

// W_8 = m_0 ... m_7 (< 2^64): the weight of the upper Horner half.
constexpr unsigned long long kW8 = [] {
  unsigned long long w = 1;
  for (int l = 0; l < 8; ++l) w *= static_cast<unsigned long long>(kG.m[l]);
  return w;
}();

// The nearest double to an unsigned 128-bit integer (ties to even): its 64 leading bits with
// a sticky LSB for everything below, one correctly rounded U64 -> F64 conversion, and an
// exact power-of-two scaling.
__device__ __forceinline__ double u128_to_double(unsigned __int128 x) {
  const uint64_t hi = uint64_t(x >> 64), lo = uint64_t(x);
  if (hi == 0) return __ull2double_rn(lo);
  const int lz = __clzll(static_cast<long long>(hi));
  const uint64_t top = lz ? (hi << lz) | (lo >> (64 - lz)) : hi;
  const uint64_t rest = lo << lz;
  const double t = __ull2double_rn(top | (rest != 0 ? 1ull : 0ull));
  return t * __longlong_as_double(static_cast<long long>(64 - lz + 1023) << 52);
}

// Garner tables for the integer digit recurrence: with t_l = (m_0 ... m_{l-1})^-1 mod m_l,
//   dig_l = sym( r_l t_l + sum_{u<l} dig_u k[l][u] ),  k[l][u] = sym(-c[l][u] t_l) mod m_l,
// where sym() is the symmetric residue mod m_l. Residues, digits, t and k are all in
// [-128, 127], so every product-sum is four-way SIMD: dp4a of int8x4 words (the four
// elements' residues against t placed in byte q; packed digits against packed k).
struct GarnerInt {
  int kw[kMods][4];    // k[l][4w .. 4w+3] packed (zero for u >= l)
  int tw[kMods][4];    // sym(t_l) in byte q, zero elsewhere
  uint32_t magic[kMods], off[kMods];
};

constexpr int sym_c(long long x, int m) {
  long long r = x % m;
  if (r < 0) r += m;
  return static_cast<int>(r > m - (m >> 1) - 1 ? r - m : r);
}

constexpr uint32_t pack_i8(int b) { return static_cast<uint32_t>(static_cast<uint8_t>(static_cast<int8_t>(b))); }

constexpr GarnerInt make_garner_int() {
  GarnerInt g{};
  for (int l = 0; l < kMods; ++l) {
    const int m = kG.m[l];
    g.magic[l] = static_cast<uint32_t>((1ull << 39) / static_cast<unsigned long long>(m) + 1);
    // m floor(2^30 / m) (a multiple of m) + floor(m / 2): x + off lies in [0, 2^31) for
    // |x| <= 2^30 - 256, and floor((x + off) / m) rounds x / m to the symmetric range
    g.off[l] = static_cast<uint32_t>(m) * ((1u << 30) / static_cast<uint32_t>(m)) + static_cast<uint32_t>(m >> 1);
    for (int q = 0; q < 4; ++q) g.tw[l][q] = static_cast<int>(pack_i8(sym_c(kG.inv[l], m)) << (8 * q));
    for (int w = 0; w < 4; ++w) {
      uint32_t word = 0;
      for (int b = 0; b < 4; ++b) {
        const int u = 4 * w + b;
        word |= pack_i8(u < l ? sym_c(-static_cast<long long>(kG.c[l][u]) * kG.inv[l], m) : 0) << (8 * b);
      }
      g.kw[l][w] = static_cast<int>(word);
    }
  }
  return g;
}

constexpr GarnerInt kGI = make_garner_int();

// sym(x) mod m_L from u = x + off_L in [0, 2^31): u - m floor(u / m) - floor(m / 2) (the
// magic division of ModMagic; integer pipes only)
template <int L>
__device__ __forceinline__ int sym_from_biased(uint32_t u) {
  constexpr uint32_t m = kG.m[L], magic = kGI.magic[L];
  const uint32_t q = __umulhi(u, magic) >> 7;
  return static_cast<int>(u - q * m) - static_cast<int>(m >> 1);
}

// sign-extended byte k of w (prmt with sign-replicating selector nibbles)
template <int K>
__device__ __forceinline__ int sbyte(uint32_t w) {
  constexpr uint32_t sel = K | ((K | 8) << 4) | ((K | 8) << 8) | ((K | 8) << 12);
  uint32_t r;
  asm("prmt.b32 %0, %1, 0, %2;" : "=r"(r) : "r"(w), "n"(sel));
  return static_cast<int>(r);
}

// w with byte K replaced by the low byte of x
template <int K>
__device__ __forceinline__ uint32_t put_byte(uint32_t w, int x) {
  constexpr uint32_t sel = (K == 0 ? 0x3214u : K == 1 ? 0x3240u : K == 2 ? 0x3410u : 0x4210u);
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(w), "r"(x), "n"(sel));
  return r;
}

// Mixed-radix digits of four residue vectors at once (res[l] = the four elements' residues
// mod m_l as int8x4), packed four digits per word: D[q][w] byte b = dig_{4w+b} of element q.
// Every step is exact integer arithmetic; the four chains are independent (ILP).
// Only the first L moduli are used (digits L .. 15 stay zero, so the value below is the
// same mixed-radix sum).
template <int L>
__device__ __forceinline__ void garner_digits4(const uint32_t (&res)[kMods], uint32_t (&D)[4][4]) {
  // dig_0 = r_0 (m_0 = 256: the stored residue is already the symmetric digit)
  D[0][0] = res[0] & 0xffu;
  D[1][0] = (res[0] >> 8) & 0xffu;
  D[2][0] = (res[0] >> 16) & 0xffu;
  D[3][0] = res[0] >> 24;
#pragma unroll
  for (int q = 0; q < 4; ++q) D[q][1] = D[q][2] = D[q][3] = 0u;
  static_for<1, L>([&](auto LL) {
    constexpr int l = decltype(LL)::value;
    int acc[4];
    static_for<0, 4>([&](auto Q) {
      constexpr int q = decltype(Q)::value;
      constexpr int tw = kGI.tw[l][q], off = static_cast<int>(kGI.off[l]);
      acc[q] = __dp4a(static_cast<int>(res[l]), tw, off);
    });
    static_for<0, (l + 3) / 4>([&](auto W) {
      constexpr int w = decltype(W)::value;
      constexpr int kw = kGI.kw[l][w];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = __dp4a(static_cast<int>(D[q][w]), kw, acc[q]);
    });
#pragma unroll
    for (int q = 0; q < 4; ++q)
      D[q][l / 4] = put_byte<l % 4>(D[q][l / 4], sym_from_biased<l>(static_cast<uint32_t>(acc[q])));
  });
}

// Exact signed value of the digits of one element (|value| < M/2), rounded to the nearest
// FP64 and scaled by 2^-es (a second rounding only for a subnormal result).
// `extra` (the split-off diagonal term Delta'_ij Z'_jj) is added before the rounding.
__device__ __forceinline__ double garner_value(const uint32_t (&D)[4], int es, __int128 extra) {
  // Digit pairs P_k = dig_2k + m_2k dig_2k+1 (|P_k| < 2^16), then value = hi * W_8 + lo with
  // each half a Horner sum over pairs, exact in int64 (|lo| < W_8 / 2, |hi| < 2^61).
  int pr[kMods / 2];
  static_for<0, kMods / 2>([&](auto K) {
    constexpr int k = decltype(K)::value;
    constexpr int m = kG.m[2 * k];
    const uint32_t w = D[k / 2];
    pr[k] = sbyte<(2 * k) % 4>(w) + m * sbyte<(2 * k + 1) % 4>(w);
  });
  long long lo = pr[3], hi = pr[7];
  static_for<0, 3>([&](auto K) {
    constexpr int k = 2 - decltype(K)::value;
    constexpr long long ml = static_cast<long long>(kG.m[2 * k]) * kG.m[2 * k + 1];
    constexpr long long mh = static_cast<long long>(kG.m[2 * k + 8]) * kG.m[2 * k + 9];
    lo = lo * ml + pr[k];
    hi = hi * mh + pr[k + 4];
  });
  const __int128 p = static_cast<__int128>(hi) * static_cast<__int128>(kW8) + lo + extra;
  const bool neg = p < 0;
  const double mg = u128_to_double(neg ? (unsigned __int128)(-p) : (unsigned __int128)p);
  return scale2(neg ? -mg : mg, -es);
}

// Reconstruct W_ij from the residues (R[l][j][i], j = column of B / Z, i = row of A) and
// apply the IPT map (mode 0) or the closing residual (mode 1) with the K1 formulas, or
// store W itself (mode 2).
// Four consecutive rows i per thread (one 4-byte load per modulus plane; ldr % 4 == 0).
template <int L>
__device__ __forceinline__ void reconstruct_body(const OzakiMapArgs& a, double (&v)[4]) {
  // n, ncols <= kOzakiMaxK: the work index fits 32 bits (32-bit division, not 64)
  const uint32_t n4 = static_cast<uint32_t>((a.n + 3) >> 2);
  const uint32_t total = n4 * static_cast<uint32_t>(a.ncols);
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    const uint32_t jj = t / n4;
    const int64_t j = jj, i0 = int64_t(t - jj * n4) << 2;
    const int eb = a.eB[j];
    const int8_t* rp = a.R + j * a.ldr + i0;
    uint32_t res[kMods];
#pragma unroll
    for (int l = 0; l < kMods; ++l) res[l] = l < L ? *reinterpret_cast<const uint32_t*>(rp + l * a.plane) : 0u;
    const int64_t jg = a.col0 + j;
    const double dj = a.mode == 0 ? a.d[jg] : 0.0;
    const long long zjj = a.dZ != nullptr ? static_cast<long long>(a.dZ[j]) : 0;
    uint32_t D[4][4];
    garner_digits4<L>(res, D);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t i = i0 + q;
      if (i >= a.n) break;
      const int ea = a.eA[i];
      double w;
      if (ea == kOzakiNonFinite || eb == kOzakiNonFinite) {
        w = __longlong_as_double(0x7ff8000000000000LL);  // NaN, as the FP64 product would give
      } else {
        __int128 extra = 0;
        if (a.dZ != nullptr) {  // Delta'_ij exactly as residues_kernel rounded it
          const long long dij = static_cast<long long>(rint(scale2(a.DT[jg * a.lddt + i], ea)));
          extra = static_cast<__int128>(dij) * zjj;
        }
        w = garner_value(D[q], ea + eb, extra);
      }
      if (a.mode == 2) {
        a.F[j * a.ldz + i] = w;
        continue;
      }
      if (a.mode >= 3) {  // complex 3M: this product is T3 = (Dr + Di)(Zr + Zi)
        const double t1 = a.T1[j * a.ldt + i], t2 = a.T2[j * a.ldt + i];
        const cd wc{t1 - t2, w - t1 - t2};
        const cd z{a.Z[j * a.ldz + i], a.Zi[j * a.ldz + i]};
        const cd di{a.d[i], a.di[i]};
        if (a.mode == 3) {
          const cd dj{a.d[jg], a.di[jg]}, wj{a.wd[j], a.wdi[j]};
          const cd f = (i == jg) ? cd{1.0, 0.0} : cdiv(csub(cmul(z, wj), wc), csub(di, dj));
          a.F[j * a.ldz + i] = f.re;
          a.Fi[j * a.ldz + i] = f.im;
          const cd df = csub(f, z);
          v[0] += df.re * df.re + df.im * df.im;
          v[1] += z.re * z.re + z.im * z.im;
          v[2] += f.re * f.re + f.im * f.im;
          v[3] = nan_max(v[3], hypot(df.re, df.im));
        } else {
          const cd r = csub(cadd(cmul(di, z), wc), cmul(z, cd{a.lam[j], a.lami[j]}));
          v[0] += r.re * r.re + r.im * r.im;
        }
        continue;
      }
      const double z = a.Z[j * a.ldz + i];
      const double di = a.d[i];
      if (a.mode == 0) {
        const double f = (i == jg) ? 1.0 : __ddiv_rn(__dsub_rn(__dmul_rn(z, a.wd[j]), w), __dsub_rn(di, dj));
        a.F[j * a.ldz + i] = f;
        const double df = __dsub_rn(f, z);
        v[0] = __fma_rn(df, df, v[0]);
        v[1] = __fma_rn(z, z, v[1]);
        v[2] = __fma_rn(f, f, v[2]);
        v[3] = nan_max(v[3], fabs(df));
      } else {
        const double rr = __dsub_rn(__dadd_rn(__dmul_rn(di, z), w), __dmul_rn(z, a.lam[j]));
        v[0] = __fma_rn(rr, rr, v[0]);
      }
    }
  }
}

__global__ void __launch_bounds__(256) reconstruct_map_kernel(OzakiMapArgs a) {
  if (a.state != nullptr && a.state->done) return;
  __shared__ double red[8][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  switch (a.moduli != nullptr ? *a.moduli : kMods) {  // uniform across the grid
    case 9: reconstruct_body<9>(a, v); break;
    case 10: reconstruct_body<10>(a, v); break;
    case 11: reconstruct_body<11>(a, v); break;
    case 12: reconstruct_body<12>(a, v); break;
    case 13: reconstruct_body<13>(a, v); break;
    case 14: reconstruct_body<14>(a, v); break;
    case 15: reconstruct_body<15>(a, v); break;
    default: reconstruct_body<16>(a, v); break;
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

// DT = A^T through 32 x 32 shared-memory tiles (coalesced both ways)
__global__ void transpose_kernel(const double* __restrict__ A, int64_t lda, int64_t n, double* __restrict__ DT,
                                 int64_t ldt) {
  __shared__ double tile[32][33];
  const int64_t bx = int64_t(blockIdx.x) * 32, by = int64_t(blockIdx.y) * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = by + y, c = bx + threadIdx.x;
    if (r < n && c < n) tile[y][threadIdx.x] = A[r * lda + c];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t r = bx + y, c = by + threadIdx.x;
    if (r < n && c < n) DT[r * ldt + c] = tile[threadIdx.x][y];
  }
}

}  // namespace

void OzakiOperand::build(cudaStream_t s, const double* X, int64_t ldx, int64_t rows_, int64_t len_, int64_t rows_pad,
                         int64_t kpad_, int64_t diag0, int* moduli) {
  rows = rows_;
  len = len_;
  kpad = kpad_;
  plane = rows_pad * kpad;
  if (res.count * 8 < size_t(kMods) * plane) res.alloc(ceil_div(int64_t(kMods) * plane, 8));  // zeroed padding rows
  if (e.count < size_t(rows_pad)) e.alloc(rows_pad);
  if (diag0 >= 0 && diag.count < size_t(rows_pad)) diag.alloc(rows_pad);
  int* ep = reinterpret_cast<int*>(e.get());
  if (moduli != nullptr) IPT_CUDA(cudaMemsetAsync(moduli, 0, sizeof(int), s));
  exponent_kernel<<<static_cast<unsigned>(ceil_div(rows, 8)), 256, 0, s>>>(X, ldx, rows, len, ep, diag0, moduli);
  residues_kernel<<<2368, 256, 0, s>>>(X, ldx, rows, len, ep, reinterpret_cast<int8_t*>(res.get()), kpad, plane,
                                       diag0, diag0 >= 0 ? diag.get() : nullptr, moduli);
  IPT_LAUNCH_CHECK();
  count_launch(2);
}

// R[l] = (Bop . Aop^T) mod m_l for all moduli: rows of the product = rows of Bop (the Z
// columns), columns = rows of Aop (the Delta rows).
// Moduli at or past *moduli (when given) are skipped on the device: their GEMMs exit at once.
void ozaki_products(cudaStream_t s, const OzakiOperand& Zop, const OzakiOperand& Aop, int64_t zrows_pad,
                    int64_t arows_pad, DevBuf& R, int64_t& plane, const int* moduli) {
  if (Zop.kpad != Aop.kpad || Zop.len > kOzakiMaxK)
    throw InvalidArgument("ozaki: inner dimension must match and be at most 65535");
  plane = zrows_pad * arows_pad;
  if (R.count * 8 < size_t(kMods) * plane) R.alloc(ceil_div(int64_t(kMods) * plane, 8), false);
  for (int l = 0; l < kMods; ++l) {
    ModStore epi{reinterpret_cast<int8_t*>(R.get()) + l * plane, arows_pad, mod_magic(kG.m[l]), moduli, l};
    launch_i8gemm(s, zrows_pad, arows_pad, Zop.kpad, reinterpret_cast<const int8_t*>(Zop.res.get()) + l * Zop.plane,
                  Zop.kpad, reinterpret_cast<const int8_t*>(Aop.res.get()) + l * Aop.plane, Aop.kpad, epi);
  }
}

void ozaki_transpose(cudaStream_t s, const double* A, int64_t lda, int64_t n, double* DT, int64_t ldt) {
  const dim3 grid(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(n, 32)));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(A, lda, n, DT, ldt);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void ozaki_reconstruct(cudaStream_t s, const OzakiMapArgs& a) {
  if (((a.n + 3) >> 2) * a.ncols >= (int64_t(1) << 32)) throw InvalidArgument("ozaki: product too large");
  reconstruct_map_kernel<<<kOzakiGrid, 256, 0, s>>>(a);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void ozaki_dgemm_device(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                        double* C, DevBuf& partials) {
  if (M <= 0 || N <= 0) return;
  if (K > kOzakiMaxK) throw InvalidArgument("ozaki_dgemm: K must be at most 65535");
  const int64_t kpad = round_up(std::max<int64_t>(K, 1), kOzakiKPad);
  // product rows = rows of A (the GEMM's M side, 256-row pair tiles), columns = rows of B
  // (N side, 512-wide tiles), so the reconstruction writes C row-major
  const int64_t mpad = round_up(M, 256), npad = round_up(N, 512);
  OzakiOperand opa, opb;
  opa.build(s, A, K, M, K, mpad, kpad);
  opb.build(s, B, K, N, K, npad, kpad);
  DevBuf R;
  int64_t plane = 0;
  ozaki_products(s, opa, opb, mpad, npad, R, plane);
  if (partials.count < size_t(kOzakiGrid) * 4) partials.alloc(size_t(kOzakiGrid) * 4, false);
  OzakiMapArgs a{};
  a.R = reinterpret_cast<const int8_t*>(R.get());
  a.plane = plane;
  a.ldr = npad;
  a.eA = opb.exps();
  a.eB = opa.exps();
  a.F = C;
  a.ldz = N;
  a.n = N;
  a.ncols = M;
  a.mode = 2;
  a.partials = partials.get();
  ozaki_reconstruct(s, a);
  IPT_CUDA(cudaStreamSynchronize(s));  // the local operand and residue buffers die here
}

}  // namespace iptb
