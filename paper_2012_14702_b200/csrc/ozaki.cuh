// FP64-accurate products on the tcgen05 INT8 datapath (Ozaki scheme II), ozaki.cu.
#pragma once

#include "ipt_internal.cuh"

namespace iptb {

constexpr int kOzakiMods = 16;
constexpr int kOzakiNonFinite = 0x7fffffff;  // exponent marker of a row / column with Inf or NaN
constexpr int kOzakiGrid = 1184;             // fixed reconstruction grid (deterministic partials)
constexpr int64_t kOzakiKPad = 128;          // K padding of the residue operands (the INT8 GEMM's BK)
constexpr int64_t kOzakiMaxK = 65535;        // |int32 sums| <= K 2^14 <= 2^30 - 2^14 (epilogue reduction range)

// One operand in residue form: rows x kpad int8 per modulus (K contiguous, zero padded),
// and the per-row binary exponent of its scaling.
struct OzakiOperand {
  DevBuf res;  // kOzakiMods planes of rows_pad x kpad bytes
  DevBuf e;    // int per row (in a double-sized buffer)
  int64_t rows = 0, len = 0, kpad = 0, plane = 0;
  void build(cudaStream_t s, const double* X, int64_t ldx, int64_t rows, int64_t len, int64_t rows_pad,
             int64_t kpad);
  const int* exps() const { return reinterpret_cast<const int*>(e.get()); }
};

struct OzakiMapArgs {
  const int8_t* R;  // residues of the product, [l][j][i]
  int64_t plane, ldr;
  const int* eA;    // per row i (Delta)
  const int* eB;    // per column j (Z)
  const double* Z;
  int64_t ldz;
  double* F;
  const double* d;
  const double* wd;
  const double* lam;
  int64_t n, ncols, col0;
  int mode;  // 0: map, 1: closing residual, 2: store W
  double* partials;
  const LoopState* state;
};

void ozaki_products(cudaStream_t s, const OzakiOperand& Zop, const OzakiOperand& Aop, int64_t zrows_pad,
                    int64_t arows_pad, DevBuf& R, int64_t& plane);
void ozaki_reconstruct(cudaStream_t s, const OzakiMapArgs& a);

// C (M x N, row-major, ldc = N) = A (M x K, row-major) . B (N x K, row-major)^T in FP64 by
// Ozaki scheme II, device pointers: each element is the correctly rounded exact dot product
// of the rows scaled to 53-bit integers (row max in [2^52, 2^53)).
void ozaki_dgemm_device(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                        double* C, DevBuf& partials);

}  // namespace iptb
