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
constexpr int kOzakiMinMods = 9;             // fewest moduli the reconstruction is instantiated for

// One operand in residue form: rows x kpad int8 per modulus (K contiguous, zero padded),
// and the per-row binary exponent of its scaling.
//
// Diagonal split (diag0 >= 0, the Z operand of the IPT map): row r's entry at k = diag0 + r
// (Z_jj = 1 for every iterate) is left out of the residues and kept as an exact integer
// in diag[r]; the product then only carries the off-diagonal part Y' = Z' - Z'_jj e_j,
// whose column 1-norm bounds |Delta' Y'| < 2^53 |Y'_j|_1. exponent_kernel turns that bound
// into the number of moduli the exact product needs (atomicMax into *moduli), and the
// GEMMs / reconstruction of moduli past it are skipped; the reconstruction adds
// Delta'_ij Z'_jj back in 128-bit integers before the single rounding, so W is the same
// correctly rounded exact product as with all 16 moduli (bitwise).
struct OzakiOperand {
  DevBuf res;   // kOzakiMods planes of rows_pad x kpad bytes
  DevBuf e;     // int per row (in a double-sized buffer)
  DevBuf diag;  // split operands: the removed diagonal entry of each row (integer-valued)
  int64_t rows = 0, len = 0, kpad = 0, plane = 0;
  void build(cudaStream_t s, const double* X, int64_t ldx, int64_t rows, int64_t len, int64_t rows_pad,
             int64_t kpad, int64_t diag0 = -1, int* moduli = nullptr);
  const int* exps() const { return reinterpret_cast<const int*>(e.get()); }
};

struct OzakiMapArgs {
  const int8_t* R;  // residues of the product, [l][j][i]
  int64_t plane, ldr;
  const int* eA;    // per row i (Delta)
  const int* eB;    // per column j (Z)
  const double* Z;
  int64_t ldz;
  const double* dZ;   // split: Z'_jj per local column (nullptr: no split)
  const double* DT;   // split: Delta transposed, DT[jg * lddt + i] = Delta_ij
  int64_t lddt;
  const int* moduli;  // device count of moduli in use (nullptr: all 16)
  double* F;
  const double* d;
  const double* wd;
  const double* lam;
  int64_t n, ncols, col0;
  // complex 3M (modes 3 / 4): this product is T3, T1 = Dr Zr and T2 = Di Zi already stored
  const double* T1;
  const double* T2;
  int64_t ldt;
  const double* Zi;
  const double* di;
  const double* wdi;
  const double* lami;
  double* Fi;
  int mode;  // 0: map, 1: closing residual, 2: store W, 3: complex map, 4: complex residual
  double* partials;
  const LoopState* state;
};

void ozaki_products(cudaStream_t s, const OzakiOperand& Zop, const OzakiOperand& Aop, int64_t zrows_pad,
                    int64_t arows_pad, DevBuf& R, int64_t& plane, const int* moduli = nullptr);
// DT (n x ldt, row-major) = A^T for A (n x n, row-major, lda)
void ozaki_transpose(cudaStream_t s, const double* A, int64_t lda, int64_t n, double* DT, int64_t ldt);
void ozaki_reconstruct(cudaStream_t s, const OzakiMapArgs& a);

// C (M x N, row-major, ldc = N) = A (M x K, row-major) . B (N x K, row-major)^T in FP64 by
// Ozaki scheme II, device pointers: each element is the correctly rounded exact dot product
// of the rows scaled to 53-bit integers (row max in [2^52, 2^53)).
void ozaki_dgemm_device(cudaStream_t s, int64_t M, int64_t N, int64_t K, const double* A, const double* B,
                        double* C, DevBuf& partials);

}  // namespace iptb
