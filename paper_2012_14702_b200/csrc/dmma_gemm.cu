// Host launchers for the K1 DMMA GEMM (dmma_gemm.cuh).
#include "dmma_gemm.cuh"
#include "ipt_internal.cuh"

namespace iptb {

namespace {
template <int MODE>
void launch_mode(const GemmParams& p, cudaStream_t s) {
  static bool configured = false;  // per-device attribute; all devices get the same value
  if (!configured) {
    IPT_CUDA(cudaFuncSetAttribute(dmma_gemm_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGemmSmemBytes)));
    configured = true;
  }
  const unsigned grid = static_cast<unsigned>(p.tiles_m) * static_cast<unsigned>(p.tiles_n);
  if (grid == 0) return;
  dmma_gemm_kernel<MODE><<<grid, kGemmThreads, kGemmSmemBytes, s>>>(p);
  IPT_LAUNCH_CHECK();
  count_launch();
}
}  // namespace

size_t gemm_tiles(int64_t rows, int64_t cols) {
  return static_cast<size_t>(ceil_div(rows, kBM) * ceil_div(cols, kBN));
}

void launch_gemm(int mode, const GemmParams& p, cudaStream_t s) {
  switch (mode) {
    case kGemmStore: launch_mode<kGemmStore>(p, s); break;
    case kGemmMap: launch_mode<kGemmMap>(p, s); break;
    case kGemmResid: launch_mode<kGemmResid>(p, s); break;
    case kGemmSub: launch_mode<kGemmSub>(p, s); break;
    default: throw InvalidArgument("launch_gemm: bad mode");
  }
}

void gemm_tn_store(cudaStream_t s, int64_t m, int64_t n, int64_t kpad, const double* A, int64_t lda,
                   const double* Bt, int64_t ldb, double* C, int64_t ldc) {
  GemmParams p{};
  p.K = kpad;
  p.A = A;
  p.lda = lda;
  p.B = Bt;
  p.ldb = ldb;
  p.C = C;
  p.ldc = ldc;
  p.tiles_m = static_cast<int>(ceil_div(m, kBM));
  p.tiles_n = static_cast<int>(ceil_div(n, kBN));
  p.n_rows = m;
  p.n_cols = n;
  launch_gemm(kGemmStore, p, s);
}

}  // namespace iptb
