// Host launchers for the K1 DMMA GEMM (dmma_gemm.cuh): TMA descriptor encoding
// (cuTensorMapEncodeTiled through the runtime's driver entry point, no -lcuda)
// and the per-mode kernel launch.
#include <cudaTypedefs.h>

#include <mutex>

#include "dmma_gemm.cuh"
#include "ipt_internal.cuh"

namespace iptb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    IPT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || p == nullptr) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// K-major operand: `outer` rows of `inner` contiguous doubles, row pitch ld doubles;
// boxes of 16 doubles (128 B, the swizzle span) x 128 rows, 128-byte swizzle.
CUtensorMap make_map(const double* base, int64_t inner, int64_t outer, int64_t ld) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld * 8) % 16 != 0)
    throw InvalidArgument("gemm: TMA operands need 16-byte aligned base and pitch");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  cuuint32_t box[2] = {kBK, kBM};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides,
                                 box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
  return m;
}

template <int MODE>
void launch_mode(const GemmParams& p, cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([] {
    IPT_CUDA(cudaFuncSetAttribute(dmma_tma_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kGemmSmemBytes)));
  });
  const unsigned grid = static_cast<unsigned>(p.tiles_m) * static_cast<unsigned>(p.tiles_n);
  if (grid == 0) return;
  const CUtensorMap ma = make_map(p.A, p.K, int64_t(p.tiles_m) * kBM, p.lda);
  const CUtensorMap mb = make_map(p.B, p.K, int64_t(p.tiles_n) * kBN, p.ldb);
  dmma_tma_kernel<MODE><<<grid, kGemmThreads, kGemmSmemBytes, s>>>(ma, mb, p);
  IPT_LAUNCH_CHECK();
  count_launch();
}

// FP64 tensor issue-rate probe: back-to-back m16n8k4 DMMAs (K1's instruction) from
// registers, 8 independent accumulators per warp, 8 warps on every SM: the roofline
// denominator of the FP64 kernels, measured in the caller's run instead of a constant.
__global__ void __launch_bounds__(256) dmma_issue_probe_kernel(double* out, int iters) {
  double acc[8][4];
  const double a0 = 1e-9 * threadIdx.x, a1 = 2e-9 * threadIdx.x, b0 = 3e-9 * threadIdx.x;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma_16x8x4(acc[j], a0, a1, b0);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 12345.678) out[0] = s;  // keeps the loop
}

}  // namespace

double fp64_issue_probe_tflops(cudaStream_t s, int device) {
  int sms = 0;
  IPT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  DevBuf out;
  out.alloc(1);
  cudaEvent_t e0, e1;
  IPT_CUDA(cudaEventCreate(&e0));
  IPT_CUDA(cudaEventCreate(&e1));
  const int iters = 20000;
  dmma_issue_probe_kernel<<<sms, 256, 0, s>>>(out.get(), iters / 10);  // warm-up / clocks up
  IPT_LAUNCH_CHECK();
  double best = 0.0;
  for (int rep = 0; rep < 3; ++rep) {
    IPT_CUDA(cudaEventRecord(e0, s));
    dmma_issue_probe_kernel<<<sms, 256, 0, s>>>(out.get(), iters);
    IPT_CUDA(cudaEventRecord(e1, s));
    IPT_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    IPT_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    // per warp and iteration: 8 DMMAs of 2 * 16 * 8 * 4 flops
    const double flops = double(sms) * 8.0 * iters * 8.0 * (2.0 * 16 * 8 * 4);
    best = std::max(best, flops / (double(ms) * 1e-3) / 1e12);
  }
  count_launch(4);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return best;
}

size_t gemm_tiles(int64_t rows, int64_t cols) {
  return static_cast<size_t>(ceil_div(rows, kBM) * ceil_div(cols, kBN));
}

void launch_gemm(int mode, const GemmParams& p, cudaStream_t s) {
  if (p.K % kBK != 0) throw InvalidArgument("launch_gemm: K must be a multiple of 16");
  switch (mode) {
    case kGemmStore: launch_mode<kGemmStore>(p, s); break;
    case kGemmMap: launch_mode<kGemmMap>(p, s); break;
    case kGemmResid: launch_mode<kGemmResid>(p, s); break;
    case kGemmSub: launch_mode<kGemmSub>(p, s); break;
    case kGemmMapC: launch_mode<kGemmMapC>(p, s); break;
    case kGemmResidC: launch_mode<kGemmResidC>(p, s); break;
    case kGemmSubC: launch_mode<kGemmSubC>(p, s); break;
    case kGemmSubAll: launch_mode<kGemmSubAll>(p, s); break;
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
