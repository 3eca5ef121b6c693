// Host side of the tcgen05 INT8 GEMM (i8gemm.cuh): tensor maps for int8 K-major operands
// and a test / measurement entry point (ipt_i8_gemm in include/ipt_cuda.h).
#include <cudaTypedefs.h>

#include <mutex>
#include <vector>

#include "i8gemm.cuh"
#include "ipt_internal.cuh"

namespace iptb {

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_i8() {
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

struct StoreI32 {
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

}  // namespace

// `rows` x `k` int8, K contiguous (pitch ld bytes), boxes of 128 bytes x box_rows rows.
CUtensorMap make_map_i8(const void* base, int64_t k, int64_t rows, int64_t ld, int box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || ld % 16 != 0)
    throw InvalidArgument("i8 gemm: TMA operands need 16-byte aligned base and pitch");
  CUtensorMap m;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld)};
  cuuint32_t box[2] = {kI8BK, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_i8()(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (int8) failed (" + std::to_string(int(r)) + ")");
  return m;
}

// C (M x N int32, row-major) = A (M x K) . B (N x K)^T, device pointers; M % 128, N % 256,
// K % 128 == 0.
void i8_gemm_device(cudaStream_t s, int64_t M, int64_t N, int64_t K, const int8_t* A, const int8_t* B, int32_t* C) {
  launch_i8gemm(s, M, N, K, A, K, B, K, StoreI32{C, N});
}

}  // namespace iptb

