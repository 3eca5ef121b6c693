// Does the TMA unit gather random z entries faster than the LSU/L1TEX path?
//
// The CSR SpMV map (K8) of config 5 is bound by the random z[col] gathers: every 8-byte use
// is one 128-byte-line wavefront in L1TEX (~1 line per clock per SM), measured ceiling
// 0.518 ms for 134 M gathers (gather_probe.cu). cp.async.bulk.tensor ... tile::gather4
// (sm_100) fetches 4 arbitrary rows of a 2D tensor into shared memory through the TMA
// engine instead. Viewing z as [N/2][2] doubles (16-byte rows, the smallest TMA box),
// one gather4 brings the 4 rows holding 4 wanted entries.
//
//   ldg    : stream cols + vals, gather z[col] with LDG (the K8 memory pattern)
//   tma<D> : stream cols + vals with LDG, gather z through TMA gather4 into a D-stage
//            per-warp ring of 4 KB stages (32 lanes x 4 rows x 16 B, each lane's 64 B at a 128 B-aligned slot), mbarrier per stage
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tma_gather_probe tma_gather_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);       \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ int4 ld_stream_i4(const int4* p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld_stream_d2(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Reference pattern: 4 consecutive entries per lane per chunk of 128, LDG gathers.
__global__ void __launch_bounds__(256) ldg_kernel(const int* __restrict__ cols, const double* __restrict__ vals,
                                                  const double* __restrict__ z, int64_t nchunks, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  double s = 0.0;
  for (int64_t ch = warp; ch < nchunks; ch += nw) {
    const int64_t e = ch * 128 + lane * 4;
    const int4 c = ld_stream_i4(reinterpret_cast<const int4*>(cols + e));
    const double2 v0 = ld_stream_d2(reinterpret_cast<const double2*>(vals + e));
    const double2 v1 = ld_stream_d2(reinterpret_cast<const double2*>(vals + e + 2));
    const double z0 = __ldg(z + c.x), z1 = __ldg(z + c.y), z2 = __ldg(z + c.z), z3 = __ldg(z + c.w);
    s = fma(v0.x, z0, s);
    s = fma(v0.y, z1, s);
    s = fma(v1.x, z2, s);
    s = fma(v1.y, z3, s);
  }
  atomicAdd(out, s);
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile(
      "{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(
          su32(b)),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* map, uint64_t* bar, int r0, int r1, int r2,
                                        int r3) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5, %6}], [%7];" ::"r"(su32(dst)),
      "l"(map), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar))
      : "memory");
}

// Each warp owns D stages of 2 KB (+ one mbarrier each) and walks its chunks of 128
// entries: stage k's gathers are issued D-1 chunks before they are consumed.
template <int D, int WARPS>
__global__ void __launch_bounds__(WARPS * 32) tma_kernel(const int* __restrict__ cols,
                                                         const double* __restrict__ vals,
                                                         const __grid_constant__ CUtensorMap zmap, int64_t nchunks,
                                                         double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* ring = reinterpret_cast<double2*>(smem) + size_t(w) * D * 256;  // D stages x 32 lanes x 8 slots (128 B aligned)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(WARPS) * D * 4096) + w * D;
  if (lane == 0)
    for (int k = 0; k < D; ++k) mbar_init(bars + k, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t warp = int64_t(blockIdx.x) * WARPS + w;
  const int64_t nw = int64_t(gridDim.x) * WARPS;
  const int64_t mine = warp < nchunks ? (nchunks - 1 - warp) / nw + 1 : 0;
  int sel[D];
  double2 va[D], vb[D];
  double s = 0.0;
  auto issue = [&](int64_t t, int slot) {
    const int64_t e = (warp + t * nw) * 128 + lane * 4;
    const int4 c = ld_stream_i4(reinterpret_cast<const int4*>(cols + e));
    va[slot] = ld_stream_d2(reinterpret_cast<const double2*>(vals + e));
    vb[slot] = ld_stream_d2(reinterpret_cast<const double2*>(vals + e + 2));
    sel[slot] = (c.x & 1) | ((c.y & 1) << 1) | ((c.z & 1) << 2) | ((c.w & 1) << 3);
    if (lane == 0) mbar_expect(bars + slot, 2048);
    __syncwarp();
    gather4(ring + (slot * 32 + lane) * 8, &zmap, bars + slot, c.x >> 1, c.y >> 1, c.z >> 1, c.w >> 1);
  };
#pragma unroll
  for (int k = 0; k < D - 1; ++k)
    if (k < mine) issue(k, k);
  for (int64_t t = 0; t < mine; t += D) {
#pragma unroll
    for (int k = 0; k < D; ++k) {
      const int64_t tk = t + k;
      if (tk < mine) {
        // issue chunk tk + D - 1 into slot (k + D - 1) % D (consumed at tk - 1: free)
        if (tk + D - 1 < mine) issue(tk + D - 1, (k + D - 1) % D);
        mbar_wait(bars + k, uint32_t((tk / D) & 1));
        const double2* r = ring + (k * 32 + lane) * 8;
        const int m = sel[k];
        const double z0 = (m & 1) ? r[0].y : r[0].x;
        const double z1 = (m & 2) ? r[1].y : r[1].x;
        const double z2 = (m & 4) ? r[2].y : r[2].x;
        const double z3 = (m & 8) ? r[3].y : r[3].x;
        s = fma(va[k].x, z0, s);
        s = fma(va[k].y, z1, s);
        s = fma(vb[k].x, z2, s);
        s = fma(vb[k].y, z3, s);
        __syncwarp();
      }
    }
  }
  atomicAdd(out, s);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <class F>
float time_ms(F f, int reps = 10) {
  f();
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <int D, int WARPS>
int run_tma(const char* name, int per_sm, int sms, const int* c, const double* v, const CUtensorMap& m,
            int64_t nchunks, int64_t nnz, double* out) {
  const size_t smem = size_t(WARPS) * D * 4096 + size_t(WARPS) * D * 8;
  CK(cudaFuncSetAttribute(tma_kernel<D, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const int grid = sms * per_sm;
  const float ms = time_ms([&] { tma_kernel<D, WARPS><<<grid, WARPS * 32, smem>>>(c, v, m, nchunks, out); });
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  printf("%-26s grid %5d smem %6zu  %7.3f ms  stream %7.1f GB/s  %.2f Ggathers/s\n", name, grid, smem, ms,
         12.0 * nnz / (ms * 1e-3) / 1e9, nnz / (ms * 1e-3) / 1e9);
  return 0;
}

int main() {
  const int64_t n = int64_t(1) << 21;
  const int64_t nchunks = 134216644 / 128;  // config 5's nnz, whole chunks of 128
  const int64_t nnz = nchunks * 128;
  std::vector<int> hc(nnz);
  std::mt19937_64 g(7);
  for (int64_t i = 0; i < nnz; ++i) hc[i] = static_cast<int>(g() % n);
  std::vector<double> hz(n), hv(nnz);
  for (int64_t i = 0; i < n; ++i) hz[i] = 1.0 + double(i % 97) * 0.5;
  for (int64_t i = 0; i < nnz; ++i) hv[i] = double((i * 7) % 13) - 6.0;
  int* c;
  double *v, *z, *out;
  CK(cudaMalloc(&c, nnz * 4));
  CK(cudaMalloc(&v, nnz * 8));
  CK(cudaMalloc(&z, n * 8));
  CK(cudaMalloc(&out, 8));
  CK(cudaMemcpy(c, hc.data(), nnz * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(v, hv.data(), nnz * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(z, hz.data(), n * 8, cudaMemcpyHostToDevice));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  CUtensorMap m;
  cuuint64_t dims[2] = {2, cuuint64_t(n / 2)};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, z, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", int(r));
  if (r != CUDA_SUCCESS) return 1;

  // correctness: the TMA kernel's total equals the LDG kernel's (same products, other order)
  {
    double a = 0, b = 0;
    CK(cudaMemset(out, 0, 8));
    ldg_kernel<<<sms * 4, 256>>>(c, v, z, nchunks, out);
    CK(cudaMemcpy(&a, out, 8, cudaMemcpyDeviceToHost));
    CK(cudaFuncSetAttribute(tma_kernel<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 4 * 4096 + 128));
    CK(cudaMemset(out, 0, 8));
    tma_kernel<4, 4><<<sms * 4, 128, 4 * 4 * 4096 + 128>>>(c, v, m, nchunks, out);
    CK(cudaGetLastError());
    CK(cudaMemcpy(&b, out, 8, cudaMemcpyDeviceToHost));
    printf("check: ldg sum %.17g tma sum %.17g rel %.3g\n", a, b, fabs(a - b) / fabs(a));
  }

  for (int per : {4, 8, 16}) {
    const int grid = sms * per;
    const float ms = time_ms([&] { ldg_kernel<<<grid, 256>>>(c, v, z, nchunks, out); });
    printf("%-26s grid %5d             %7.3f ms  stream %7.1f GB/s  %.2f Ggathers/s\n", "ldg u4", grid, ms,
           12.0 * nnz / (ms * 1e-3) / 1e9, nnz / (ms * 1e-3) / 1e9);
  }
  run_tma<4, 4>("tma D4 w4", 4, sms, c, v, m, nchunks, nnz, out);
  run_tma<4, 4>("tma D4 w4", 8, sms, c, v, m, nchunks, nnz, out);
  run_tma<8, 4>("tma D8 w4", 4, sms, c, v, m, nchunks, nnz, out);
  run_tma<8, 4>("tma D8 w4", 6, sms, c, v, m, nchunks, nnz, out);
  run_tma<4, 8>("tma D4 w8", 4, sms, c, v, m, nchunks, nnz, out);
  run_tma<4, 8>("tma D4 w8", 6, sms, c, v, m, nchunks, nnz, out);
  run_tma<2, 4>("tma D2 w4", 8, sms, c, v, m, nchunks, nnz, out);
  run_tma<2, 8>("tma D2 w8", 8, sms, c, v, m, nchunks, nnz, out);
  return 0;
}
