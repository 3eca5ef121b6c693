// Ceiling probe for the CSR SpMV map (K8): the same memory traffic without the row
// structure. nnz = 134,216,644 (config 5), z = 2^21 doubles (16 MB, L2-resident).
//   stream : read cols (int32) + vals (fp64) once            -> HBM roofline of 12 B/nnz
//   gather : stream + z[col] gather, sum of vals * z[col]    -> the SpMV memory ceiling
// Columns uniform random in [0, 2^21) like the config 5 construction.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ double ld_stream_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream_s32(const int* p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// z gather load flavours: 0 ld.global.nc (L1 allocate), 1 nc + L1::no_allocate, 2 ld.global.cg (L2 only),
// 3 ld.global.nc + L1::evict_first
template <int KIND>
__device__ __forceinline__ double ld_gather(const double* p) {
  double v;
  if (KIND == 0) v = __ldg(p);
  else if (KIND == 1) asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else if (KIND == 2) asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::evict_first.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

template <int U, bool GATHER, int KIND = 0>
__global__ void __launch_bounds__(256) probe(const int* __restrict__ cols, const double* __restrict__ vals,
                                             const double* __restrict__ z, int64_t nnz, double* out) {
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (; e + (U - 1) * stride < nnz; e += U * stride) {
    int c[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = ld_stream_s32(cols + e + u * stride);
      v[u] = ld_stream_f64(vals + e + u * stride);
    }
    if (GATHER) {
      double zz[U];
#pragma unroll
      for (int u = 0; u < U; ++u) zz[u] = ld_gather<KIND>(z + c[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) s = fma(v[u], zz[u], s);
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) s += v[u] + c[u];
    }
  }
  for (; e < nnz; e += stride) s += GATHER ? vals[e] * z[cols[e]] : vals[e] + cols[e];
  if (s == 1234.5678) out[0] = s;
}

template <int U, bool G, int KIND = 0>
void run(const char* name, int grid, const int* c, const double* v, const double* z, int64_t nnz, double* out) {
  probe<U, G, KIND><<<grid, 256>>>(c, v, z, nnz, out);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 10;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) probe<U, G, KIND><<<grid, 256>>>(c, v, z, nnz, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  ms /= reps;
  const double bytes = 12.0 * nnz;
  printf("%-22s grid %6d  %7.3f ms  stream %7.1f GB/s  gathered sectors %7.1f GB/s  err=%s\n", name, grid, ms,
         bytes / (ms * 1e-3) / 1e9, G ? 32.0 * nnz / (ms * 1e-3) / 1e9 : 0.0, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t nnz = 134216644, n = int64_t(1) << 21;
  std::vector<int> hc(nnz);
  std::mt19937_64 g(7);
  for (int64_t i = 0; i < nnz; ++i) hc[i] = static_cast<int>(g() % n);
  int* c;
  double *v, *z, *out;
  cudaMalloc(&c, nnz * 4);
  cudaMalloc(&v, nnz * 8);
  cudaMalloc(&z, n * 8);
  cudaMalloc(&out, 8);
  cudaMemcpy(c, hc.data(), nnz * 4, cudaMemcpyHostToDevice);
  cudaMemset(v, 0, nnz * 8);
  cudaMemset(z, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {4, 8, 16}) {
    run<4, false>("stream u4", sms * per, c, v, z, nnz, out);
    run<4, true>("gather u4", sms * per, c, v, z, nnz, out);
    run<8, true>("gather u8", sms * per, c, v, z, nnz, out);
    run<4, true, 1>("gather u4 noalloc", sms * per, c, v, z, nnz, out);
    run<4, true, 2>("gather u4 cg", sms * per, c, v, z, nnz, out);
    run<4, true, 3>("gather u4 evict1st", sms * per, c, v, z, nnz, out);
  }
  return 0;
}
