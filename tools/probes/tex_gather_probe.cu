// Does the texture path gather faster than LDG? The CSR SpMV's z gather is bound by the
// L1TEX wavefront rate (one 128 B line per clock per SM for a fully divergent LDG,
// B300_MICROARCH.md "L1tex wavefront queue"), not by L2 or HBM. This probe times the
// same traffic as gather_probe.cu with z read (a) by LDG, (b) by tex1Dfetch<int2> from a
// linear-memory texture object, and the gather alone (indices hashed in registers).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tex_gather_probe tex_gather_probe.cu
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

template <int KIND>
__device__ __forceinline__ double gather(const double* z, cudaTextureObject_t t, int c) {
  if (KIND == 0) return __ldg(z + c);
  const int2 w = tex1Dfetch<int2>(t, c);
  return __hiloint2double(w.y, w.x);
}

template <int U, int KIND>
__global__ void __launch_bounds__(256) spmv_like(const int* __restrict__ cols, const double* __restrict__ vals,
                                                 const double* __restrict__ z, cudaTextureObject_t t, int64_t nnz,
                                                 double* out) {
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  for (; e + (U - 1) * stride < nnz; e += U * stride) {
    int c[U];
    double v[U], zz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = ld_stream_s32(cols + e + u * stride);
      v[u] = ld_stream_f64(vals + e + u * stride);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) zz[u] = gather<KIND>(z, t, c[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) s = fma(v[u], zz[u], s);
  }
  if (s == 1234.5678) out[0] = s;
}

// the gather alone: indices from a register hash, no matrix stream
template <int U, int KIND>
__global__ void __launch_bounds__(256) gather_only(const double* __restrict__ z, cudaTextureObject_t t, int64_t count,
                                                   uint32_t mask, double* out) {
  double s = 0.0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u + 12345u;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < count; e += U * stride) {
    double zz[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      h = h * 1664525u + 1013904223u;
      zz[u] = gather<KIND>(z, t, int((h >> 8) & mask));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) s += zz[u];
  }
  if (s == 1234.5678) out[0] = s;
}

template <typename F>
float time_ms(F launch) {
  launch();
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int reps = 10;
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
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
  cudaResourceDesc rd = {};
  rd.resType = cudaResourceTypeLinear;
  rd.res.linear.devPtr = z;
  rd.res.linear.desc = cudaCreateChannelDesc<int2>();
  rd.res.linear.sizeInBytes = n * 8;
  cudaTextureDesc td = {};
  td.readMode = cudaReadModeElementType;
  cudaTextureObject_t tex = 0;
  cudaError_t err = cudaCreateTextureObject(&tex, &rd, &td, nullptr);
  printf("texture object: %s\n", cudaGetErrorString(err));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per : {4, 8, 16}) {
    const int grid = sms * per;
    float ms;
    ms = time_ms([&] { spmv_like<4, 0><<<grid, 256>>>(c, v, z, tex, nnz, out); });
    printf("spmv-like LDG u4   grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { spmv_like<4, 1><<<grid, 256>>>(c, v, z, tex, nnz, out); });
    printf("spmv-like TEX u4   grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { spmv_like<8, 1><<<grid, 256>>>(c, v, z, tex, nnz, out); });
    printf("spmv-like TEX u8   grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { gather_only<8, 0><<<grid, 256>>>(z, tex, nnz, uint32_t(n - 1), out); });
    printf("gather-only LDG u8 grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { gather_only<8, 1><<<grid, 256>>>(z, tex, nnz, uint32_t(n - 1), out); });
    printf("gather-only TEX u8 grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
    // a small table (L1-resident, 4096 doubles = 32 KB): the L1TEX front-end rate without L2
    ms = time_ms([&] { gather_only<8, 0><<<grid, 256>>>(z, tex, nnz, 4095u, out); });
    printf("gather-only LDG u8 (32 KB table) grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
    ms = time_ms([&] { gather_only<8, 1><<<grid, 256>>>(z, tex, nnz, 4095u, out); });
    printf("gather-only TEX u8 (32 KB table) grid %5d  %7.3f ms  %6.1f G gathers/s\n", grid, ms, nnz / (ms * 1e-3) / 1e9);
  }
  printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
