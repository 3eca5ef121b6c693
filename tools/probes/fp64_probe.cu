// FP64 issue-rate probe for sm_100a: DMMA (mma.sync f64) vs DFMA throughput per SM.
// Used once to pick the GEMM datapath; results are committed under profiles/.
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_k16(double* out, int iters) {
  double acc[NACC][4];
  double a[8], b[4];
  for (int i = 0; i < 8; ++i) a[i] = 1e-9 * (threadIdx.x + i);
  for (int i = 0; i < 4; ++i) b[i] = 1e-9 * (threadIdx.x - i);
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5,%6,%7,%8,%9,%10,%11},{%12,%13,%14,%15},{%0,%1,%2,%3};\n"
        : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
        : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
          "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0; for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma_k4(double* out, int iters) {
  double acc[NACC][4];
  double a0 = 1e-9 * threadIdx.x, a1 = 2e-9 * threadIdx.x, b0 = 3e-9 * threadIdx.x;
  for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) acc[j][i] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3},{%4,%5},{%6},{%0,%1,%2,%3};\n"
        : "+d"(acc[j][0]), "+d"(acc[j][1]), "+d"(acc[j][2]), "+d"(acc[j][3])
        : "d"(a0), "d"(a1), "d"(b0));
    }
  }
  double s = 0; for (int j = 0; j < NACC; ++j) for (int i = 0; i < 4; ++i) s += acc[j][i];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double acc[NACC];
  double a = 1.0000001, b = 1e-9 * threadIdx.x;
  for (int j = 0; j < NACC; ++j) acc[j] = j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < NACC; ++j) acc[j] = fma(acc[j], a, b);
  }
  double s = 0; for (int j = 0; j < NACC; ++j) s += acc[j];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
double run(K kern, int grid, int block, int iters, double flops_per_warp_iter, const char* name) {
  double* out; cudaMalloc(&out, 8);
  kern<<<grid, block>>>(out, iters / 10);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<grid, block>>>(out, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)grid * block / 32;
  double tf = warps * iters * flops_per_warp_iter / (ms * 1e-3) / 1e12;
  printf("%-28s grid=%5d block=%4d  %8.3f ms  %7.2f TFLOP/s  err=%s\n", name, grid, block, ms, tf,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out);
  return tf;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs=%d clock=%d kHz\n", sms, clk);
  const int it = 20000;
  for (int bw : {4, 8, 16}) {
    run(dmma_k16<4>, sms, bw * 32, it, 4 * 2.0 * 16 * 8 * 16, "dmma m16n8k16 nacc4");
    run(dmma_k16<8>, sms, bw * 32, it, 8 * 2.0 * 16 * 8 * 16, "dmma m16n8k16 nacc8");
    run(dmma_k4<8>, sms, bw * 32, it * 4, 8 * 2.0 * 16 * 8 * 4, "dmma m16n8k4 nacc8");
  }
  for (int bw : {8, 16, 32})
    run(dfma_loop<16>, sms * 2, bw * 32, it * 8, 16 * 2.0 * 32, "dfma nacc16");
  // latency: one warp, one accumulator
  run(dmma_k16<1>, 1, 32, it, 2.0 * 16 * 8 * 16, "dmma k16 latency-bound");
  return 0;
}
