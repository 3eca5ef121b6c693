// Shared device/host helpers for the IPT hot path on sm_100a.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace iptb {

constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    throw CudaError(std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what + " at " +
                    file + ":" + std::to_string(line));
  }
}
#define IPT_CUDA(x) ::iptb::cuda_check((x), #x, __FILE__, __LINE__)
#define IPT_LAUNCH_CHECK() ::iptb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

__host__ __device__ constexpr int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
__host__ __device__ constexpr int64_t ceil_div(int64_t x, int64_t m) { return (x + m - 1) / m; }

// Per-iteration decision state of a device-resident fixed-point loop. Written
// only by the single-thread decide kernels; every other kernel of an iteration
// reads `done` first and exits, so the host can enqueue iterations ahead of
// the decision without a per-iteration round trip.
struct LoopState {
  int32_t iterations;   // number of map applications performed
  int32_t status;       // 0 converged, 1 max iterations, 2 diverged
  int32_t done;
  int32_t pad;
  double final_step;    // relative step of the last map application
  double final_max_abs; // max |F - Z| of the last map application
  double sums[4];       // last reduced {sum|F-Z|^2, sum|Z|^2, sum|F|^2, max|F-Z|}
  double scale_ak;      // continuation schedule alpha^k (single pair)
};

enum StopRule : int32_t { kStopRelFro = 0, kStopMaxAbs = 1 };
enum Status : int32_t { kConverged = 0, kMaxIterations = 1, kDiverged = 2 };

// Deterministic block reduction of 4 values: lanes combine with a fixed xor
// tree, warps in index order. v[3] is a NaN-propagating max.
__device__ __forceinline__ double nan_max(double a, double b) {
  return (a != a || b != b) ? (a + b) : (a > b ? a : b);
}

template <int NWARPS>
__device__ __forceinline__ void block_reduce4(double v[4], double (*smem)[4]) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    v[0] += __shfl_xor_sync(0xffffffffu, v[0], off);
    v[1] += __shfl_xor_sync(0xffffffffu, v[1], off);
    v[2] += __shfl_xor_sync(0xffffffffu, v[2], off);
    v[3] = nan_max(v[3], __shfl_xor_sync(0xffffffffu, v[3], off));
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    smem[warp][0] = v[0];
    smem[warp][1] = v[1];
    smem[warp][2] = v[2];
    smem[warp][3] = v[3];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = smem[0][0], b = smem[0][1], c = smem[0][2], m = smem[0][3];
#pragma unroll
    for (int w = 1; w < NWARPS; ++w) {
      a += smem[w][0];
      b += smem[w][1];
      c += smem[w][2];
      m = nan_max(m, smem[w][3]);
    }
    v[0] = a;
    v[1] = b;
    v[2] = c;
    v[3] = m;
  }
}

// Complex scalars of the complex paths: the reference's std::complex<double> arithmetic
// (products as written, scaled division like libgcc's __divdc3 for finite inputs).
struct cd {
  double re, im;
};
__device__ __forceinline__ cd cmul(cd a, cd b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ cd csub(cd a, cd b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cd cadd(cd a, cd b) { return {a.re + b.re, a.im + b.im}; }
// Scaled complex division (robust like libgcc's __divdc3 for finite inputs).
__device__ __forceinline__ cd cdiv(cd a, cd b) {
  if (b.im == 0.0) return {a.re / b.re, a.im / b.re};
  if (fabs(b.re) >= fabs(b.im)) {
    const double r = b.im / b.re, den = b.re + b.im * r;
    return {(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  }
  const double r = b.re / b.im, den = b.re * r + b.im;
  return {(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}

}  // namespace iptb
