// Small device utilities: buffers, transposes, deterministic partial reduction.
#include "ipt_internal.cuh"

namespace iptb {

std::atomic<int64_t> g_launches{0};

void DevBuf::alloc(size_t n, bool zero) {
  release();
  if (n == 0) n = 1;
  IPT_CUDA(cudaMalloc(&p, n * sizeof(double)));
  count = n;
  if (zero) {
    // The library stream is non-blocking w.r.t. the legacy stream: finish the memset
    // before any copy or kernel on the library stream can touch the buffer.
    IPT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(double), nullptr));
    IPT_CUDA(cudaStreamSynchronize(nullptr));
  }
}
void DevBuf::release() {
  if (p) cudaFree(p);
  p = nullptr;
  count = 0;
}

// 32x32 tiles through shared memory; src column-major (element (r, c) at c*ld_src + r),
// dst row-major (element (r, c) at r*ld_dst + c).
__global__ void transpose_kernel(const double* __restrict__ src, int64_t ld_src, int64_t rows,
                                 int64_t cols, double* __restrict__ dst, int64_t ld_dst,
                                 double sign) {
  __shared__ double tile[32][33];
  const int64_t r0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[c * ld_src + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < rows && c < cols) dst[r * ld_dst + c] = sign * tile[threadIdx.x][k];
  }
}

void transpose_to_rowmajor(cudaStream_t s, const double* src, int64_t ld_src, int64_t rows,
                           int64_t cols, double* dst, int64_t ld_dst, double sign) {
  if (rows == 0 || cols == 0) return;
  dim3 grid(static_cast<unsigned>(ceil_div(rows, 32)), static_cast<unsigned>(ceil_div(cols, 32)));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(src, ld_src, rows, cols, dst, ld_dst, sign);
  IPT_LAUNCH_CHECK();
  count_launch();
}

void fill_zero(cudaStream_t s, double* p, size_t count) {
  IPT_CUDA(cudaMemsetAsync(p, 0, count * sizeof(double), s));
}

__global__ void scale_copy_kernel(const double* __restrict__ src, double* __restrict__ dst, size_t n,
                                  double f) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = f * src[i];
}
void scale_copy(cudaStream_t s, const double* src, double* dst, size_t count, double factor) {
  if (count == 0) return;
  const unsigned grid = static_cast<unsigned>(std::min<size_t>(ceil_div(count, 256), 148 * 16));
  scale_copy_kernel<<<grid, 256, 0, s>>>(src, dst, count, factor);
  IPT_LAUNCH_CHECK();
  count_launch();
}

// Sum the per-CTA partials in a fixed order (thread t takes t, t+512, ...; then
// the fixed block tree), so the reduced scalars are run-to-run identical.
__global__ void reduce_partials_kernel(const double* __restrict__ partials, int64_t count,
                                       double* __restrict__ out4, const LoopState* state) {
  if (state != nullptr && state->done) return;
  __shared__ double red[16][4];
  double v[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    v[0] += partials[4 * i + 0];
    v[1] += partials[4 * i + 1];
    v[2] += partials[4 * i + 2];
    v[3] = nan_max(v[3], partials[4 * i + 3]);
  }
  block_reduce4<16>(v, red);
  if (threadIdx.x == 0) {
    out4[0] = v[0];
    out4[1] = v[1];
    out4[2] = v[2];
    out4[3] = v[3];
  }
}

void reduce_partials(cudaStream_t s, const double* partials, int64_t count, double* out4,
                     const LoopState* state) {
  reduce_partials_kernel<<<1, 512, 0, s>>>(partials, count, out4, state);
  IPT_LAUNCH_CHECK();
  count_launch();
}

}  // namespace iptb
