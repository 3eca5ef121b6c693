// Latency of the C++ drop-in API calls at small N (what acceptance criterion 9 measures).
#include <chrono>
#include <cstdio>

#include "ipt/kernels.hpp"
#include "ipt/solver.hpp"

using namespace ipt;
static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main(int argc, char** argv) {
  const std::size_t n = argc > 1 ? std::atoi(argv[1]) : 1024;
  cvec v(n * n);
  for (std::size_t i = 0; i < n; ++i)
    for (std::size_t j = 0; j < n; ++j) v[i * n + j] = (i == j) ? cplx(double(i + 1)) : cplx(0.01 * std::sin(1.0 + i * 7 + j * 3));
  ComplexMatrix m = ComplexMatrix::dense(n, n, v);
  const Partition p = partition(m);
  const InverseGaps g = build_gaps(p);
  ComplexMatrix c = ComplexMatrix::dense(n, n);
  kernels::matmul(p.delta, m, c);  // warm (context creation)
  for (int rep = 0; rep < 3; ++rep) {
    double t0 = now();
    kernels::matmul(p.delta, m, c);
    double t1 = now();
    SpectrumResult r = solve_full(p, g);
    double t2 = now();
    cvec x(n, cplx(1.0)), y(n);
    kernels::matvec(p.delta, x.data(), y.data());
    double t3 = now();
    std::printf("n=%zu matmul %.2f ms | solve_full %.2f ms (%d it, %ld products) | matvec %.2f ms | T_eig/T_mm per product %.2f\n",
                n, 1e3 * (t1 - t0), 1e3 * (t2 - t1), r.iterations, r.matmul_count, 1e3 * (t3 - t2),
                (t2 - t1) / (t1 - t0) / r.matmul_count);
  }
  return 0;
}
