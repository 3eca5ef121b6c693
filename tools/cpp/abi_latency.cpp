// Phase breakdown of one C-ABI solve_full at small N (device events from ipt_stats + host wall).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ipt_cuda.h"

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? std::atoll(argv[1]) : 1024;
  std::vector<double> d(n), a(n * n), z(n * n), lam(n);
  for (int64_t i = 0; i < n; ++i) {
    d[i] = double(i + 1);
    for (int64_t j = 0; j < n; ++j) a[i * n + j] = i == j ? 0.0 : 0.01 * std::sin(1.0 + i * 7 + j * 3);
  }
  ipt_ctx* ctx = nullptr;
  if (ipt_ctx_create(0, &ctx) != IPT_OK) return 1;
  ipt_params prm;
  ipt_default_params(&prm);
  for (int rep = 0; rep < 4; ++rep) {
    ipt_stats st{};
    const double t0 = now();
    const int rc = ipt_full_solve(ctx, n, d.data(), nullptr, a.data(), nullptr, nullptr, nullptr, &prm, z.data(),
                                  nullptr, lam.data(), nullptr, &st);
    const double t1 = now();
    std::printf("n=%lld rc=%d wall %.2f ms | upload %.2f loop %.2f (%d it) final %.2f sigma %.2f download %.2f ms\n",
                (long long)n, rc, 1e3 * (t1 - t0), st.ms_upload, st.ms_loop, st.iterations, st.ms_final, st.ms_sigma,
                st.ms_download);
  }
  ipt_ctx_destroy(ctx);
  return 0;
}
