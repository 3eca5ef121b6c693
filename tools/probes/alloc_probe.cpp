// Host result-carrier allocation: time to get a zero-filled std::vector<std::complex<double>>
// of 1 GB (config 2's Z) by value-initialisation, parallel first touch, and THP advice.
//   g++ -O2 -std=c++17 -pthread -o alloc_probe alloc_probe.cpp
#include <sys/mman.h>

#include <chrono>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

using cvec = std::vector<std::complex<double>>;
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

static void touch(char* c, size_t bytes, unsigned t) {
    const size_t pages = bytes / 4096, step = (pages + t - 1) / t;
    std::vector<std::thread> th;
    for (unsigned k = 0; k < t; ++k) {
        size_t b = k * step, e = std::min(pages, b + step);
        if (b < e) th.emplace_back([=] { for (size_t i = b; i < e; ++i) c[i * 4096] = 0; });
    }
    for (auto& x : th) x.join();
}

int main(int argc, char** argv) {
    const size_t n = argc > 1 ? std::atoll(argv[1]) : (size_t(1) << 26);
    std::printf("THP: "); std::fflush(stdout);
    std::system("cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag");
    for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        { cvec v(n); v[n / 2] = 1.0; }
        double t1 = now();
        { cvec v; v.reserve(n); touch(reinterpret_cast<char*>(v.data()), n * 16, 16); v.resize(n); }
        double t2 = now();
        { cvec v; v.reserve(n);
          uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + 0x1fffff) & ~uintptr_t(0x1fffff);
          madvise(reinterpret_cast<void*>(a), n * 16 - (a - reinterpret_cast<uintptr_t>(v.data())) - 0x200000, MADV_HUGEPAGE);
          v.resize(n); }
        double t3 = now();
        { cvec v; v.reserve(n);
          uintptr_t a = (reinterpret_cast<uintptr_t>(v.data()) + 0x1fffff) & ~uintptr_t(0x1fffff);
          madvise(reinterpret_cast<void*>(a), n * 16 - (a - reinterpret_cast<uintptr_t>(v.data())) - 0x200000, MADV_HUGEPAGE);
          touch(reinterpret_cast<char*>(v.data()), n * 16, 16); v.resize(n); }
        double t4 = now();
        { cvec v; v.reserve(n); touch(reinterpret_cast<char*>(v.data()), n * 16, 4); v.resize(n); }
        double t5 = now();
        std::printf("%zu entries: value-init %.1f ms | 16-thread touch + resize %.1f | THP advice + resize %.1f | THP + 16-thread touch + resize %.1f | 4-thread touch + resize %.1f\n",
                    n, 1e3 * (t1 - t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2), 1e3 * (t4 - t3), 1e3 * (t5 - t4));
    }
    return 0;
}
