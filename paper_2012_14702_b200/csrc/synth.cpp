// Seeded synthetic inputs for BASELINE.json's configurations (include/ipt_synth.h).
// Host-side harness code: multithreaded where the draw order allows it.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "../../include/ipt_synth.h"

namespace {

// xoshiro256++ seeded by splitmix64 with Box-Muller normals: the generator the
// reference documents in proj/include/ipt/rng.hpp:13-82 (restated, same stream).
class Xoshiro {
 public:
  explicit Xoshiro(uint64_t seed) {
    uint64_t x = seed;
    for (auto& w : s_) w = splitmix(x);
  }
  static uint64_t splitmix(uint64_t& x) {
    x += 0x9e3779b97f4a7c15ull;
    uint64_t z = x;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  }
  static uint64_t stream(uint64_t seed, uint64_t id) {
    uint64_t x = seed ^ (0x5851f42d4c957f2dull * (id + 1));
    return splitmix(x);
  }
  uint64_t next() {
    const uint64_t out = rotl(s_[0] + s_[3], 23) + s_[0];
    const uint64_t t = s_[1] << 17;
    s_[2] ^= s_[0];
    s_[3] ^= s_[1];
    s_[1] ^= s_[2];
    s_[0] ^= s_[3];
    s_[2] ^= t;
    s_[3] = rotl(s_[3], 45);
    return out;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t bound) {
    const uint64_t limit = bound * (UINT64_MAX / bound);
    uint64_t r;
    do r = next();
    while (r >= limit);
    return r % bound;
  }
  double normal() {
    if (spare_ok_) {
      spare_ok_ = false;
      return spare_;
    }
    double u1;
    do u1 = uniform();
    while (u1 == 0.0);
    const double u2 = uniform();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 6.283185307179586476925286766559 * u2;
    spare_ = r * std::sin(a);
    spare_ok_ = true;
    return r * std::cos(a);
  }

 private:
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t s_[4];
  double spare_ = 0.0;
  bool spare_ok_ = false;
};

int hw_threads(int t) {
  if (t > 0) return t;
  const unsigned h = std::thread::hardware_concurrency();
  return h ? static_cast<int>(h) : 8;
}

template <typename F>
void parallel_for(int64_t n, int threads, F&& f) {
  threads = std::max(1, std::min<int>(threads, static_cast<int>(std::max<int64_t>(n, 1))));
  std::vector<std::thread> pool;
  std::exception_ptr err;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (int64_t i = t; i < n; i += threads) f(i);
      } catch (...) {
        err = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Copy the strict upper triangle onto the lower one (64x64 tiles, tile rows in parallel).
void mirror_upper(int64_t n, double* a, int threads) {
  const int64_t B = 64, nb = (n + B - 1) / B;
  parallel_for(nb, threads, [&](int64_t bi) {
    for (int64_t bj = bi; bj < nb; ++bj)
      for (int64_t i = bi * B; i < std::min(n, bi * B + B); ++i)
        for (int64_t j = std::max(i + 1, bj * B); j < std::min(n, bj * B + B); ++j) a[j * n + i] = a[i * n + j];
  });
  for (int64_t i = 0; i < n; ++i) a[i * n + i] = 0.0;
}

void radix_sort_u64(std::vector<uint64_t>& v, int bits) {
  std::vector<uint64_t> tmp(v.size());
  const int R = 16;
  for (int shift = 0; shift < bits; shift += R) {
    std::vector<size_t> cnt((1u << R) + 1, 0);
    for (uint64_t x : v) ++cnt[((x >> shift) & ((1u << R) - 1)) + 1];
    for (size_t i = 1; i < cnt.size(); ++i) cnt[i] += cnt[i - 1];
    for (uint64_t x : v) tmp[cnt[(x >> shift) & ((1u << R) - 1)]++] = x;
    v.swap(tmp);
  }
}

struct CsrPlan {
  int64_t n = 0;
  uint64_t seed = 0;
  std::vector<uint64_t> keys;  // sorted unique min*n+max
};

}  // namespace

extern "C" {

int ipt_synth_dense_uniform(int64_t n, double eps, uint64_t seed, double* d, double* delta) {
  try {
    if (n <= 0) return -1;
    for (int64_t i = 0; i < n; ++i) d[i] = static_cast<double>(i + 1);
    Xoshiro rng(Xoshiro::stream(seed, 0));
    for (int64_t i = 0; i < n; ++i) {
      double* row = delta + i * n;
      for (int64_t j = i + 1; j < n; ++j) row[j] = eps * (2.0 * rng.uniform() - 1.0);
    }
    mirror_upper(n, delta, hw_threads(0));
    return 0;
  } catch (...) {
    return -5;
  }
}

int ipt_synth_dense_normal(int64_t n, double sigma, uint64_t seed, int threads, double* d, double* delta) {
  try {
    if (n <= 0) return -1;
    {
      Xoshiro r0(Xoshiro::stream(seed, 0));
      for (int64_t i = 0; i < n; ++i) d[i] = static_cast<double>(n) * r0.uniform();
      std::sort(d, d + n);
      for (int64_t i = 0; i < n; ++i) d[i] += static_cast<double>(i);
    }
    parallel_for(n, hw_threads(threads), [&](int64_t i) {
      Xoshiro r(Xoshiro::stream(seed, static_cast<uint64_t>(i) + 1));
      double* row = delta + i * n;
      for (int64_t j = i + 1; j < n; ++j) row[j] = sigma * r.normal();
    });
    mirror_upper(n, delta, hw_threads(threads));
    return 0;
  } catch (...) {
    return -5;
  }
}

int ipt_synth_csr_ci_plan(int64_t n, int per_row, uint64_t seed, void** handle, int64_t* nnz) {
  try {
    if (n < 2 || per_row < 0 || per_row >= n) return -1;
    auto* plan = new CsrPlan();
    plan->n = n;
    plan->seed = seed;
    Xoshiro pos(Xoshiro::stream(seed, 1));
    plan->keys.reserve(static_cast<size_t>(n) * per_row);
    std::vector<uint64_t> row;
    for (int64_t i = 0; i < n; ++i) {
      row.clear();
      while (static_cast<int>(row.size()) < per_row) {
        const uint64_t j = pos.below(static_cast<uint64_t>(n));
        if (j == static_cast<uint64_t>(i)) continue;
        if (std::find(row.begin(), row.end(), j) != row.end()) continue;
        row.push_back(j);
      }
      for (uint64_t j : row) {
        const uint64_t a = std::min<uint64_t>(i, j), b = std::max<uint64_t>(i, j);
        plan->keys.push_back(a * static_cast<uint64_t>(n) + b);
      }
    }
    int bits = 1;
    while ((uint64_t(1) << bits) < static_cast<uint64_t>(n) * static_cast<uint64_t>(n)) ++bits;
    radix_sort_u64(plan->keys, bits);
    plan->keys.erase(std::unique(plan->keys.begin(), plan->keys.end()), plan->keys.end());
    *nnz = static_cast<int64_t>(plan->keys.size()) * 2;
    *handle = plan;
    return 0;
  } catch (...) {
    return -5;
  }
}

int ipt_synth_csr_ci_fill(void* handle, double sigma, double* d, int64_t* rowptr, int32_t* cols, double* vals) {
  auto* plan = static_cast<CsrPlan*>(handle);
  try {
    const int64_t n = plan->n;
    const uint64_t un = static_cast<uint64_t>(n);
    {
      Xoshiro e(Xoshiro::stream(plan->seed, 0));
      for (int64_t i = 0; i < n; ++i) d[i] = 10.0 * std::log1p(static_cast<double>(i)) + 0.5 * e.uniform();
      std::sort(d, d + n);
    }
    std::vector<int64_t> fill(n + 1, 0);
    for (uint64_t k : plan->keys) {
      ++fill[k / un + 1];
      ++fill[k % un + 1];
    }
    for (int64_t i = 0; i < n; ++i) fill[i + 1] += fill[i];
    std::memcpy(rowptr, fill.data(), sizeof(int64_t) * (n + 1));
    // Keys ascend by (min, max): row r receives its partners below r (from keys
    // (c, r)) before those above r (keys (r, c)), each ascending -> sorted rows.
    Xoshiro val(Xoshiro::stream(plan->seed, 2));
    for (uint64_t k : plan->keys) {
      const int64_t a = static_cast<int64_t>(k / un), b = static_cast<int64_t>(k % un);
      const double v = sigma * val.normal();
      cols[fill[a]] = static_cast<int32_t>(b);
      vals[fill[a]++] = v;
      cols[fill[b]] = static_cast<int32_t>(a);
      vals[fill[b]++] = v;
    }
    delete plan;
    return 0;
  } catch (...) {
    delete plan;
    return -5;
  }
}

void ipt_synth_rng_draws(uint64_t seed, uint64_t stream, int use_stream, int kind, uint64_t bound,
                         int64_t count, void* out) {
  Xoshiro rng(use_stream ? Xoshiro::stream(seed, stream) : seed);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) static_cast<uint64_t*>(out)[i] = rng.next();
    else if (kind == 1) static_cast<double*>(out)[i] = rng.uniform();
    else if (kind == 2) static_cast<double*>(out)[i] = rng.normal();
    else static_cast<uint64_t*>(out)[i] = rng.below(bound);
  }
}

}  // extern "C"
