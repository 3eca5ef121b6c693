// Shared glue of the C++ drop-in API: per-thread device context, C-ABI error
// mapping to the reference's exception types, and the one-time layout
// conversion std::complex (interleaved) <-> planar re / im at the boundary.
#pragma once

#include <atomic>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <memory>
#include <utility>
#include <stdexcept>
#include <string>
#include <thread>
#include <functional>
#include <vector>

#include "ipt/complex_matrix.hpp"
#include "ipt_cuda.h"

namespace ipt::api {

ipt_ctx* context();  // thread-local, created on first use
void set_device(int device);
// Several GPUs in this process (IPT_DEVICES, b200::set_devices): the device list, the
// calling thread's contexts joined by the in-process communicator (empty below two ranks),
// and f(rank, ctx) on one host thread per rank (rank 0 on the caller's), rethrowing the
// first rank's own error.
void set_devices(const std::vector<int>& devices);
std::vector<int> devices();
std::vector<ipt_ctx*> group_contexts();
void run_ranks(const std::vector<ipt_ctx*>& ctxs, const std::function<void(int, ipt_ctx*)>& f);

inline void check(int rc) {
    if (rc == IPT_OK) return;
    const std::string msg = ipt_last_error();
    if (rc == IPT_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

// Host scratch buffer drawn from a thread-local pool: the layout conversions at the
// boundary reuse pages that are already faulted in instead of first-touching fresh
// memory on every call (buffers above kPoolMax doubles are not retained).
// std::allocator that leaves doubles uninitialised on resize: every Vec is an output the
// device path overwrites or a conversion target filled right away, so the zero fill of
// std::vector (a single-threaded pass over fresh pages) is pure cost.
template <typename T>
struct NoInitAllocator : std::allocator<T> {
    template <typename U>
    struct rebind {
        using other = NoInitAllocator<U>;
    };
    NoInitAllocator() = default;
    template <typename U>
    NoInitAllocator(const NoInitAllocator<U>&) noexcept {}
    template <typename U>
    void construct(U* p) noexcept {
        ::new (static_cast<void*>(p)) U;
    }
    template <typename U, typename... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};

class Vec {
public:
    explicit Vec(std::size_t n = 0) { acquire(n); }
    ~Vec() { release(); }
    Vec(const Vec&) = delete;
    Vec& operator=(const Vec&) = delete;
    Vec(Vec&& o) noexcept : v_(std::move(o.v_)) {}
    Vec& operator=(Vec&& o) noexcept {
        release();
        v_ = std::move(o.v_);
        return *this;
    }
    void resize(std::size_t n) {
        release();
        acquire(n);
    }
    double* data() { return v_.data(); }
    const double* data() const { return v_.data(); }
    std::size_t size() const { return v_.size(); }
    double& operator[](std::size_t i) { return v_[i]; }
    const double& operator[](std::size_t i) const { return v_[i]; }
    double* begin() { return v_.data(); }
    double* end() { return v_.data() + v_.size(); }

private:
    static constexpr std::size_t kPoolMax = std::size_t(1) << 25;  // 256 MB
    static constexpr std::size_t kPoolSlots = 16;
    using Store = std::vector<double, NoInitAllocator<double>>;
    static std::vector<Store>& pool() {
        thread_local std::vector<Store> p;
        return p;
    }
    void acquire(std::size_t n) {
        auto& p = pool();
        std::size_t best = p.size();
        for (std::size_t i = 0; i < p.size(); ++i)
            if (p[i].capacity() >= n && (best == p.size() || p[i].capacity() < p[best].capacity())) best = i;
        if (best < p.size()) {
            v_ = std::move(p[best]);
            p.erase(p.begin() + static_cast<std::ptrdiff_t>(best));
        }
        v_.resize(n);
    }
    void release() {
        if (v_.capacity() == 0) return;
        auto& p = pool();
        if (v_.capacity() <= kPoolMax && p.size() < kPoolSlots) p.push_back(std::move(v_));
        v_ = Store();
    }
    Store v_;
};

struct Planar {
    Vec re, im;
    bool any_im = false;
    const double* im_or_null() const { return any_im ? im.data() : nullptr; }
};

// Large conversions are split over host threads (IPT_THREADS, default all cores).
unsigned host_threads();

template <typename F>
void parallel_chunks(std::size_t count, F&& f) {
    const unsigned t = count < (std::size_t(1) << 20) ? 1u : host_threads();
    if (t <= 1) {
        f(std::size_t{0}, count);
        return;
    }
    std::vector<std::thread> pool;
    const std::size_t step = (count + t - 1) / t;
    for (unsigned k = 0; k < t; ++k) {
        const std::size_t b = k * step, e = std::min(count, b + step);
        if (b < e) pool.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& th : pool) th.join();
}

// Planar copy of interleaved complex data; the imaginary plane is only materialised when
// some imaginary part is nonzero (real inputs: one pass, half the host memory).
inline Planar split(const cplx* v, std::size_t count) {
    Planar p;
    p.re.resize(count);
    std::atomic<bool> any_im{false};
    parallel_chunks(count, [&](std::size_t b, std::size_t e) {
        bool any = false;
        for (std::size_t i = b; i < e; ++i) {
            p.re[i] = v[i].real();
            any = any || v[i].imag() != 0.0;
        }
        if (any) any_im.store(true, std::memory_order_relaxed);
    });
    p.any_im = any_im.load();
    if (p.any_im) {
        p.im.resize(count);
        parallel_chunks(count, [&](std::size_t b, std::size_t e) {
            for (std::size_t i = b; i < e; ++i) p.im[i] = v[i].imag();
        });
    }
    return p;
}

inline void merge(const Vec& re, const Vec& im, cplx* out) {
    parallel_chunks(re.size(), [&](std::size_t b, std::size_t e) {
        for (std::size_t i = b; i < e; ++i) out[i] = cplx(re[i], im[i]);
    });
}

struct Csr {
    std::vector<int64_t> rowptr;
    std::vector<int32_t, NoInitAllocator<int32_t>> cols;
    Planar val;
};

// Mixes ~2048 evenly spaced entries (and the CSR structure at the same stride): catches
// contents changed through a raw pointer taken before the previous product.
inline std::uint64_t fingerprint(const cplx* v, std::size_t count, const std::size_t* idx) {
    std::uint64_t h = 0xcbf29ce484222325ull ^ count;
    auto mix = [&h](std::uint64_t w) { h ^= w + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2); };
    const std::size_t step = std::max<std::size_t>(1, count / 2048);
    auto mix_at = [&](std::size_t t) {
        std::uint64_t w[2];
        std::memcpy(w, v + t, sizeof w);
        mix(w[0]);
        mix(w[1]);
        if (idx) mix(idx[t]);
    };
    for (std::size_t t = 0; t < count; t += step) mix_at(t);
    if (count) mix_at(count - 1);
    return h;
}

// solve_single's device-resident problem (solver.cpp): freed with the resident operators.
void release_resident_single();

// The carrier's CSR (size_t columns, interleaved complex values) in the C ABI's form
// (int32 columns, planar values), converted over the host threads.
inline Csr to_csr(const ComplexMatrix& a) {
    if (a.rows() >= (std::size_t(1) << 31)) throw std::invalid_argument("csr: more than 2^31 columns");
    Csr c;
    c.rowptr.assign(a.row_offsets().begin(), a.row_offsets().end());
    const std::size_t nnz = a.col_indices().size();
    c.cols.resize(nnz);
    const std::size_t* src = a.col_indices().data();
    parallel_chunks(nnz, [&](std::size_t b, std::size_t e) {
        for (std::size_t q = b; q < e; ++q) c.cols[q] = static_cast<int32_t>(src[q]);
    });
    c.val = split(a.values().data(), a.values().size());
    return c;
}

}  // namespace ipt::api
