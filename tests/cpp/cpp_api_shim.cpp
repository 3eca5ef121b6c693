// Test shim: the C++ drop-in API (include/ipt/*.hpp) behind a few extern "C" calls on
// interleaved complex arrays, so tests/parity_fuzz.py can drive the reference's own entry
// points -- ComplexMatrix carriers, Partition, build_gaps, ipt::solve_full / solve_single /
// solve_single_continuation / kernels::matvec / kernels::matmul, ipt::b200::set_devices --
// on the same random inputs it gives the Python mirror and the reference build.
// Test infrastructure (built into paper_2012_14702_b200/_build), not part of the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ipt/kernels.hpp"
#include "ipt/partition.hpp"
#include "ipt/solver.hpp"

namespace {

thread_local std::string g_err;

ipt::ComplexMatrix dense_from(const double* v, std::size_t n) {
    ipt::cvec c(n * n);
    std::memcpy(c.data(), v, sizeof(ipt::cplx) * n * n);
    return ipt::ComplexMatrix::dense(n, n, std::move(c));
}

// M = diag(d) + Delta, Delta dense (csr = 0) or built from its nonzeros as CSR (csr = 1)
ipt::Partition make_partition(int64_t n, const double* d, const double* delta, int csr) {
    const std::size_t m = static_cast<std::size_t>(n);
    if (!csr) {
        ipt::ComplexMatrix a = dense_from(delta, m);
        for (std::size_t i = 0; i < m; ++i) a.at(i, i) = ipt::cplx(d[2 * i], d[2 * i + 1]);
        return ipt::partition(a);
    }
    std::vector<ipt::Triplet> t;
    for (std::size_t i = 0; i < m; ++i) {
        t.push_back({i, i, ipt::cplx(d[2 * i], d[2 * i + 1])});
        for (std::size_t j = 0; j < m; ++j) {
            if (i == j) continue;
            const ipt::cplx v(delta[2 * (i * m + j)], delta[2 * (i * m + j) + 1]);
            if (v != ipt::cplx{}) t.push_back({i, j, v});
        }
    }
    return ipt::partition(ipt::ComplexMatrix::sparse_from_triplets(m, m, std::move(t)));
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

void set_devices(int ndev, const int* devs) {
    ipt::b200::set_devices(ndev > 0 ? std::vector<int>(devs, devs + ndev) : std::vector<int>{});
}

}  // namespace

extern "C" {

const char* shim_last_error() { return g_err.c_str(); }

// out_stats: iterations, status, final_step, residual, sigma_min
int shim_solve_full(int64_t n, const double* d, const double* delta, int csr, double tol, int max_iter,
                    int ndev, const int* devs, double* z_out, double* lam_out, double* stats) {
    return guarded([&] {
        set_devices(ndev, devs);
        const ipt::Partition p = make_partition(n, d, delta, csr);
        ipt::IterationConfig cfg;
        cfg.tolerance = tol;
        cfg.max_iterations = max_iter;
        const ipt::SpectrumResult r = ipt::solve_full(p, ipt::build_gaps(p), cfg);
        set_devices(0, nullptr);
        std::memcpy(z_out, r.Z.data(), sizeof(ipt::cplx) * r.Z.rows() * r.Z.cols());
        std::memcpy(lam_out, r.eigenvalues.data(), sizeof(ipt::cplx) * r.eigenvalues.size());
        stats[0] = r.iterations;
        stats[1] = static_cast<int>(r.status);
        stats[2] = r.final_step;
        stats[3] = r.residual_frobenius;
        stats[4] = r.min_singular_value_estimate;
    });
}

// mode 0 plain, 1 continuation (alpha); repeat > 1 calls it again on the same Partition
// (the device-resident problem) and returns the last result
int shim_solve_single(int64_t n, const double* d, const double* delta, int csr, int64_t anchor, double tol,
                      int max_iter, int mode, double alpha, int repeat, int ndev, const int* devs, double* z_out,
                      double* lam_out, double* stats) {
    return guarded([&] {
        set_devices(ndev, devs);
        const ipt::Partition p = make_partition(n, d, delta, csr);
        const ipt::InverseGaps g = ipt::build_gaps(p);
        ipt::IterationConfig cfg;
        cfg.tolerance = tol;
        cfg.max_iterations = max_iter;
        ipt::EigenpairResult r;
        for (int k = 0; k < std::max(1, repeat); ++k)
            r = mode == 1 ? ipt::solve_single_continuation(p, g, static_cast<std::size_t>(anchor), cfg, alpha)
                          : ipt::solve_single(p, g, static_cast<std::size_t>(anchor), cfg);
        set_devices(0, nullptr);
        std::memcpy(z_out, r.z.data(), sizeof(ipt::cplx) * r.z.size());
        lam_out[0] = r.eigenvalue.real();
        lam_out[1] = r.eigenvalue.imag();
        stats[0] = r.iterations;
        stats[1] = static_cast<int>(r.status);
        stats[2] = r.final_step;
        stats[3] = r.residual;
    });
}

int shim_matvec(int64_t n, const double* a, int csr, const double* x, double* y) {
    return guarded([&] {
        const std::size_t m = static_cast<std::size_t>(n);
        ipt::ComplexMatrix A = dense_from(a, m);
        if (csr) A = A.to_sparse();
        ipt::cvec xv(m), yv(m);
        std::memcpy(xv.data(), x, sizeof(ipt::cplx) * m);
        ipt::kernels::matvec(A, xv.data(), yv.data());
        std::memcpy(y, yv.data(), sizeof(ipt::cplx) * m);
    });
}

int shim_matmul(int64_t n, const double* a, const double* b, double* c) {
    return guarded([&] {
        const std::size_t m = static_cast<std::size_t>(n);
        const ipt::ComplexMatrix A = dense_from(a, m), B = dense_from(b, m);
        ipt::ComplexMatrix C = ipt::ComplexMatrix::dense(m, m);
        ipt::kernels::matmul(A, B, C);
        std::memcpy(c, C.data(), sizeof(ipt::cplx) * m * m);
    });
}

}  // extern "C"
