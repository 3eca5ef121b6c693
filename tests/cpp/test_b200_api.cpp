// C++ tests of the B200 additions to the drop-in API (include/ipt/solver.hpp,
// namespace ipt::b200): the Ozaki/tcgen05 product and the max-abs stop rule through
// the C++ entry point, against the DMMA product and the reference-compatible calls.
// Built by paper_2012_14702_b200/Makefile (target cpp_tests), run on the B200 by
// tests/test_gpu_cpp_api.py.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"

#include <cmath>
#include <cstdint>
#include <cstdlib>

#include <ipt/complex_matrix.hpp>
#include <ipt/partition.hpp>
#include <ipt/solver.hpp>

namespace {

// M = diag(1..n) + eps * (symmetric uniform[-1, 1], zero diagonal), a fixed LCG stream
ipt::Partition near_diagonal(std::size_t n, double eps, std::uint64_t seed) {
    ipt::ComplexMatrix m = ipt::ComplexMatrix::dense(n, n);
    std::uint64_t x = seed;
    auto uni = [&x] {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return double(x >> 11) * 0x1p-53;
    };
    for (std::size_t i = 0; i < n; ++i) {
        m.at(i, i) = double(i + 1);
        for (std::size_t j = i + 1; j < n; ++j) {
            const double v = eps * (2.0 * uni() - 1.0);
            m.at(i, j) = v;
            m.at(j, i) = v;
        }
    }
    return ipt::partition(m);
}

double max_abs_diff(const ipt::ComplexMatrix& a, const ipt::ComplexMatrix& b) {
    double d = 0.0;
    for (std::size_t i = 0; i < a.rows(); ++i)
        for (std::size_t j = 0; j < a.cols(); ++j) d = std::fmax(d, std::abs(a.get(i, j) - b.get(i, j)));
    return d;
}

}  // namespace

TEST_CASE("b200::solve_full with the Ozaki product matches the DMMA product") {
    for (std::size_t n : {7u, 130u, 700u}) {
        const ipt::Partition p = near_diagonal(n, 0.3 / std::sqrt(double(n)), 17 + n);
        const ipt::InverseGaps g = ipt::build_gaps(p);
        ipt::IterationConfig cfg;
        cfg.tolerance = 1e-13;
        ipt::b200::FullOptions dmma, oz;
        oz.product = ipt::b200::Product::Ozaki;
        const ipt::SpectrumResult a = ipt::b200::solve_full(p, g, cfg, dmma);
        const ipt::SpectrumResult b = ipt::b200::solve_full(p, g, cfg, oz);
        CHECK(a.status == ipt::SolveStatus::Converged);
        CHECK(b.status == ipt::SolveStatus::Converged);
        CHECK(a.iterations == b.iterations);
        CHECK(max_abs_diff(a.Z, b.Z) <= 1e-13);
        for (std::size_t j = 0; j < n; ++j) {
            CHECK(std::abs(a.eigenvalues[j] - b.eigenvalues[j]) <= 1e-13 * std::abs(a.eigenvalues[j]));
            CHECK(b.Z.get(j, j) == ipt::cplx(1.0, 0.0));  // anchor entries exactly 1
        }
        CHECK(b.matmul_count == b.iterations + 1);
    }
}

TEST_CASE("b200::solve_full default options equal ipt::solve_full") {
    const ipt::Partition p = near_diagonal(300, 0.01, 5);
    const ipt::InverseGaps g = ipt::build_gaps(p);
    const ipt::SpectrumResult a = ipt::solve_full(p, g);
    const ipt::SpectrumResult b = ipt::b200::solve_full(p, g, ipt::IterationConfig{}, ipt::b200::FullOptions{});
    CHECK(a.iterations == b.iterations);
    CHECK(max_abs_diff(a.Z, b.Z) == 0.0);  // same device path, deterministic
}

TEST_CASE("b200::solve_full max-abs stop rule") {
    const ipt::Partition p = near_diagonal(256, 0.02, 9);
    const ipt::InverseGaps g = ipt::build_gaps(p);
    ipt::IterationConfig cfg;
    cfg.tolerance = 1e-12;
    ipt::b200::FullOptions o;
    o.stop_rule = ipt::b200::StopRule::MaxAbs;
    o.product = ipt::b200::Product::Ozaki;
    const ipt::SpectrumResult r = ipt::b200::solve_full(p, g, cfg, o);
    CHECK(r.status == ipt::SolveStatus::Converged);
    CHECK(r.final_step < 1e-12);  // (relative step; the rule itself stopped on max|F - Z| < tol)
}

TEST_CASE("IPT_PRODUCT=ozaki routes the drop-in ipt::solve_full to the tcgen05 product") {
    const ipt::Partition p = near_diagonal(400, 0.02, 23);
    const ipt::InverseGaps g = ipt::build_gaps(p);
    ipt::b200::FullOptions oz;
    oz.product = ipt::b200::Product::Ozaki;
    const ipt::SpectrumResult want = ipt::b200::solve_full(p, g, ipt::IterationConfig{}, oz);
    setenv("IPT_PRODUCT", "ozaki", 1);
    const ipt::SpectrumResult got = ipt::solve_full(p, g);
    unsetenv("IPT_PRODUCT");
    const ipt::SpectrumResult dmma = ipt::solve_full(p, g);
    CHECK(max_abs_diff(got.Z, want.Z) == 0.0);  // the same (deterministic) Ozaki path
    CHECK(got.iterations == want.iterations);
    CHECK(max_abs_diff(dmma.Z, want.Z) <= 1e-13);
}
