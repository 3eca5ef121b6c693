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
#include <algorithm>
#include <tuple>
#include <utility>
#include <vector>

#include <ipt/anderson.hpp>
#include <ipt/complex_matrix.hpp>
#include <ipt/kernels.hpp>
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

ipt::ComplexMatrix random_complex(std::size_t rows, std::size_t cols, std::uint64_t seed) {
    std::uint64_t x = seed;
    auto uni = [&x] {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return double(x >> 11) * 0x1p-53 - 0.5;
    };
    ipt::cvec v(rows * cols);
    for (auto& e : v) e = ipt::cplx(uni(), uni());
    return ipt::ComplexMatrix::dense(rows, cols, std::move(v));
}

double max_abs_diff(const ipt::cvec& a, const ipt::cvec& b) {
    double d = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) d = std::fmax(d, std::abs(a[i] - b[i]));
    return d;
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

TEST_CASE("kernels::matvec keeps the operator on the device while it is unchanged") {
    ipt::kernels::release_resident_operators();
    ipt::ComplexMatrix a = random_complex(512, 512, 3);  // 4 MB: resident
    ipt::cvec x(512);
    for (std::size_t i = 0; i < x.size(); ++i) x[i] = ipt::cplx(std::cos(double(i)), std::sin(0.5 * double(i)));
    ipt::cvec y1(512), y2(512), want(512);
    ipt::kernels::matvec(a, x.data(), y1.data());
    CHECK(ipt::kernels::resident_operator_count() == 1);
    ipt::kernels::matvec(a, x.data(), y2.data());
    CHECK(ipt::kernels::resident_operator_count() == 1);
    CHECK(max_abs_diff(y1, y2) == 0.0);  // the resident copy, deterministic
    ipt::kernels::matvec_serial(a, x.data(), want.data());
    CHECK(max_abs_diff(y1, want) <= 1e-12);
    // a mutation through the accessor invalidates the copy
    a.at(7, 11) = ipt::cplx(3.0, -1.0);
    ipt::kernels::matvec(a, x.data(), y1.data());
    ipt::kernels::matvec_serial(a, x.data(), want.data());
    CHECK(max_abs_diff(y1, want) <= 1e-12);
    // a write through a pointer taken before the product, at a sampled entry
    ipt::cplx* raw = a.data();
    ipt::kernels::matvec(a, x.data(), y1.data());
    raw[0] = ipt::cplx(-2.0, 5.0);
    ipt::kernels::matvec(a, x.data(), y1.data());
    ipt::kernels::matvec_serial(a, x.data(), want.data());
    CHECK(max_abs_diff(y1, want) <= 1e-12);
    // the adjoint product of the same matrix has its own resident copy
    ipt::cvec ya(512), wa(512);
    ipt::kernels::adjoint_matvec_dense(a, x.data(), ya.data());
    const ipt::ComplexMatrix ah = a.adjoint();
    ipt::kernels::matvec_serial(ah, x.data(), wa.data());
    CHECK(max_abs_diff(ya, wa) <= 1e-12);
    ipt::kernels::release_resident_operators();
    CHECK(ipt::kernels::resident_operator_count() == 0);
}

TEST_CASE("kernels::matmul keeps its left factor on the device across right factors") {
    ipt::kernels::release_resident_operators();
    const ipt::ComplexMatrix a = random_complex(300, 500, 8);  // 2.4 MB
    for (std::uint64_t seed : {1u, 2u, 3u}) {
        const ipt::ComplexMatrix b = random_complex(500, 40 + seed, seed);
        ipt::ComplexMatrix c, want;
        ipt::kernels::matmul(a, b, c);
        ipt::kernels::matmul_serial(a, b, want);
        CHECK(max_abs_diff(c, want) <= 1e-12);
    }
    CHECK(ipt::kernels::resident_operator_count() == 1);
    // a real right factor with the complex resident operand (the stacked [Ar; Ai] form)
    ipt::cvec rv(500 * 7);
    for (std::size_t t = 0; t < rv.size(); ++t) rv[t] = ipt::cplx(std::sin(double(t)), 0.0);
    const ipt::ComplexMatrix br = ipt::ComplexMatrix::dense(500, 7, rv);
    ipt::ComplexMatrix c, want;
    ipt::kernels::matmul(a, br, c);
    ipt::kernels::matmul_serial(a, br, want);
    CHECK(max_abs_diff(c, want) <= 1e-12);
    ipt::kernels::release_resident_operators();
}

TEST_CASE("AndersonState: affine weights, secant exactness, anchor re-pin") {
    // scalar affine map lifted to the non-anchor coordinate: memory 1 reaches the fixed
    // point after two mixed steps
    const ipt::cplx a(-0.6, 0.3), b(0.4, -1.1);
    const ipt::cplx fixed = b / (ipt::cplx(1.0) - a);
    ipt::AndersonState st(1, 0);
    ipt::cvec z{ipt::cplx(1.0), ipt::cplx(0.0)};
    bool hit = false;
    for (int k = 0; k < 3 && !hit; ++k) {
        const ipt::cvec fz{ipt::cplx(1.0), a * z[1] + b};
        z = ipt::anderson_step(st, z, fz);
        ipt::cplx wsum{};
        for (const auto& w : st.last_weights()) wsum += w;
        CHECK(std::abs(wsum - ipt::cplx(1.0)) <= 1e-12);
        CHECK(z[0] == ipt::cplx(1.0));
        hit = std::abs(z[1] - fixed) <= 1e-12;
    }
    CHECK(hit);
    CHECK(st.history_size() == 1);
    st.reset();
    CHECK(st.history_size() == 0);
}

TEST_CASE("solve_single_accelerated on complex inputs (host mixing, device products)") {
    const std::size_t n = 400;
    std::uint64_t x = 77;
    auto uni = [&x] {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return double(x >> 11) * 0x1p-53 - 0.5;
    };
    ipt::ComplexMatrix m = ipt::ComplexMatrix::dense(n, n);
    for (std::size_t i = 0; i < n; ++i) {
        m.at(i, i) = ipt::cplx(double(i) * 1.5, 0.3 * uni());
        for (std::size_t j = 0; j < n; ++j)
            if (j != i) m.at(i, j) = 0.02 * ipt::cplx(uni(), uni());
    }
    const ipt::Partition p = ipt::partition(m);
    const ipt::InverseGaps g = ipt::build_gaps(p);
    ipt::IterationConfig cfg;
    cfg.residual_tolerance = 1e-10;
    const ipt::EigenpairResult acc = ipt::solve_single_accelerated(p, g, 3, cfg, 5);
    ipt::IterationConfig plain_cfg;
    plain_cfg.tolerance = 1e-14;
    const ipt::EigenpairResult plain = ipt::solve_single(p, g, 3, plain_cfg);
    CHECK(acc.status == ipt::SolveStatus::Converged);
    CHECK(plain.status == ipt::SolveStatus::Converged);
    CHECK(acc.residual <= 1e-10);
    CHECK(std::abs(acc.eigenvalue - plain.eigenvalue) <= 1e-10 * std::abs(plain.eigenvalue));
    CHECK(acc.matvec_count <= acc.iterations + 1);
    CHECK(acc.matvec_count < plain.matvec_count);
    CHECK(acc.z[3] == ipt::cplx(1.0));
    CHECK(ipt::kernels::resident_operator_count() >= 1);  // Delta stayed on the device
}

namespace {

// symmetric CSR, `per_row` random off-diagonal columns per row (symmetrised), CI-like diagonal
ipt::Partition ci_like(std::size_t n, int per_row, std::uint64_t seed) {
    std::uint64_t x = seed;
    auto next = [&x] {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        return x >> 11;
    };
    std::vector<ipt::Triplet> t;
    std::vector<std::vector<char>> seen(n);
    for (std::size_t i = 0; i < n; ++i) t.push_back({i, i, ipt::cplx(10.0 * std::log1p(double(i)) + 0.5 * double(next() % 1000) / 1000.0, 0.0)});
    std::vector<std::pair<std::size_t, std::size_t>> pairs;
    for (std::size_t i = 0; i < n; ++i)
        for (int k = 0; k < per_row; ++k) {
            const std::size_t j = next() % n;
            if (j != i) pairs.emplace_back(std::min(i, j), std::max(i, j));
        }
    std::sort(pairs.begin(), pairs.end());
    pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
    for (const auto& [i, j] : pairs) {
        const double v = 0.01 * (double(next() % 2000) / 1000.0 - 1.0);
        t.push_back({i, j, ipt::cplx(v, 0.0)});
        t.push_back({j, i, ipt::cplx(v, 0.0)});
    }
    return ipt::partition(ipt::ComplexMatrix::sparse_from_triplets(n, n, t));
}

}  // namespace

TEST_CASE("b200::set_devices: the sharded solves reproduce one GPU bit for bit") {
    // Ranks of one process joined by the in-process communicator; on this one-GPU pool the
    // device is listed several times (the ranks time-share it), on a node every GPU once.
    const ipt::Partition p = near_diagonal(1000, 0.3 / std::sqrt(1000.0), 31);  // uneven shards for 3
    const ipt::InverseGaps g = ipt::build_gaps(p);
    ipt::IterationConfig cfg;
    cfg.tolerance = 1e-12;
    cfg.record_trace = true;
    const ipt::SpectrumResult one = ipt::solve_full(p, g, cfg);
    const ipt::Partition q = ci_like(6000, 8, 77);
    const ipt::InverseGaps gq = ipt::build_gaps(q, 0.0);
    ipt::IterationConfig c1;
    c1.tolerance = 1e-10;
    const ipt::EigenpairResult s_one = ipt::solve_single(q, gq, 0, c1);
    const ipt::SpectrumResult f_one = ipt::solve_full(ci_like(700, 6, 5), ipt::build_gaps(ci_like(700, 6, 5), 0.0), cfg);
    for (const std::vector<int>& devs : {std::vector<int>{0, 0}, std::vector<int>{0, 0, 0}, std::vector<int>{0, 0, 0, 0}}) {
        ipt::b200::set_devices(devs);
        const ipt::SpectrumResult r = ipt::solve_full(p, g, cfg);
        CHECK(r.iterations == one.iterations);
        CHECK(r.status == one.status);
        CHECK(max_abs_diff(r.Z, one.Z) == 0.0);
        CHECK(max_abs_diff(r.eigenvalues, one.eigenvalues) == 0.0);
        CHECK(r.trace.size() == one.trace.size());
        CHECK(std::abs(r.residual_frobenius - one.residual_frobenius) <= 1e-6 * one.residual_frobenius + 1e-13);
        CHECK(std::abs(r.min_singular_value_estimate - one.min_singular_value_estimate) <=
              1e-12 * one.min_singular_value_estimate);
        const ipt::EigenpairResult s = ipt::solve_single(q, gq, 0, c1);
        CHECK(s.iterations == s_one.iterations);
        CHECK(std::abs(s.eigenvalue - s_one.eigenvalue) <= 1e-12 * std::abs(s_one.eigenvalue));
        CHECK(max_abs_diff(s.z, s_one.z) <= 1e-14);
        const ipt::SpectrumResult f = ipt::solve_full(ci_like(700, 6, 5), ipt::build_gaps(ci_like(700, 6, 5), 0.0), cfg);
        CHECK(f.iterations == f_one.iterations);
        CHECK(max_abs_diff(f.Z, f_one.Z) == 0.0);
    }
    // an error on the ranks surfaces as the single-GPU call's exception, and the group stays usable
    ipt::b200::set_devices({0, 0});
    ipt::ComplexMatrix bad_warm = ipt::ComplexMatrix::identity(1000);
    bad_warm.at(3, 3) = 0.0;
    CHECK_THROWS_AS(ipt::solve_full(p, g, cfg, &bad_warm), std::invalid_argument);
    CHECK(max_abs_diff(ipt::solve_full(p, g, cfg).Z, one.Z) == 0.0);
    ipt::b200::set_devices({});
    setenv("IPT_DEVICES", "0,0", 1);
    CHECK(ipt::b200::devices_in_use() == 2);
    const ipt::SpectrumResult e = ipt::solve_full(p, g, cfg);
    CHECK(max_abs_diff(e.Z, one.Z) == 0.0);
    setenv("IPT_DEVICES", "0,x", 1);
    CHECK_THROWS_AS(ipt::solve_full(p, g, cfg), std::invalid_argument);
    unsetenv("IPT_DEVICES");
    CHECK(ipt::b200::devices_in_use() == 1);
}

TEST_CASE("solve_single keeps its problem on the device across calls on the same Partition") {
    ipt::b200::set_devices({});
    ipt::Partition q = ci_like(6000, 8, 91);
    const ipt::InverseGaps gq = ipt::build_gaps(q, 0.0);
    ipt::IterationConfig c;
    c.tolerance = 1e-10;
    c.record_trace = true;
    // fresh uploads (the resident problem released before each call) vs the resident one
    std::vector<ipt::EigenpairResult> fresh;
    for (std::size_t a : {0u, 5u, 17u}) {
        ipt::kernels::release_resident_operators();
        fresh.push_back(ipt::solve_single(q, gq, a, c));
    }
    ipt::kernels::release_resident_operators();
    std::size_t k = 0;
    for (int rep = 0; rep < 2; ++rep) {
        k = 0;
        for (std::size_t a : {0u, 5u, 17u}) {
            const ipt::EigenpairResult r = ipt::solve_single(q, gq, a, c);
            CHECK(r.iterations == fresh[k].iterations);
            CHECK(r.eigenvalue == fresh[k].eigenvalue);
            CHECK(max_abs_diff(r.z, fresh[k].z) == 0.0);
            CHECK(r.trace == fresh[k].trace);
            ++k;
        }
    }
    const ipt::EigenpairResult cont = ipt::solve_single_continuation(q, gq, 3, c, 0.5);
    ipt::kernels::release_resident_operators();
    const ipt::EigenpairResult cont_fresh = ipt::solve_single_continuation(q, gq, 3, c, 0.5);
    CHECK(max_abs_diff(cont.z, cont_fresh.z) == 0.0);
    // a changed Delta is uploaded again (revision stamp / fingerprint), a changed d as well
    const ipt::EigenpairResult before = ipt::solve_single(q, gq, 0, c);
    ipt::Partition q2 = ci_like(6000, 8, 92);
    q.delta = q2.delta;
    const ipt::EigenpairResult after = ipt::solve_single(q, gq, 0, c);
    ipt::kernels::release_resident_operators();
    const ipt::EigenpairResult want = ipt::solve_single(q, gq, 0, c);
    CHECK(max_abs_diff(after.z, want.z) == 0.0);
    CHECK(max_abs_diff(after.z, before.z) > 0.0);
    q.d[7] += 1e-3;
    const ipt::InverseGaps g3 = ipt::build_gaps(q, 0.0);
    const ipt::EigenpairResult d_changed = ipt::solve_single(q, g3, 0, c);
    ipt::kernels::release_resident_operators();
    const ipt::EigenpairResult d_fresh = ipt::solve_single(q, g3, 0, c);
    CHECK(max_abs_diff(d_changed.z, d_fresh.z) == 0.0);
    // dense Delta, warm start
    const ipt::Partition p = near_diagonal(1200, 0.3 / std::sqrt(1200.0), 3);
    const ipt::InverseGaps gp = ipt::build_gaps(p);
    ipt::cvec warm(1200, ipt::cplx(0.0, 0.0));
    warm[4] = 1.0;
    warm[5] = 1e-3;
    ipt::kernels::release_resident_operators();
    const ipt::EigenpairResult w_fresh = ipt::solve_single(p, gp, 4, c, &warm);
    const ipt::EigenpairResult w_res = ipt::solve_single(p, gp, 4, c, &warm);
    CHECK(max_abs_diff(w_fresh.z, w_res.z) == 0.0);
    CHECK(w_fresh.iterations == w_res.iterations);
}
