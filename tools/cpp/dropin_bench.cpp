// Time to solution through the C++ drop-in API (include/ipt/*.hpp) with the reference's
// own phase method (proj/src/bench.cpp:50-99: T_eig = solve_full, T_mm = matmul(Delta, B),
// T_eigs = solve_single, T_mv = matvec, medians over repetitions), on BASELINE's configs:
// the caller holds std::complex ComplexMatrix carriers, so the interleaved <-> planar
// conversion at the boundary is inside every number.
//
//   dropin_bench 2   : configs[1] dense N = 8192 (T_eig, T_mm, T_eigs, T_mv)
//   dropin_bench 3   : configs[2] dense N = 32768 (T_eig; ~70 GB of host memory)
//   dropin_bench 5   : configs[4] CSR N = 2^21 (T_eigs, T_mv)
//
// Inputs come from the library's seeded generator (include/ipt_synth.h, the reference's
// Rng and draw orders). One JSON line per config on stdout.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ipt/kernels.hpp"
#include "ipt/partition.hpp"
#include "ipt/solver.hpp"
#include "ipt_synth.h"

using namespace ipt;

namespace {

double now() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

template <typename F>
double timed(F&& f) {
    const double t0 = now();
    f();
    return now() - t0;
}

double median(std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0.0 : v[v.size() / 2];
}

Partition dense_config(std::size_t n) {
    std::vector<double> d(n), delta(n * n);
    if (ipt_synth_dense_uniform(static_cast<int64_t>(n), 0.32 / std::sqrt(double(n)), 42, d.data(), delta.data()))
        std::abort();
    Partition p;
    p.d.resize(n);
    for (std::size_t i = 0; i < n; ++i) p.d[i] = d[i];
    cvec v(n * n);
    for (std::size_t t = 0; t < n * n; ++t) v[t] = delta[t];
    std::vector<double>().swap(delta);
    p.delta = ComplexMatrix::dense(n, n, std::move(v));
    return p;
}

Partition csr_config5() {
    const int64_t n = int64_t(1) << 21;
    void* h = nullptr;
    int64_t nnz = 0;
    if (ipt_synth_csr_ci_plan(n, 32, 42, &h, &nnz)) std::abort();
    std::vector<double> d(n), vals(nnz);
    std::vector<int64_t> rowptr(n + 1);
    std::vector<int32_t> cols(nnz);
    if (ipt_synth_csr_ci_fill(h, 0.01, d.data(), rowptr.data(), cols.data(), vals.data())) std::abort();
    std::vector<Triplet> t(static_cast<std::size_t>(nnz));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t q = rowptr[i]; q < rowptr[i + 1]; ++q)
            t[static_cast<std::size_t>(q)] = Triplet{std::size_t(i), std::size_t(cols[q]), cplx(vals[q], 0.0)};
    Partition p;
    p.d.assign(d.begin(), d.end());
    p.delta = ComplexMatrix::sparse_from_triplets(n, n, std::move(t));
    return p;
}

}  // namespace

int main(int argc, char** argv) {
    const int which = argc > 1 ? std::atoi(argv[1]) : 2;
    const int reps = argc > 2 ? std::atoi(argv[2]) : 3;
    IterationConfig cfg;
    if (which == 2 || which == 3) {
        const std::size_t n = which == 2 ? 8192 : 32768;
        double t0 = now();
        const Partition p = dense_config(n);
        const double t_gen = now() - t0;
        const InverseGaps g = build_gaps(p);
        cfg.tolerance = 1e-12;
        std::vector<double> te, tm, ts, tv;
        SpectrumResult full;
        EigenpairResult one;
        ComplexMatrix b, c;
        cvec x(n), y(n);
        for (std::size_t i = 0; i < n; ++i) x[i] = cplx(std::sin(0.1 * double(i)), 0.0);
        if (which == 2) {
            cvec bv(n * n);
            for (std::size_t t = 0; t < n * n; ++t) bv[t] = cplx(std::cos(1e-3 * double(t)), 0.0);
            b = ComplexMatrix::dense(n, n, std::move(bv));
        }
        {  // warm: context creation, pools
            SpectrumResult w = solve_full(dense_config(256), build_gaps(dense_config(256)), cfg);
            (void)w;
        }
        for (int r = 0; r < reps; ++r) {
            te.push_back(timed([&] { full = solve_full(p, g, cfg); }));
            if (which == 2) {
                tm.push_back(timed([&] { kernels::matmul(p.delta, b, c); }));
                ts.push_back(timed([&] { one = solve_single(p, g, 0, cfg); }));
                tv.push_back(timed([&] { kernels::matvec(p.delta, x.data(), y.data()); }));
            }
        }
        std::printf("{\"config\": %d, \"n\": %zu, \"reps\": %d, \"generate_s\": %.3f, \"T_eig_s\": %.4f, "
                    "\"iterations\": %d, \"matmul_count\": %ld, \"lambda0\": %.15f, \"residual\": %.3e",
                    which, n, reps, t_gen, median(te), full.iterations, full.matmul_count,
                    full.eigenvalues[0].real(), full.residual_frobenius);
        if (which == 2)
            std::printf(", \"T_mm_s\": %.4f, \"T_eigs_s\": %.4f, \"T_mv_s\": %.5f, \"T_eig_over_T_mm_per_product\": %.3f",
                        median(tm), median(ts), median(tv), median(te) / median(tm) / double(full.matmul_count));
        std::printf(", \"T_eig_all_s\": [");
        for (std::size_t i = 0; i < te.size(); ++i) std::printf("%s%.4f", i ? ", " : "", te[i]);
        std::printf("]}\n");
    } else if (which == 5) {
        double t0 = now();
        const Partition p = csr_config5();
        const double t_gen = now() - t0;
        const InverseGaps g = build_gaps(p, 0.0);
        cfg.tolerance = 1e-10;
        const std::size_t n = p.size();
        cvec x(n, cplx(1.0)), y(n);
        std::vector<double> ts, tv;
        EigenpairResult one;
        for (int r = 0; r < reps; ++r) {
            ts.push_back(timed([&] { one = solve_single(p, g, 0, cfg); }));
            tv.push_back(timed([&] { kernels::matvec(p.delta, x.data(), y.data()); }));
        }
        std::printf("{\"config\": 5, \"n\": %zu, \"nnz\": %zu, \"reps\": %d, \"generate_s\": %.3f, \"T_eigs_s\": %.4f, "
                    "\"T_mv_s\": %.5f, \"T_mv_first_s\": %.4f, \"iterations\": %d, \"eigenvalue\": %.15f, "
                    "\"T_eigs_all_s\": [",
                    n, p.delta.values().size(), reps, t_gen, median(ts), median(tv), tv.front(), one.iterations,
                    one.eigenvalue.real());
        for (std::size_t i = 0; i < ts.size(); ++i) std::printf("%s%.4f", i ? ", " : "", ts[i]);
        std::printf("]}\n");
    }
    return 0;
}
