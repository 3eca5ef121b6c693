// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the *unmodified* reference library (compiled from the
// sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libipt_ref.so). It lets pytest / bench.py drive the reference's
// own solver entry points on plain interleaved-complex buffers:
//   solve_full        proj/src/solver.cpp:180-273
//   solve_single      proj/src/solver.cpp:132-136 (run_single :49-93)
//   continuation      proj/src/solver.cpp:138-154
//   accelerated       proj/src/anderson.cpp:184-247
//   apply_map_*       proj/src/solver.cpp:122-130, :156-178
//   kernels::matmul   proj/src/kernels.cpp:175-181 ; matvec :112-140
//   sigma_min         proj/src/solver.cpp:275-297
// The max-abs stop rule of BASELINE.json is not in the reference; it is
// driven here as a loop over the reference's own apply_map_full.
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "ipt/anderson.hpp"
#include "ipt/kernels.hpp"
#include "ipt/partition.hpp"
#include "ipt/refine.hpp"
#include "ipt/rng.hpp"
#include "ipt/solver.hpp"
#include "ipt/testgen.hpp"

#define REF_API extern "C" __attribute__((visibility("default")))

using namespace ipt;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const DegenerateDiagonal& e) {
    g_err = e.what();
    return -3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return -1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

cvec to_cvec(const double* p, std::size_t n) {
  cvec v(n);
  std::memcpy(static_cast<void*>(v.data()), p, n * sizeof(cplx));
  return v;
}
void from_cvec(const cvec& v, double* out) {
  std::memcpy(out, static_cast<const void*>(v.data()), v.size() * sizeof(cplx));
}
ComplexMatrix dense_from(const double* p, std::size_t r, std::size_t c) {
  return ComplexMatrix::dense(r, c, to_cvec(p, r * c));
}
ComplexMatrix csr_from(std::size_t n, const int64_t* rowptr, const int64_t* cols, const double* vals) {
  std::vector<Triplet> t;
  t.reserve(static_cast<std::size_t>(rowptr[n]));
  for (std::size_t i = 0; i < n; ++i)
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k)
      t.push_back({i, static_cast<std::size_t>(cols[k]), cplx(vals[2 * k], vals[2 * k + 1])});
  return ComplexMatrix::sparse_from_triplets(n, n, std::move(t));
}
Partition make_partition(std::size_t n, const double* d, int is_csr, const double* dense,
                         const int64_t* rowptr, const int64_t* cols, const double* vals) {
  Partition p;
  p.d = to_cvec(d, n);
  p.delta = is_csr ? csr_from(n, rowptr, cols, vals) : dense_from(dense, n, n);
  return p;
}
IterationConfig make_cfg(double tol, int max_iter, double div_thr, int record_trace) {
  IterationConfig c;
  c.tolerance = tol;
  c.max_iterations = max_iter;
  c.divergence_threshold = div_thr;
  c.record_trace = record_trace != 0;
  return c;
}
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

REF_API const char* ref_last_error() { return g_err.c_str(); }

// stats: [0]=iterations [1]=status(0 conv,1 maxit,2 div) [2]=final_step [3]=residual_frobenius
//        [4]=sigma_min [5]=matmul_count [6]=seconds [7]=final max|dZ| (max-abs rule only)
REF_API int ref_solve_full(int64_t n, const double* d, const double* delta, double degeneracy_tol,
                           double tol, int max_iter, double div_thr, int record_trace,
                           const double* warm, double* z_out, double* lam_out, double* stats,
                           double* trace) {
  return guarded([&] {
    Partition p = make_partition(n, d, 0, delta, nullptr, nullptr, nullptr);
    const InverseGaps g = build_gaps(p, degeneracy_tol);
    const IterationConfig cfg = make_cfg(tol, max_iter, div_thr, record_trace);
    ComplexMatrix w;
    if (warm) w = dense_from(warm, n, n);
    const double t0 = now_s();
    const SpectrumResult r = solve_full(p, g, cfg, warm ? &w : nullptr);
    const double t1 = now_s();
    from_cvec(cvec(r.Z.data(), r.Z.data() + n * n), z_out);
    from_cvec(r.eigenvalues, lam_out);
    stats[0] = r.iterations;
    stats[1] = static_cast<double>(static_cast<int>(r.status));
    stats[2] = r.final_step;
    stats[3] = r.residual_frobenius;
    stats[4] = r.min_singular_value_estimate;
    stats[5] = static_cast<double>(r.matmul_count);
    stats[6] = t1 - t0;
    stats[7] = 0.0;
    if (trace)
      for (std::size_t k = 0; k < r.trace.size(); ++k) trace[k] = r.trace[k];
  });
}

// solve_full on a CSR Delta: the reference's sparse product path (kernels.cpp:88-108).
// vals interleaved complex (re, im) per nonzero.
REF_API int ref_solve_full_csr(int64_t n, const double* d, const int64_t* rowptr, const int64_t* cols,
                               const double* vals, double tol, int max_iter, double div_thr,
                               double* z_out, double* lam_out, double* stats) {
  return guarded([&] {
    Partition p = make_partition(n, d, 1, nullptr, rowptr, cols, vals);
    const InverseGaps g = build_gaps(p, 0.0);
    const IterationConfig cfg = make_cfg(tol, max_iter, div_thr, 0);
    const double t0 = now_s();
    const SpectrumResult r = solve_full(p, g, cfg, nullptr);
    const double t1 = now_s();
    from_cvec(cvec(r.Z.data(), r.Z.data() + n * n), z_out);
    from_cvec(r.eigenvalues, lam_out);
    stats[0] = r.iterations;
    stats[1] = static_cast<double>(static_cast<int>(r.status));
    stats[2] = r.final_step;
    stats[3] = r.residual_frobenius;
    stats[4] = r.min_singular_value_estimate;
    stats[5] = static_cast<double>(r.matmul_count);
    stats[6] = t1 - t0;
    stats[7] = 0.0;
  });
}

REF_API int ref_apply_map_full_csr(int64_t n, const double* d, const int64_t* rowptr, const int64_t* cols,
                                   const double* vals, const double* z, double* out) {
  return guarded([&] {
    Partition p = make_partition(n, d, 1, nullptr, rowptr, cols, vals);
    const InverseGaps g = build_gaps(p, 0.0);
    const ComplexMatrix f = apply_map_full(p, g, dense_from(z, n, n));
    from_cvec(cvec(f.data(), f.data() + n * n), out);
  });
}

// Dense LU of the reference (lu.cpp): packed factors, permutation, singular flag.
REF_API int ref_lu_factor(int64_t n, const double* a, double* lu_out, int64_t* perm_out, int* singular) {
  return guarded([&] {
    const LuFactors f = lu_factor(dense_from(a, n, n));
    from_cvec(f.lu, lu_out);
    for (int64_t i = 0; i < n; ++i) perm_out[i] = static_cast<int64_t>(f.perm[i]);
    *singular = f.singular ? 1 : 0;
  });
}

// X = A^{-1} B (lu_solve_matrix), B n x r row-major; adjoint != 0: column-wise A^{-H} b.
REF_API int ref_lu_solve(int64_t n, const double* a, int64_t r, const double* b, int adjoint, double* x_out) {
  return guarded([&] {
    const LuFactors f = lu_factor(dense_from(a, n, n));
    if (!adjoint) {
      const ComplexMatrix x = lu_solve_matrix(f, dense_from(b, n, r));
      from_cvec(cvec(x.data(), x.data() + n * r), x_out);
    } else {
      const cvec bb = to_cvec(b, n * r);
      cvec out(n * r);
      for (int64_t c = 0; c < r; ++c) {
        cvec col(n);
        for (int64_t i = 0; i < n; ++i) col[i] = bb[i * r + c];
        const cvec xc = lu_solve_adjoint(f, col);
        for (int64_t i = 0; i < n; ++i) out[i * r + c] = xc[i];
      }
      from_cvec(out, x_out);
    }
  });
}

REF_API double ref_condition_estimate(int64_t n, const double* a) {
  const ComplexMatrix m = dense_from(a, n, n);
  return condition_estimate_1norm(lu_factor(m), m);
}

// Max-abs stop rule (BASELINE.json configs): Z_{k+1} = apply_map_full(Z_k) until
// max|Z_{k+1}-Z_k| < tol, divergence tested first on |Z_{k+1}|_F exactly as solve_full
// does; then the reference's closing product for Lambda and |MZ-ZL|_F.
REF_API int ref_solve_full_maxabs(int64_t n, const double* d, const double* delta,
                                  double tol, int max_iter, double div_thr, double* z_out,
                                  double* lam_out, double* stats, double* trace) {
  return guarded([&] {
    Partition p = make_partition(n, d, 0, delta, nullptr, nullptr, nullptr);
    const InverseGaps g = build_gaps(p, 0.0);
    const std::size_t N = static_cast<std::size_t>(n);
    ComplexMatrix z = ComplexMatrix::identity(N);
    int it = 0, status = 1;
    double step = 0.0, mx = 0.0;
    const double t0 = now_s();
    for (int k = 0; k < max_iter; ++k) {
      ComplexMatrix f = apply_map_full(p, g, z);
      double diff2 = 0.0, cur2 = 0.0, new2 = 0.0;
      mx = 0.0;
      for (std::size_t t = 0; t < N * N; ++t) {
        const cplx a = f.data()[t], b = z.data()[t];
        diff2 += std::norm(a - b);
        cur2 += std::norm(b);
        new2 += std::norm(a);
        mx = std::max(mx, std::abs(a - b));
      }
      step = std::sqrt(diff2) / std::sqrt(cur2);
      z = std::move(f);
      it = k + 1;
      if (trace) trace[k] = mx;
      const double zn = std::sqrt(new2);
      if (!std::isfinite(zn) || zn > div_thr) { status = 2; break; }
      if (mx < tol) { status = 0; break; }
    }
    ComplexMatrix w = ComplexMatrix::dense(N, N);
    kernels::matmul(p.delta, z, w);
    cvec lam(N);
    for (std::size_t j = 0; j < N; ++j) lam[j] = p.d[j] + w.at(j, j);
    double r2 = 0.0;
    for (std::size_t i = 0; i < N; ++i)
      for (std::size_t j = 0; j < N; ++j)
        r2 += std::norm(p.d[i] * z.at(i, j) + w.at(i, j) - z.at(i, j) * lam[j]);
    const double t1 = now_s();
    from_cvec(cvec(z.data(), z.data() + N * N), z_out);
    from_cvec(lam, lam_out);
    stats[0] = it;
    stats[1] = status;
    stats[2] = step;
    stats[3] = std::sqrt(r2);
    stats[4] = 0.0;
    stats[5] = it + 1;
    stats[6] = t1 - t0;
    stats[7] = mx;
  });
}

// mode 0 = solve_single, 1 = solve_single_continuation(alpha), 2 = solve_single_accelerated(memory)
// stats: [0]=iterations [1]=status [2]=final_step [3]=residual [4]=matvec_count [5]=seconds
REF_API int ref_solve_single(int64_t n, const double* d, int is_csr, const double* dense,
                             const int64_t* rowptr, const int64_t* cols, const double* vals,
                             double degeneracy_tol, int64_t anchor, double tol, int max_iter,
                             double div_thr, double residual_tol, int record_trace, int mode,
                             double alpha, int memory, const double* warm, double* z_out,
                             double* lam_out, double* stats, double* trace) {
  return guarded([&] {
    Partition p = make_partition(n, d, is_csr, dense, rowptr, cols, vals);
    const InverseGaps g = build_gaps(p, degeneracy_tol);
    IterationConfig cfg = make_cfg(tol, max_iter, div_thr, record_trace);
    cfg.residual_tolerance = residual_tol;
    cvec w;
    if (warm) w = to_cvec(warm, n);
    const double t0 = now_s();
    EigenpairResult r;
    if (mode == 0)
      r = solve_single(p, g, anchor, cfg, warm ? &w : nullptr);
    else if (mode == 1)
      r = solve_single_continuation(p, g, anchor, cfg, alpha);
    else
      r = solve_single_accelerated(p, g, anchor, cfg, memory);
    const double t1 = now_s();
    from_cvec(r.z, z_out);
    lam_out[0] = r.eigenvalue.real();
    lam_out[1] = r.eigenvalue.imag();
    stats[0] = r.iterations;
    stats[1] = static_cast<double>(static_cast<int>(r.status));
    stats[2] = r.final_step;
    stats[3] = r.residual;
    stats[4] = static_cast<double>(r.matvec_count);
    stats[5] = t1 - t0;
    if (trace)
      for (std::size_t k = 0; k < r.trace.size(); ++k) trace[k] = r.trace[k];
  });
}

// solve_single for several anchors on one partition (column route of SURVEY §8c):
// z_out is count x n (row k = anchor k's eigenvector), meta count x 4 =
// {iterations, status, Re lambda, Im lambda}.
REF_API int ref_solve_single_multi(int64_t n, const double* d, const double* dense,
                                   const int64_t* anchors, int64_t count, double tol, int max_iter,
                                   double* z_out, double* meta) {
  return guarded([&] {
    Partition p = make_partition(n, d, 0, dense, nullptr, nullptr, nullptr);
    const InverseGaps g = build_gaps(p, -1.0);
    const IterationConfig cfg = make_cfg(tol, max_iter, 1e8, 0);
    for (int64_t k = 0; k < count; ++k) {
      const EigenpairResult r = solve_single(p, g, static_cast<std::size_t>(anchors[k]), cfg);
      from_cvec(r.z, z_out + 2 * k * n);
      meta[4 * k + 0] = r.iterations;
      meta[4 * k + 1] = static_cast<double>(static_cast<int>(r.status));
      meta[4 * k + 2] = r.eigenvalue.real();
      meta[4 * k + 3] = r.eigenvalue.imag();
    }
  });
}

REF_API int ref_apply_map_full(int64_t n, const double* d, const double* delta, const double* z,
                               double* out) {
  return guarded([&] {
    Partition p = make_partition(n, d, 0, delta, nullptr, nullptr, nullptr);
    const InverseGaps g = build_gaps(p, 0.0);
    const ComplexMatrix f = apply_map_full(p, g, dense_from(z, n, n));
    from_cvec(cvec(f.data(), f.data() + n * n), out);
  });
}

REF_API int ref_apply_map_single(int64_t n, const double* d, const double* delta, int64_t anchor,
                                 const double* z, double* out) {
  return guarded([&] {
    Partition p = make_partition(n, d, 0, delta, nullptr, nullptr, nullptr);
    const InverseGaps g = build_gaps(p, 0.0);
    from_cvec(apply_map_single(p, g, anchor, to_cvec(z, n)), out);
  });
}

// C(m x n) = A(m x k) B(k x n), all row-major complex; serial=1 uses matmul_serial.
REF_API int ref_matmul(int64_t m, int64_t k, int64_t n, const double* a, const double* b, double* c,
                       int serial) {
  return guarded([&] {
    const ComplexMatrix A = dense_from(a, m, k), B = dense_from(b, k, n);
    ComplexMatrix C = ComplexMatrix::dense(m, n);
    if (serial) kernels::matmul_serial(A, B, C); else kernels::matmul(A, B, C);
    from_cvec(cvec(C.data(), C.data() + m * n), c);
  });
}

REF_API int ref_matvec(int64_t n, int is_csr, const double* dense, const int64_t* rowptr,
                       const int64_t* cols, const double* vals, const double* x, double* y) {
  return guarded([&] {
    const ComplexMatrix A = is_csr ? csr_from(n, rowptr, cols, vals) : dense_from(dense, n, n);
    cvec xv = to_cvec(x, n), yv(n);
    kernels::matvec(A, xv.data(), yv.data());
    from_cvec(yv, y);
  });
}

REF_API double ref_sigma_min(int64_t n, const double* z, int max_iters, double tol) {
  double out = -1.0;
  guarded([&] { out = smallest_singular_value_estimate(dense_from(z, n, n), max_iters, tol); });
  return out;
}

REF_API int ref_gen_near_diagonal(int64_t n, double eps, int symmetric, uint64_t seed, double* out) {
  return guarded([&] {
    const ComplexMatrix m = gen_near_diagonal({static_cast<std::size_t>(n), eps, symmetric != 0, {}, false, seed});
    from_cvec(cvec(m.data(), m.data() + n * n), out);
  });
}

REF_API int ref_dense_eigenvalues(int64_t n, const double* m, double* vals_out) {
  return guarded([&] {
    const EigDecomp e = dense_eigensolve(dense_from(m, n, n));
    if (!e.converged) throw std::runtime_error("dense_eigensolve did not converge");
    from_cvec(e.values, vals_out);
  });
}

REF_API int ref_build_gaps(int64_t n, const double* d, double tol, int64_t* ij) {
  g_err.clear();
  try {
    Partition p;
    p.d = to_cvec(d, n);
    (void)build_gaps(p, tol);
    return 0;
  } catch (const DegenerateDiagonal& e) {
    ij[0] = static_cast<int64_t>(e.i);
    ij[1] = static_cast<int64_t>(e.j);
    g_err = e.what();
    return -3;
  }
}

// Raw draws of the reference's xoshiro256++ (rng.hpp) for pinning our generator port.
// kind 0 = next(), 1 = uniform(), 2 = normal(), 3 = below(bound)
REF_API void ref_rng_draws(uint64_t seed, uint64_t stream, int use_stream, int kind, uint64_t bound,
                           int64_t count, void* out) {
  Rng rng(use_stream ? Rng::stream_seed(seed, stream) : seed);
  for (int64_t i = 0; i < count; ++i) {
    if (kind == 0) static_cast<uint64_t*>(out)[i] = rng.next();
    else if (kind == 1) static_cast<double*>(out)[i] = rng.uniform();
    else if (kind == 2) static_cast<double*>(out)[i] = rng.normal();
    else static_cast<uint64_t*>(out)[i] = rng.below(bound);
  }
}

// The reference's CI-like sparse generator (testgen.cpp:174-194) as CSR arrays (partition
// applied: d = diagonal, delta = off-diagonal). Call with rowptr == nullptr to get nnz.
REF_API int ref_gen_fci_like(int64_t n, double density, double gap_scale, uint64_t seed, int64_t* nnz_out,
                             double* d, int64_t* rowptr, int64_t* cols, double* vals) {
  return guarded([&] {
    const Partition p = partition(gen_fci_like(static_cast<std::size_t>(n), density, gap_scale, seed));
    *nnz_out = static_cast<int64_t>(p.delta.values().size());
    if (rowptr == nullptr) return;
    for (int64_t i = 0; i < n; ++i) d[i] = p.d[i].real();
    for (int64_t i = 0; i <= n; ++i) rowptr[i] = static_cast<int64_t>(p.delta.row_offsets()[i]);
    for (int64_t k = 0; k < *nnz_out; ++k) {
      cols[k] = static_cast<int64_t>(p.delta.col_indices()[k]);
      vals[k] = p.delta.values()[k].real();
    }
  });
}
