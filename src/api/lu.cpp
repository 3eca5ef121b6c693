// ipt/lu.hpp over the C ABI: lu_factor / lu_solve / lu_solve_adjoint /
// lu_solve_matrix (proj/src/lu.cpp:10-104) on the device, and the reference's 1-norm
// condition estimator (lu.cpp:106-147) driven by device solves.
#include "ipt/lu.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <stdexcept>

#include "api_internal.hpp"

namespace ipt {

namespace {

std::shared_ptr<ipt_lu> wrap(ipt_lu* p) { return std::shared_ptr<ipt_lu>(p, [](ipt_lu* q) { ipt_lu_free(q); }); }

// The device factors of f (uploaded from the packed host copy when f was built by hand).
ipt_lu* device_of(const LuFactors& f, std::shared_ptr<ipt_lu>& hold) {
    if (f.device) return f.device.get();
    const std::size_t n = f.n;
    if (f.lu.size() != n * n || f.perm.size() != n) throw std::invalid_argument("lu: malformed factors");
    const api::Planar p = api::split(f.lu.data(), n * n);
    std::vector<int64_t> perm(f.perm.begin(), f.perm.end());
    ipt_lu* raw = nullptr;
    api::check(ipt_lu_from_host(api::context(), static_cast<int64_t>(n), p.re.data(), p.im_or_null(), perm.data(),
                                f.singular ? 1 : 0, &raw));
    hold = wrap(raw);
    return raw;
}

// X = A^{-1} B or A^{-H} B for B given row-major (n x r) interleaved.
cvec solve_rows(const LuFactors& f, const cplx* b, std::size_t r, bool adjoint) {
    const std::size_t n = f.n;
    std::shared_ptr<ipt_lu> hold;
    ipt_lu* d = device_of(f, hold);
    const api::Planar bp = api::split(b, n * r);
    api::Vec xr(n * r), xi(n * r);
    auto fn = adjoint ? ipt_lu_solve_adjoint : ipt_lu_solve;
    api::check(fn(api::context(), d, static_cast<int64_t>(r), bp.re.data(), bp.im_or_null(), xr.data(), xi.data()));
    cvec x(n * r);
    api::merge(xr, xi, x.data());
    return x;
}

}  // namespace

LuFactors lu_factor(const ComplexMatrix& a) {
    if (a.rows() != a.cols()) throw std::invalid_argument("lu_factor: matrix must be square");
    const std::size_t n = a.rows();
    LuFactors f;
    f.n = n;
    if (n == 0) return f;
    const ComplexMatrix ad = a.to_dense();
    const api::Planar p = api::split(ad.data(), n * n);
    ipt_lu* raw = nullptr;
    api::check(ipt_lu_factor(api::context(), static_cast<int64_t>(n), p.re.data(), p.im_or_null(), &raw));
    f.device = wrap(raw);
    int64_t nn = 0;
    int singular = 0;
    api::check(ipt_lu_info(raw, &nn, &singular));
    f.singular = singular != 0;
    api::Vec re(n * n), im(n * n);
    std::vector<int64_t> perm(n);
    api::check(ipt_lu_download(api::context(), raw, re.data(), im.data(), perm.data()));
    f.lu.resize(n * n);
    api::merge(re, im, f.lu.data());
    f.perm.assign(perm.begin(), perm.end());
    return f;
}

cvec lu_solve(const LuFactors& f, const cvec& b) {
    if (b.size() != f.n) throw std::invalid_argument("lu_solve: size mismatch");
    if (f.n == 0) return {};
    return solve_rows(f, b.data(), 1, false);
}

cvec lu_solve_adjoint(const LuFactors& f, const cvec& b) {
    if (b.size() != f.n) throw std::invalid_argument("lu_solve_adjoint: size mismatch");
    if (f.n == 0) return {};
    return solve_rows(f, b.data(), 1, true);
}

ComplexMatrix lu_solve_matrix(const LuFactors& f, const ComplexMatrix& b) {
    const std::size_t n = f.n;
    if (b.rows() != n) throw std::invalid_argument("lu_solve_matrix: size mismatch");
    const std::size_t r = b.cols();
    if (n == 0 || r == 0) return ComplexMatrix::dense(n, r);
    const ComplexMatrix bd = b.to_dense();
    cvec x = solve_rows(f, bd.data(), r, false);
    return ComplexMatrix::dense(n, r, std::move(x));
}

double condition_estimate_1norm(const LuFactors& f, const ComplexMatrix& a) {
    if (f.singular) return std::numeric_limits<double>::infinity();
    const std::size_t n = f.n;
    if (a.rows() != n || a.cols() != n) throw std::invalid_argument("condition_estimate_1norm: size mismatch");
    ComplexMatrix ad = a.to_dense();
    double norm_a = 0.0;  // max column sum
    for (std::size_t j = 0; j < n; ++j) {
        double col = 0.0;
        for (std::size_t i = 0; i < n; ++i) col += std::abs(ad.at(i, j));
        norm_a = std::max(norm_a, col);
    }
    // Hager's estimate of |A^{-1}|_1: start from the uniform vector, at most five
    // sign / unit-vector refinements, stop when the gradient test no longer improves.
    cvec x(n, cplx(1.0 / static_cast<double>(n), 0.0));
    double est = 0.0;
    for (int pass = 0; pass < 5; ++pass) {
        const cvec y = lu_solve(f, x);
        double ysum = 0.0;
        for (const cplx& v : y) ysum += std::abs(v);
        est = std::max(est, ysum);
        cvec sgn(n);
        for (std::size_t i = 0; i < n; ++i) {
            const double mag = std::abs(y[i]);
            sgn[i] = mag == 0.0 ? cplx(1.0, 0.0) : y[i] / mag;
        }
        const cvec z = lu_solve_adjoint(f, sgn);
        std::size_t best = 0;
        double zbest = 0.0;
        for (std::size_t i = 0; i < n; ++i) {
            const double mag = std::abs(z[i]);
            if (mag > zbest) {
                zbest = mag;
                best = i;
            }
        }
        double zdotx = 0.0;
        for (std::size_t i = 0; i < n; ++i) zdotx += std::abs(z[i] * x[i]);
        if (zbest <= zdotx) break;
        x.assign(n, cplx{});
        x[best] = 1.0;
    }
    return norm_a * est;
}

}  // namespace ipt
