// ipt/lu.hpp over the C ABI: lu_factor / lu_solve / lu_solve_adjoint /
// lu_solve_matrix (proj/src/lu.cpp:10-104) on the device, and the 1-norm condition
// estimate (Hager's method, the reference's condition_estimate_1norm contract) driven by
// device solves.
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

// kappa_1 = |A|_1 * est(|A^{-1}|_1). The estimate is Hager's convex maximisation of
// |A^{-1} x|_1 over |x|_1 = 1 (Hager 1984; Higham's complex form): from the centroid of the
// simplex, one ascent step per round -- the subgradient A^{-H} sign(A^{-1} x) names the
// vertex e_j to move to -- until the subgradient certifies a local maximum (at most five
// rounds). Each round is one forward and one adjoint solve with the device factors.
double condition_estimate_1norm(const LuFactors& f, const ComplexMatrix& a) {
    if (f.singular) return std::numeric_limits<double>::infinity();
    const std::size_t n = f.n;
    if (a.rows() != n || a.cols() != n) throw std::invalid_argument("condition_estimate_1norm: size mismatch");
    std::vector<double> colsum(n, 0.0);
    if (a.is_dense()) {
        const cplx* v = a.data();
        for (std::size_t i = 0; i < n; ++i)
            for (std::size_t j = 0; j < n; ++j) colsum[j] += std::abs(v[i * n + j]);
    } else {
        for (std::size_t q = 0; q < a.values().size(); ++q) colsum[a.col_indices()[q]] += std::abs(a.values()[q]);
    }
    const double a_norm1 = n ? *std::max_element(colsum.begin(), colsum.end()) : 0.0;

    auto norm1 = [](const cvec& v) {
        double s = 0.0;
        for (const cplx& x : v) s += std::abs(x);
        return s;
    };
    auto unit_phase = [](cplx v) {
        const double r = std::abs(v);
        return r > 0.0 ? v / r : cplx(1.0, 0.0);
    };
    cvec x(n, cplx(1.0 / static_cast<double>(n), 0.0));
    double best = 0.0;
    for (int round = 0; round < 5; ++round) {
        const cvec y = lu_solve(f, x);
        best = std::max(best, norm1(y));
        cvec s(n);
        std::transform(y.begin(), y.end(), s.begin(), unit_phase);
        const cvec grad = lu_solve_adjoint(f, s);
        std::size_t jmax = 0;
        double gmax = -1.0, gx = 0.0;
        for (std::size_t i = 0; i < n; ++i) {
            const double gi = std::abs(grad[i]);
            if (gi > gmax) {
                gmax = gi;
                jmax = i;
            }
            gx += std::abs(grad[i] * x[i]);
        }
        if (gmax <= gx) break;  // no vertex ascends: local maximum reached
        std::fill(x.begin(), x.end(), cplx{});
        x[jmax] = 1.0;
    }
    return a_norm1 * best;
}

}  // namespace ipt
