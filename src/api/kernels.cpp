// kernels:: of the drop-in API (proj/include/ipt/kernels.hpp). matvec / matmul /
// adjoint_matvec_dense run on the B200 through the C ABI; the *_serial oracles and
// the norms are host loops, as in the reference.
#include "ipt/kernels.hpp"

#include <cmath>
#include <cstdint>
#include <string>

#include "api_internal.hpp"

namespace ipt::kernels {

using api::Planar;
using api::Vec;

void matvec(const ComplexMatrix& a, const cplx* x, cplx* y) {
    const std::size_t m = a.rows(), n = a.cols();
    if (m == 0) return;
    const Planar px = api::split(x, n);
    Vec yr(m), yi(m);
    if (a.is_dense()) {
        const Planar pa = api::split(a.data(), m * n);
        api::check(ipt_matvec_dense(api::context(), static_cast<int64_t>(m), static_cast<int64_t>(n), pa.re.data(),
                                    pa.im_or_null(), px.re.data(), px.im_or_null(), yr.data(), yi.data()));
    } else {
        if (m != n) {
            matvec(a.to_dense(), x, y);
            return;
        }
        const api::Csr c = api::to_csr(a);
        api::check(ipt_matvec_csr(api::context(), static_cast<int64_t>(m), static_cast<int64_t>(n), c.rowptr.data(),
                                  c.cols.data(), c.val.re.data(), c.val.im_or_null(), px.re.data(),
                                  px.im_or_null(), yr.data(), yi.data()));
    }
    for (std::size_t i = 0; i < m; ++i) y[i] = cplx(yr[i], yi[i]);
}

void matvec_serial(const ComplexMatrix& a, const cplx* x, cplx* y) {
    for (std::size_t i = 0; i < a.rows(); ++i) {
        cplx s{};
        if (a.is_dense()) {
            const cplx* r = a.row(i);
            for (std::size_t j = 0; j < a.cols(); ++j) s += r[j] * x[j];
        } else {
            for (std::size_t k = a.row_offsets()[i]; k < a.row_offsets()[i + 1]; ++k)
                s += a.values()[k] * x[a.col_indices()[k]];
        }
        y[i] = s;
    }
}

void adjoint_matvec_dense(const ComplexMatrix& a, const cplx* x, cplx* y) {
    if (!a.is_dense()) throw std::invalid_argument("adjoint_matvec_dense: sparse input");
    // y = A^H x  <=>  y^T = x^T conj(A): one 1 x m by m x n product on the device.
    const std::size_t m = a.rows(), n = a.cols();
    if (n == 0) return;
    const Planar px = api::split(x, m);
    Planar pa = api::split(a.data(), m * n);
    for (double& v : pa.im) v = -v;
    Vec yr(n), yi(n);
    api::check(ipt_gemm(api::context(), 1, static_cast<int64_t>(m), static_cast<int64_t>(n), px.re.data(),
                        px.im_or_null(), pa.re.data(), pa.im_or_null(), yr.data(), yi.data()));
    for (std::size_t j = 0; j < n; ++j) y[j] = cplx(yr[j], yi[j]);
}

void matmul(const ComplexMatrix& a, const ComplexMatrix& b, ComplexMatrix& c) {
    if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
    if (!b.is_dense()) throw std::invalid_argument("matmul: right factor must be dense");
    if (!c.is_dense() || c.rows() != a.rows() || c.cols() != b.cols()) c = ComplexMatrix::dense(a.rows(), b.cols());
    const std::size_t m = a.rows(), k = a.cols(), n = b.cols();
    if (m == 0 || n == 0) return;
    ComplexMatrix densified;  // only a CSR left factor is densified
    const cplx* av = a.is_dense() ? a.data() : (densified = a.to_dense()).data();
    const Planar pa = api::split(av, m * k), pb = api::split(b.data(), k * n);
    Vec cr(m * n), ci(m * n);
    api::check(ipt_gemm(api::context(), static_cast<int64_t>(m), static_cast<int64_t>(k), static_cast<int64_t>(n),
                        pa.re.data(), pa.im_or_null(), pb.re.data(), pb.im_or_null(), cr.data(), ci.data()));
    api::merge(cr, ci, c.data());
}

void matmul_serial(const ComplexMatrix& a, const ComplexMatrix& b, ComplexMatrix& c) {
    if (a.cols() != b.rows()) throw std::invalid_argument("matmul: inner dimensions differ");
    if (!b.is_dense()) throw std::invalid_argument("matmul: right factor must be dense");
    c = ComplexMatrix::dense(a.rows(), b.cols());
    for (std::size_t i = 0; i < a.rows(); ++i) {
        cplx* ci = c.row(i);
        auto axpy = [&](cplx s, std::size_t p) {
            const cplx* bp = b.row(p);
            for (std::size_t j = 0; j < b.cols(); ++j) ci[j] += s * bp[j];
        };
        if (a.is_dense())
            for (std::size_t p = 0; p < a.cols(); ++p) axpy(a.row(i)[p], p);
        else
            for (std::size_t k = a.row_offsets()[i]; k < a.row_offsets()[i + 1]; ++k)
                axpy(a.values()[k], a.col_indices()[k]);
    }
}

double frobenius_norm(const ComplexMatrix& m) {
    const cvec* v = nullptr;
    cvec tmp;
    if (m.is_dense()) {
        tmp.assign(m.data(), m.data() + m.rows() * m.cols());
        v = &tmp;
    } else {
        v = &m.values();
    }
    double s = 0.0;
    for (const cplx& x : *v) s += std::norm(x);
    return std::sqrt(s);
}

double nrm2(const cplx* v, std::size_t n) {
    double s = 0.0;
    for (std::size_t i = 0; i < n; ++i) s += std::norm(v[i]);
    return std::sqrt(s);
}

double nrm2(const cvec& v) { return nrm2(v.data(), v.size()); }

double max_abs(const cvec& v) {
    double s = 0.0;
    for (const cplx& x : v) s = std::max(s, std::abs(x));
    return s;
}

}  // namespace ipt::kernels
