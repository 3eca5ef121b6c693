// Anderson-accelerated single pair of the drop-in API (contract: include/ipt/anderson.hpp;
// reference semantics: proj/include/ipt/anderson.hpp, solve_single_accelerated).
//
// AndersonState is the host mixing step (it takes and returns host vectors). The solve
// itself runs on the B200: real problems entirely on the device (the fused kMvAccel map +
// device Gram-Schmidt of ipt_single.cu, via ipt::b200::solve_single_accelerated); complex
// problems mix on the host with each product taken against the device-resident operator
// (kernels::matvec keeps Delta on the device between passes).
#include "ipt/anderson.hpp"

#include <algorithm>
#include <cmath>

#include "ipt/kernels.hpp"
#include "ipt/partition.hpp"

namespace ipt {

namespace {

cplx dot(const cvec& a, const cvec& b) {  // a^H b
    cplx s{};
    for (std::size_t t = 0; t < a.size(); ++t) s += std::conj(a[t]) * b[t];
    return s;
}

// min_gamma |rhs - D gamma|_2 for the columns D[0..h): modified Gram-Schmidt with one
// reorthogonalisation sweep, then R gamma = Q^H rhs. False when a column falls below
// 1e-13 |D|_F after orthogonalisation (numerically dependent history).
bool lsq_qr(const std::vector<cvec>& D, const cvec& rhs, cvec& gamma) {
    const std::size_t h = D.size();
    double fro2 = 0.0;
    for (const cvec& c : D)
        for (const cplx& v : c) fro2 += std::norm(v);
    const double floor = 1e-13 * std::sqrt(fro2);
    std::vector<cvec> Q;
    Q.reserve(h);
    std::vector<cplx> R(h * h, cplx{});  // upper triangle, row-major
    for (std::size_t j = 0; j < h; ++j) {
        cvec v = D[j];
        for (int sweep = 0; sweep < 2; ++sweep)
            for (std::size_t i = 0; i < j; ++i) {
                const cplx c = dot(Q[i], v);
                R[i * h + j] += c;
                for (std::size_t t = 0; t < v.size(); ++t) v[t] -= c * Q[i][t];
            }
        const double nv = kernels::nrm2(v);
        if (!(nv > floor)) return false;
        R[j * h + j] = nv;
        for (cplx& x : v) x /= nv;
        Q.push_back(std::move(v));
    }
    gamma.assign(h, cplx{});
    for (std::size_t i = h; i-- > 0;) {
        cplx s = dot(Q[i], rhs);
        for (std::size_t j = i + 1; j < h; ++j) s -= R[i * h + j] * gamma[j];
        gamma[i] = s / R[i * h + i];
    }
    return true;
}

// Tikhonov fallback: (D^H D + lambda I) gamma = D^H rhs, lambda = factor * max_i |(D^H D)_ii|,
// by Gaussian elimination with partial pivoting (h <= memory, a handful of unknowns).
bool lsq_tikhonov(const std::vector<cvec>& D, const cvec& rhs, double factor, cvec& gamma) {
    const std::size_t h = D.size();
    std::vector<cplx> A(h * h);
    cvec b(h);
    double dmax = 0.0;
    for (std::size_t i = 0; i < h; ++i) {
        for (std::size_t j = 0; j < h; ++j) A[i * h + j] = dot(D[i], D[j]);
        dmax = std::max(dmax, std::abs(A[i * h + i]));
        b[i] = dot(D[i], rhs);
    }
    for (std::size_t i = 0; i < h; ++i) A[i * h + i] += factor * dmax;
    for (std::size_t k = 0; k < h; ++k) {
        std::size_t piv = k;
        for (std::size_t i = k + 1; i < h; ++i)
            if (std::abs(A[i * h + k]) > std::abs(A[piv * h + k])) piv = i;
        if (A[piv * h + k] == cplx{}) return false;
        if (piv != k) {
            for (std::size_t j = 0; j < h; ++j) std::swap(A[k * h + j], A[piv * h + j]);
            std::swap(b[k], b[piv]);
        }
        for (std::size_t i = k + 1; i < h; ++i) {
            const cplx l = A[i * h + k] / A[k * h + k];
            for (std::size_t j = k; j < h; ++j) A[i * h + j] -= l * A[k * h + j];
            b[i] -= l * b[k];
        }
    }
    gamma.assign(h, cplx{});
    for (std::size_t i = h; i-- > 0;) {
        cplx s = b[i];
        for (std::size_t j = i + 1; j < h; ++j) s -= A[i * h + j] * gamma[j];
        gamma[i] = s / A[i * h + i];
        if (!std::isfinite(gamma[i].real()) || !std::isfinite(gamma[i].imag())) return false;
    }
    return true;
}

}  // namespace

AndersonState::AndersonState(int memory, std::size_t anchor, double regularization)
    : depth_(memory), pin_(anchor), tikhonov_(regularization) {
    if (memory < 0) throw std::invalid_argument("AndersonState: memory must be >= 0");
    ring_.resize(static_cast<std::size_t>(memory));
}

void AndersonState::reset() {
    head_ = count_ = 0;
    rising_ = 0;
    last_res_norm_ = -1.0;
}

cvec AndersonState::step(const cvec& z, const cvec& fz) {
    const std::size_t n = z.size();
    cvec res(n);
    for (std::size_t t = 0; t < n; ++t) res[t] = fz[t] - z[t];
    const double rn = kernels::nrm2(res);
    // three growing fixed-point residuals in a row: the history points across a basin
    // boundary, start it over
    if (last_res_norm_ >= 0.0 && rn > last_res_norm_) {
        if (++rising_ >= 3) {
            head_ = count_ = 0;
            rising_ = 0;
        }
    } else {
        rising_ = 0;
    }
    last_res_norm_ = rn;

    const std::size_t h = count_;
    auto slot = [this](std::size_t k) -> Pair& { return ring_[(head_ + k) % ring_.size()]; };
    auto remember = [&](cvec img, cvec r) {
        if (depth_ == 0) return;
        if (count_ < ring_.size()) {
            slot(count_) = Pair{std::move(img), std::move(r)};
            ++count_;
        } else {  // full: overwrite the oldest
            ring_[head_] = Pair{std::move(img), std::move(r)};
            head_ = (head_ + 1) % ring_.size();
        }
    };
    if (depth_ == 0 || h == 0) {
        mix_.assign(1, cplx(1.0));
        remember(fz, std::move(res));
        return fz;
    }

    // D_j = res_{j+1} - res_j over the history extended by the current pair
    std::vector<cvec> D(h, cvec(n));
    for (std::size_t j = 0; j < h; ++j) {
        const cvec& ra = slot(j).res;
        const cvec& rb = j + 1 < h ? slot(j + 1).res : res;
        for (std::size_t t = 0; t < n; ++t) D[j][t] = rb[t] - ra[t];
    }
    cvec gamma;
    const bool solved = lsq_qr(D, res, gamma) || lsq_tikhonov(D, res, tikhonov_ > 0.0 ? tikhonov_ : 1e-12, gamma);

    cvec next;
    if (!solved) {
        mix_.assign(1, cplx(1.0));
        next = fz;
    } else {
        // affine weights of the images: g_0, g_j - g_{j-1}, 1 - g_{h-1}
        mix_.resize(h + 1);
        mix_[0] = gamma[0];
        for (std::size_t j = 1; j < h; ++j) mix_[j] = gamma[j] - gamma[j - 1];
        mix_[h] = cplx(1.0) - gamma[h - 1];
        next.assign(n, cplx{});
        for (std::size_t j = 0; j <= h; ++j) {
            const cvec& img = j < h ? slot(j).img : fz;
            for (std::size_t t = 0; t < n; ++t) next[t] += mix_[j] * img[t];
        }
    }
    // the chart coordinate: exact in exact arithmetic, re-pinned against rounding drift
    const cplx za = next[pin_];
    if (za != cplx{} && za != cplx(1.0))
        for (cplx& v : next) v /= za;
    next[pin_] = 1.0;
    remember(fz, std::move(res));
    return next;
}

cvec anderson_step(AndersonState& state, const cvec& z, const cvec& fz) { return state.step(z, fz); }

EigenpairResult solve_single_accelerated(const Partition& p, const InverseGaps& g, std::size_t anchor,
                                         const IterationConfig& config, int memory) {
    if (!(config.tolerance > 0.0)) throw std::invalid_argument("config: tolerance must be positive");
    if (config.max_iterations <= 0) throw std::invalid_argument("config: max_iterations must be positive");
    if (p.size() != g.size()) throw std::invalid_argument("solver: partition/gaps size mismatch");
    if (anchor >= p.size()) throw std::invalid_argument("solver: anchor out of range");
    if (memory < 0) throw std::invalid_argument("AndersonState: memory must be >= 0");

    bool complex_input = false;
    for (const cplx& v : p.d) complex_input = complex_input || v.imag() != 0.0;
    const cvec* vals = nullptr;
    cvec dense_copy;
    if (p.delta.is_sparse()) {
        vals = &p.delta.values();
    } else {
        for (std::size_t t = 0; t < p.size() * p.size() && !complex_input; ++t)
            complex_input = p.delta.data()[t].imag() != 0.0;
    }
    if (vals)
        for (const cplx& v : *vals) complex_input = complex_input || v.imag() != 0.0;
    if (!complex_input && memory <= 16) return b200::solve_single_accelerated(p, g, anchor, config, memory);

    // complex (or very deep) mixing: host mixing, device products
    const std::size_t n = p.size();
    const cvec gcol = g.column(anchor);
    AndersonState mixer(memory, anchor);
    EigenpairResult r;
    r.anchor = anchor;
    r.z.assign(n, cplx{});
    r.z[anchor] = 1.0;
    cvec w(n), fz(n);
    auto residual = [&](const cplx lambda, double& rnorm, double& znorm) {
        double rs = 0.0, zs = 0.0;
        for (std::size_t j = 0; j < n; ++j) {
            rs += std::norm(p.d[j] * r.z[j] + w[j] - lambda * r.z[j]);
            zs += std::norm(r.z[j]);
        }
        rnorm = std::sqrt(rs);
        znorm = std::sqrt(zs);
    };
    bool done = false;
    for (int k = 0; k < config.max_iterations && !done; ++k) {
        kernels::matvec(p.delta, r.z.data(), w.data());
        ++r.matvec_count;
        r.iterations = k + 1;
        const cplx lambda = p.d[anchor] + w[anchor];
        double rnorm = 0.0, znorm = 0.0;
        residual(lambda, rnorm, znorm);
        if (rnorm <= config.residual_tolerance) {
            r.eigenvalue = lambda;
            r.residual = rnorm / znorm;
            r.status = SolveStatus::Converged;
            done = true;
            break;
        }
        const cplx wa = w[anchor];
        double diff = 0.0, base = 0.0;
        for (std::size_t j = 0; j < n; ++j) {
            fz[j] = j == anchor ? cplx(1.0) : gcol[j] * (r.z[j] * wa - w[j]);
            diff += std::norm(r.z[j] - fz[j]);
            base += std::norm(r.z[j]);
        }
        const double step = std::sqrt(diff) / std::sqrt(base);
        r.z = mixer.step(r.z, fz);
        r.final_step = step;
        if (config.record_trace) r.trace.push_back(step);
        const double zn = kernels::nrm2(r.z);
        if (!std::isfinite(zn) || zn > config.divergence_threshold) {
            r.status = SolveStatus::Diverged;
            break;
        }
    }
    if (!done) {
        kernels::matvec(p.delta, r.z.data(), w.data());
        ++r.matvec_count;
        r.eigenvalue = p.d[anchor] + w[anchor];
        double rnorm = 0.0, znorm = 0.0;
        residual(r.eigenvalue, rnorm, znorm);
        r.residual = rnorm / znorm;
    }
    return r;
}

}  // namespace ipt
