// Solver entry points of the drop-in API (proj/include/ipt/solver.hpp) on the B200.
// Validation and exception behaviour follow proj/src/solver.cpp:18-45; every
// product, map application and reduction runs on the device via include/ipt_cuda.h.
#include "ipt/solver.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <future>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "api_internal.hpp"
#include "ipt/kernels.hpp"

namespace ipt {

namespace api {

namespace {
thread_local int t_device = -1;
struct CtxHolder {
    ipt_ctx* ctx = nullptr;
    int device = -1;
    ~CtxHolder() {
        if (ctx) ipt_ctx_destroy(ctx);
    }
};
thread_local CtxHolder t_ctx;
}  // namespace

void set_device(int device) { t_device = device; }

// ---- one process, several GPUs (IPT_DEVICES / b200::set_devices) -----------------------
// The column-sharded full spectrum and the row-sharded CSR single pair run with the ranks
// as contexts of this process, one host thread per rank, joined by the library's in-process
// communicator (peer copies / peer stores over NVLink between devices; collectives are
// event-ordered, so a device may also host several ranks). Each rank writes its own
// columns of Z straight into the caller's result (IPT_OUTPUT_LOCAL_COLUMNS).
namespace {
thread_local bool t_devices_set = false;
thread_local std::vector<int> t_devices;
struct GroupHolder {
    std::vector<int> devices;
    std::vector<ipt_ctx*> ctxs;
    ipt_local_group* group = nullptr;
    void reset() {
        for (ipt_ctx* c : ctxs) ipt_ctx_destroy(c);
        ctxs.clear();
        if (group) ipt_local_group_destroy(group);  // after every member context
        group = nullptr;
        devices.clear();
    }
    ~GroupHolder() { reset(); }
};
thread_local GroupHolder t_group;
}  // namespace

void set_devices(const std::vector<int>& devices) {
    t_devices = devices;
    t_devices_set = !devices.empty();  // an empty list returns to $IPT_DEVICES
}

std::vector<int> devices() {
    if (t_devices_set) return t_devices;
    std::vector<int> out;
    const char* env = std::getenv("IPT_DEVICES");
    if (env == nullptr || *env == 0) return out;
    const std::string s(env);
    if (s == "all") {
        int count = 0;
        check(ipt_device_count(&count));
        for (int d = 0; d < count; ++d) out.push_back(d);
        return out;
    }
    std::stringstream ss(s);
    std::string item;
    while (std::getline(ss, item, ',')) {
        std::size_t used = 0;
        int d = -1;
        try {
            d = std::stoi(item, &used);
        } catch (const std::exception&) {
            used = 0;
        }
        if (used == 0 || used != item.size() || d < 0)
            throw std::invalid_argument("IPT_DEVICES: expected 'all' or a comma-separated list of device indices");
        out.push_back(d);
    }
    return out;
}

std::vector<ipt_ctx*> group_contexts() {
    const std::vector<int> devs = devices();
    if (devs.size() < 2) return {};
    if (t_group.devices != devs) {
        t_group.reset();
        check(ipt_local_group_create(static_cast<int>(devs.size()), &t_group.group));
        for (std::size_t r = 0; r < devs.size(); ++r) {
            ipt_ctx* c = nullptr;
            check(ipt_ctx_create(devs[r], &c));
            t_group.ctxs.push_back(c);
            check(ipt_ctx_init_local_comm(c, t_group.group, static_cast<int>(r)));
        }
        t_group.devices = devs;
    }
    return t_group.ctxs;
}

void run_ranks(const std::vector<ipt_ctx*>& ctxs, const std::function<void(int, ipt_ctx*)>& f) {
    const std::size_t g = ctxs.size();
    std::vector<std::exception_ptr> err(g);
    std::vector<std::thread> th;
    for (std::size_t r = 1; r < g; ++r)
        th.emplace_back([&, r] {
            try {
                f(static_cast<int>(r), ctxs[r]);
            } catch (...) {
                err[r] = std::current_exception();
            }
        });
    try {
        f(0, ctxs[0]);
    } catch (...) {
        err[0] = std::current_exception();
    }
    for (auto& t : th) t.join();
    // report the rank that failed first-hand, not the ranks its abort released
    std::exception_ptr first, any;
    for (auto& e : err) {
        if (!e) continue;
        if (!any) any = e;
        try {
            std::rethrow_exception(e);
        } catch (const std::exception& x) {
            if (!first && std::string(x.what()).find("aborted") == std::string::npos) first = e;
        } catch (...) {
            if (!first) first = e;
        }
    }
    // an error aborts the in-process communicator: the next call opens a fresh group
    if (any) t_group.reset();
    if (first) std::rethrow_exception(first);
    if (any) std::rethrow_exception(any);
}

ipt_ctx* context() {
    int dev = t_device;
    if (dev < 0) {
        const char* env = std::getenv("IPT_DEVICE");
        dev = env ? std::atoi(env) : 0;
    }
    if (t_ctx.ctx == nullptr || t_ctx.device != dev) {
        if (t_ctx.ctx) {
            // device-resident operators / problems belong to this context: drop them before
            // it goes (a new context could reuse its address)
            kernels::release_resident_operators();
            ipt_ctx_destroy(t_ctx.ctx);
        }
        t_ctx.ctx = nullptr;
        check(ipt_ctx_create(dev, &t_ctx.ctx));
        t_ctx.device = dev;
    }
    return t_ctx.ctx;
}

unsigned host_threads() {
    static const unsigned t = [] {
        const char* env = std::getenv("IPT_THREADS");
        const int v = env ? std::atoi(env) : 0;
        if (v > 0) return static_cast<unsigned>(v);
        const unsigned h = std::thread::hardware_concurrency();
        return h ? h : 8u;
    }();
    return t;
}

}  // namespace api

namespace {

using api::Planar;
using api::Vec;

void validate(const IterationConfig& cfg) {
    if (!(cfg.tolerance > 0.0)) throw std::invalid_argument("config: tolerance must be positive");
    if (cfg.max_iterations <= 0) throw std::invalid_argument("config: max_iterations must be positive");
    if (!(cfg.divergence_threshold > 1.0)) throw std::invalid_argument("config: divergence_threshold must exceed 1");
}

void check_anchor(const Partition& p, const InverseGaps& g, std::size_t anchor) {
    if (p.size() != g.size()) throw std::invalid_argument("solver: partition/gaps size mismatch");
    if (p.delta.rows() != p.size() || p.delta.cols() != p.size())
        throw std::invalid_argument("solver: residual must be square of matching size");
    if (anchor >= p.size()) throw std::invalid_argument("solver: anchor out of range");
}

ipt_params to_params(const IterationConfig& cfg) {
    ipt_params prm;
    ipt_default_params(&prm);
    prm.tolerance = cfg.tolerance;
    prm.max_iterations = cfg.max_iterations;
    prm.divergence_threshold = cfg.divergence_threshold;
    prm.record_trace = cfg.record_trace ? 1 : 0;
    return prm;
}

cvec combine(const Vec& re, const Vec& im) {
    cvec out(re.size());
    api::merge(re, im, out.data());
    return out;
}

// Delta as a dense planar operator (apply_map_single and the dense full path).
Planar dense_delta(const Partition& p) {
    if (p.delta.is_dense()) return api::split(p.delta.data(), p.size() * p.size());
    const ComplexMatrix dd = p.delta.to_dense();
    return api::split(dd.data(), p.size() * p.size());
}

// solve_single's problem stays on the device between calls on the same Partition (several
// anchors of one matrix, repeated solves): Delta and d are uploaded once and each further
// call only resets the anchor, iterates and downloads z. Kept while Delta's storage,
// ComplexMatrix::revision() and a sampled content fingerprint match and d is unchanged
// (compared in full); within IPT_OPERATOR_CACHE_MB (default 16384) like the resident
// kernels:: operators, and freed with them (kernels::release_resident_operators).
struct ResidentSingle {
    const void* storage = nullptr;
    std::uint64_t revision = 0, fingerprint = 0;
    std::size_t n = 0, count = 0;
    bool sparse = false;
    ipt_ctx* ctx = nullptr;
    ipt_single_problem* prob = nullptr;
    cvec d;         // the diagonal it was opened with
    Planar dense;   // the host sources anchor rows are rebuilt from (referenced by the problem)
    api::Csr csr;
    void release() {
        if (prob) ipt_single_free(prob);
        prob = nullptr;
        storage = nullptr;
        d = cvec();
        dense = Planar();
        csr = api::Csr();
    }
    ~ResidentSingle() { release(); }
};
thread_local ResidentSingle t_single;

std::int64_t resident_budget() {
    static const std::int64_t b = [] {
        const char* e = std::getenv("IPT_OPERATOR_CACHE_MB");
        return (e ? std::atoll(e) : 16384LL) << 20;
    }();
    return b;
}

// The device-resident problem for p, opened now if need be; nullptr when it is not kept
// (small, complex Delta or d, or over the budget).
ipt_single_problem* resident_single(const Partition& p) {
    const std::size_t n = p.size();
    const bool sparse = p.delta.is_sparse();
    const std::size_t count = sparse ? p.delta.values().size() : n * n;
    const std::int64_t bytes = sparse ? std::int64_t(count) * 12 + 8 * std::int64_t(n + 1) : std::int64_t(count) * 8;
    if (bytes < (std::int64_t(1) << 20) || bytes > resident_budget()) return nullptr;
    ipt_ctx* ctx = api::context();
    const cplx* vals = sparse ? p.delta.values().data() : p.delta.data();
    const std::uint64_t rev = p.delta.revision();
    const std::uint64_t fp = api::fingerprint(vals, count, sparse ? p.delta.col_indices().data() : nullptr);
    ResidentSingle& r = t_single;
    if (r.prob && r.storage == vals && r.revision == rev && r.fingerprint == fp && r.n == n && r.count == count &&
        r.sparse == sparse && r.ctx == ctx && r.d == p.d)
        return r.prob;
    r.release();
    const Planar d = api::split(p.d.data(), n);
    if (d.any_im) return nullptr;
    ipt_single_problem* h = nullptr;
    if (sparse) {
        r.csr = api::to_csr(p.delta);
        if (r.csr.val.any_im) {
            r.csr = api::Csr();
            return nullptr;
        }
        api::check(ipt_single_upload_csr_shared(ctx, static_cast<int64_t>(n), d.re.data(), nullptr,
                                                r.csr.rowptr.data(), r.csr.cols.data(), r.csr.val.re.data(), nullptr,
                                                &h));
    } else {
        r.dense = api::split(vals, count);
        if (r.dense.any_im) {
            r.dense = Planar();
            return nullptr;
        }
        api::check(ipt_single_upload_dense(ctx, static_cast<int64_t>(n), d.re.data(), nullptr, r.dense.re.data(),
                                           nullptr, &h));
    }
    r.prob = h;
    r.storage = vals;
    r.revision = rev;
    r.fingerprint = fp;
    r.n = n;
    r.count = count;
    r.sparse = sparse;
    r.ctx = ctx;
    r.d = p.d;
    return h;
}

EigenpairResult run_single(const Partition& p, std::size_t anchor, const IterationConfig& cfg, const cvec* warm,
                           int schedule, double alpha) {
    const std::size_t n = p.size();
    Planar d;  // split only where Delta is uploaded (not for the resident problem)
    Planar w;
    if (warm) {
        if (warm->size() != n) throw std::invalid_argument("solver: warm start size mismatch");
        if ((*warm)[anchor] == cplx{}) throw std::invalid_argument("solver: warm start has zero anchor coordinate");
        w = api::split(warm->data(), n);
    }
    ipt_params prm = to_params(cfg);
    prm.schedule = schedule;
    prm.shrink_alpha = alpha;
    ipt_stats st{};
    std::vector<double> trace(cfg.record_trace ? cfg.max_iterations : 0);
    st.trace = cfg.record_trace ? trace.data() : nullptr;
    Vec zr(n), zi(n);
    const double* wre = warm ? w.re.data() : nullptr;
    const double* wim = warm ? w.im_or_null() : nullptr;
    const std::vector<ipt_ctx*> ranks = p.delta.is_sparse() ? api::group_contexts() : std::vector<ipt_ctx*>{};
    if (!ranks.empty()) {
        d = api::split(p.d.data(), n);
        // CSR rows sharded over the multi-device group; the iterate is all-gathered every
        // step (fused peer stores), so every rank ends with all of z: rank 0's is returned
        const api::Csr c = api::to_csr(p.delta);
        std::vector<ipt_stats> sts(ranks.size());
        std::vector<std::vector<double>> traces(ranks.size(), trace);
        std::vector<Vec> zrs(ranks.size()), zis(ranks.size());
        api::run_ranks(ranks, [&](int rank, ipt_ctx* ctx) {
            ipt_stats& s = sts[rank];
            s = ipt_stats{};
            s.trace = cfg.record_trace ? traces[rank].data() : nullptr;
            Vec& r_re = rank == 0 ? zr : zrs[rank];
            Vec& r_im = rank == 0 ? zi : zis[rank];
            if (rank != 0) {
                r_re.resize(n);
                r_im.resize(n);
            }
            api::check(ipt_single_solve_csr(ctx, static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                            c.rowptr.data(), c.cols.data(), c.val.re.data(), c.val.im_or_null(),
                                            static_cast<int64_t>(anchor), wre, wim, &prm, r_re.data(), r_im.data(),
                                            &s));
        });
        st = sts[0];
        trace = traces[0];
    } else if (ipt_single_problem* h = (w.any_im ? nullptr : resident_single(p))) {
        ipt_ctx* ctx = api::context();
        api::check(ipt_single_reset(ctx, h, static_cast<int64_t>(anchor), schedule == IPT_SCHEDULE_CONTINUATION ? nullptr : wre,
                                    schedule == IPT_SCHEDULE_CONTINUATION ? nullptr : wim));
        api::check(ipt_single_iterate(ctx, h, &prm, &st));
        api::check(ipt_single_finalize(ctx, h, &st));
        api::check(ipt_single_download(ctx, h, zr.data(), zi.data()));
    } else if (p.delta.is_sparse()) {
        d = api::split(p.d.data(), n);
        const api::Csr c = api::to_csr(p.delta);
        api::check(ipt_single_solve_csr(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                        c.rowptr.data(), c.cols.data(), c.val.re.data(), c.val.im_or_null(),
                                        static_cast<int64_t>(anchor), wre, wim, &prm, zr.data(), zi.data(), &st));
    } else {
        d = api::split(p.d.data(), n);
        const Planar a = api::split(p.delta.data(), n * n);
        api::check(ipt_single_solve_dense(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                          a.re.data(), a.im_or_null(), static_cast<int64_t>(anchor), wre, wim, &prm,
                                          zr.data(), zi.data(), &st));
    }
    EigenpairResult r;
    r.z = combine(zr, zi);
    r.eigenvalue = cplx(st.eigenvalue_re, st.eigenvalue_im);
    r.anchor = anchor;
    r.iterations = st.iterations;
    r.final_step = st.final_step;
    r.residual = st.residual;
    r.status = static_cast<SolveStatus>(st.status);
    r.matvec_count = static_cast<long>(st.product_count);
    if (cfg.record_trace) r.trace.assign(trace.begin(), trace.begin() + st.iterations);
    return r;
}


// solve_full with the columns sharded over the calling thread's multi-device group: every
// rank runs the same C-ABI solve on its context, writes its own columns of Z and Lambda into
// the shared result, and reports the same global scalars (all-reduced).
SpectrumResult solve_full_ranks(const Partition& p, const IterationConfig& config, ipt_params prm,
                                const ComplexMatrix* warm_dense, const Planar& warm_planar,
                                const std::vector<ipt_ctx*>& ranks) {
    const std::size_t n = p.size();
    const std::size_t g = ranks.size();
    prm.output_mode = IPT_OUTPUT_LOCAL_COLUMNS;
    std::vector<ipt_stats> sts(g);
    std::vector<std::vector<double>> traces(g, std::vector<double>(config.record_trace ? config.max_iterations : 0));
    SpectrumResult r;
    if (p.delta.is_dense()) {
        cvec zv;
        std::shared_future<void> zready = std::async(std::launch::async, [&zv, n] { zv = cvec(n * n); }).share();
        r.eigenvalues.resize(n);
        api::run_ranks(ranks, [&](int rank, ipt_ctx* c) {
            ipt_stats& st = sts[rank];
            st = ipt_stats{};
            st.trace = config.record_trace ? traces[rank].data() : nullptr;
            ipt_full_problem* h = nullptr;
            const int rc = ipt_full_solve_interleaved_start(
                c, static_cast<int64_t>(n), reinterpret_cast<const double*>(p.d.data()),
                reinterpret_cast<const double*>(p.delta.data()),
                warm_dense ? reinterpret_cast<const double*>(warm_dense->data()) : nullptr, &prm, &h, &st);
            zready.get();
            api::check(rc);
            std::unique_ptr<ipt_full_problem, void (*)(ipt_full_problem*)> hold(h, ipt_full_free);
            api::check(ipt_full_solve_interleaved_finish(c, h, &prm, reinterpret_cast<double*>(zv.data()),
                                                         reinterpret_cast<double*>(r.eigenvalues.data()), &st));
        });
        zready.get();
        r.Z = ComplexMatrix::dense(n, n, std::move(zv));
    } else {  // CSR Delta: the sparse-Delta map per rank
        const Planar d = api::split(p.d.data(), n);
        const api::Csr c = api::to_csr(p.delta);
        Vec zr(n * n), zi(n * n), lr(n), li(n);
        const double* wre = warm_dense ? warm_planar.re.data() : nullptr;
        const double* wim = warm_dense ? warm_planar.im_or_null() : nullptr;
        api::run_ranks(ranks, [&](int rank, ipt_ctx* ctx) {
            ipt_stats& st = sts[rank];
            st = ipt_stats{};
            st.trace = config.record_trace ? traces[rank].data() : nullptr;
            api::check(ipt_full_solve_csr(ctx, static_cast<int64_t>(n), d.re.data(), d.im_or_null(), c.rowptr.data(),
                                          c.cols.data(), c.val.re.data(), c.val.im_or_null(), wre, wim, &prm,
                                          zr.data(), zi.data(), lr.data(), li.data(), &st));
        });
        r.Z = ComplexMatrix::dense(n, n);
        api::merge(zr, zi, r.Z.data());
        r.eigenvalues = combine(lr, li);
    }
    const ipt_stats& st = sts[0];
    r.iterations = st.iterations;
    r.final_step = st.final_step;
    r.residual_frobenius = st.residual;
    r.min_singular_value_estimate = st.min_singular_value_estimate;
    r.status = static_cast<SolveStatus>(st.status);
    r.matmul_count = static_cast<long>(st.product_count);
    if (config.record_trace) r.trace.assign(traces[0].begin(), traces[0].begin() + st.iterations);
    return r;
}

}  // namespace

const char* to_string(SolveStatus s) {
    switch (s) {
        case SolveStatus::Converged: return "converged";
        case SolveStatus::MaxIterations: return "max_iterations";
        case SolveStatus::Diverged: return "diverged";
    }
    return "unknown";
}

cvec apply_map_single(const Partition& p, const InverseGaps& g, std::size_t anchor, const cvec& z) {
    check_anchor(p, g, anchor);
    const std::size_t n = p.size();
    if (z.size() != n) throw std::invalid_argument("apply_map_single: size mismatch");
    const Planar d = api::split(p.d.data(), n), a = dense_delta(p), zz = api::split(z.data(), n);
    Vec fr(n), fi(n);
    api::check(ipt_apply_map_single_dense(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                          a.re.data(), a.im_or_null(), static_cast<int64_t>(anchor), zz.re.data(),
                                          zz.im_or_null(), fr.data(), fi.data()));
    return combine(fr, fi);
}

EigenpairResult solve_single(const Partition& p, const InverseGaps& g, std::size_t anchor,
                             const IterationConfig& config, const cvec* warm_start) {
    validate(config);
    check_anchor(p, g, anchor);
    return run_single(p, anchor, config, warm_start, IPT_SCHEDULE_PLAIN, 0.9);
}

EigenpairResult solve_single_continuation(const Partition& p, const InverseGaps& g, std::size_t anchor,
                                          const IterationConfig& config, double shrink_alpha) {
    if (!(shrink_alpha >= 0.0 && shrink_alpha < 1.0))
        throw std::invalid_argument("continuation: shrink factor must lie in [0, 1)");
    validate(config);
    check_anchor(p, g, anchor);
    return run_single(p, anchor, config, nullptr, IPT_SCHEDULE_CONTINUATION, shrink_alpha);
}

ComplexMatrix apply_map_full(const Partition& p, const InverseGaps& g, const ComplexMatrix& Z) {
    check_anchor(p, g, 0);
    if (Z.rows() != p.size() || Z.cols() != p.size()) throw std::invalid_argument("apply_map_full: size mismatch");
    const std::size_t n = p.size();
    const ComplexMatrix zd = Z.to_dense();
    const Planar d = api::split(p.d.data(), n), zz = api::split(zd.data(), n * n);
    Vec fr(n * n), fi(n * n);
    if (p.delta.is_sparse()) {  // CSR Delta: the device SpMM map (kernels.cpp:88-108)
        const api::Csr c = api::to_csr(p.delta);
        api::check(ipt_apply_map_full_csr(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                          c.rowptr.data(), c.cols.data(), c.val.re.data(), c.val.im_or_null(),
                                          zz.re.data(), zz.im_or_null(), fr.data(), fi.data()));
    } else {
        const Planar a = dense_delta(p);
        api::check(ipt_apply_map_full(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                      a.re.data(), a.im_or_null(), zz.re.data(), zz.im_or_null(), fr.data(),
                                      fi.data()));
    }
    ComplexMatrix out = ComplexMatrix::dense(n, n);
    api::merge(fr, fi, out.data());
    return out;
}

namespace b200 {

void set_device(int device) { api::set_device(device); }
void set_devices(const std::vector<int>& devices) { api::set_devices(devices); }
int devices_in_use() { return std::max<int>(1, static_cast<int>(api::devices().size())); }

EigenpairResult solve_single_accelerated(const Partition& p, const InverseGaps& g, std::size_t anchor,
                                         const IterationConfig& config, int memory) {
    if (!(config.tolerance > 0.0)) throw std::invalid_argument("config: tolerance must be positive");
    if (config.max_iterations <= 0) throw std::invalid_argument("config: max_iterations must be positive");
    check_anchor(p, g, anchor);
    const std::size_t n = p.size();
    const Planar d = api::split(p.d.data(), n);
    ipt_params prm = to_params(config);
    ipt_stats st{};
    std::vector<double> trace(config.record_trace ? config.max_iterations : 0);
    st.trace = config.record_trace ? trace.data() : nullptr;
    Vec z(n);
    if (p.delta.is_sparse()) {
        const api::Csr c = api::to_csr(p.delta);
        if (d.any_im || c.val.any_im) throw std::invalid_argument("solve_single_accelerated (device): real inputs only");
        api::check(ipt_single_solve_accelerated_csr(api::context(), static_cast<int64_t>(n), d.re.data(),
                                                    c.rowptr.data(), c.cols.data(), c.val.re.data(),
                                                    static_cast<int64_t>(anchor), &prm, memory,
                                                    config.residual_tolerance, z.data(), &st));
    } else {
        const Planar a = api::split(p.delta.data(), n * n);
        if (d.any_im || a.any_im) throw std::invalid_argument("solve_single_accelerated (device): real inputs only");
        api::check(ipt_single_solve_accelerated_dense(api::context(), static_cast<int64_t>(n), d.re.data(),
                                                      a.re.data(), static_cast<int64_t>(anchor), &prm, memory,
                                                      config.residual_tolerance, z.data(), &st));
    }
    EigenpairResult r;
    r.z.resize(n);
    for (std::size_t i = 0; i < n; ++i) r.z[i] = cplx(z[i], 0.0);
    r.eigenvalue = cplx(st.eigenvalue_re, 0.0);
    r.anchor = anchor;
    r.iterations = st.iterations;
    r.final_step = st.final_step;
    r.residual = st.residual;
    r.status = static_cast<SolveStatus>(st.status);
    r.matvec_count = static_cast<long>(st.product_count);
    if (config.record_trace) {
        const int kept = st.iterations - (r.status == SolveStatus::Converged ? 1 : 0);
        r.trace.assign(trace.begin(), trace.begin() + std::max(kept, 0));
    }
    return r;
}

SpectrumResult solve_full(const Partition& p, const InverseGaps& g, const IterationConfig& config,
                          const FullOptions& options, const ComplexMatrix* warm_start) {
    validate(config);
    check_anchor(p, g, 0);
    const std::size_t n = p.size();
    const Planar d = api::split(p.d.data(), n);
    Planar w;
    ComplexMatrix wd;
    if (warm_start) {
        wd = warm_start->to_dense();
        if (wd.rows() != n || wd.cols() != n) throw std::invalid_argument("solve_full: warm start size mismatch");
        if (p.delta.is_sparse()) w = api::split(wd.data(), n * n);
    }
    ipt_params prm = to_params(config);
    prm.stop_rule = options.stop_rule == StopRule::MaxAbs ? IPT_STOP_MAX_ABS : IPT_STOP_REL_FRO;
    prm.want_sigma_min = options.want_sigma_min ? 1 : 0;
    prm.product = options.product == Product::Ozaki ? IPT_PRODUCT_OZAKI : IPT_PRODUCT_DMMA;
    ipt_stats st{};
    std::vector<double> trace(config.record_trace ? config.max_iterations : 0);
    st.trace = config.record_trace ? trace.data() : nullptr;
    const std::vector<ipt_ctx*> ranks = api::group_contexts();
    if (!ranks.empty()) return solve_full_ranks(p, config, prm, warm_start ? &wd : nullptr, w, ranks);
    if (p.delta.is_dense()) {
        // The carrier's interleaved std::complex arrays go to the C ABI as they are (the
        // de-interleave happens inside the pinned staging pass); the result carrier is
        // allocated and zero-filled on a host thread while the device iterates, and Z is
        // interleaved straight into it while the closing product runs.
        const bool prof = std::getenv("IPT_PROFILE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        auto zbuf = std::async(std::launch::async, [n] { return cvec(n * n); });
        ipt_full_problem* h = nullptr;
        const int rc = ipt_full_solve_interleaved_start(
            api::context(), static_cast<int64_t>(n), reinterpret_cast<const double*>(p.d.data()),
            reinterpret_cast<const double*>(p.delta.data()),
            warm_start ? reinterpret_cast<const double*>(wd.data()) : nullptr, &prm, &h, &st);
        const auto t1 = std::chrono::steady_clock::now();
        cvec zv = zbuf.get();
        const auto t2 = std::chrono::steady_clock::now();
        api::check(rc);
        std::unique_ptr<ipt_full_problem, void (*)(ipt_full_problem*)> hold(h, ipt_full_free);
        SpectrumResult r;
        r.eigenvalues.resize(n);
        api::check(ipt_full_solve_interleaved_finish(api::context(), h, &prm, reinterpret_cast<double*>(zv.data()),
                                                     reinterpret_cast<double*>(r.eigenvalues.data()), &st));
        if (prof) {
            const auto t3 = std::chrono::steady_clock::now();
            auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
            std::fprintf(stderr, "[ipt] C++ solve_full ms: start %.1f, result carrier wait %.1f, finish %.1f\n",
                         ms(t0, t1), ms(t1, t2), ms(t2, t3));
        }
        r.Z = ComplexMatrix::dense(n, n, std::move(zv));
        r.iterations = st.iterations;
        r.final_step = st.final_step;
        r.residual_frobenius = st.residual;
        r.min_singular_value_estimate = st.min_singular_value_estimate;
        r.status = static_cast<SolveStatus>(st.status);
        r.matmul_count = static_cast<long>(st.product_count);
        if (config.record_trace) r.trace.assign(trace.begin(), trace.begin() + st.iterations);
        return r;
    }
    Vec zr(n * n), zi(n * n), lr(n), li(n);
    const double* wre = warm_start ? w.re.data() : nullptr;
    const double* wim = warm_start ? w.im_or_null() : nullptr;
    if (p.delta.is_sparse()) {  // CSR Delta: fused SpMM map on the device (real), else densified
        const api::Csr c = api::to_csr(p.delta);
        api::check(ipt_full_solve_csr(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(),
                                      c.rowptr.data(), c.cols.data(), c.val.re.data(), c.val.im_or_null(), wre, wim,
                                      &prm, zr.data(), zi.data(), lr.data(), li.data(), &st));
    } else {
        const Planar a = dense_delta(p);
        api::check(ipt_full_solve(api::context(), static_cast<int64_t>(n), d.re.data(), d.im_or_null(), a.re.data(),
                                  a.im_or_null(), wre, wim, &prm, zr.data(), zi.data(), lr.data(), li.data(), &st));
    }
    SpectrumResult r;
    r.Z = ComplexMatrix::dense(n, n);
    api::merge(zr, zi, r.Z.data());
    r.eigenvalues = combine(lr, li);
    r.iterations = st.iterations;
    r.final_step = st.final_step;
    r.residual_frobenius = st.residual;
    r.min_singular_value_estimate = st.min_singular_value_estimate;
    r.status = static_cast<SolveStatus>(st.status);
    r.matmul_count = static_cast<long>(st.product_count);
    if (config.record_trace) r.trace.assign(trace.begin(), trace.begin() + st.iterations);
    return r;
}

}  // namespace b200

SpectrumResult solve_full(const Partition& p, const InverseGaps& g, const IterationConfig& config,
                          const ComplexMatrix* warm_start) {
    // IPT_PRODUCT=ozaki lets unmodified reference callers (refine, cli, bench) take the
    // FP64-accurate tcgen05 product; the default is the DMMA product
    b200::FullOptions options;
    const char* e = std::getenv("IPT_PRODUCT");
    if (e && std::string(e) == "ozaki") options.product = b200::Product::Ozaki;
    return b200::solve_full(p, g, config, options, warm_start);
}

double smallest_singular_value_estimate(const ComplexMatrix& z, int max_iters, double tol) {
    const std::size_t n = z.rows();
    if (n == 0 || z.cols() != n) throw std::invalid_argument("smallest_singular_value_estimate: square input required");
    const ComplexMatrix zd = z.to_dense();
    const Planar zz = api::split(zd.data(), n * n);
    double out = 0.0;
    api::check(ipt_sigma_min(api::context(), static_cast<int64_t>(n), zz.re.data(), zz.im_or_null(), max_iters, tol,
                             &out));
    return out;
}

namespace api {
void release_resident_single() { t_single.release(); }
}  // namespace api

}  // namespace ipt
