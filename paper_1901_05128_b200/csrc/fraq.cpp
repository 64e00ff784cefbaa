// fraq.cpp -- C++ mirror of the reference `fraq` API on the B200 C ABI (see fraq.hpp).
#include "fraq.hpp"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

namespace fraq {

namespace {

std::string last_error() {
    char buf[1024];
    fraq_last_error(buf, sizeof(buf));
    return buf;
}

}  // namespace

void check(int st) {
    if (st == FRAQ_OK) return;
    const std::string msg = last_error();
    switch (st) {
        case FRAQ_EINVAL: throw std::invalid_argument(msg);
        case FRAQ_ELOGIC: throw std::logic_error(msg);
        case FRAQ_ERANGE: throw std::out_of_range(msg);
        case FRAQ_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

int default_device() {
    const char* e = std::getenv("FRAQ_DEVICE");
    return e ? std::atoi(e) : 0;
}

fraq_ctx default_context() {
    static std::mutex mu;
    static fraq_ctx ctx = nullptr;
    std::lock_guard<std::mutex> lock(mu);
    if (!ctx) check(fraq_ctx_create(default_device(), nullptr, &ctx));
    return ctx;
}

// ------------------------------------------------------------------ gauss_jacobi
double gamma_fn(double x) { return fraq_gamma(x); }
double inv_gamma_product(double alpha) { return fraq_inv_gamma_product(alpha); }

double jacobi_moment0(double a, double b) { return jacobi_moment(a, b, 0); }

double jacobi_moment(double a, double b, int k) {
    double out = 0.0;
    check(fraq_jacobi_moment(a, b, k, &out));
    return out;
}

JacobiRule gauss_jacobi(double a, double b, int n) {
    JacobiRule r;
    r.exponent_a = a;
    r.exponent_b = b;
    const int cap = n > 0 ? n : 1;
    r.nodes.resize(cap);
    r.weights.resize(cap);
    check(fraq_gauss_jacobi(default_context(), a, b, n, r.nodes.data(), r.weights.data()));
    r.nodes.resize(n);
    r.weights.resize(n);
    return r;
}

// ------------------------------------------------------------------ cq_weights
WeightTable be_weights(double alpha, double tau, long n_max) {
    WeightTable t;
    t.scheme = CqScheme::BE;
    t.alpha = alpha;
    t.tau = tau;
    t.weights.resize(n_max >= 0 ? n_max + 1 : 1);
    check(fraq_be_weights(default_context(), alpha, tau, n_max, t.weights.data(), FRAQ_HOST));
    return t;
}

WeightTable sbd_weights(double alpha, double tau, long n_max) {
    WeightTable t;
    t.scheme = CqScheme::SBD;
    t.alpha = alpha;
    t.tau = tau;
    t.weights.resize(n_max >= 0 ? n_max + 1 : 1);
    check(fraq_sbd_weights(default_context(), alpha, tau, n_max, t.weights.data(), FRAQ_HOST));
    return t;
}

double coupling_from_transition(double m) {
    double a = 0.0;
    check(fraq_coupling_from_transition(m, &a));
    return a;
}

// ------------------------------------------------------------------ kernels
fraq_kernel_t to_flat(const FastKernelBE& k) {
    fraq_kernel_t f;
    std::memset(&f, 0, sizeof(f));
    if (k.ratios.size() > FRAQ_MAX_POINTS || k.node_weights.size() != k.ratios.size())
        throw std::invalid_argument("FastKernelBE: malformed node tables");
    f.sbd = 0;
    f.gamma = k.alpha;
    f.tau = k.tau;
    f.n_head = 2;
    f.head[0] = k.head[0];
    f.head[1] = k.head[1];
    f.np1 = (int)k.ratios.size();
    f.np2 = 0;
    std::memcpy(f.m1, k.node_weights.data(), sizeof(double) * f.np1);
    std::memcpy(f.r1, k.ratios.data(), sizeof(double) * f.np1);
    return f;
}

fraq_kernel_t to_flat(const FastKernelSBD& k) {
    fraq_kernel_t f;
    std::memset(&f, 0, sizeof(f));
    if (k.ratio1.size() > FRAQ_MAX_POINTS || k.ratio2.size() > FRAQ_MAX_POINTS ||
        k.mult1.size() != k.ratio1.size() || k.mult2.size() != k.ratio2.size() ||
        k.head.size() > FRAQ_MAX_HEAD || (int)k.head.size() < k.n_head)
        throw std::invalid_argument("FastKernelSBD: malformed tables");
    f.sbd = 1;
    f.gamma = k.alpha;
    f.tau = k.tau;
    f.n_head = k.n_head;
    std::memcpy(f.head, k.head.data(), sizeof(double) * k.n_head);
    f.np1 = (int)k.ratio1.size();
    f.np2 = (int)k.ratio2.size();
    std::memcpy(f.m1, k.mult1.data(), sizeof(double) * f.np1);
    std::memcpy(f.r1, k.ratio1.data(), sizeof(double) * f.np1);
    std::memcpy(f.m2, k.mult2.data(), sizeof(double) * f.np2);
    std::memcpy(f.r2, k.ratio2.data(), sizeof(double) * f.np2);
    return f;
}

FastKernelBE be_from_flat(const fraq_kernel_t& f) {
    FastKernelBE k;
    k.alpha = f.gamma;
    k.tau = f.tau;
    k.head[0] = f.head[0];
    k.head[1] = f.head[1];
    k.node_weights.assign(f.m1, f.m1 + f.np1);
    k.ratios.assign(f.r1, f.r1 + f.np1);
    return k;
}

FastKernelSBD sbd_from_flat(const fraq_kernel_t& f) {
    FastKernelSBD k;
    k.alpha = f.gamma;
    k.tau = f.tau;
    k.n_head = f.n_head;
    k.head.assign(f.head, f.head + f.n_head);
    k.mult1.assign(f.m1, f.m1 + f.np1);
    k.ratio1.assign(f.r1, f.r1 + f.np1);
    k.mult2.assign(f.m2, f.m2 + f.np2);
    k.ratio2.assign(f.r2, f.r2 + f.np2);
    return k;
}

namespace {
double recon_one(const fraq_kernel_t& f, long i) {
    double out = 0.0;
    check(fraq_reconstruct(default_context(), &f, 1, &i, &out));
    return out;
}

KernelErrorReport report(const fraq_kernel_t& f, long n_max) {
    KernelErrorReport r;
    r.alpha = f.gamma;
    r.tau = f.tau;
    r.head_len = f.sbd ? f.n_head : 2;
    r.max_index = n_max;
    r.eps.assign(n_max >= 0 ? n_max + 1 : 1, 0.0);
    check(fraq_kernel_error_report(default_context(), &f, n_max, r.eps.data(), &r.max_eps,
                                   &r.argmax));
    return r;
}
}  // namespace

double FastKernelBE::reconstruct(long i) const { return recon_one(to_flat(*this), i); }
double FastKernelSBD::reconstruct(long i) const { return recon_one(to_flat(*this), i); }

FastKernelBE build_be_kernel(double alpha, double tau, int n_points) {
    fraq_kernel_t f;
    check(fraq_build_be_kernel(default_context(), alpha, tau, n_points, &f));
    return be_from_flat(f);
}

FastKernelSBD build_sbd_kernel(double alpha, double tau, int n1, int n2, int n_head) {
    fraq_kernel_t f;
    check(fraq_build_sbd_kernel(default_context(), alpha, tau, n1, n2, n_head, &f));
    return sbd_from_flat(f);
}

int default_sbd_head(double alpha) { return fraq_default_sbd_head(alpha); }
namespace {
FastKernelSBD fold_flat(const fraq_kernel_t& f, int max_head, int* levels) {
    fraq_kernel_t o;
    int M = 0;
    check(fraq_fold_kernel(&f, max_head, &o, &M));
    if (levels) *levels = M;
    if (!o.sbd) {
        // nothing folded in a BE kernel: the same kernel in the generic-head format
        // (feed w = m' r^(n_head - 3) with n_head = 2: m' = w r)
        o.sbd = 1;
        for (int j = 0; j < o.np1; ++j) o.m1[j] *= o.r1[j];
    }
    return sbd_from_flat(o);
}
}  // namespace
FastKernelSBD fold_kernel(const FastKernelBE& k, int max_head, int* levels) {
    return fold_flat(to_flat(k), max_head, levels);
}
FastKernelSBD fold_kernel(const FastKernelSBD& k, int max_head, int* levels) {
    return fold_flat(to_flat(k), max_head, levels);
}

KernelErrorReport kernel_error_report(const FastKernelBE& k, long n_max) {
    return report(to_flat(k), n_max);
}
KernelErrorReport kernel_error_report(const FastKernelSBD& k, long n_max) {
    return report(to_flat(k), n_max);
}

FastKernelBE build_be_kernel_auto(double alpha, double tau, KernelBudget& b) {
    fraq_budget_t fb{b.horizon, b.eps_tol, b.max_points, b.max_head, 0.0};
    fraq_kernel_t f;
    check(fraq_build_be_kernel_auto(default_context(), alpha, tau, &fb, &f));
    b.horizon = fb.horizon;
    b.achieved_eps = fb.achieved_eps;
    return be_from_flat(f);
}

FastKernelSBD build_sbd_kernel_auto(double alpha, double tau, KernelBudget& b) {
    fraq_budget_t fb{b.horizon, b.eps_tol, b.max_points, b.max_head, 0.0};
    fraq_kernel_t f;
    check(fraq_build_sbd_kernel_auto(default_context(), alpha, tau, &fb, &f));
    b.horizon = fb.horizon;
    b.achieved_eps = fb.achieved_eps;
    return sbd_from_flat(f);
}

// ------------------------------------------------------------------ histories
DeviceHistory::DeviceHistory(const std::vector<fraq_kernel_t>& kernels,
                             const std::vector<long>& dims, HistoryVariant variant) {
    std::vector<const fraq_kernel_t*> kp;
    long total = 0;
    for (std::size_t g = 0; g < kernels.size(); ++g) {
        kp.push_back(&kernels[g]);
        total += dims[g];
    }
    check(fraq_hist_create(default_context(), (int)kernels.size(), kp.data(), dims.data(),
                           variant == HistoryVariant::standalone ? FRAQ_STANDALONE : FRAQ_SCHEME,
                           &h_));
    dim_ = (std::size_t)total;
    n_groups_ = kernels.size();
    lag_.resize(dim_);
}

DeviceHistory::~DeviceHistory() {
    if (h_) fraq_hist_destroy(h_);
}

DeviceHistory::DeviceHistory(DeviceHistory&& o) noexcept
    : h_(o.h_), dim_(o.dim_), n_groups_(o.n_groups_), lag_(std::move(o.lag_)) {
    o.h_ = nullptr;
}

DeviceHistory& DeviceHistory::operator=(DeviceHistory&& o) noexcept {
    if (this != &o) {
        if (h_) fraq_hist_destroy(h_);
        h_ = o.h_;
        dim_ = o.dim_;
        n_groups_ = o.n_groups_;
        lag_ = std::move(o.lag_);
        o.h_ = nullptr;
    }
    return *this;
}

static void check_dim(std::size_t have, std::size_t want, const char* what) {
    if (have != want) throw std::invalid_argument(std::string(what) + ": wrong dimension");
}

void DeviceHistory::push(std::span<const double> v) {
    check_dim(v.size(), dim_, "History::append");
    check(fraq_hist_push(h_, v.data(), FRAQ_HOST));
}
void DeviceHistory::advance() { check(fraq_hist_advance(h_)); }
void DeviceHistory::append(std::span<const double> v) {
    check_dim(v.size(), dim_, "History::append");
    check(fraq_hist_append(h_, v.data(), FRAQ_HOST));
}
long DeviceHistory::level() const {
    long l = 0;
    check(fraq_hist_info(h_, &l, nullptr, nullptr));
    return l;
}
long DeviceHistory::appended() const {
    long a = 0;
    check(fraq_hist_info(h_, nullptr, &a, nullptr));
    return a;
}
void DeviceHistory::history_sum(std::span<double> out) const {
    check_dim(out.size(), dim_, "History::history_sum");
    check(fraq_hist_history_sum(h_, out.data(), FRAQ_HOST));
}
void DeviceHistory::derivative(std::span<double> out) const {
    check_dim(out.size(), dim_, "History::derivative");
    check(fraq_hist_derivative(h_, out.data(), FRAQ_HOST));
}
std::span<const double> DeviceHistory::lagged(long depth) const {
    check(fraq_hist_lagged(h_, depth, lag_.data(), FRAQ_HOST));
    return {lag_.data(), dim_};
}
void DeviceHistory::run(const double* U, long ldu, long n_steps, double* D, long ldd, int mem) {
    check(fraq_hist_run(h_, U, ldu, n_steps, D, ldd, mem));
}
int DeviceHistory::last_path() const { return fraq_hist_last_path(h_); }
std::vector<long> DeviceHistory::launches() const {
    std::vector<long> out(6, 0);
    check(fraq_hist_path_info(h_, out.data(), 0, nullptr));
    return out;
}
std::vector<int> DeviceHistory::fir_info() const {
    std::vector<int> out(3 * n_groups_, 0);
    check(fraq_hist_path_info(h_, nullptr, (int)n_groups_, out.data()));
    return out;
}

BeHistory::BeHistory(const FastKernelBE& k, HistoryVariant v, std::size_t dim)
    : DeviceHistory({to_flat(k)}, {(long)dim}, v) {}

SbdHistory::SbdHistory(const FastKernelSBD& k, HistoryVariant v, std::size_t dim)
    : DeviceHistory({to_flat(k)}, {(long)dim}, v) {}

// ------------------------------------------------------------------ fpfp
Scheme scheme_from_name(const std::string& name) {
    if (name == "be") return Scheme::BE;
    if (name == "fastbe" || name == "fbe") return Scheme::FastBE;
    if (name == "sbd") return Scheme::SBD;
    if (name == "fastsbd" || name == "fsbd") return Scheme::FastSBD;
    throw std::invalid_argument("unknown scheme: " + name);
}

std::string scheme_name(Scheme s) {
    switch (s) {
        case Scheme::BE: return "be";
        case Scheme::FastBE: return "fastbe";
        case Scheme::SBD: return "sbd";
        case Scheme::FastSBD: return "fastsbd";
    }
    return "?";
}

bool scheme_is_fast(Scheme s) { return s == Scheme::FastBE || s == Scheme::FastSBD; }
bool scheme_is_sbd(Scheme s) { return s == Scheme::SBD || s == Scheme::FastSBD; }

StateField initial_field(const ProblemSpec& spec) {
    StateField f;
    const int m = spec.grid_m;
    f.g1.resize(m);
    f.g2.resize(m);
    const double h = spec.h();
    for (int j = 0; j < m; ++j) {
        const double x = (j + 1) * h;
        switch (spec.initial) {
            case InitialData::poly_sin:
                f.g1[j] = x * (1.0 - x);
                f.g2[j] = std::sin(x);
                break;
            case InitialData::indicator:
                f.g1[j] = x > 0.5 ? 1.0 - x : 0.0;
                f.g2[j] = x < 0.5 ? x : 0.0;
                break;
            case InitialData::custom:
                if ((int)spec.custom_g1.size() != m || (int)spec.custom_g2.size() != m)
                    throw std::invalid_argument(
                        "initial_field: custom samples must have grid_m entries");
                f.g1 = spec.custom_g1;
                f.g2 = spec.custom_g2;
                break;
        }
    }
    return f;
}

double l2_norm(std::span<const double> v, double h) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return std::sqrt(h * s);
}

namespace {
fraq_spec_t flat_spec(const ProblemSpec& s) {
    fraq_spec_t f;
    f.alpha1 = s.alpha1;
    f.alpha2 = s.alpha2;
    f.coupling_a = s.coupling_a;
    f.length = s.length;
    f.t_final = s.t_final;
    f.grid_m = s.grid_m;
    f.n_steps = s.n_steps;
    f.initial = s.initial == InitialData::poly_sin
                    ? FRAQ_POLY_SIN
                    : (s.initial == InitialData::indicator ? FRAQ_INDICATOR : FRAQ_CUSTOM);
    f.custom_g1 = s.custom_g1.empty() ? nullptr : s.custom_g1.data();
    f.custom_g2 = s.custom_g2.empty() ? nullptr : s.custom_g2.data();
    return f;
}
fraq_kconf_t flat_kconf(const KernelConfig& k) {
    return fraq_kconf_t{k.be_points, k.sbd_points_1, k.sbd_points_2, k.sbd_head, k.eps_tol,
                        k.auto_size ? 1 : 0, k.solver};
}
int flat_scheme(Scheme s) {
    switch (s) {
        case Scheme::BE: return FRAQ_BE;
        case Scheme::FastBE: return FRAQ_FASTBE;
        case Scheme::SBD: return FRAQ_SBD;
        default: return FRAQ_FASTSBD;
    }
}
struct ObsCtx {
    const std::function<void(long, const StateField&)>* fn;
    StateField f;
};
void obs_tramp(long n, const double* g1, const double* g2, int m, void* user) {
    auto* o = static_cast<ObsCtx*>(user);
    o->f.g1.assign(g1, g1 + m);
    o->f.g2.assign(g2, g2 + m);
    o->f.step = n;
    (*o->fn)(n, o->f);
}
}  // namespace

RunResult run_on(fraq_ctx ctx, const ProblemSpec& spec, Scheme scheme, const KernelConfig& kconf,
                 const std::function<void(long, const StateField&)>& observer) {
    if (spec.initial == InitialData::custom &&
        ((int)spec.custom_g1.size() != spec.grid_m || (int)spec.custom_g2.size() != spec.grid_m))
        throw std::invalid_argument("initial_field: custom samples must have grid_m entries");
    const fraq_spec_t fs = flat_spec(spec);
    const fraq_kconf_t kc = flat_kconf(kconf);
    RunResult rr;
    rr.final_state.g1.resize(spec.grid_m > 0 ? spec.grid_m : 1);
    rr.final_state.g2.resize(spec.grid_m > 0 ? spec.grid_m : 1);
    fraq_run_info_t info{};
    if (observer) {
        ObsCtx oc{&observer, {}};
        check(fraq_run_observed(ctx, &fs, flat_scheme(scheme), &kc, obs_tramp, &oc,
                                rr.final_state.g1.data(), rr.final_state.g2.data(), &info));
    } else {
        check(fraq_run(ctx, &fs, 1, flat_scheme(scheme), &kc, rr.final_state.g1.data(),
                       rr.final_state.g2.data(), &info));
    }
    rr.final_state.step = spec.n_steps;
    rr.loop_seconds = info.loop_seconds;
    rr.setup_seconds = info.setup_seconds;
    rr.kernel_eps1 = info.kernel_eps1;
    rr.kernel_eps2 = info.kernel_eps2;
    return rr;
}

RunResult run(const ProblemSpec& spec, Scheme scheme, const KernelConfig& kconf,
              const std::function<void(long, const StateField&)>& observer) {
    return run_on(default_context(), spec, scheme, kconf, observer);
}

RunResult run_2d(double alpha1, double alpha2, double coupling_a, int grid_m, double t_final,
                 long n_steps, Scheme scheme, const std::vector<double>& g1_0,
                 const std::vector<double>& g2_0, const KernelConfig& kconf) {
    const size_t mm = (size_t)grid_m * (size_t)grid_m;
    if (g1_0.size() != mm || g2_0.size() != mm)
        throw std::invalid_argument("run_2d: initial data must have grid_m^2 entries");
    const fraq_kconf_t kc = flat_kconf(kconf);
    RunResult rr;
    rr.final_state.g1.resize(mm);
    rr.final_state.g2.resize(mm);
    fraq_run_info_t info{};
    check(fraq_run_2d(default_context(), alpha1, alpha2, coupling_a, grid_m, t_final, n_steps,
                      flat_scheme(scheme), &kc, g1_0.data(), g2_0.data(), rr.final_state.g1.data(),
                      rr.final_state.g2.data(), &info));
    rr.final_state.step = n_steps;
    rr.loop_seconds = info.loop_seconds;
    rr.setup_seconds = info.setup_seconds;
    rr.kernel_eps1 = info.kernel_eps1;
    rr.kernel_eps2 = info.kernel_eps2;
    return rr;
}

void dst2d(int grid_m, int n_fields, const double* in, double* out, bool inverse, int mem) {
    check(fraq_dst2d(default_context(), grid_m, n_fields, in, out, inverse ? 1 : 0, mem));
}

void dst_cols(int grid_m, long n_cols, const double* in, double* out, bool inverse, int mem) {
    check(fraq_dst_cols(default_context(), grid_m, n_cols, in, out, inverse ? 1 : 0, mem));
}

RunResult modal_run(double alpha1, double alpha2, double coupling_a, double t_final,
                    long n_steps, Scheme scheme, long n_modes, const double* lam,
                    const double* c0, double* cN, int mem, const KernelConfig& kconf) {
    const fraq_kconf_t kc = flat_kconf(kconf);
    fraq_run_info_t info{};
    check(fraq_modal_run(default_context(), alpha1, alpha2, coupling_a, t_final, n_steps,
                         flat_scheme(scheme), &kc, n_modes, lam, c0, cN, mem, &info));
    RunResult rr;
    rr.final_state.step = n_steps;
    rr.loop_seconds = info.loop_seconds;
    rr.setup_seconds = info.setup_seconds;
    rr.kernel_eps1 = info.kernel_eps1;
    rr.kernel_eps2 = info.kernel_eps2;
    return rr;
}

std::vector<RunResult> run_batch(const std::vector<ProblemSpec>& specs, Scheme scheme,
                                 const KernelConfig& kconf) {
    std::vector<fraq_spec_t> fs;
    for (const auto& s : specs) fs.push_back(flat_spec(s));
    const fraq_kconf_t kc = flat_kconf(kconf);
    const int n = (int)specs.size();
    if (n == 0) return {};
    const int m = specs[0].grid_m;
    std::vector<double> g1((size_t)n * m), g2((size_t)n * m);
    fraq_run_info_t info{};
    check(fraq_run(default_context(), fs.data(), n, flat_scheme(scheme), &kc, g1.data(), g2.data(),
                   &info));
    std::vector<RunResult> out(n);
    for (int i = 0; i < n; ++i) {
        out[i].final_state.g1.assign(g1.begin() + (size_t)i * m, g1.begin() + (size_t)(i + 1) * m);
        out[i].final_state.g2.assign(g2.begin() + (size_t)i * m, g2.begin() + (size_t)(i + 1) * m);
        out[i].final_state.step = specs[i].n_steps;
        out[i].loop_seconds = info.loop_seconds;
        out[i].setup_seconds = info.setup_seconds;
    }
    return out;
}

// ------------------------------------------------------------------ block_solver.hpp
void DiscreteLaplacian::apply(std::span<const double> x, std::span<double> y) const {
    if ((int)x.size() < grid_m || (int)y.size() < grid_m)
        throw std::invalid_argument("DiscreteLaplacian::apply: spans shorter than grid_m");
    check(fraq_laplacian_apply(default_context(), grid_m, h, x.data(), y.data(), FRAQ_HOST));
}

double DiscreteLaplacian::eigenvalue(int k, double length) const {
    // block_solver.cpp:21-24 (closed form; a test oracle in the reference)
    const double s = std::sin(k * 3.14159265358979323846 * h / (2.0 * length));
    return 4.0 / (h * h) * s * s;
}

BandedLU::BandedLU(int n, int kl, int ku)
    : n_(n), kl_(kl), ku_(ku), ldab_(2 * kl + ku + 1),
      ab_(static_cast<std::size_t>(2 * kl + ku + 1) * (n > 0 ? n : 0), 0.0) {
    check(fraq_banded_create(default_context(), n, kl, ku, &b_));
}
BandedLU::~BandedLU() {
    if (b_) fraq_banded_destroy(b_);
}
BandedLU::BandedLU(BandedLU&& o) noexcept
    : n_(o.n_), kl_(o.kl_), ku_(o.ku_), ldab_(o.ldab_), factored_(o.factored_),
      ab_(std::move(o.ab_)), b_(o.b_) {
    o.b_ = nullptr;
}
BandedLU& BandedLU::operator=(BandedLU&& o) noexcept {
    if (this != &o) {
        if (b_) fraq_banded_destroy(b_);
        n_ = o.n_;
        kl_ = o.kl_;
        ku_ = o.ku_;
        ldab_ = o.ldab_;
        factored_ = o.factored_;
        ab_ = std::move(o.ab_);
        b_ = o.b_;
        o.b_ = nullptr;
    }
    return *this;
}
double& BandedLU::at(int row, int col) {
    if (row < 0 || row >= n_ || col < 0 || col >= n_ || col - row > ku_ || row - col > kl_)
        throw std::out_of_range("BandedLU::at: outside the band");
    return ab_[static_cast<std::size_t>(col) * ldab_ + (kl_ + ku_ + row - col)];
}
void BandedLU::factorize() {
    // hand the assembled band to the device object, factor there
    check(fraq_banded_assign(b_, ab_.data()));
    check(fraq_banded_factorize(b_));
    factored_ = true;
}
void BandedLU::solve(std::span<double> rhs) const {
    if (!factored_) throw std::logic_error("BandedLU::solve before factorize");
    if ((int)rhs.size() < n_) throw std::invalid_argument("BandedLU::solve: rhs shorter than n");
    check(fraq_banded_solve(b_, rhs.data(), FRAQ_HOST));
}

BlockSystem::BlockSystem(double d01, double d02, double coupling_a, double tau,
                         const DiscreteLaplacian& lap, double bdf_lead)
    : m_(lap.grid_m) {
    check(fraq_block_create(default_context(), d01, d02, coupling_a, tau, lap.grid_m, lap.h,
                            bdf_lead, &b_));
}
BlockSystem::~BlockSystem() {
    if (b_) fraq_block_destroy(b_);
}
BlockSystem::BlockSystem(BlockSystem&& o) noexcept : m_(o.m_), b_(o.b_) { o.b_ = nullptr; }
BlockSystem& BlockSystem::operator=(BlockSystem&& o) noexcept {
    if (this != &o) {
        if (b_) fraq_block_destroy(b_);
        m_ = o.m_;
        b_ = o.b_;
        o.b_ = nullptr;
    }
    return *this;
}
void BlockSystem::solve(std::span<const double> rhs1, std::span<const double> rhs2,
                        std::span<double> g1, std::span<double> g2) const {
    if ((int)rhs1.size() < m_ || (int)rhs2.size() < m_ || (int)g1.size() < m_ ||
        (int)g2.size() < m_)
        throw std::invalid_argument("BlockSystem::solve: spans shorter than grid_m");
    check(fraq_block_solve(b_, rhs1.data(), rhs2.data(), g1.data(), g2.data(), FRAQ_HOST));
}

void solve_block_system(double d01, double d02, double coupling_a, double tau,
                        const DiscreteLaplacian& lap, std::span<const double> rhs1,
                        std::span<const double> rhs2, std::span<double> g1,
                        std::span<double> g2, double bdf_lead) {
    BlockSystem sys(d01, d02, coupling_a, tau, lap, bdf_lead);
    sys.solve(rhs1, rhs2, g1, g2);
}

// ------------------------------------------------------------------ steppers (fpfp.hpp:80-140)
namespace {
fraq_stepper make_stepper(const ProblemSpec& spec, int scheme, const KernelConfig* kconf) {
    if (spec.initial == InitialData::custom &&
        ((int)spec.custom_g1.size() != spec.grid_m || (int)spec.custom_g2.size() != spec.grid_m))
        throw std::invalid_argument("initial_field: custom samples must have grid_m entries");
    const fraq_spec_t fs = flat_spec(spec);
    fraq_kconf_t kc;
    if (kconf)
        kc = flat_kconf(*kconf);
    else
        fraq_kconf_default(&kc);
    fraq_stepper st = nullptr;
    check(fraq_stepper_create(default_context(), &fs, scheme, &kc, &st));
    return st;
}
void refresh(fraq_stepper st, StateField& f, long& at, long step, int m) {
    if (at == step) return;
    f.g1.resize(m);
    f.g2.resize(m);
    long n = 0;
    check(fraq_stepper_state(st, f.g1.data(), f.g2.data(), &n));
    f.step = n;
    at = step;
}
}  // namespace

ClassicalStepper::ClassicalStepper(const ProblemSpec& spec, bool sbd)
    : st_(make_stepper(spec, sbd ? FRAQ_SBD : FRAQ_BE, nullptr)) {
    state_.g1.resize(spec.grid_m);
}
ClassicalStepper::~ClassicalStepper() {
    if (st_) fraq_stepper_destroy(st_);
}
void ClassicalStepper::step() {
    check(fraq_stepper_step(st_, 1));
    ++step_;
}
const StateField& ClassicalStepper::state() const {
    refresh(st_, state_, state_at_, step_, (int)state_.g1.size());
    return state_;
}

FastStepper::FastStepper(const ProblemSpec& spec, bool sbd, const KernelConfig& kconf)
    : st_(make_stepper(spec, sbd ? FRAQ_FASTSBD : FRAQ_FASTBE, &kconf)) {
    state_.g1.resize(spec.grid_m);
    check(fraq_stepper_kernel_eps(st_, &eps1_, &eps2_));
}
FastStepper::~FastStepper() {
    if (st_) fraq_stepper_destroy(st_);
}
void FastStepper::step() { step_n(1); }
void FastStepper::step_n(long n) {
    check(fraq_stepper_step(st_, n));
    step_ += n;
}
std::pair<double, double> FastStepper::time_split(long n) {
    double a = 0.0, b = 0.0;
    check(fraq_stepper_time_split(st_, n, &a, &b));
    step_ += n;
    return {a, b};
}
const StateField& FastStepper::state() const {
    refresh(st_, state_, state_at_, step_, (int)state_.g1.size());
    return state_;
}

}  // namespace fraq
