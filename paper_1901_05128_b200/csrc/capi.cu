// capi.cu -- extern "C" entry points of libfraqcu (declared in include/fraqcu.h).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>

#include "history.cuh"
#include "internal.cuh"

namespace fraqcu {

thread_local std::string g_last_error;
void set_last_error(const std::string& m) { g_last_error = m; }

// history.cu
void hist_create(fraq_ctx c, int n_groups, const fraq_kernel_t* const* ks, const long* dims,
                 int variant, fraq_hist* out);
void hist_destroy(fraq_hist h);
void hist_info(fraq_hist h, long* level, long* appended, long* dim);
void hist_push(fraq_hist h, const double* v, int mem);
void hist_advance(fraq_hist h);
void hist_append(fraq_hist h, const double* v, int mem);
void hist_output(fraq_hist h, int mode, double* out, int mem);
void hist_lagged(fraq_hist h, long depth, double* out, int mem);
void hist_run(fraq_hist h, const double* U, long ldu, long n_steps, double* D, long ldd, int mem);
int hist_last_path(fraq_hist h);
void hist_path_info(fraq_hist h, long* launches, int n_groups, int* fir);
fraq_ctx hist_ctx(fraq_hist h);
void dst2d(fraq_ctx c, int M, int n_fields, const double* in, double* out, bool inverse, int mem);
void dst_cols(fraq_ctx c, int M, long n_cols, const double* in, double* out, bool inverse, int mem);
void modal_run_modes(fraq_ctx c, double alpha1, double alpha2, double a, double t_final, long N,
                     int scheme, const fraq_kconf_t* kc, long n_modes, const double* lam,
                     const double* c0, double* cN, int mem, fraq_run_info_t* info);
void ffpe_run_2d(fraq_ctx c, double alpha1, double alpha2, double a, int m, double t_final,
                 long N, int scheme, const fraq_kconf_t* kc, const double* g1_0,
                 const double* g2_0, double* g1, double* g2, fraq_run_info_t* info);
// ffpe.cu
void ffpe_run(fraq_ctx c, const fraq_spec_t* specs, int n_inst, int scheme,
              const fraq_kconf_t* kc, double* g1, double* g2, fraq_run_info_t* info,
              fraq_observer_fn obs, void* user);

// ffpe.cu: single-step API objects
struct PhysStepper;
struct BlockDev;
struct BandedDev;
void stepper_create(fraq_ctx c, const fraq_spec_t* spec, int scheme, const fraq_kconf_t* kc,
                    PhysStepper** out);
void stepper_step(PhysStepper* st, long n);
void stepper_state(PhysStepper* st, double* g1, double* g2, long* step);
void stepper_eps(PhysStepper* st, double* e1, double* e2);
void stepper_time_split(PhysStepper* st, long n, double* ms_hist, double* ms_solve);
void stepper_destroy(PhysStepper* st);
void block_create(fraq_ctx c, double d01, double d02, double a, double tau, int m, double h,
                  double lead, BlockDev** out);
void block_solve(BlockDev* b, const double* rhs1, const double* rhs2, double* g1, double* g2,
                 int mem);
void block_destroy(BlockDev* b);
void laplacian_apply(fraq_ctx c, int m, double h, const double* x, double* y, int mem);
void banded_create(fraq_ctx c, int n, int kl, int ku, BandedDev** out);
double* banded_at(BandedDev* b, int row, int col);
void banded_factorize(BandedDev* b);
void banded_assign(BandedDev* b, const double* ab);
void banded_solve(BandedDev* b, double* rhs, int mem);
void banded_destroy(BandedDev* b);

namespace {
constexpr double kPi = 3.14159265358979323846;

double host_gamma(double x) {  // gauss_jacobi.cpp:108-123 (host scalar helper for the ABI)
    static const double c[9] = {0.99999999999980993,  676.5203681218851,     -1259.1392167224028,
                                771.32342877765313,   -176.61502916214059,   12.507343278686905,
                                -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7};
    if (x < 0.5) return kPi / (std::sin(kPi * x) * host_gamma(1.0 - x));
    x -= 1.0;
    double acc = c[0];
    for (int i = 1; i < 9; ++i) acc += c[i] / (x + i);
    const double t = x + 7.5;
    return std::sqrt(2.0 * kPi) * std::pow(t, x + 0.5) * std::exp(-t) * acc;
}

// A history is bound to its context: calls serialise on that context's lock.
template <class F>
int guarded_hist(fraq_hist h, F&& f) {
    if (!h) return guarded([] { fail(FRAQ_EINVAL, "null history"); });
    return guarded(hist_ctx(h), f);
}

void check_exps(double a, double b) {
    if (!(a > -1.0) || !(b > -1.0))
        fail(FRAQ_EINVAL, "jacobi exponents must be > -1, got a=" + std::to_string(a) +
                              " b=" + std::to_string(b));
}
}  // namespace

}  // namespace fraqcu

using namespace fraqcu;

extern "C" {

int fraq_version(void) { return 10000; }

int fraq_last_error(char* buf, size_t n) {
    if (buf && n) {
        std::strncpy(buf, g_last_error.c_str(), n - 1);
        buf[n - 1] = 0;
    }
    return (int)g_last_error.size();
}

int fraq_ctx_create(int device, void* stream, fraq_ctx* out) {
    return guarded([&] {
        if (!out) fail(FRAQ_EINVAL, "fraq_ctx_create: null out");
        int count = 0;
        cudaError_t e = cudaGetDeviceCount(&count);
        if (e != cudaSuccess || count == 0)
            fail(FRAQ_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
        if (device < 0 || device >= count) fail(FRAQ_EINVAL, "fraq_ctx_create: bad device");
        FRAQ_CUDA(cudaSetDevice(device));
        auto* c = new fraq_ctx_s();
        c->device = device;
        if (stream) {
            c->stream = (cudaStream_t)stream;
        } else {
            cudaError_t es = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
            if (es != cudaSuccess) {
                delete c;
                fail(FRAQ_ECUDA, cudaGetErrorString(es));
            }
            c->own_stream = true;
        }
        cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
        *out = c;
    });
}

int fraq_ctx_destroy(fraq_ctx c) {
    // the caller guarantees no concurrent use of c (it is being destroyed); wait for any call
    // in flight on another thread, then release outside the lock
    if (!c) return FRAQ_OK;
    { std::lock_guard<std::recursive_mutex> lock(c->mu); }
    return guarded([&] {
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        if (c->own_stream) cudaStreamDestroy(c->stream);
        delete c;
    });
}

int fraq_ctx_synchronize(fraq_ctx c) {
    return guarded(c, [&] {
        check_ctx(c);
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    });
}

void* fraq_ctx_stream(fraq_ctx c) { return c ? (void*)c->stream : nullptr; }

// ------------------------------------------------------------------ L0
double fraq_gamma(double x) { return host_gamma(x); }
double fraq_inv_gamma_product(double g) { return std::sin(kPi * g) / kPi; }

int fraq_jacobi_moment(double a, double b, int k, double* out) {
    // gauss_jacobi.cpp:135-149 (scalar, host: a test oracle in the reference)
    return guarded([&] {
        check_exps(a, b);
        if (k < 0) fail(FRAQ_EINVAL, "jacobi_moment: k must be >= 0");
        const double m0 = std::pow(2.0, a + b + 1.0) * host_gamma(a + 1.0) * host_gamma(b + 1.0) /
                          host_gamma(a + b + 2.0);
        double prev = m0;
        if (k == 0) {
            *out = prev;
            return;
        }
        double cur = (b - a) / (a + b + 2.0) * prev;
        for (int j = 1; j < k; ++j) {
            const double nxt = ((b - a) * cur + j * prev) / (a + b + 2.0 + j);
            prev = cur;
            cur = nxt;
        }
        *out = cur;
    });
}

int fraq_gauss_jacobi(fraq_ctx c, double a, double b, int n, double* nodes, double* weights) {
    return guarded(c, [&] {
        check_ctx(c);
        gauss_jacobi_dev(c, a, b, n, nodes, weights);
    });
}

// ------------------------------------------------------------------ L1
static int weights_common(fraq_ctx c, bool sbd, double g, double tau, long n_max, double* out,
                          int mem) {
    return guarded(c, [&] {
        check_ctx(c);
        if (mem == FRAQ_DEVICE) {
            if (sbd)
                sbd_weights_dev(c, g, tau, n_max, out);
            else
                be_weights_dev(c, g, tau, n_max, out);
            return;
        }
        check_weight_args(g, tau);
        if (n_max < 0) fail(FRAQ_EINVAL, sbd ? "sbd_weights: n_max must be >= 0"
                                            : "be_weights: n_max must be >= 0");
        DevBuf<double> d((size_t)n_max + 1);
        if (sbd)
            sbd_weights_dev(c, g, tau, n_max, d.p);
        else
            be_weights_dev(c, g, tau, n_max, d.p);
        FRAQ_CUDA(cudaMemcpy(out, d.p, sizeof(double) * (n_max + 1), cudaMemcpyDeviceToHost));
    });
}

int fraq_be_weights(fraq_ctx c, double g, double tau, long n_max, double* out, int mem) {
    return weights_common(c, false, g, tau, n_max, out, mem);
}
int fraq_sbd_weights(fraq_ctx c, double g, double tau, long n_max, double* out, int mem) {
    return weights_common(c, true, g, tau, n_max, out, mem);
}

int fraq_coupling_from_transition(double m, double* out) {
    // cq_weights.cpp:61-67
    return guarded([&] {
        if (!(m > 0.0) || !(m <= 1.0))
            fail(FRAQ_EINVAL,
                 "coupling_from_transition: m must be in (0,1], got " + std::to_string(m));
        if (m == 0.5)
            fail(FRAQ_EINVAL,
                 "coupling_from_transition: m = 1/2 makes the transition matrix singular");
        *out = (1.0 - m) / (2.0 * m - 1.0);
    });
}

// ------------------------------------------------------------------ L2 kernels
int fraq_build_be_kernel(fraq_ctx c, double g, double tau, int np, fraq_kernel_t* out) {
    return guarded(c, [&] {
        check_ctx(c);
        build_be_kernel_dev(c, g, tau, np, out);
    });
}

int fraq_build_sbd_kernel(fraq_ctx c, double g, double tau, int np1, int np2, int nh,
                          fraq_kernel_t* out) {
    return guarded(c, [&] {
        check_ctx(c);
        build_sbd_kernel_dev(c, g, tau, np1, np2, nh, out);
    });
}

int fraq_default_sbd_head(double g) { return g <= 0.5 ? 15 : 17; }

int fraq_fold_kernel(const fraq_kernel_t* k, int max_head, fraq_kernel_t* out, int* fold_levels) {
    return guarded([&] {
        if (!k || !out) fail(FRAQ_EINVAL, "fold_kernel: null kernel");
        if (k->np1 < 0 || k->np2 < 0 || k->np1 > FRAQ_MAX_POINTS || k->np2 > FRAQ_MAX_POINTS ||
            k->n_head < 2 || k->n_head > FRAQ_MAX_HEAD)
            fail(FRAQ_EINVAL, "fold_kernel: malformed kernel tables");
        fraq_kernel_t tmp;
        const int M = fold_kernel(*k, max_head, &tmp);
        if (M > 0)
            *out = tmp;
        else if (out != k)
            *out = *k;
        if (fold_levels) *fold_levels = M;
    });
}

int fraq_build_be_kernel_auto(fraq_ctx c, double g, double tau, fraq_budget_t* b,
                              fraq_kernel_t* out) {
    return guarded(c, [&] {
        check_ctx(c);
        build_kernel_auto_dev(c, false, 1, &g, tau, b, out);
    });
}

int fraq_build_sbd_kernel_auto(fraq_ctx c, double g, double tau, fraq_budget_t* b,
                               fraq_kernel_t* out) {
    return guarded(c, [&] {
        check_ctx(c);
        build_kernel_auto_dev(c, true, 1, &g, tau, b, out);
    });
}

int fraq_build_kernels_auto(fraq_ctx c, int sbd, int n, const double* gammas, double tau,
                            fraq_budget_t* budgets, fraq_kernel_t* out) {
    return guarded(c, [&] {
        check_ctx(c);
        build_kernel_auto_dev(c, sbd != 0, n, gammas, tau, budgets, out);
    });
}

int fraq_reconstruct(fraq_ctx c, const fraq_kernel_t* k, long n, const long* idx, double* out) {
    return guarded(c, [&] {
        check_ctx(c);
        reconstruct_dev(c, k, n, idx, out);
    });
}

int fraq_kernel_error_report(fraq_ctx c, const fraq_kernel_t* k, long n_max, double* eps,
                             double* max_eps, long* argmax) {
    return guarded(c, [&] {
        check_ctx(c);
        kernel_error_report_dev(c, k, n_max, eps, max_eps, argmax);
    });
}

// ------------------------------------------------------------------ L2 histories
int fraq_hist_create(fraq_ctx c, int n_groups, const fraq_kernel_t* const* kernels,
                     const long* dims, int variant, fraq_hist* out) {
    return guarded(c, [&] { hist_create(c, n_groups, kernels, dims, variant, out); });
}
int fraq_hist_destroy(fraq_hist h) {
    return guarded_hist(h, [&] { hist_destroy(h); });
}
int fraq_hist_info(fraq_hist h, long* level, long* appended, long* dim) {
    return guarded_hist(h, [&] { hist_info(h, level, appended, dim); });
}
int fraq_hist_push(fraq_hist h, const double* v, int mem) {
    return guarded_hist(h, [&] { hist_push(h, v, mem); });
}
int fraq_hist_advance(fraq_hist h) {
    return guarded_hist(h, [&] { hist_advance(h); });
}
int fraq_hist_append(fraq_hist h, const double* v, int mem) {
    return guarded_hist(h, [&] { hist_append(h, v, mem); });
}
int fraq_hist_history_sum(fraq_hist h, double* out, int mem) {
    return guarded_hist(h, [&] { hist_output(h, 1, out, mem); });
}
int fraq_hist_derivative(fraq_hist h, double* out, int mem) {
    return guarded_hist(h, [&] { hist_output(h, 2, out, mem); });
}
int fraq_hist_lagged(fraq_hist h, long depth, double* out, int mem) {
    return guarded_hist(h, [&] { hist_lagged(h, depth, out, mem); });
}
int fraq_hist_run(fraq_hist h, const double* U, long ldu, long n_steps, double* D, long ldd,
                  int mem) {
    return guarded_hist(h, [&] { hist_run(h, U, ldu, n_steps, D, ldd, mem); });
}
int fraq_hist_last_path(fraq_hist h) {
    if (!h) return -1;
    std::lock_guard<std::recursive_mutex> lock(hist_ctx(h)->mu);
    return hist_last_path(h);
}

int fraq_hist_path_info(fraq_hist h, long* launches, int n_groups, int* fir) {
    return guarded_hist(h, [&] { hist_path_info(h, launches, n_groups, fir); });
}

// ------------------------------------------------------------------ direct CQ
int fraq_direct_cq(fraq_ctx c, int sbd, double g, double tau, const double* U, long ldu,
                   long n_steps, long dim, double* D, long ldd, int mem) {
    return guarded(c, [&] {
        check_ctx(c);
        check_weight_args(g, tau);
        if (n_steps < 0 || dim < 0 || ldu < dim || ldd < dim)
            fail(FRAQ_EINVAL, "direct_cq: bad shape");
        if (mem == FRAQ_DEVICE) {
            direct_cq_dev(c, sbd, g, tau, U, ldu, n_steps, dim, D, ldd);
            return;
        }
        DevBuf<double> du((size_t)n_steps * dim), dd((size_t)n_steps * dim);
        FRAQ_CUDA(cudaMemcpy2DAsync(du.p, dim * 8, U, ldu * 8, dim * 8, n_steps,
                                    cudaMemcpyHostToDevice, c->stream));
        direct_cq_dev(c, sbd, g, tau, du.p, dim, n_steps, dim, dd.p, dim);
        FRAQ_CUDA(cudaMemcpy2DAsync(D, ldd * 8, dd.p, dim * 8, dim * 8, n_steps,
                                    cudaMemcpyDeviceToHost, c->stream));
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// ------------------------------------------------------------------ L4
void fraq_kconf_default(fraq_kconf_t* c) {
    c->be_points = 64;
    c->sbd_points_1 = 41;
    c->sbd_points_2 = 41;
    c->sbd_head = 0;
    c->eps_tol = 1e-12;
    c->auto_size = 1;
    c->solver = FRAQ_SOLVER_AUTO;
}

int fraq_run_2d(fraq_ctx c, double alpha1, double alpha2, double coupling_a, int grid_m,
                double t_final, long n_steps, int scheme, const fraq_kconf_t* kconf,
                const double* g1_0, const double* g2_0, double* g1, double* g2,
                fraq_run_info_t* info) {
    return guarded(c, [&] {
        check_ctx(c);
        ffpe_run_2d(c, alpha1, alpha2, coupling_a, grid_m, t_final, n_steps, scheme, kconf, g1_0,
                    g2_0, g1, g2, info);
    });
}

int fraq_dst2d(fraq_ctx c, int grid_m, int n_fields, const double* in, double* out, int inverse,
               int mem) {
    return guarded(c, [&] {
        check_ctx(c);
        dst2d(c, grid_m, n_fields, in, out, inverse != 0, mem);
    });
}

int fraq_dst_cols(fraq_ctx c, int grid_m, long n_cols, const double* in, double* out, int inverse,
                  int mem) {
    return guarded(c, [&] {
        check_ctx(c);
        dst_cols(c, grid_m, n_cols, in, out, inverse != 0, mem);
    });
}

int fraq_modal_run(fraq_ctx c, double alpha1, double alpha2, double coupling_a, double t_final,
                   long n_steps, int scheme, const fraq_kconf_t* kconf, long n_modes,
                   const double* lam, const double* c0, double* cN, int mem,
                   fraq_run_info_t* info) {
    return guarded(c, [&] {
        check_ctx(c);
        modal_run_modes(c, alpha1, alpha2, coupling_a, t_final, n_steps, scheme, kconf, n_modes,
                        lam, c0, cN, mem, info);
    });
}

int fraq_run(fraq_ctx c, const fraq_spec_t* specs, int n_inst, int scheme,
             const fraq_kconf_t* kconf, double* g1, double* g2, fraq_run_info_t* info) {
    return guarded(c, [&] {
        check_ctx(c);
        ffpe_run(c, specs, n_inst, scheme, kconf, g1, g2, info, nullptr, nullptr);
    });
}

int fraq_run_observed(fraq_ctx c, const fraq_spec_t* spec, int scheme, const fraq_kconf_t* kconf,
                      fraq_observer_fn fn, void* user, double* g1, double* g2,
                      fraq_run_info_t* info) {
    return guarded(c, [&] {
        check_ctx(c);
        ffpe_run(c, spec, 1, scheme, kconf, g1, g2, info, fn, user);
    });
}

// ------------------------------------------------------------------ single-step API
}  // extern "C"

struct fraq_stepper_s {
    fraq_ctx ctx;
    PhysStepper* p;
};
struct fraq_block_s {
    fraq_ctx ctx;
    BlockDev* p;
};
struct fraq_banded_s {
    fraq_ctx ctx;
    BandedDev* p;
};

namespace {
template <class H, class F>
int guarded_obj(H h, const char* what, F&& f) {
    if (!h) return guarded([&] { fail(FRAQ_EINVAL, std::string("null ") + what); });
    return guarded(h->ctx, [&] {
        check_ctx(h->ctx);
        f();
    });
}
}  // namespace

extern "C" {

int fraq_stepper_create(fraq_ctx c, const fraq_spec_t* spec, int scheme,
                        const fraq_kconf_t* kconf, fraq_stepper* out) {
    return guarded(c, [&] {
        check_ctx(c);
        if (!spec || !out) fail(FRAQ_EINVAL, "stepper: null argument");
        PhysStepper* p = nullptr;
        stepper_create(c, spec, scheme, kconf, &p);
        *out = new fraq_stepper_s{c, p};
    });
}
int fraq_stepper_step(fraq_stepper st, long n_steps) {
    return guarded_obj(st, "stepper", [&] { stepper_step(st->p, n_steps); });
}
int fraq_stepper_state(fraq_stepper st, double* g1, double* g2, long* step) {
    return guarded_obj(st, "stepper", [&] { stepper_state(st->p, g1, g2, step); });
}
int fraq_stepper_kernel_eps(fraq_stepper st, double* eps1, double* eps2) {
    return guarded_obj(st, "stepper", [&] { stepper_eps(st->p, eps1, eps2); });
}
int fraq_stepper_time_split(fraq_stepper st, long n_steps, double* ms_hist, double* ms_solve) {
    return guarded_obj(st, "stepper", [&] {
        if (!ms_hist || !ms_solve) fail(FRAQ_EINVAL, "stepper: null output");
        stepper_time_split(st->p, n_steps, ms_hist, ms_solve);
    });
}
int fraq_stepper_destroy(fraq_stepper st) {
    if (!st) return FRAQ_OK;
    const int r = guarded_obj(st, "stepper", [&] { stepper_destroy(st->p); });
    delete st;
    return r;
}

int fraq_block_create(fraq_ctx c, double d01, double d02, double coupling_a, double tau,
                      int grid_m, double h, double bdf_lead, fraq_block* out) {
    return guarded(c, [&] {
        check_ctx(c);
        if (!out) fail(FRAQ_EINVAL, "BlockSystem: null out");
        BlockDev* p = nullptr;
        block_create(c, d01, d02, coupling_a, tau, grid_m, h, bdf_lead, &p);
        *out = new fraq_block_s{c, p};
    });
}
int fraq_block_solve(fraq_block b, const double* rhs1, const double* rhs2, double* g1,
                     double* g2, int mem) {
    return guarded_obj(b, "BlockSystem", [&] { block_solve(b->p, rhs1, rhs2, g1, g2, mem); });
}
int fraq_block_destroy(fraq_block b) {
    if (!b) return FRAQ_OK;
    const int r = guarded_obj(b, "BlockSystem", [&] { block_destroy(b->p); });
    delete b;
    return r;
}
int fraq_laplacian_apply(fraq_ctx c, int grid_m, double h, const double* x, double* y, int mem) {
    return guarded(c, [&] {
        check_ctx(c);
        laplacian_apply(c, grid_m, h, x, y, mem);
    });
}

int fraq_banded_create(fraq_ctx c, int n, int kl, int ku, fraq_banded* out) {
    return guarded(c, [&] {
        check_ctx(c);
        if (!out) fail(FRAQ_EINVAL, "BandedLU: null out");
        BandedDev* p = nullptr;
        banded_create(c, n, kl, ku, &p);
        *out = new fraq_banded_s{c, p};
    });
}
int fraq_banded_set(fraq_banded b, int row, int col, double value) {
    return guarded_obj(b, "BandedLU", [&] { *banded_at(b->p, row, col) = value; });
}
int fraq_banded_get(fraq_banded b, int row, int col, double* value) {
    return guarded_obj(b, "BandedLU", [&] { *value = *banded_at(b->p, row, col); });
}
int fraq_banded_assign(fraq_banded b, const double* ab) {
    return guarded_obj(b, "BandedLU", [&] { banded_assign(b->p, ab); });
}
int fraq_banded_factorize(fraq_banded b) {
    return guarded_obj(b, "BandedLU", [&] { banded_factorize(b->p); });
}
int fraq_banded_solve(fraq_banded b, double* rhs, int mem) {
    return guarded_obj(b, "BandedLU", [&] { banded_solve(b->p, rhs, mem); });
}
int fraq_banded_destroy(fraq_banded b) {
    if (!b) return FRAQ_OK;
    const int r = guarded_obj(b, "BandedLU", [&] { banded_destroy(b->p); });
    delete b;
    return r;
}

}  // extern "C"
