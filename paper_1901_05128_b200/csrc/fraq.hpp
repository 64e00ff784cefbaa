// fraq.hpp -- C++ mirror of the reference `fraq` headers (proj/include/fraq/*.hpp) on top of the
// B200 C ABI (include/fraqcu.h).
//
// Same namespace, class, function and field names, argument meaning and exception types as the
// reference (gauss_jacobi.hpp, cq_weights.hpp, fast_kernel.hpp, fpfp.hpp), so reference call
// sites compile unchanged against this header.  Every compute call runs on the GPU through the
// C ABI; there is no CPU fallback (no CUDA device -> std::runtime_error).
//
// Differences, all additive:
//   * BeHistory / SbdHistory own a device history (fraq_hist); lagged() returns a span into a
//     host mirror that stays valid until the next call on the object;
//   * run(U, n_steps, D) batched evaluation (host or device pointers) on the histories;
//   * run_batch() solves many FFPE instances at once (BASELINE C5).
#pragma once

#include <cstddef>
#include <functional>
#include <memory>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "fraqcu.h"

namespace fraq {

// ------------------------------------------------------------------ runtime
/// Device of the process-wide context: FRAQ_DEVICE, else 0.
int default_device();
/// Process-wide context on default_device(), created lazily.
fraq_ctx default_context();
/// Throws the reference exception type matching a fraqcu status code.
void check(int status);

// ------------------------------------------------------------------ gauss_jacobi.hpp
struct JacobiRule {
    double exponent_a = 0.0;
    double exponent_b = 0.0;
    std::vector<double> nodes;
    std::vector<double> weights;
    std::size_t size() const { return nodes.size(); }
};

double gamma_fn(double x);
double inv_gamma_product(double alpha);
double jacobi_moment0(double exponent_a, double exponent_b);
double jacobi_moment(double exponent_a, double exponent_b, int k);
JacobiRule gauss_jacobi(double exponent_a, double exponent_b, int n_points);

// ------------------------------------------------------------------ cq_weights.hpp
enum class CqScheme { BE, SBD };

struct WeightTable {
    CqScheme scheme = CqScheme::BE;
    double alpha = 0.0;
    double tau = 1.0;
    std::vector<double> weights;
    double operator[](std::size_t i) const { return weights[i]; }
    std::size_t size() const { return weights.size(); }
};

WeightTable be_weights(double alpha, double tau, long n_max);
WeightTable sbd_weights(double alpha, double tau, long n_max);
double coupling_from_transition(double m);

// ------------------------------------------------------------------ fast_kernel.hpp
struct FastKernelBE {
    double alpha = 0.0;
    double tau = 1.0;
    double head[2] = {0.0, 0.0};
    std::vector<double> node_weights;
    std::vector<double> ratios;
    std::size_t n_points() const { return ratios.size(); }
    double reconstruct(long i) const;
};

struct FastKernelSBD {
    double alpha = 0.0;
    double tau = 1.0;
    int n_head = 3;
    std::vector<double> head;
    std::vector<double> mult1;
    std::vector<double> ratio1;
    std::vector<double> mult2;
    std::vector<double> ratio2;
    double reconstruct(long i) const;
};

struct KernelErrorReport {
    double alpha = 0.0;
    double tau = 1.0;
    long head_len = 0;
    long max_index = 0;
    std::vector<double> eps;
    double max_eps = 0.0;
    long argmax = 0;
};

FastKernelBE build_be_kernel(double alpha, double tau, int n_points);
FastKernelSBD build_sbd_kernel(double alpha, double tau, int n_points_1, int n_points_2,
                               int n_head);
int default_sbd_head(double alpha);
/// B200 addition (fraq_fold_kernel): the fast-decaying nodes folded into a longer exact head; the
/// result is an SBD-format kernel equal to `k` below fp64 rounding (`levels`: head levels added).
FastKernelSBD fold_kernel(const FastKernelBE& k, int max_head = 96, int* levels = nullptr);
FastKernelSBD fold_kernel(const FastKernelSBD& k, int max_head = 96, int* levels = nullptr);
KernelErrorReport kernel_error_report(const FastKernelBE& k, long n_max);
KernelErrorReport kernel_error_report(const FastKernelSBD& k, long n_max);

struct KernelBudget {
    long horizon = 0;
    double eps_tol = 1e-12;
    int max_points = 256;
    int max_head = 256;
    double achieved_eps = 0.0;
};

FastKernelBE build_be_kernel_auto(double alpha, double tau, KernelBudget& budget);
FastKernelSBD build_sbd_kernel_auto(double alpha, double tau, KernelBudget& budget);

enum class HistoryVariant { standalone, scheme };

// flat conversions (the ABI's value type)
fraq_kernel_t to_flat(const FastKernelBE& k);
fraq_kernel_t to_flat(const FastKernelSBD& k);
FastKernelBE be_from_flat(const fraq_kernel_t& f);
FastKernelSBD sbd_from_flat(const fraq_kernel_t& f);

/// Common device history implementation (one or several DOF groups).
class DeviceHistory {
public:
    DeviceHistory(const std::vector<fraq_kernel_t>& kernels, const std::vector<long>& dims,
                  HistoryVariant variant);
    ~DeviceHistory();
    DeviceHistory(const DeviceHistory&) = delete;
    DeviceHistory& operator=(const DeviceHistory&) = delete;
    DeviceHistory(DeviceHistory&&) noexcept;
    DeviceHistory& operator=(DeviceHistory&&) noexcept;

    void push(std::span<const double> value);
    void advance();
    void append(std::span<const double> value);
    long level() const;
    long appended() const;
    std::size_t dim() const { return dim_; }
    void history_sum(std::span<double> out) const;
    void derivative(std::span<double> out) const;
    std::span<const double> lagged(long depth) const;
    /// n_steps x (push U row; derivative -> D row).  mem: FRAQ_HOST or FRAQ_DEVICE.
    void run(const double* U, long ldu, long n_steps, double* D, long ldd, int mem = FRAQ_HOST);
    int last_path() const;
    /// kernels launched by path (fraq_hist_path_info) and K5e's per-group (M, long nodes, window)
    std::vector<long> launches() const;
    std::vector<int> fir_info() const;
    fraq_hist handle() const { return h_; }

private:
    fraq_hist h_ = nullptr;
    std::size_t dim_ = 0;
    std::size_t n_groups_ = 0;
    mutable std::vector<double> lag_;
};

/// BeHistory (fast_kernel.hpp:87-116) on the device.
class BeHistory : public DeviceHistory {
public:
    BeHistory(const FastKernelBE& kernel, HistoryVariant variant, std::size_t dim);
};

/// SbdHistory (fast_kernel.hpp:120-146) on the device.
class SbdHistory : public DeviceHistory {
public:
    SbdHistory(const FastKernelSBD& kernel, HistoryVariant variant, std::size_t dim);
};

// ------------------------------------------------------------------ block_solver.hpp
/// Tridiagonal stencil (-1, 2, -1)/h^2 on M interior nodes, homogeneous Dirichlet
/// (block_solver.hpp:10-22).  apply() runs on the device.
struct DiscreteLaplacian {
    int grid_m = 1;
    double h = 0.5;

    DiscreteLaplacian() = default;
    DiscreteLaplacian(int m, double length) : grid_m(m), h(length / (m + 1)) {}

    /// y = A x
    void apply(std::span<const double> x, std::span<double> y) const;

    /// lambda_k = (4/h^2) sin^2(k pi h / (2L)), k = 1..M.  Test oracle.
    double eigenvalue(int k, double length) const;
};

/// General banded LU with partial pivoting, LAPACK gbtrf storage (block_solver.hpp:25-36).
/// at() assembles into a host copy; factorize() and solve() run on the device.
class BandedLU {
public:
    BandedLU(int n, int kl, int ku);
    ~BandedLU();
    BandedLU(const BandedLU&) = delete;
    BandedLU& operator=(const BandedLU&) = delete;
    BandedLU(BandedLU&&) noexcept;
    BandedLU& operator=(BandedLU&&) noexcept;

    double& at(int row, int col);  // assembly access, |row-col| <= kl/ku
    void factorize();              // throws on zero pivot
    void solve(std::span<double> rhs) const;

private:
    int n_, kl_, ku_, ldab_;
    bool factored_ = false;
    std::vector<double> ab_;
    fraq_banded b_ = nullptr;
};

/// One implicit solve of the coupled two-field block system (block_solver.hpp:38-58):
///   [ lead/tau + d01 (a + A) , -a d02 I ; -a d01 I , lead/tau + d02 (a + A) ],
/// reduced once on construction (block cyclic reduction / block Thomas), solved on the device.
class BlockSystem {
public:
    BlockSystem(double d01, double d02, double coupling_a, double tau,
                const DiscreteLaplacian& lap, double bdf_lead);
    ~BlockSystem();
    BlockSystem(const BlockSystem&) = delete;
    BlockSystem& operator=(const BlockSystem&) = delete;
    BlockSystem(BlockSystem&&) noexcept;
    BlockSystem& operator=(BlockSystem&&) noexcept;

    /// Solves into g1, g2 (each grid_m long).
    void solve(std::span<const double> rhs1, std::span<const double> rhs2,
               std::span<double> g1, std::span<double> g2) const;

private:
    int m_;
    fraq_block b_ = nullptr;
};

/// The one-shot form shared by all steppers: assemble, factorize, solve (block_solver.hpp:60-65).
void solve_block_system(double d01, double d02, double coupling_a, double tau,
                        const DiscreteLaplacian& lap, std::span<const double> rhs1,
                        std::span<const double> rhs2, std::span<double> g1,
                        std::span<double> g2, double bdf_lead = 1.0);

// ------------------------------------------------------------------ fpfp.hpp
enum class Scheme { BE, FastBE, SBD, FastSBD };
Scheme scheme_from_name(const std::string& name);
std::string scheme_name(Scheme s);
bool scheme_is_fast(Scheme s);
bool scheme_is_sbd(Scheme s);

enum class InitialData { poly_sin, indicator, custom };

struct ProblemSpec {
    double alpha1 = 0.5;
    double alpha2 = 0.5;
    double coupling_a = 0.0;
    int grid_m = 255;
    double length = 1.0;
    double t_final = 1.0;
    long n_steps = 100;
    InitialData initial = InitialData::poly_sin;
    std::vector<double> custom_g1, custom_g2;
    double tau() const { return t_final / double(n_steps); }
    double h() const { return length / double(grid_m + 1); }
};

struct StateField {
    std::vector<double> g1, g2;
    long step = 0;
};

struct KernelConfig {
    int be_points = 64;
    int sbd_points_1 = 41;
    int sbd_points_2 = 41;
    int sbd_head = 0;
    double eps_tol = 1e-12;
    bool auto_size = true;
    // addition: spatial solver of the fast schemes, FRAQ_SOLVER_PHYSICAL (reference-shaped
    // stencil + block solve), FRAQ_SOLVER_MODAL (DST eigenbasis, independent modes) or
    // FRAQ_SOLVER_AUTO (modal where it applies)
    int solver = FRAQ_SOLVER_AUTO;
};

struct RunResult {
    StateField final_state;
    double loop_seconds = 0.0;
    double setup_seconds = 0.0;
    double kernel_eps1 = 0.0;
    double kernel_eps2 = 0.0;
};

StateField initial_field(const ProblemSpec& spec);
double l2_norm(std::span<const double> v, double h);

/// fpfp.cpp:351-381 on the device.  The observer, when set, sees the initial state and every
/// accepted step (fpfp.cpp:360-375): the run then uses the physical solver and copies each level
/// back to the host (fraq_run_observed).
RunResult run(const ProblemSpec& spec, Scheme scheme, const KernelConfig& kconf = {},
              const std::function<void(long, const StateField&)>& observer = nullptr);

/// addition: run() on a caller-owned context (its own stream), e.g. one per worker thread --
/// calls on different contexts proceed concurrently on the device.
RunResult run_on(fraq_ctx ctx, const ProblemSpec& spec, Scheme scheme,
                 const KernelConfig& kconf = {},
                 const std::function<void(long, const StateField&)>& observer = nullptr);

/// 2D FFPE on the unit square (grid_m^2 interior points, five-point Laplacian), fast schemes,
/// stepped in the 2D DST eigenbasis.  Data row-major (x fastest).  No reference counterpart.
RunResult run_2d(double alpha1, double alpha2, double coupling_a, int grid_m, double t_final,
                 long n_steps, Scheme scheme, const std::vector<double>& g1_0,
                 const std::vector<double>& g2_0, const KernelConfig& kconf = {});

/// 2D DST of n_fields grid_m^2 arrays: forward coefficients c[ky][kx] = (2/(M+1))^2 S G S, or the
/// inverse synthesis G = S c S.  mem: FRAQ_HOST or FRAQ_DEVICE for in / out.
void dst2d(int grid_m, int n_fields, const double* in, double* out, bool inverse,
           int mem = FRAQ_HOST);

/// 1D pass of the same transform along the leading axis of a grid_m x n_cols array (forward
/// scale 2/(M+1), inverse 1): the slab-local step of the transposed, mode-sharded 2D DST.
void dst_cols(int grid_m, long n_cols, const double* in, double* out, bool inverse,
              int mem = FRAQ_HOST);

/// One instance (fast BE / BDF2) stepped over n_modes modes with eigenvalues lam; c0 / cN are
/// [2][n_modes] (field-major).  The per-rank work of the mode-sharded 2D solve.
RunResult modal_run(double alpha1, double alpha2, double coupling_a, double t_final,
                    long n_steps, Scheme scheme, long n_modes, const double* lam,
                    const double* c0, double* cN, int mem = FRAQ_HOST,
                    const KernelConfig& kconf = {});

// --- single-step entry points (fpfp.hpp:80-140); the state lives on the device ---

/// Classical stepper (fpfp.hpp:82-101): full solution history on the device, O(n) direct CQ
/// sums per step, block solve.  spec.n_steps is the last reachable step.
class ClassicalStepper {
public:
    ClassicalStepper(const ProblemSpec& spec, bool sbd);
    ~ClassicalStepper();
    ClassicalStepper(const ClassicalStepper&) = delete;
    ClassicalStepper& operator=(const ClassicalStepper&) = delete;
    void step();  // advances by one time level
    const StateField& state() const;
    long step_index() const { return step_; }

private:
    fraq_stepper st_ = nullptr;
    long step_ = 0;
    mutable StateField state_;
    mutable long state_at_ = -1;
};

/// Fast stepper (fpfp.hpp:103-140): exact heads, per-node accumulators (K5), factored blocks,
/// reconstructed SBD correction weights -- the reference's physical-space algorithm on the GPU.
class FastStepper {
public:
    FastStepper(const ProblemSpec& spec, bool sbd, const KernelConfig& kconf);
    ~FastStepper();
    FastStepper(const FastStepper&) = delete;
    FastStepper& operator=(const FastStepper&) = delete;
    void step();
    const StateField& state() const;
    long step_index() const { return step_; }
    double kernel_eps1() const { return eps1_; }
    double kernel_eps2() const { return eps2_; }
    /// addition: advance n levels in one stream-ordered call
    void step_n(long n);
    /// addition (diagnostics): advance n levels timing each kernel; returns {ms K5, ms K6}
    std::pair<double, double> time_split(long n);

private:
    fraq_stepper st_ = nullptr;
    long step_ = 0;
    double eps1_ = 0.0, eps2_ = 0.0;
    mutable StateField state_;
    mutable long state_at_ = -1;
};

/// Many independent instances (same grid_m, n_steps, t_final) solved together.
std::vector<RunResult> run_batch(const std::vector<ProblemSpec>& specs, Scheme scheme,
                                 const KernelConfig& kconf = {});

}  // namespace fraq
