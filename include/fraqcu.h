/*
 * fraqcu.h -- C ABI of the B200-native fast convolution-quadrature (CQ) path of arXiv 1901.05128.
 *
 * Drop-in boundary for the reference `fraq` library (/root/reference/proj).  The reference
 * exposes a C++20 header API plus a pybind11 module `_fraq`; it has no C FFI.
 * Every entry point below replaces one reference function or method, cited as path:line under
 * /root/reference/proj.  The C++ mirror of the reference headers (namespace fraq, same class and
 * function names, same exception types) and the Python module `_fraq` are thin layers over this
 * ABI: paper_1901_05128_b200/csrc/fraq.hpp and fraq_py.cpp.  INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - plain C types only: double / long / int / pointers + sizes; no torch or CUDA types;
 *   - `mem` arguments say where a buffer lives: FRAQ_HOST (pageable or pinned host memory) or
 *     FRAQ_DEVICE (a device pointer on the context's GPU, zero-copy);
 *   - all arithmetic is IEEE fp64 on the device (sm_100a); there is no CPU fallback: without a
 *     CUDA device every compute entry point returns FRAQ_ECUDA;
 *   - status codes map 1:1 onto the reference's exception types:
 *       FRAQ_EINVAL  -> std::invalid_argument    FRAQ_ELOGIC   -> std::logic_error
 *       FRAQ_ERANGE  -> std::out_of_range        FRAQ_ERUNTIME -> std::runtime_error
 *     FRAQ_ECUDA / FRAQ_ENOMEM are device failures.  fraq_last_error() returns the message of the
 *     last failure on the calling thread;
 *   - a context is bound to one device and one CUDA stream; all work is stream-ordered; calls
 *     that return values in host memory synchronize the stream.
 */
#ifndef FRAQCU_H
#define FRAQCU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FRAQ_MAX_POINTS 512 /* gauss_jacobi cap, gauss_jacobi.cpp:13 */
#define FRAQ_MAX_HEAD 512

enum {
    FRAQ_OK = 0,
    FRAQ_EINVAL = -1,
    FRAQ_ELOGIC = -2,
    FRAQ_ERANGE = -3,
    FRAQ_ERUNTIME = -4,
    FRAQ_ECUDA = -5,
    FRAQ_ENOMEM = -6
};
enum { FRAQ_HOST = 0, FRAQ_DEVICE = 1 };
/* HistoryVariant, fast_kernel.hpp:79-82 */
enum { FRAQ_STANDALONE = 0, FRAQ_SCHEME = 1 };
/* Scheme, fpfp.hpp:14 */
enum { FRAQ_BE = 0, FRAQ_FASTBE = 1, FRAQ_SBD = 2, FRAQ_FASTSBD = 3 };
/* InitialData, fpfp.hpp:21 */
enum { FRAQ_POLY_SIN = 0, FRAQ_INDICATOR = 1, FRAQ_CUSTOM = 2 };

typedef struct fraq_ctx_s* fraq_ctx;
typedef struct fraq_hist_s* fraq_hist;
typedef struct fraq_stepper_s* fraq_stepper;
typedef struct fraq_block_s* fraq_block;
typedef struct fraq_banded_s* fraq_banded;

/* Compressed kernel tables: FastKernelBE (sbd = 0; m1 = node_weights, r1 = ratios, head[0..1])
 * or FastKernelSBD (sbd = 1; families (m1, r1) and (m2, r2), head[0..n_head-1]).
 * fast_kernel.hpp:13-39.  Plain value type; the device copy is made when a history uses it. */
typedef struct {
    int sbd;
    double gamma; /* the CQ exponent ("alpha" in the reference kernel structs) */
    double tau;
    int n_head; /* 2 for BE */
    int np1, np2;
    double head[FRAQ_MAX_HEAD];
    double m1[FRAQ_MAX_POINTS], r1[FRAQ_MAX_POINTS];
    double m2[FRAQ_MAX_POINTS], r2[FRAQ_MAX_POINTS];
} fraq_kernel_t;

/* KernelBudget, fast_kernel.hpp:68-74. */
typedef struct {
    long horizon;
    double eps_tol;
    int max_points;
    int max_head;
    double achieved_eps; /* out */
} fraq_budget_t;

/* ProblemSpec, fpfp.hpp:27-41. */
typedef struct {
    double alpha1, alpha2, coupling_a, length, t_final;
    int grid_m;
    long n_steps;
    int initial;              /* FRAQ_POLY_SIN / FRAQ_INDICATOR / FRAQ_CUSTOM */
    const double* custom_g1;  /* host, grid_m values (custom only) */
    const double* custom_g2;
} fraq_spec_t;

/* KernelConfig, fpfp.hpp:50-57, plus the spatial solver of the fast schemes (addition):
 * FRAQ_SOLVER_PHYSICAL (0) = the reference's physical-space stepper (stencil RHS + 2x2-block
 * tridiagonal solve per level); FRAQ_SOLVER_MODAL (1) = the same scheme stepped in the DST
 * eigenbasis (the reference's mode-space oracle, test_fpfp.cpp:21-180), every mode an independent
 * 2x2 recursion -- exact in exact arithmetic, better conditioned in fp64; FRAQ_SOLVER_AUTO (2,
 * default) = MODAL for the fast schemes without an observer (PHYSICAL if the modal path rejects
 * the kernels, e.g. a head window over 56 levels), PHYSICAL otherwise. */
enum { FRAQ_SOLVER_PHYSICAL = 0, FRAQ_SOLVER_MODAL = 1, FRAQ_SOLVER_AUTO = 2 };
typedef struct {
    int be_points, sbd_points_1, sbd_points_2, sbd_head;
    double eps_tol;
    int auto_size;
    int solver;
} fraq_kconf_t;

/* RunResult minus the state, fpfp.hpp:59-65, plus the chosen table sizes. */
typedef struct {
    double loop_seconds, setup_seconds;
    double kernel_eps1, kernel_eps2;
    int np[4];     /* field 1 (np1, np2), field 2 (np1, np2) */
    int n_head[2];
} fraq_run_info_t;

/* ---------------------------------------------------------------- context / errors */
int fraq_ctx_create(int device, void* cuda_stream /* cudaStream_t, NULL = own stream */,
                    fraq_ctx* out);
int fraq_ctx_destroy(fraq_ctx ctx);
int fraq_ctx_synchronize(fraq_ctx ctx);
void* fraq_ctx_stream(fraq_ctx ctx);
int fraq_last_error(char* buf, size_t n);
int fraq_version(void);

/* ---------------------------------------------------------------- L0 quadrature
 * gauss_jacobi.hpp:19-35 / gauss_jacobi.cpp:108-204.  Nodes by Sturm bisection on the Jacobi
 * matrix (one thread per eigenvalue), one guarded Newton polish, Christoffel weights: device
 * setup kernel K2.  Output in host memory (n values each). */
double fraq_gamma(double x);
double fraq_inv_gamma_product(double g);
int fraq_jacobi_moment(double a, double b, int k, double* out);
int fraq_gauss_jacobi(fraq_ctx ctx, double a, double b, int n, double* nodes, double* weights);

/* ---------------------------------------------------------------- L1 classical weights
 * cq_weights.hpp:23-33 / cq_weights.cpp:19-67: device kernel K1.  out holds n_max+1 values. */
int fraq_be_weights(fraq_ctx ctx, double g, double tau, long n_max, double* out, int mem);
int fraq_sbd_weights(fraq_ctx ctx, double g, double tau, long n_max, double* out, int mem);
int fraq_coupling_from_transition(double m, double* out);

/* ---------------------------------------------------------------- L2 compressed kernels
 * fast_kernel.hpp:53-77 / fast_kernel.cpp:38-256: device kernels K2 (rules), K3 (fold),
 * K4 (error scan + auto sizing, same growth sequence and caps as the reference). */
int fraq_build_be_kernel(fraq_ctx ctx, double g, double tau, int n_points, fraq_kernel_t* out);
int fraq_build_sbd_kernel(fraq_ctx ctx, double g, double tau, int n_points_1, int n_points_2,
                          int n_head, fraq_kernel_t* out);
int fraq_default_sbd_head(double g);
int fraq_build_be_kernel_auto(fraq_ctx ctx, double g, double tau, fraq_budget_t* budget,
                              fraq_kernel_t* out);
int fraq_build_sbd_kernel_auto(fraq_ctx ctx, double g, double tau, fraq_budget_t* budget,
                               fraq_kernel_t* out);
/* Batched auto sizing for parameter sweeps: n kernels at once (one CTA per exponent). */
int fraq_build_kernels_auto(fraq_ctx ctx, int sbd, int n, const double* gammas, double tau,
                            fraq_budget_t* budgets, fraq_kernel_t* out);
/* FastKernel*::reconstruct (fast_kernel.cpp:38-52) at n indices. */
int fraq_reconstruct(fraq_ctx ctx, const fraq_kernel_t* k, long n, const long* idx, double* out);
/* kernel_error_report (fast_kernel.cpp:126-180): eps (nullable, host, n_max+1 values). */
int fraq_kernel_error_report(fraq_ctx ctx, const fraq_kernel_t* k, long n_max, double* eps,
                             double* max_eps, long* argmax);

/* The short-node fold as a kernel rewrite (host only; no reference counterpart -- it rewrites
 * the reference's FastKernelBE / FastKernelSBD tables, fast_kernel.hpp:13-39, into an equivalent
 * kernel): a node with |r_j|^M <= 2^-70 has forgotten everything older than M levels, so the
 * kernel (head d_0..d_(L-1); nodes fed at lag L) equals, to below fp64 rounding, the kernel with
 * the head c_0..c_(L+M-1), c_i = reconstruct(i) (fast_kernel.cpp:38-52) for i >= L, and only the
 * slow nodes.  `out` is in the SBD table format (generic head; the feed convention
 * mult * ratio^(n_head - 3), fast_kernel.cpp:337-340, absorbs r^M).  M is the multiple of 8 with
 * L + M <= max_head that minimises the bytes a per-level history pass moves; *fold_levels = 0
 * and `out` = *k when nothing folds.  The physical FFPE stepper builds its histories from such
 * kernels; K5e / K5f / K13 use the same node split. */
int fraq_fold_kernel(const fraq_kernel_t* k, int max_head, fraq_kernel_t* out, int* fold_levels);

/* ---------------------------------------------------------------- L2 history states
 * BeHistory / SbdHistory (fast_kernel.hpp:87-146, fast_kernel.cpp:261-409) on the device.
 * A history holds n_groups contiguous DOF groups, group g having dims[g] DOFs and its own kernel
 * (one group = the reference object with dim = dims[0]).  State layout: per group
 * y[node][dof] (DOF contiguous, padded), lag ring [cap][dof].  Sequencing checks and error codes
 * follow the reference exactly; state-observing calls run the fused step kernel K5. */
int fraq_hist_create(fraq_ctx ctx, int n_groups, const fraq_kernel_t* const* kernels,
                     const long* dims, int variant, fraq_hist* out);
int fraq_hist_destroy(fraq_hist h);
int fraq_hist_info(fraq_hist h, long* level, long* appended, long* dim);
int fraq_hist_push(fraq_hist h, const double* value, int mem);
int fraq_hist_advance(fraq_hist h);
int fraq_hist_append(fraq_hist h, const double* value, int mem);
int fraq_hist_history_sum(fraq_hist h, double* out, int mem);
int fraq_hist_derivative(fraq_hist h, double* out, int mem);
int fraq_hist_lagged(fraq_hist h, long depth, double* out, int mem);
/* Batched standalone evaluation: pushes U[n * ldu + 0 .. dim) for n = 0..n_steps-1 and writes the
 * derivative after each push to D[n * ldd + ...] (NaN where the reference would throw
 * "too early"); D may be NULL.  Equivalent to n_steps x (push; derivative).  Uses the
 * temporally blocked kernel K5d (8-level block GEMMs on the fp64 tensor cores, the history kept
 * on chip across the whole call); mem = FRAQ_HOST streams U / D through pinned staging buffers
 * with the copies overlapping the kernels. */
int fraq_hist_run(fraq_hist h, const double* U, long ldu, long n_steps, double* D, long ldd,
                  int mem);
/* Which kernel the last fraq_hist_run used: 0 = per-level K5 (calls under 4 levels, or more than
 * 512 nodes), 2 = K5c (lane-per-DOF DFMA blocked: FRAQ_K5C=1, or head windows over 32 levels),
 * 3 = K5d (DMMA block GEMMs; the first levels of a history and ragged tails), 4 = K5e (K5d's
 * block GEMMs on the slow nodes + the fast-decaying nodes as an exact FIR window; the steady
 * state, default).  (1 was the retired warp-per-4-DOF kernel K5b.) */
int fraq_hist_last_path(fraq_hist h);
/* Diagnostics of this history's kernels.  launches[0..5]: kernels launched so far by path
 * (0 per-level K5, 1 short-state rebuilds after K5e / K5f, 2 K5c, 3 K5d, 4 K5e, 5 K5f: the
 * per-level step in K5e's folded form -- push / derivative / history_sum in the steady state of
 * a pure push sequence, FRAQ_NO_K5F=1 keeps them on K5).  fir[3 g + 0..2]
 * for group g < n_groups: K5e's FIR length M (levels; 0 = no node folded), the nodes kept as
 * recurrences, the combined input window (rows) -- zeros while K5e has no plan.  Either pointer
 * may be NULL. */
int fraq_hist_path_info(fraq_hist h, long* launches, int n_groups, int* fir);

/* ---------------------------------------------------------------- direct CQ (K10)
 * The classical O(N^2) CQ sum D[n] = sum_{i<=n} d_i U[n-i] with the exact weights of
 * be_weights / sbd_weights (the reference's direct harness sum, test_fast_kernel.cpp:27-41,
 * acceptance_main.cpp:158-159) as a lower-triangular Toeplitz x signal GEMM on the fp64 tensor
 * cores (DMMA).  U rows n = 0..n_steps-1 of dim values (leading dim ldu), D likewise. */
int fraq_direct_cq(fraq_ctx ctx, int sbd, double g, double tau, const double* U, long ldu,
                   long n_steps, long dim, double* D, long ldd, int mem);

/* ---------------------------------------------------------------- L4 FFPE
 * run() (fpfp.cpp:351-381) for n_inst independent instances (BASELINE C3: 1, C5: 4096) solved
 * together on the device.  kconf->solver selects the spatial solver of the fast schemes:
 * PHYSICAL = histories K5 for both fields, RHS + 2x2-block tridiagonal solve K6, SBD correction
 * sequence K7 (the reference's FastStepper shape); MODAL / AUTO (default) = DST (K12, DMMA),
 * per-mode stepping on DMMA (K13), inverse DST.  Classical schemes always run physically.
 * g1/g2: host, n_inst * grid_m values (row per instance). */
void fraq_kconf_default(fraq_kconf_t* c);
int fraq_run(fraq_ctx ctx, const fraq_spec_t* specs, int n_inst, int scheme,
             const fraq_kconf_t* kconf, double* g1, double* g2, fraq_run_info_t* info);
/* run() with the reference's per-step observer (fpfp.cpp:360-365): fn(n, g1, g2, grid_m, user)
 * sees the initial state (n = 0) and every accepted level; single instance.  Each call copies
 * the level back to the host, so the loop time includes those copies. */
typedef void (*fraq_observer_fn)(long n, const double* g1, const double* g2, int grid_m,
                                 void* user);
/* Two-dimensional FFPE on the unit square (BASELINE C4; no reference capability -- the reference
 * is 1D only): grid_m x grid_m interior points, five-point Laplacian, homogeneous Dirichlet, fast
 * BE / BDF2 in time, stepped in the 2D DST eigenbasis (lambda_k + lambda_l).  g1_0 / g2_0 and the
 * outputs g1 / g2 are grid_m * grid_m values, row-major (x fastest).  Scheme FRAQ_FASTBE or
 * FRAQ_FASTSBD. */
int fraq_run_2d(fraq_ctx ctx, double alpha1, double alpha2, double coupling_a, int grid_m,
                double t_final, long n_steps, int scheme, const fraq_kconf_t* kconf,
                const double* g1_0, const double* g2_0, double* g1, double* g2,
                fraq_run_info_t* info);
/* Building blocks of the mode-sharded 2D solve, no reference counterpart:
 * fraq_dst2d: n_fields grid_m x grid_m arrays; forward (inverse = 0) c[ky][kx] =
 * (2/(M+1))^2 sum_y,x S[ky][y] S[kx][x] G[y][x], inverse (1) G = S c S, S[k][j] =
 * sin((k+1)(j+1) pi/(M+1)) -- the mode basis of the reference's mode-space oracle
 * (test_fpfp.cpp:39-54) in 2D.  fraq_modal_run: one instance stepped over n_modes modes with
 * eigenvalues lam[] (fast BE/BDF2, the FastStepper algebra fpfp.cpp:259-349 per mode);
 * c0 / cN: [2][n_modes] field-major.  mem: FRAQ_HOST or FRAQ_DEVICE for all arrays. */
int fraq_dst2d(fraq_ctx ctx, int grid_m, int n_fields, const double* in, double* out, int inverse,
               int mem);
/* fraq_dst_cols: the 1D pass of the same transform along the leading axis of a grid_m x n_cols
 * row-major array, out[k][c] = s sum_j S[k][j] in[j][c] with s = 2/(M+1) (forward) or 1
 * (inverse) -- K12 (one DMMA GEMM).  The slab-local step of the transposed 2D DST of the
 * mode-sharded C4 driver (x pass, NCCL all-to-all transpose, y pass). */
int fraq_dst_cols(fraq_ctx ctx, int grid_m, long n_cols, const double* in, double* out,
                  int inverse, int mem);
int fraq_modal_run(fraq_ctx ctx, double alpha1, double alpha2, double coupling_a, double t_final,
                   long n_steps, int scheme, const fraq_kconf_t* kconf, long n_modes,
                   const double* lam, const double* c0, double* cN, int mem,
                   fraq_run_info_t* info);
int fraq_run_observed(fraq_ctx ctx, const fraq_spec_t* spec, int scheme,
                      const fraq_kconf_t* kconf, fraq_observer_fn fn, void* user, double* g1,
                      double* g2, fraq_run_info_t* info);

/* ---------------------------------------------------------------- single-step API
 * ClassicalStepper / FastStepper (fpfp.hpp:96-140, fpfp.cpp:81-349): one instance in physical
 * space, advanced level by level -- the reference's stepper algorithm on the device (histories
 * K5 + RHS and 2x2-block solve K6; classical schemes: full device history and O(n) sums).
 * spec->n_steps sizes the kernels (auto sizing horizon) and is the last reachable level.
 * fraq_stepper_step(st, k): advances k levels (stream-ordered, asynchronous); the reference's
 * step() is k = 1.  fraq_stepper_state: G^n of both fields (host, grid_m values each; nullable)
 * and the step index n (state() / step_index(), fpfp.hpp:100-101,112-113); synchronizes.
 * fraq_stepper_kernel_eps: kernel_eps1() / kernel_eps2() (fpfp.hpp:114-115; 0 for classical). */
int fraq_stepper_create(fraq_ctx ctx, const fraq_spec_t* spec, int scheme,
                        const fraq_kconf_t* kconf, fraq_stepper* out);
int fraq_stepper_step(fraq_stepper st, long n_steps);
int fraq_stepper_state(fraq_stepper st, double* g1, double* g2, long* step);
int fraq_stepper_kernel_eps(fraq_stepper st, double* eps1, double* eps2);
int fraq_stepper_destroy(fraq_stepper st);
/* diagnostics: advance n_steps levels with CUDA events around every kernel; *ms_hist = summed
 * device time of the history kernels (K5, or the classical sums), *ms_solve = of the RHS +
 * block solves (K6).  The physical path's time split for bench.py. */
int fraq_stepper_time_split(fraq_stepper st, long n_steps, double* ms_hist, double* ms_solve);

/* BlockSystem (block_solver.hpp:38-58, block_solver.cpp:95-153): the coupled two-field system
 *   [ lead/tau + d01 (a + A) , -a d02 I ; -a d01 I , lead/tau + d02 (a + A) ],
 * A the Dirichlet stencil (-1, 2, -1)/h^2 on grid_m points, reduced once at creation (block
 * cyclic reduction for grid_m = 2^K - 1, else block Thomas), solved on the device.
 * fraq_block_solve: rhs1/rhs2 in, g1/g2 out (grid_m values each; mem FRAQ_HOST or FRAQ_DEVICE). */
int fraq_block_create(fraq_ctx ctx, double d01, double d02, double coupling_a, double tau,
                      int grid_m, double h, double bdf_lead, fraq_block* out);
int fraq_block_solve(fraq_block b, const double* rhs1, const double* rhs2, double* g1,
                     double* g2, int mem);
int fraq_block_destroy(fraq_block b);
/* DiscreteLaplacian::apply (block_solver.cpp:10-19): y = A x on grid_m points, spacing h. */
int fraq_laplacian_apply(fraq_ctx ctx, int grid_m, double h, const double* x, double* y, int mem);
/* BandedLU (block_solver.hpp:25-36, block_solver.cpp:28-93): general band matrix with kl sub-
 * and ku super-diagonals, LAPACK gbtrf storage.  fraq_banded_set assembles one entry (at(),
 * FRAQ_ERANGE outside the band); factorize uses partial pivoting (FRAQ_ERUNTIME on a zero
 * pivot); solve before factorize is FRAQ_ELOGIC.  Factorization and substitution run on the
 * device (sequential: the reference's general-purpose utility, not on the FFPE path). */
int fraq_banded_create(fraq_ctx ctx, int n, int kl, int ku, fraq_banded* out);
int fraq_banded_set(fraq_banded b, int row, int col, double value);
int fraq_banded_get(fraq_banded b, int row, int col, double* value);
/* the whole band at once: ab[(kl+ku+row-col) + col*(2kl+ku+1)], n*(2kl+ku+1) values (host) */
int fraq_banded_assign(fraq_banded b, const double* ab);
int fraq_banded_factorize(fraq_banded b);
int fraq_banded_solve(fraq_banded b, double* rhs, int mem);
int fraq_banded_destroy(fraq_banded b);

/* ---------------------------------------------------------------- diagnostics
 * Measured fp64 FMA throughput of the context's GPU (TFLOP/s, 2 flops per DFMA): the roofline
 * denominator of the fp64-bound temporally blocked history kernel. */
int fraq_diag_fp64_peak(fraq_ctx ctx, double* tflops);
/* fp64 tensor-core (DMMA) throughput: tflops[0] alone, tflops[1] DMMA + DFMA interleaved. */
int fraq_diag_dmma_peak(fraq_ctx ctx, double* tflops);

#ifdef __cplusplus
}
#endif
#endif /* FRAQCU_H */
