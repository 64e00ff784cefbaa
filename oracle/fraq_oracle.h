/*
 * fraq_oracle.h -- CPU restatement of the reference fast-CQ path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the parity checker for the B200 path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_1901_05128_b200) never links or calls it.
 *
 * Every function restates a function of the reference (arXiv 1901.05128, `fraq`), cited as
 * path:line under /root/reference/proj.  Parity pin: tests/test_oracle_pin.py checks this
 * restatement against the reference itself compiled from its own sources (oracle/_ref, built
 * by oracle/Makefile) and against the golden values frozen in the reference's tests
 * (tests/golden/).
 *
 * Error convention (mirrors the reference's exception types):
 *   FO_OK 0, FO_EINVAL -1 (std::invalid_argument), FO_ELOGIC -2 (std::logic_error),
 *   FO_ERANGE -3 (std::out_of_range), FO_ERUNTIME -4 (std::runtime_error).
 */
#ifndef FRAQ_ORACLE_H
#define FRAQ_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

enum { FO_OK = 0, FO_EINVAL = -1, FO_ELOGIC = -2, FO_ERANGE = -3, FO_ERUNTIME = -4 };

/* ---- L0 quadrature (gauss_jacobi.cpp) ---- */
double fo_gamma(double x);
double fo_inv_gamma_product(double g);
int fo_jacobi_moment0(double a, double b, double* out);
int fo_jacobi_moment(double a, double b, int k, double* out);
int fo_gauss_jacobi(double a, double b, int n, double* nodes, double* weights);

/* ---- L1 classical CQ weights (cq_weights.cpp) ---- */
int fo_be_weights(double g, double tau, long nmax, double* out);  /* out[nmax+1] */
int fo_sbd_weights(double g, double tau, long nmax, double* out); /* out[nmax+1] */
int fo_coupling_from_transition(double m, double* out);

/* ---- L2 compressed kernels (fast_kernel.cpp) ----
 * One struct for both schemes.  BE: n_head = 2, family 1 = (node_weights, ratios), np2 = 0.
 * SBD: two families with ratios (s+1)/(s+5) and (s+1)/2. */
typedef struct {
    int sbd;
    double gamma, tau;
    int n_head;
    double head[512];
    int np1, np2;
    double m1[512], r1[512];
    double m2[512], r2[512];
} fo_kernel;

int fo_build_be_kernel(double g, double tau, int np, fo_kernel* k);
int fo_build_sbd_kernel(double g, double tau, int np1, int np2, int n_head, fo_kernel* k);
int fo_default_sbd_head(double g);
double fo_reconstruct(const fo_kernel* k, long i);
int fo_kernel_error_report(const fo_kernel* k, long nmax, double* eps, double* max_eps,
                           long* argmax);
int fo_build_be_kernel_auto(double g, double tau, long* horizon, double eps_tol, int max_points,
                            int max_head, fo_kernel* k, double* achieved);
int fo_build_sbd_kernel_auto(double g, double tau, long* horizon, double eps_tol,
                             int max_points, int max_head, fo_kernel* k, double* achieved);

/* ---- L2 history states (fast_kernel.cpp:261-409) ---- */
typedef struct {
    const fo_kernel* k;
    long lo, dim, level, appended, cap;
    double* feed1; /* SBD: mult*ratio^(n_head-3); BE: node weights */
    double* feed2;
    double* acc1; /* [np1][dim] */
    double* acc2; /* [np2][dim] */
    double* ring; /* [cap][dim] */
} fo_hist;

int fo_hist_init(fo_hist* h, const fo_kernel* k, int scheme_variant, long dim);
void fo_hist_free(fo_hist* h);
int fo_hist_advance(fo_hist* h);
int fo_hist_append(fo_hist* h, const double* v);
int fo_hist_push(fo_hist* h, const double* v);
void fo_hist_history_sum(const fo_hist* h, double* out);
int fo_hist_lagged(const fo_hist* h, long depth, const double** out);
int fo_hist_derivative(const fo_hist* h, double* out);

/* Batched driver: pushes U[n][dim] for n = 0..n_steps-1 and writes D[n][dim] after every push
 * whose derivative is defined (NaN otherwise). */
int fo_hist_run(const fo_kernel* k, int scheme_variant, long dim, long n_steps, const double* U,
                double* D);

/* ---- direct (O(N^2)) CQ: harness sum of test_fast_kernel.cpp:27-41 over the classical table */
int fo_direct_cq(int sbd, double g, double tau, long dim, long n_steps, const double* U,
                 double* D);

/* ---- L3 spatial operator + block solve (block_solver.cpp) ---- */
void fo_laplacian_apply(int m, double h, const double* x, double* y);
double fo_laplacian_eigenvalue(int m, double h, int k, double length);
typedef struct {
    int m;
    int n, kl, ku, ldab;
    double* ab;
    int* piv;
    double d01, d02, a, lead_tau, ih2;
} fo_block;
int fo_block_init(fo_block* b, double d01, double d02, double a, double tau, int m, double h,
                  double lead);
void fo_block_free(fo_block* b);
void fo_block_solve(const fo_block* b, const double* rhs1, const double* rhs2, double* g1,
                    double* g2);

/* ---- L4 FFPE steppers (fpfp.cpp) ---- */
enum { FO_BE = 0, FO_FASTBE = 1, FO_SBD = 2, FO_FASTSBD = 3 };
typedef struct {
    double alpha1, alpha2, a, length, t_final;
    int grid_m;
    long n_steps;
    int initial; /* 0 poly_sin, 1 indicator, 2 custom */
    const double* custom_g1;
    const double* custom_g2;
} fo_spec;
typedef struct {
    int be_points, sbd_points_1, sbd_points_2, sbd_head;
    double eps_tol;
    int auto_size;
} fo_kconf;
void fo_kconf_default(fo_kconf* c);
int fo_initial_field(const fo_spec* s, double* g1, double* g2);
double fo_l2_norm(const double* v, long n, double h);
/* Runs the scheme; writes the final state.  Optional trace: if trace_every > 0, G1/G2 at
 * n % trace_every == 0 are appended to trace[...] (2*grid_m per row). */
int fo_run(const fo_spec* s, int scheme, const fo_kconf* kc, double* g1_out, double* g2_out,
           double* eps1, double* eps2, int* np_out /* [4]: np1 field1, np2 field1, ... */,
           int* nhead_out /* [2] */);

/* ---- mode-space fast FFPE stepping (test_fpfp.cpp:79-134 with fast histories) ---- */
int fo_modal_run(const fo_kernel* k1, const fo_kernel* k2, double a, double tau, long N,
                 long n_modes, const double* lam, const double* u0, const double* v0, double* uN,
                 double* vN);

#ifdef __cplusplus
}
#endif
/* extended-precision mode-space anchor on sampled modes (fraq_anchor_ld.c) */
int fo_anchor_ld(const fo_kernel* k1, const fo_kernel* k2, double a, double tau, long N, int M,
                 long nm, const int* modes, const double* g1, const double* g2, double* uN,
                 double* vN);
int fo_anchor_modes_ld(const fo_kernel* k1, const fo_kernel* k2, double a, double tau, long N,
                       long nm, const double* lam2, const double* u02, const double* v02,
                       double* uN, double* vN);

#endif
