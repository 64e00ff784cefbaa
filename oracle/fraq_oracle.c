/*
 * fraq_oracle.c -- CPU restatement of the reference fast-CQ path.
 *
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's CPU legs
 * as the checker.  Never part of the product path.  See fraq_oracle.h for the pinning story.
 *
 * Citations are path:line under /root/reference/proj.
 */
#include "fraq_oracle.h"

#include <float.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FO_PI 3.14159265358979323846

/* ===================================================================== L0 quadrature */

/* Lanczos approximation, g = 7, nine published coefficients; reflection below 1/2.
 * Follows gauss_jacobi.cpp:108-123. */
double fo_gamma(double x) {
    static const double c[9] = {0.99999999999980993,  676.5203681218851,     -1259.1392167224028,
                                771.32342877765313,   -176.61502916214059,   12.507343278686905,
                                -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7};
    if (x < 0.5) return FO_PI / (sin(FO_PI * x) * fo_gamma(1.0 - x));
    const double z = x - 1.0;
    double s = c[0];
    for (int i = 1; i < 9; ++i) s += c[i] / (z + i);
    const double t = z + 7.5;
    return sqrt(2.0 * FO_PI) * pow(t, z + 0.5) * exp(-t) * s;
}

/* 1/(Gamma(1-g) Gamma(g)) = sin(pi g)/pi  (gauss_jacobi.cpp:125-127). */
double fo_inv_gamma_product(double g) { return sin(FO_PI * g) / FO_PI; }

static int exps_ok(double a, double b) { return (a > -1.0) && (b > -1.0); }

/* mu0 = 2^(a+b+1) G(a+1) G(b+1) / G(a+b+2)  (gauss_jacobi.cpp:129-133). */
int fo_jacobi_moment0(double a, double b, double* out) {
    if (!exps_ok(a, b)) return FO_EINVAL;
    *out = pow(2.0, a + b + 1.0) * fo_gamma(a + 1.0) * fo_gamma(b + 1.0) / fo_gamma(a + b + 2.0);
    return FO_OK;
}

/* Moments of s^k by the three-term recurrence in k (gauss_jacobi.cpp:135-149). */
int fo_jacobi_moment(double a, double b, int k, double* out) {
    if (!exps_ok(a, b) || k < 0) return FO_EINVAL;
    double m0;
    fo_jacobi_moment0(a, b, &m0);
    if (k == 0) {
        *out = m0;
        return FO_OK;
    }
    double prev = m0, cur = (b - a) / (a + b + 2.0) * m0;
    for (int j = 1; j < k; ++j) {
        const double nxt = ((b - a) * cur + j * prev) / (a + b + 2.0 + j);
        prev = cur;
        cur = nxt;
    }
    *out = cur;
    return FO_OK;
}

/* Monic Jacobi recurrence p_{k+1} = (x - A_k) p_k - B_k p_{k-1}  (gauss_jacobi.cpp:23-36). */
static double rec_a(double a, double b, int k) {
    if (k == 0) return (b - a) / (a + b + 2.0);
    const double s = 2.0 * k + a + b;
    return (b * b - a * a) / (s * (s + 2.0));
}
static double rec_b(double a, double b, int k) {
    if (k == 0) {
        double m0;
        fo_jacobi_moment0(a, b, &m0);
        return m0;
    }
    const double s = 2.0 * k + a + b;
    if (k == 1) return 4.0 * (a + 1.0) * (b + 1.0) / (s * s * (s + 1.0));
    return 4.0 * k * (k + a) * (k + b) * (k + a + b) / (s * s * (s + 1.0) * (s - 1.0));
}

/* Implicit QL with Wilkinson-type shift on the symmetric tridiagonal (diag d, offdiag e[1..n-1]).
 * Eigenvalues only: the reference accumulates eigenvectors (gauss_jacobi.cpp:74-78) but never
 * reads them, and the rotations on z do not feed back into d/e, so the eigenvalues are the same
 * bits.  Deflation test, 60-iteration cap and the r == 0 early exit follow gauss_jacobi.cpp:40-87. */
static int ql_eigenvalues(double* d, double* e, int n) {
    for (int i = 1; i < n; ++i) e[i - 1] = e[i];
    e[n - 1] = 0.0;
    for (int l = 0; l < n; ++l) {
        int it = 0, m;
        for (;;) {
            for (m = l; m < n - 1; ++m) {
                const double dd = fabs(d[m]) + fabs(d[m + 1]);
                if (fabs(e[m]) <= 1e-300 || fabs(e[m]) <= 2.3e-16 * dd) break;
            }
            if (m == l) break;
            if (it++ == 60) return FO_ERUNTIME;
            double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
            double r = hypot(g, 1.0);
            g = d[m] - d[l] + e[l] / (g + (g >= 0 ? fabs(r) : -fabs(r)));
            double s = 1.0, c = 1.0, p = 0.0;
            int early = 0;
            for (int i = m - 1; i >= l; --i) {
                const double f = s * e[i];
                const double bb = c * e[i];
                r = hypot(f, g);
                e[i + 1] = r;
                if (r == 0.0) {
                    d[i + 1] -= p;
                    e[m] = 0.0;
                    early = 1;
                    break;
                }
                s = f / r;
                c = g / r;
                g = d[i + 1] - p;
                r = (d[i] - g) * s + 2.0 * c * bb;
                p = s * r;
                d[i + 1] = g + p;
                g = c * r - bb;
            }
            (void)early;
            if (r == 0.0 && m - 1 >= l) continue;
            d[l] -= p;
            e[l] = g;
            e[m] = 0.0;
        }
    }
    return FO_OK;
}

static int cmp_dbl(const void* x, const void* y) {
    const double a = *(const double*)x, b = *(const double*)y;
    return (a > b) - (a < b);
}

/* Golub-Welsch nodes, one guarded Newton polish on the monic P_n, Christoffel weights
 * (gauss_jacobi.cpp:151-204).  Cap 512 points (gauss_jacobi.cpp:13,154). */
int fo_gauss_jacobi(double a, double b, int n, double* nodes, double* weights) {
    if (!exps_ok(a, b) || n < 1 || n > 512) return FO_EINVAL;
    double mu0;
    fo_jacobi_moment0(a, b, &mu0);
    double* d = (double*)malloc(sizeof(double) * n);
    double* e = (double*)malloc(sizeof(double) * n);
    for (int k = 0; k < n; ++k) d[k] = rec_a(a, b, k);
    e[0] = 0.0;
    for (int k = 1; k < n; ++k) e[k] = sqrt(rec_b(a, b, k));
    int st = ql_eigenvalues(d, e, n);
    if (st) {
        free(d);
        free(e);
        return st;
    }
    qsort(d, n, sizeof(double), cmp_dbl);
    for (int i = 0; i < n; ++i) {
        double x = d[i];
        /* value and derivative of the monic P_n at x */
        double p = 1.0, dp = 0.0, pm = 0.0, dpm = 0.0;
        for (int k = 0; k < n; ++k) {
            const double ak = rec_a(a, b, k), bk = (k == 0) ? 0.0 : rec_b(a, b, k);
            const double pn = (x - ak) * p - bk * pm;
            const double dpn = p + (x - ak) * dp - bk * dpm;
            pm = p;
            dpm = dp;
            p = pn;
            dp = dpn;
        }
        if (dp != 0.0) {
            const double step = p / dp;
            if (fabs(step) < 1e-8) x -= step;
        }
        nodes[i] = x;
        /* orthonormal recurrence, w = 1 / sum p_k^2 */
        double q_prev = 0.0, q = 1.0 / sqrt(mu0), sum = q * q, bprev = 0.0;
        for (int k = 0; k < n - 1; ++k) {
            const double bk1 = sqrt(rec_b(a, b, k + 1));
            const double qn = ((x - rec_a(a, b, k)) * q - bprev * q_prev) / bk1;
            q_prev = q;
            q = qn;
            bprev = bk1;
            sum += q * q;
        }
        weights[i] = 1.0 / sum;
    }
    free(d);
    free(e);
    return FO_OK;
}

/* ===================================================================== L1 weights */

static int check_gt(double g, double tau) {
    if (!(g > 0.0) || !(g <= 1.0) || !(tau > 0.0)) return FO_EINVAL;
    return FO_OK;
}

/* Coefficients of (1 - x z)^g: c_i = c_{i-1} ((i-1-g)/i) x  (cq_weights.cpp:19-25). */
static void binom_series(double g, double x, long nmax, double* c) {
    c[0] = 1.0;
    for (long i = 1; i <= nmax; ++i) c[i] = c[i - 1] * ((i - 1 - g) / i) * x;
}

/* d_i of ((1-z)/tau)^g  (cq_weights.cpp:29-40). */
int fo_be_weights(double g, double tau, long nmax, double* out) {
    if (check_gt(g, tau) || nmax < 0) return FO_EINVAL;
    binom_series(g, 1.0, nmax, out);
    const double sc = pow(tau, -g);
    for (long i = 0; i <= nmax; ++i) out[i] *= sc;
    return FO_OK;
}

/* (3/(2 tau))^g * Cauchy product of (1-z)^g and (1-z/3)^g  (cq_weights.cpp:42-59). */
int fo_sbd_weights(double g, double tau, long nmax, double* out) {
    if (check_gt(g, tau) || nmax < 0) return FO_EINVAL;
    double* c1 = (double*)malloc(sizeof(double) * (nmax + 1));
    double* c2 = (double*)malloc(sizeof(double) * (nmax + 1));
    binom_series(g, 1.0, nmax, c1);
    binom_series(g, 1.0 / 3.0, nmax, c2);
    const double sc = pow(1.5 / tau, g);
    for (long i = 0; i <= nmax; ++i) {
        double s = 0.0;
        for (long j = 0; j <= i; ++j) s += c1[j] * c2[i - j];
        out[i] = sc * s;
    }
    free(c1);
    free(c2);
    return FO_OK;
}

/* a = (1-m)/(2m-1)  (cq_weights.cpp:61-67). */
int fo_coupling_from_transition(double m, double* out) {
    if (!(m > 0.0) || !(m <= 1.0) || m == 0.5) return FO_EINVAL;
    *out = (1.0 - m) / (2.0 * m - 1.0);
    return FO_OK;
}

/* ===================================================================== L2 kernels */

static int kernel_gamma_ok(double g) { return (g > 0.0) && (g < 1.0); }

/* BE fold: head = d_0, d_1; w_j = -(sin(pi g)/pi)/(4 tau^g) W_j; r_j = (s_j+1)/2
 * (fast_kernel.cpp:54-74). */
int fo_build_be_kernel(double g, double tau, int np, fo_kernel* k) {
    if (!kernel_gamma_ok(g) || np < 2) return FO_EINVAL;
    if (np > 512) return FO_EINVAL;
    double nodes[512], wts[512];
    int st = fo_gauss_jacobi(g, 1.0 - g, np, nodes, wts);
    if (st) return st;
    memset(k, 0, sizeof(*k));
    k->sbd = 0;
    k->gamma = g;
    k->tau = tau;
    k->n_head = 2;
    double h[2];
    st = fo_be_weights(g, tau, 1, h);
    if (st) return st;
    k->head[0] = h[0];
    k->head[1] = h[1];
    const double pref = -fo_inv_gamma_product(g) / (4.0 * pow(tau, g));
    k->np1 = np;
    k->np2 = 0;
    for (int j = 0; j < np; ++j) {
        k->m1[j] = pref * wts[j];
        k->r1[j] = 0.5 * (nodes[j] + 1.0);
    }
    return FO_OK;
}

int fo_default_sbd_head(double g) { return g <= 0.5 ? 15 : 17; }

/* SBD fold, two families (fast_kernel.cpp:78-124).  Family 1 keeps Re[c1 w_j q^4] with
 * c1 = -2^(2+2g) e^{-i pi g} sin(pi g)/(pi tau^g), q = 1/(s+5); family 2 multiplies by the
 * principal-branch real part of (1+3s)^g. */
int fo_build_sbd_kernel(double g, double tau, int np1, int np2, int n_head, fo_kernel* k) {
    if (!kernel_gamma_ok(g) || np1 < 1 || np2 < 1 || n_head < 3) return FO_EINVAL;
    if (np1 > 512 || np2 > 512 || n_head > 512) return FO_EINVAL;
    double n1[512], w1[512], n2[512], w2[512];
    int st = fo_gauss_jacobi(g, 2.0 - 2.0 * g, np1, n1, w1);
    if (st) return st;
    st = fo_gauss_jacobi(g, 2.0 - 2.0 * g, np2, n2, w2);
    if (st) return st;
    memset(k, 0, sizeof(*k));
    k->sbd = 1;
    k->gamma = g;
    k->tau = tau;
    k->n_head = n_head;
    st = fo_sbd_weights(g, tau, n_head - 1, k->head);
    if (st) return st;
    const double igg = fo_inv_gamma_product(g);
    const double ta = pow(tau, g);
    /* complex c1 = -2^(2+2g) * (cos(pi g) - i sin(pi g)) * igg / ta, as (re, im) */
    const double mag = -pow(2.0, 2.0 + 2.0 * g);
    const double c1re = mag * cos(-FO_PI * g) * igg / ta;
    const double c1im = mag * sin(-FO_PI * g) * igg / ta;
    k->np1 = np1;
    for (int j = 0; j < np1; ++j) {
        const double s = n1[j];
        const double q = 1.0 / (s + 5.0);
        const double q4 = q * q * q * q;
        /* (c1 * w) * q4, real part: complex*real multiplies both parts */
        (void)c1im;
        k->m1[j] = (c1re * w1[j]) * q4;
        k->r1[j] = (s + 1.0) / (s + 5.0);
    }
    const double c2 = -pow(2.0, -g - 3.0) * igg / ta;
    k->np2 = np2;
    for (int j = 0; j < np2; ++j) {
        const double s = n2[j];
        const double w = 1.0 + 3.0 * s;
        const double rp = (w >= 0.0) ? pow(w, g) : pow(-w, g) * cos(FO_PI * g);
        k->m2[j] = c2 * w2[j] * rp;
        k->r2[j] = 0.5 * (s + 1.0);
    }
    return FO_OK;
}

/* Reconstructed weight via pow (fast_kernel.cpp:38-52). */
double fo_reconstruct(const fo_kernel* k, long i) {
    double acc = 0.0;
    const double sh = k->sbd ? 3.0 : 2.0;
    for (int j = 0; j < k->np1; ++j) acc += k->m1[j] * pow(k->r1[j], (double)i - sh);
    for (int j = 0; j < k->np2; ++j) acc += k->m2[j] * pow(k->r2[j], (double)i - sh);
    return acc;
}

/* Incremental-power reconstruction scan over [i_lo, nmax] vs the table; powers start at
 * r^(i_lo - shift) (pow for SBD, 1 for BE) and advance by one multiply per index
 * (fast_kernel.cpp:22-34,126-180,182-256). */
static void eps_scan(const fo_kernel* k, const double* table, long i_lo, long nmax, double* eps,
                     double* worst, long* arg) {
    double p1[512], p2[512];
    for (int j = 0; j < k->np1; ++j) p1[j] = k->sbd ? pow(k->r1[j], (double)(i_lo - 3)) : 1.0;
    for (int j = 0; j < k->np2; ++j) p2[j] = pow(k->r2[j], (double)(i_lo - 3));
    double w = 0.0;
    long am = i_lo;
    for (long i = i_lo; i <= nmax; ++i) {
        double rec = 0.0;
        for (int j = 0; j < k->np1; ++j) {
            rec += k->m1[j] * p1[j];
            p1[j] *= k->r1[j];
        }
        for (int j = 0; j < k->np2; ++j) {
            rec += k->m2[j] * p2[j];
            p2[j] *= k->r2[j];
        }
        const double e = fabs(rec - table[i]);
        if (eps) eps[i] = e;
        if (e > w) {
            w = e;
            am = i;
        }
    }
    *worst = w;
    *arg = am;
}

int fo_kernel_error_report(const fo_kernel* k, long nmax, double* eps, double* max_eps,
                           long* argmax) {
    if (!k->sbd && nmax < 2) return FO_EINVAL;
    if (k->sbd && nmax < k->n_head) return FO_EINVAL;
    double* t = (double*)malloc(sizeof(double) * (nmax + 1));
    int st = k->sbd ? fo_sbd_weights(k->gamma, k->tau, nmax, t)
                    : fo_be_weights(k->gamma, k->tau, nmax, t);
    if (st) {
        free(t);
        return st;
    }
    if (eps)
        for (long i = 0; i <= nmax; ++i) eps[i] = 0.0;
    long lo = k->sbd ? k->n_head : 2;
    /* reference report starts its max at 0 and argmax at 0 (KernelErrorReport defaults) */
    double w;
    long am;
    eps_scan(k, t, lo, nmax, eps, &w, &am);
    *max_eps = w;
    *argmax = (w > 0.0) ? am : 0;
    free(t);
    return FO_OK;
}

/* np grows 64 -> x1.5 up to max_points until eps <= eps_tol tau^-g (fast_kernel.cpp:182-205). */
int fo_build_be_kernel_auto(double g, double tau, long* horizon, double eps_tol, int max_points,
                            int max_head, fo_kernel* k, double* achieved) {
    (void)max_head;
    if (*horizon < 4) *horizon = 4;
    const long H = *horizon;
    double* t = (double*)malloc(sizeof(double) * (H + 1));
    int st = fo_be_weights(g, tau, H, t);
    if (st) {
        free(t);
        return st;
    }
    const double tol = eps_tol * pow(tau, -g);
    int np = 64;
    for (;;) {
        if (np > max_points) np = max_points;
        st = fo_build_be_kernel(g, tau, np, k);
        if (st) break;
        double w;
        long am;
        eps_scan(k, t, 2, H, NULL, &w, &am);
        *achieved = w;
        if (w <= tol || np >= max_points) break;
        np = np + np / 2;
    }
    free(t);
    return st;
}

/* SBD: grow both point counts from 41 (tail eps from min(H, 8 head0)), then the head by x1.5
 * while the argmax sits below 8 head0 (fast_kernel.cpp:207-256). */
int fo_build_sbd_kernel_auto(double g, double tau, long* horizon, double eps_tol,
                             int max_points, int max_head, fo_kernel* k, double* achieved) {
    if (*horizon < 8) *horizon = 8;
    const long H = *horizon;
    double* t = (double*)malloc(sizeof(double) * (H + 1));
    int st = fo_sbd_weights(g, tau, H, t);
    if (st) {
        free(t);
        return st;
    }
    const double tol = eps_tol * pow(tau, -g);
    const int head0 = fo_default_sbd_head(g);
    int np = 41;
    double w;
    long am;
    for (;;) {
        if (np > max_points) np = max_points;
        st = fo_build_sbd_kernel(g, tau, np, np, head0, k);
        if (st) {
            free(t);
            return st;
        }
        long tail_from = 8L * head0;
        if (H < tail_from) tail_from = H;
        eps_scan(k, t, tail_from, H, NULL, &w, &am);
        if (w <= tol || np >= max_points) break;
        np = np + np / 2;
    }
    int head = head0;
    eps_scan(k, t, head, H, NULL, &w, &am);
    while (w > tol && am < 8L * head0 && head < max_head && head < H) {
        int nh = head + head / 2;
        if (nh > max_head) nh = max_head;
        if (nh > H) nh = (int)H;
        head = nh;
        eps_scan(k, t, head, H, NULL, &w, &am);
    }
    *achieved = w;
    if (head != head0) st = fo_build_sbd_kernel(g, tau, np, np, head, k);
    free(t);
    return st;
}

/* ===================================================================== L2 histories */

/* BeHistory / SbdHistory ctors (fast_kernel.cpp:261-266,327-341).  One struct: BE has lag 2
 * and feed = node weights; SBD has lag n_head and feed = mult * ratio^(n_head-3). */
int fo_hist_init(fo_hist* h, const fo_kernel* k, int scheme_variant, long dim) {
    memset(h, 0, sizeof(*h));
    h->k = k;
    h->lo = scheme_variant ? 1 : 0;
    h->dim = dim;
    h->cap = k->sbd ? (k->n_head > 2 ? k->n_head : 2) : 2;
    h->feed1 = (double*)malloc(sizeof(double) * (k->np1 + 1));
    h->feed2 = (double*)malloc(sizeof(double) * (k->np2 + 1));
    for (int j = 0; j < k->np1; ++j)
        h->feed1[j] = k->sbd ? k->m1[j] * pow(k->r1[j], (double)(k->n_head - 3)) : k->m1[j];
    for (int j = 0; j < k->np2; ++j)
        h->feed2[j] = k->m2[j] * pow(k->r2[j], (double)(k->n_head - 3));
    h->acc1 = (double*)calloc((size_t)k->np1 * dim + 1, sizeof(double));
    h->acc2 = (double*)calloc((size_t)k->np2 * dim + 1, sizeof(double));
    h->ring = (double*)calloc((size_t)h->cap * dim + 1, sizeof(double));
    return FO_OK;
}

void fo_hist_free(fo_hist* h) {
    free(h->feed1);
    free(h->feed2);
    free(h->acc1);
    free(h->acc2);
    free(h->ring);
    memset(h, 0, sizeof(*h));
}

/* Level n+1 consumes G(t_{n+1-lag}) when it lies in [lo, appended-1]; otherwise decay only.
 * Evicted feed -> logic_error (fast_kernel.cpp:268-289,343-365). */
int fo_hist_advance(fo_hist* h) {
    const fo_kernel* k = h->k;
    const long lag = k->sbd ? k->n_head : 2;
    const long fi = h->level + 1 - lag;
    h->level += 1;
    if (fi >= h->lo && fi < h->appended - h->cap) return FO_ELOGIC;
    const int feed = (fi >= h->lo) && (fi <= h->appended - 1);
    const double* v = feed ? h->ring + (size_t)(fi % h->cap) * h->dim : NULL;
    const long D = h->dim;
    for (int f = 0; f < 2; ++f) {
        const int np = f ? k->np2 : k->np1;
        const double* r = f ? k->r2 : k->r1;
        const double* c = f ? h->feed2 : h->feed1;
        double* acc = f ? h->acc2 : h->acc1;
        for (int j = 0; j < np; ++j) {
            double* a = acc + (size_t)j * D;
            if (feed)
                for (long m = 0; m < D; ++m) a[m] = r[j] * a[m] + c[j] * v[m];
            else
                for (long m = 0; m < D; ++m) a[m] *= r[j];
        }
    }
    return FO_OK;
}

int fo_hist_append(fo_hist* h, const double* v) {
    memcpy(h->ring + (size_t)(h->appended % h->cap) * h->dim, v, sizeof(double) * h->dim);
    h->appended += 1;
    return FO_OK;
}

int fo_hist_push(fo_hist* h, const double* v) {
    if (h->appended > 0) {
        int st = fo_hist_advance(h);
        if (st) return st;
    }
    return fo_hist_append(h, v);
}

/* Serial node order, family 1 then family 2 (fast_kernel.cpp:302-308,378-388). */
void fo_hist_history_sum(const fo_hist* h, double* out) {
    const long D = h->dim;
    for (long m = 0; m < D; ++m) out[m] = 0.0;
    for (int j = 0; j < h->k->np1; ++j) {
        const double* a = h->acc1 + (size_t)j * D;
        for (long m = 0; m < D; ++m) out[m] += a[m];
    }
    for (int j = 0; j < h->k->np2; ++j) {
        const double* a = h->acc2 + (size_t)j * D;
        for (long m = 0; m < D; ++m) out[m] += a[m];
    }
}

int fo_hist_lagged(const fo_hist* h, long depth, const double** out) {
    const long idx = h->appended - 1 - depth;
    if (idx < 0 || depth < 0 || depth >= h->cap) return FO_ERANGE;
    *out = h->ring + (size_t)(idx % h->cap) * h->dim;
    return FO_OK;
}

/* BE: needs two pushes; d_0 G_n + d_1 G_{n-1} + sum (fast_kernel.cpp:317-325).
 * SBD: head FIR over i <= min(n_head-1, bound), bound = n or n-1 (fast_kernel.cpp:397-409). */
int fo_hist_derivative(const fo_hist* h, double* out) {
    const fo_kernel* k = h->k;
    const long D = h->dim;
    if (!k->sbd) {
        if (h->appended < 2) return FO_ELOGIC;
        fo_hist_history_sum(h, out);
        const double *g0, *g1;
        fo_hist_lagged(h, 0, &g0);
        fo_hist_lagged(h, 1, &g1);
        for (long m = 0; m < D; ++m) out[m] += k->head[0] * g0[m] + k->head[1] * g1[m];
        return FO_OK;
    }
    if (h->appended < 1) return FO_ELOGIC;
    fo_hist_history_sum(h, out);
    const long n = h->appended - 1;
    const long bound = (h->lo == 0) ? n : n - 1;
    const long top = (k->n_head - 1 < bound) ? k->n_head - 1 : bound;
    for (long i = 0; i <= top; ++i) {
        const double* g;
        fo_hist_lagged(h, i, &g);
        const double d = k->head[i];
        for (long m = 0; m < D; ++m) out[m] += d * g[m];
    }
    return FO_OK;
}

int fo_hist_run(const fo_kernel* k, int scheme_variant, long dim, long n_steps, const double* U,
                double* D) {
    fo_hist h;
    fo_hist_init(&h, k, scheme_variant, dim);
    int st = FO_OK;
    for (long n = 0; n < n_steps; ++n) {
        st = fo_hist_push(&h, U + (size_t)n * dim);
        if (st) break;
        double* o = D + (size_t)n * dim;
        if (fo_hist_derivative(&h, o) != FO_OK)
            for (long m = 0; m < dim; ++m) o[m] = NAN;
    }
    fo_hist_free(&h);
    return st;
}

/* Classical O(N^2) CQ sum sum_{i=0..n} d_i u_{n-i} over the full table (the harness direct
 * sum of test_fast_kernel.cpp:27-41 / acceptance_main.cpp:158-159 with exact weights). */
int fo_direct_cq(int sbd, double g, double tau, long dim, long n_steps, const double* U,
                 double* D) {
    double* t = (double*)malloc(sizeof(double) * (n_steps + 1));
    int st = sbd ? fo_sbd_weights(g, tau, n_steps, t) : fo_be_weights(g, tau, n_steps, t);
    if (st) {
        free(t);
        return st;
    }
    for (long n = 0; n < n_steps; ++n)
        for (long m = 0; m < dim; ++m) {
            double s = 0.0;
            for (long i = 0; i <= n; ++i) s += t[i] * U[(size_t)(n - i) * dim + m];
            D[(size_t)n * dim + m] = s;
        }
    free(t);
    return FO_OK;
}

/* ===================================================================== L3 operator + solve */

/* (2 x_i - x_{i-1} - x_{i+1}) / h^2, Dirichlet (block_solver.cpp:10-19). */
void fo_laplacian_apply(int m, double h, const double* x, double* y) {
    const double ih2 = 1.0 / (h * h);
    for (int i = 0; i < m; ++i) {
        double v = 2.0 * x[i];
        if (i > 0) v -= x[i - 1];
        if (i + 1 < m) v -= x[i + 1];
        y[i] = v * ih2;
    }
}

double fo_laplacian_eigenvalue(int m, double h, int k, double length) {
    (void)m;
    const double s = sin(k * FO_PI * h / (2.0 * length));
    return 4.0 / (h * h) * s * s;
}

#define AB(b, row, col) ((b)->ab[(size_t)(col) * (b)->ldab + ((b)->kl + (b)->ku + (row) - (col))])

/* Band LU with partial pivoting in LAPACK gbtrf storage (block_solver.cpp:28-93) assembled for
 * the interleaved (G1_k, G2_k) system (block_solver.cpp:95-117). */
int fo_block_init(fo_block* b, double d01, double d02, double a, double tau, int m, double h,
                  double lead) {
    memset(b, 0, sizeof(*b));
    b->m = m;
    b->n = 2 * m;
    b->kl = 2;
    b->ku = 2;
    b->ldab = 2 * b->kl + b->ku + 1;
    b->ab = (double*)calloc((size_t)b->ldab * b->n, sizeof(double));
    b->piv = (int*)calloc(b->n, sizeof(int));
    b->d01 = d01;
    b->d02 = d02;
    b->a = a;
    b->lead_tau = lead / tau;
    b->ih2 = 1.0 / (h * h);
    const double ih2 = b->ih2;
    for (int k = 0; k < m; ++k) {
        const int r1 = 2 * k, r2 = 2 * k + 1;
        AB(b, r1, r1) = lead / tau + d01 * (a + 2.0 * ih2);
        AB(b, r2, r2) = lead / tau + d02 * (a + 2.0 * ih2);
        AB(b, r1, r2) = -a * d02;
        AB(b, r2, r1) = -a * d01;
        if (k > 0) {
            AB(b, r1, r1 - 2) = -d01 * ih2;
            AB(b, r2, r2 - 2) = -d02 * ih2;
        }
        if (k + 1 < m) {
            AB(b, r1, r1 + 2) = -d01 * ih2;
            AB(b, r2, r2 + 2) = -d02 * ih2;
        }
    }
    const int n = b->n, kl = b->kl, kv = b->kl + b->ku, ld = b->ldab;
    double* ab = b->ab;
    for (int j = 0; j < n; ++j) {
        const int jmax = (n - 1 < j + kl) ? n - 1 : j + kl;
        int pr = j;
        double pmax = fabs(ab[(size_t)j * ld + kv]);
        for (int i = j + 1; i <= jmax; ++i) {
            const double v = fabs(ab[(size_t)j * ld + kv + (i - j)]);
            if (v > pmax) {
                pmax = v;
                pr = i;
            }
        }
        if (pmax == 0.0) return FO_ERUNTIME;
        b->piv[j] = pr;
        const int cmax = (n - 1 < j + kv) ? n - 1 : j + kv;
        if (pr != j)
            for (int c = j; c <= cmax; ++c) {
                const size_t base = (size_t)c * ld + kv;
                const double t = ab[base + (j - c)];
                ab[base + (j - c)] = ab[base + (pr - c)];
                ab[base + (pr - c)] = t;
            }
        const double dinv = 1.0 / ab[(size_t)j * ld + kv];
        for (int i = j + 1; i <= jmax; ++i) {
            double* lij = &ab[(size_t)j * ld + kv + (i - j)];
            *lij *= dinv;
            const double l = *lij;
            for (int c = j + 1; c <= cmax; ++c) {
                const size_t base = (size_t)c * ld + kv;
                ab[base + (i - c)] -= l * ab[base + (j - c)];
            }
        }
    }
    return FO_OK;
}

void fo_block_free(fo_block* b) {
    free(b->ab);
    free(b->piv);
    memset(b, 0, sizeof(*b));
}

void fo_block_solve(const fo_block* b, const double* rhs1, const double* rhs2, double* g1,
                    double* g2) {
    const int n = b->n, kl = b->kl, kv = b->kl + b->ku, ld = b->ldab;
    double* w = (double*)malloc(sizeof(double) * n);
    for (int k = 0; k < b->m; ++k) {
        w[2 * k] = rhs1[k];
        w[2 * k + 1] = rhs2[k];
    }
    for (int j = 0; j < n; ++j) {
        if (b->piv[j] != j) {
            const double t = w[j];
            w[j] = w[b->piv[j]];
            w[b->piv[j]] = t;
        }
        const int imax = (n - 1 < j + kl) ? n - 1 : j + kl;
        const double xj = w[j];
        for (int i = j + 1; i <= imax; ++i) w[i] -= b->ab[(size_t)j * ld + kv + (i - j)] * xj;
    }
    for (int j = n - 1; j >= 0; --j) {
        double v = w[j];
        const int cm = (n - 1 < j + kv) ? n - 1 : j + kv;
        for (int c = j + 1; c <= cm; ++c) v -= b->ab[(size_t)c * ld + kv + (j - c)] * w[c];
        w[j] = v / b->ab[(size_t)j * ld + kv];
    }
    for (int k = 0; k < b->m; ++k) {
        g1[k] = w[2 * k];
        g2[k] = w[2 * k + 1];
    }
    free(w);
}

/* ===================================================================== L4 FFPE */

void fo_kconf_default(fo_kconf* c) {
    c->be_points = 64;
    c->sbd_points_1 = 41;
    c->sbd_points_2 = 41;
    c->sbd_head = 0;
    c->eps_tol = 1e-12;
    c->auto_size = 1;
}

/* poly_sin / indicator (open at 1/2) / custom samples (fpfp.cpp:40-70). */
int fo_initial_field(const fo_spec* s, double* g1, double* g2) {
    const int m = s->grid_m;
    const double h = s->length / (double)(m + 1);
    for (int j = 0; j < m; ++j) {
        const double x = (j + 1) * h;
        if (s->initial == 0) {
            g1[j] = x * (1.0 - x);
            g2[j] = sin(x);
        } else if (s->initial == 1) {
            g1[j] = x > 0.5 ? 1.0 - x : 0.0;
            g2[j] = x < 0.5 ? x : 0.0;
        } else {
            if (!s->custom_g1 || !s->custom_g2) return FO_EINVAL;
            g1[j] = s->custom_g1[j];
            g2[j] = s->custom_g2[j];
        }
    }
    return FO_OK;
}

double fo_l2_norm(const double* v, long n, double h) {
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(h * s);
}

/* rhs_i = lead_part_i - a s_i - (A s)_i + a s_other  (fpfp.cpp:123-126, 277-279, 339-344). */
static void assemble_rhs(int m, double h, double a, const double* lead1, const double* lead2,
                         const double* s1, const double* s2, double* rhs1, double* rhs2,
                         double* as) {
    fo_laplacian_apply(m, h, s1, as);
    for (int k = 0; k < m; ++k) rhs1[k] = lead1[k] - a * s1[k] - as[k] + a * s2[k];
    fo_laplacian_apply(m, h, s2, as);
    for (int k = 0; k < m; ++k) rhs2[k] = lead2[k] - a * s2[k] - as[k] + a * s1[k];
}

/* SBD first step: 2/3-1/3 system (fpfp.cpp:136-149, 293-308). */
static void sbd_first_rhs(int m, double h, double a, double tau, double d10, double d20,
                          const double* u0, const double* v0, double* rhs1, double* rhs2,
                          double* as) {
    fo_laplacian_apply(m, h, u0, as);
    for (int k = 0; k < m; ++k)
        rhs1[k] = u0[k] / tau - (d10 / 3.0) * (a * u0[k] + as[k]) + (a * d20 / 3.0) * v0[k];
    fo_laplacian_apply(m, h, v0, as);
    for (int k = 0; k < m; ++k)
        rhs2[k] = v0[k] / tau - (d20 / 3.0) * (a * v0[k] + as[k]) + (a * d10 / 3.0) * u0[k];
}

/* CorrPowers::value_at: running powers r^e, one multiply per exponent (fpfp.cpp:240-250). */
typedef struct {
    double p1[512], p2[512];
    long e;
} corr_pw;
static double corr_value(corr_pw* c, const fo_kernel* k, long e) {
    while (c->e < e) {
        for (int j = 0; j < k->np1; ++j) c->p1[j] *= k->r1[j];
        for (int j = 0; j < k->np2; ++j) c->p2[j] *= k->r2[j];
        c->e += 1;
    }
    double v = 0.0;
    for (int j = 0; j < k->np1; ++j) v += k->m1[j] * c->p1[j];
    for (int j = 0; j < k->np2; ++j) v += k->m2[j] * c->p2[j];
    return v;
}

/* run(): classical (full history, fpfp.cpp:81-175) or fast (fpfp.cpp:180-349) steppers. */
int fo_run(const fo_spec* s, int scheme, const fo_kconf* kc, double* g1_out, double* g2_out,
           double* eps1, double* eps2, int* np_out, int* nhead_out) {
    const int m = s->grid_m;
    const long N = s->n_steps;
    const double tau = s->t_final / (double)N, h = s->length / (double)(m + 1), a = s->a;
    const double o1 = 1.0 - s->alpha1, o2 = 1.0 - s->alpha2;
    const int sbd = (scheme == FO_SBD || scheme == FO_FASTSBD);
    const int fast = (scheme == FO_FASTBE || scheme == FO_FASTSBD);
    int st = FO_OK;
    double *g1 = malloc(sizeof(double) * m), *g2 = malloc(sizeof(double) * m);
    double *rhs1 = malloc(sizeof(double) * m), *rhs2 = malloc(sizeof(double) * m);
    double *as = malloc(sizeof(double) * m), *s1 = malloc(sizeof(double) * m),
           *s2 = malloc(sizeof(double) * m);
    double *l1 = malloc(sizeof(double) * m), *l2 = malloc(sizeof(double) * m);
    st = fo_initial_field(s, g1, g2);
    if (st) goto done;
    if (eps1) *eps1 = 0.0;
    if (eps2) *eps2 = 0.0;

    if (!fast) {
        double *t1 = malloc(sizeof(double) * (N + 1)), *t2 = malloc(sizeof(double) * (N + 1));
        double* H1 = malloc(sizeof(double) * (size_t)(N + 1) * m);
        double* H2 = malloc(sizeof(double) * (size_t)(N + 1) * m);
        st = sbd ? fo_sbd_weights(o1, tau, N, t1) : fo_be_weights(o1, tau, N, t1);
        if (!st) st = sbd ? fo_sbd_weights(o2, tau, N, t2) : fo_be_weights(o2, tau, N, t2);
        fo_block sys, sys1;
        memset(&sys1, 0, sizeof(sys1));
        if (!st) st = fo_block_init(&sys, t1[0], t2[0], a, tau, m, h, sbd ? 1.5 : 1.0);
        if (!st && sbd) st = fo_block_init(&sys1, 2.0 / 3.0 * t1[0], 2.0 / 3.0 * t2[0], a, tau, m, h, 1.0);
        if (!st) {
            memcpy(H1, g1, sizeof(double) * m);
            memcpy(H2, g2, sizeof(double) * m);
            for (long n = 1; n <= N; ++n) {
                double* u_nm1 = H1 + (size_t)(n - 1) * m;
                double* v_nm1 = H2 + (size_t)(n - 1) * m;
                if (sbd && n == 1) {
                    sbd_first_rhs(m, h, a, tau, t1[0], t2[0], H1, H2, rhs1, rhs2, as);
                    fo_block_solve(&sys1, rhs1, rhs2, g1, g2);
                } else {
                    for (int k = 0; k < m; ++k) {
                        s1[k] = sbd ? 0.5 * t1[n - 1] * H1[k] : 0.0;
                        s2[k] = sbd ? 0.5 * t2[n - 1] * H2[k] : 0.0;
                    }
                    for (long i = 1; i <= n - 1; ++i) {
                        const double w1 = t1[i], w2 = t2[i];
                        const double* u = H1 + (size_t)(n - i) * m;
                        const double* v = H2 + (size_t)(n - i) * m;
                        for (int k = 0; k < m; ++k) {
                            s1[k] += w1 * u[k];
                            s2[k] += w2 * v[k];
                        }
                    }
                    for (int k = 0; k < m; ++k) {
                        if (sbd) {
                            l1[k] = (2.0 * u_nm1[k] - 0.5 * H1[(size_t)(n - 2) * m + k]) / tau;
                            l2[k] = (2.0 * v_nm1[k] - 0.5 * H2[(size_t)(n - 2) * m + k]) / tau;
                        } else {
                            l1[k] = u_nm1[k] / tau;
                            l2[k] = v_nm1[k] / tau;
                        }
                    }
                    assemble_rhs(m, h, a, l1, l2, s1, s2, rhs1, rhs2, as);
                    fo_block_solve(&sys, rhs1, rhs2, g1, g2);
                }
                memcpy(H1 + (size_t)n * m, g1, sizeof(double) * m);
                memcpy(H2 + (size_t)n * m, g2, sizeof(double) * m);
            }
            fo_block_free(&sys);
            if (sbd) fo_block_free(&sys1);
        }
        free(t1);
        free(t2);
        free(H1);
        free(H2);
        goto done;
    }

    /* fast steppers */
    {
        fo_kernel* k1 = malloc(sizeof(fo_kernel));
        fo_kernel* k2 = malloc(sizeof(fo_kernel));
        double e1 = 0.0, e2 = 0.0;
        if (kc->auto_size) {
            long H1 = N, H2 = N;
            if (sbd) {
                st = fo_build_sbd_kernel_auto(o1, tau, &H1, kc->eps_tol, 256, 256, k1, &e1);
                if (!st) st = fo_build_sbd_kernel_auto(o2, tau, &H2, kc->eps_tol, 256, 256, k2, &e2);
            } else {
                st = fo_build_be_kernel_auto(o1, tau, &H1, kc->eps_tol, 256, 256, k1, &e1);
                if (!st) st = fo_build_be_kernel_auto(o2, tau, &H2, kc->eps_tol, 256, 256, k2, &e2);
            }
        } else {
            long am;
            if (sbd) {
                const int h1 = kc->sbd_head > 0 ? kc->sbd_head : fo_default_sbd_head(o1);
                const int h2 = kc->sbd_head > 0 ? kc->sbd_head : fo_default_sbd_head(o2);
                st = fo_build_sbd_kernel(o1, tau, kc->sbd_points_1, kc->sbd_points_2, h1, k1);
                if (!st) st = fo_build_sbd_kernel(o2, tau, kc->sbd_points_1, kc->sbd_points_2, h2, k2);
                if (!st) st = fo_kernel_error_report(k1, N > 8 ? N : 8, NULL, &e1, &am);
                if (!st) st = fo_kernel_error_report(k2, N > 8 ? N : 8, NULL, &e2, &am);
            } else {
                st = fo_build_be_kernel(o1, tau, kc->be_points, k1);
                if (!st) st = fo_build_be_kernel(o2, tau, kc->be_points, k2);
                if (!st) st = fo_kernel_error_report(k1, N > 2 ? N : 2, NULL, &e1, &am);
                if (!st) st = fo_kernel_error_report(k2, N > 2 ? N : 2, NULL, &e2, &am);
            }
        }
        if (st) {
            free(k1);
            free(k2);
            goto done;
        }
        if (eps1) *eps1 = e1;
        if (eps2) *eps2 = e2;
        if (np_out) {
            np_out[0] = k1->np1;
            np_out[1] = k1->np2;
            np_out[2] = k2->np1;
            np_out[3] = k2->np2;
        }
        if (nhead_out) {
            nhead_out[0] = k1->n_head;
            nhead_out[1] = k2->n_head;
        }
        fo_hist hh1, hh2;
        fo_hist_init(&hh1, k1, 1, m);
        fo_hist_init(&hh2, k2, 1, m);
        fo_block sys, sys1;
        memset(&sys1, 0, sizeof(sys1));
        st = fo_block_init(&sys, k1->head[0], k2->head[0], a, tau, m, h, sbd ? 1.5 : 1.0);
        if (!st && sbd)
            st = fo_block_init(&sys1, 2.0 / 3.0 * k1->head[0], 2.0 / 3.0 * k2->head[0], a, tau, m, h, 1.0);
        double *G01 = malloc(sizeof(double) * m), *G02 = malloc(sizeof(double) * m);
        memcpy(G01, g1, sizeof(double) * m);
        memcpy(G02, g2, sizeof(double) * m);
        fo_hist_append(&hh1, g1);
        fo_hist_append(&hh2, g2);
        corr_pw* cp1 = calloc(1, sizeof(corr_pw));
        corr_pw* cp2 = calloc(1, sizeof(corr_pw));
        for (int j = 0; j < 512; ++j) cp1->p1[j] = cp1->p2[j] = cp2->p1[j] = cp2->p2[j] = 1.0;
        for (long n = 1; !st && n <= N; ++n) {
            st = fo_hist_advance(&hh1);
            if (!st) st = fo_hist_advance(&hh2);
            if (st) break;
            const double *u1, *v1;
            fo_hist_lagged(&hh1, 0, &u1);
            fo_hist_lagged(&hh2, 0, &v1);
            if (!sbd) {
                /* fpfp.cpp:259-284 */
                fo_hist_history_sum(&hh1, s1);
                fo_hist_history_sum(&hh2, s2);
                if (n >= 2)
                    for (int k = 0; k < m; ++k) {
                        s1[k] += k1->head[1] * u1[k];
                        s2[k] += k2->head[1] * v1[k];
                    }
                for (int k = 0; k < m; ++k) {
                    l1[k] = u1[k] / tau;
                    l2[k] = v1[k] / tau;
                }
                assemble_rhs(m, h, a, l1, l2, s1, s2, rhs1, rhs2, as);
                fo_block_solve(&sys, rhs1, rhs2, g1, g2);
            } else if (n == 1) {
                sbd_first_rhs(m, h, a, tau, k1->head[0], k2->head[0], u1, v1, rhs1, rhs2, as);
                fo_block_solve(&sys1, rhs1, rhs2, g1, g2);
            } else {
                /* fpfp.cpp:309-345 */
                fo_hist_history_sum(&hh1, s1);
                fo_hist_history_sum(&hh2, s2);
                for (int f = 0; f < 2; ++f) {
                    const fo_kernel* kk = f ? k2 : k1;
                    fo_hist* hh = f ? &hh2 : &hh1;
                    double* ss = f ? s2 : s1;
                    const long top = (kk->n_head - 1 < n - 1) ? kk->n_head - 1 : n - 1;
                    for (long i = 1; i <= top; ++i) {
                        const double* u;
                        fo_hist_lagged(hh, i - 1, &u);
                        const double w = kk->head[i];
                        for (int k = 0; k < m; ++k) ss[k] += w * u[k];
                    }
                }
                const double c1 = (n - 1 < k1->n_head) ? k1->head[n - 1] : corr_value(cp1, k1, n - 4);
                const double c2 = (n - 1 < k2->n_head) ? k2->head[n - 1] : corr_value(cp2, k2, n - 4);
                for (int k = 0; k < m; ++k) {
                    s1[k] += 0.5 * c1 * G01[k];
                    s2[k] += 0.5 * c2 * G02[k];
                }
                const double *u2, *v2;
                fo_hist_lagged(&hh1, 1, &u2);
                fo_hist_lagged(&hh2, 1, &v2);
                for (int k = 0; k < m; ++k) {
                    l1[k] = (2.0 * u1[k] - 0.5 * u2[k]) / tau;
                    l2[k] = (2.0 * v1[k] - 0.5 * v2[k]) / tau;
                }
                assemble_rhs(m, h, a, l1, l2, s1, s2, rhs1, rhs2, as);
                fo_block_solve(&sys, rhs1, rhs2, g1, g2);
            }
            fo_hist_append(&hh1, g1);
            fo_hist_append(&hh2, g2);
        }
        free(cp1);
        free(cp2);
        free(G01);
        free(G02);
        fo_block_free(&sys);
        if (sbd) fo_block_free(&sys1);
        fo_hist_free(&hh1);
        fo_hist_free(&hh2);
        free(k1);
        free(k2);
    }
done:
    if (!st) {
        memcpy(g1_out, g1, sizeof(double) * m);
        memcpy(g2_out, g2, sizeof(double) * m);
    }
    free(g1);
    free(g2);
    free(rhs1);
    free(rhs2);
    free(as);
    free(s1);
    free(s2);
    free(l1);
    free(l2);
    return st;
}

/* ---- Mode-space fast FFPE stepping (TEST INFRASTRUCTURE) ----
 * The reference's mode-space oracle (test_fpfp.cpp:79-134: mode_be / mode_sbd, solve2x2) with the
 * O(n) history sums replaced by the fast histories of fast_kernel.cpp (scheme variant, one lane per
 * mode), i.e. FastStepper (fpfp.cpp:259-349) with the discrete Laplacian replaced by its
 * eigenvalues lam[k] (block_solver.cpp:21-24; in 2D lam_k + lam_l).  u0/v0 are the initial DST
 * coefficients of both fields; uN/vN receive the coefficients after N levels. */
static void solve2x2(double a11, double a12, double a21, double a22, double r1, double r2,
                     double* x1, double* x2) {
    const double det = a11 * a22 - a12 * a21;
    *x1 = (r1 * a22 - a12 * r2) / det;
    *x2 = (a11 * r2 - a21 * r1) / det;
}

int fo_modal_run(const fo_kernel* k1, const fo_kernel* k2, double a, double tau, long N,
                 long nm, const double* lam, const double* u0, const double* v0, double* uN,
                 double* vN) {
    if (N < 1 || nm < 1 || k1->sbd != k2->sbd) return FO_EINVAL;
    const int sbd = k1->sbd;
    fo_hist hh1, hh2;
    int st = fo_hist_init(&hh1, k1, 1, nm);
    if (!st) st = fo_hist_init(&hh2, k2, 1, nm);
    if (st) return st;
    double *s1 = malloc(sizeof(double) * nm), *s2 = malloc(sizeof(double) * nm);
    double *x1 = malloc(sizeof(double) * nm), *x2 = malloc(sizeof(double) * nm);
    corr_pw* cp1 = calloc(1, sizeof(corr_pw));
    corr_pw* cp2 = calloc(1, sizeof(corr_pw));
    for (int j = 0; j < 512; ++j) cp1->p1[j] = cp1->p2[j] = cp2->p1[j] = cp2->p2[j] = 1.0;
    const double d10 = k1->head[0], d20 = k2->head[0];
    fo_hist_append(&hh1, u0);
    fo_hist_append(&hh2, v0);
    for (long n = 1; !st && n <= N; ++n) {
        st = fo_hist_advance(&hh1);
        if (!st) st = fo_hist_advance(&hh2);
        if (st) break;
        const double *u1, *v1;
        fo_hist_lagged(&hh1, 0, &u1);
        fo_hist_lagged(&hh2, 0, &v1);
        if (sbd && n == 1) {
            for (long k = 0; k < nm; ++k) {
                const double al = a + lam[k];
                const double r1 = u1[k] / tau - (d10 / 3.0) * al * u1[k] + (a * d20 / 3.0) * v1[k];
                const double r2 = v1[k] / tau - (d20 / 3.0) * al * v1[k] + (a * d10 / 3.0) * u1[k];
                solve2x2(1.0 / tau + (2.0 / 3.0) * d10 * al, -(2.0 / 3.0) * a * d20,
                         -(2.0 / 3.0) * a * d10, 1.0 / tau + (2.0 / 3.0) * d20 * al, r1, r2,
                         &x1[k], &x2[k]);
            }
        } else {
            fo_hist_history_sum(&hh1, s1);
            fo_hist_history_sum(&hh2, s2);
            const double* u2 = NULL;
            const double* v2 = NULL;
            if (!sbd) {
                if (n >= 2)
                    for (long k = 0; k < nm; ++k) {
                        s1[k] += k1->head[1] * u1[k];
                        s2[k] += k2->head[1] * v1[k];
                    }
            } else {
                for (int f = 0; f < 2; ++f) {
                    const fo_kernel* kk = f ? k2 : k1;
                    fo_hist* hh = f ? &hh2 : &hh1;
                    double* ss = f ? s2 : s1;
                    const long top = (kk->n_head - 1 < n - 1) ? kk->n_head - 1 : n - 1;
                    for (long i = 1; i <= top; ++i) {
                        const double* u;
                        fo_hist_lagged(hh, i - 1, &u);
                        for (long k = 0; k < nm; ++k) ss[k] += kk->head[i] * u[k];
                    }
                }
                const double c1 = (n - 1 < k1->n_head) ? k1->head[n - 1] : corr_value(cp1, k1, n - 4);
                const double c2 = (n - 1 < k2->n_head) ? k2->head[n - 1] : corr_value(cp2, k2, n - 4);
                for (long k = 0; k < nm; ++k) {
                    s1[k] += 0.5 * c1 * u0[k];
                    s2[k] += 0.5 * c2 * v0[k];
                }
                fo_hist_lagged(&hh1, 1, &u2);
                fo_hist_lagged(&hh2, 1, &v2);
            }
            const double lead = sbd ? 1.5 : 1.0;
            for (long k = 0; k < nm; ++k) {
                const double al = a + lam[k];
                const double l1 = sbd ? (2.0 * u1[k] - 0.5 * u2[k]) / tau : u1[k] / tau;
                const double l2 = sbd ? (2.0 * v1[k] - 0.5 * v2[k]) / tau : v1[k] / tau;
                const double r1 = l1 - al * s1[k] + a * s2[k];
                const double r2 = l2 - al * s2[k] + a * s1[k];
                solve2x2(lead / tau + d10 * al, -a * d20, -a * d10, lead / tau + d20 * al, r1, r2,
                         &x1[k], &x2[k]);
            }
        }
        fo_hist_append(&hh1, x1);
        fo_hist_append(&hh2, x2);
    }
    if (!st) {
        memcpy(uN, x1, sizeof(double) * nm);
        memcpy(vN, x2, sizeof(double) * nm);
    }
    free(s1);
    free(s2);
    free(x1);
    free(x2);
    free(cp1);
    free(cp2);
    fo_hist_free(&hh1);
    fo_hist_free(&hh2);
    return st;
}
