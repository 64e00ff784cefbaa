/* fraq_anchor_ld.c -- TEST INFRASTRUCTURE: an extended-precision (x87 long double) anchor for the
 * 1D FFPE fast schemes at full size, on sampled DST modes.
 *
 * The exact discrete solution of the reference's FastBE / FastSBD scheme (fpfp.cpp:259-349) with
 * the node tables it uses (fp64 values, taken as exact) is diagonal in the sine basis of the
 * Dirichlet stencil (block_solver.cpp:10-24; the reference's own mode-space oracle,
 * test_fpfp.cpp:21-180).  This evaluates it on a sample of modes with every operation in long
 * double: the projection of G0 (test_fpfp.cpp:39-47 normalisation 2/(M+1)), the exact eigenvalues
 * lambda_k = 4 (M+1)^2 sin^2(k pi / (2 (M+1))) (unit interval), the per-node history recurrences
 * (fast_kernel.cpp:261-409, scheme variant), the SBD G0 correction with running powers
 * (fpfp.cpp:240-250, 325-334) and the 2x2 solves (test_fpfp.cpp:79-84).  It is the truth against
 * which the physical-space solvers (the reference's and the B200 one) are measured: their block
 * system at M = 4095 has cond ~1.4e6, and the fp64 rounding of its constant diagonal shifts the
 * whole solution (profiles/r02/physical_bisect.txt).  Never linked into the product.
 *
 *   fo_anchor_ld(k1, k2, a, tau, N, M, nm, modes[nm], g1[M], g2[M], uN[nm], vN[nm])
 * modes are 1-based DST indices; uN / vN receive the coefficients after N levels. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fraq_oracle.h"

typedef long double LD;

typedef struct {
    const fo_kernel* k;
    int cap, lag;
    long level, appended, nm;
    LD *feed, *acc, *ring; /* nodes np1 + np2; acc [J][nm]; ring [cap][nm] */
    LD *pw;                /* running powers for the SBD correction */
    long pw_e;
} ld_hist;

static int ld_init(ld_hist* h, const fo_kernel* k, long nm) {
    memset(h, 0, sizeof(*h));
    h->k = k;
    h->nm = nm;
    h->cap = k->sbd ? (k->n_head > 2 ? k->n_head : 2) : 2;
    h->lag = k->sbd ? k->n_head : 2;
    const int J = k->np1 + k->np2;
    h->feed = calloc(J + 1, sizeof(LD));
    h->pw = calloc(J + 1, sizeof(LD));
    h->acc = calloc((size_t)J * nm + 1, sizeof(LD));
    h->ring = calloc((size_t)h->cap * nm + 1, sizeof(LD));
    if (!h->feed || !h->pw || !h->acc || !h->ring) return FO_EINVAL;
    for (int j = 0; j < J; ++j) {
        const LD m = j < k->np1 ? k->m1[j] : k->m2[j - k->np1];
        const LD r = j < k->np1 ? k->r1[j] : k->r2[j - k->np1];
        h->feed[j] = k->sbd ? m * powl(r, (LD)(k->n_head - 3)) : m;
        h->pw[j] = 1.0L;
    }
    return FO_OK;
}

static void ld_free(ld_hist* h) {
    free(h->feed);
    free(h->pw);
    free(h->acc);
    free(h->ring);
}

static LD ld_r(const fo_kernel* k, int j) { return j < k->np1 ? k->r1[j] : k->r2[j - k->np1]; }

/* advance() of the scheme variant (lo = 1): feed G^{level+1-lag} when 1 <= it <= appended-1 */
static void ld_advance(ld_hist* h) {
    const long fi = h->level + 1 - h->lag;
    h->level += 1;
    const int feed = fi >= 1 && fi <= h->appended - 1;
    const LD* v = feed ? h->ring + (size_t)(fi % h->cap) * h->nm : NULL;
    const int J = h->k->np1 + h->k->np2;
    for (int j = 0; j < J; ++j) {
        const LD r = ld_r(h->k, j), c = h->feed[j];
        LD* a = h->acc + (size_t)j * h->nm;
        for (long m = 0; m < h->nm; ++m) a[m] = feed ? r * a[m] + c * v[m] : r * a[m];
    }
}

static void ld_append(ld_hist* h, const LD* v) {
    memcpy(h->ring + (size_t)(h->appended % h->cap) * h->nm, v, sizeof(LD) * h->nm);
    h->appended += 1;
}

static const LD* ld_lagged(const ld_hist* h, long depth) {
    return h->ring + (size_t)((h->appended - 1 - depth) % h->cap) * h->nm;
}

static void ld_sum(const ld_hist* h, LD* out) {
    const int J = h->k->np1 + h->k->np2;
    for (long m = 0; m < h->nm; ++m) out[m] = 0.0L;
    for (int j = 0; j < J; ++j) {
        const LD* a = h->acc + (size_t)j * h->nm;
        for (long m = 0; m < h->nm; ++m) out[m] += a[m];
    }
}

/* sum_j m_j r_j^e with running powers (CorrPowers::value_at, fpfp.cpp:240-250) */
static LD ld_corr(ld_hist* h, long e) {
    const fo_kernel* k = h->k;
    const int J = k->np1 + k->np2;
    while (h->pw_e < e) {
        for (int j = 0; j < J; ++j) h->pw[j] *= ld_r(k, j);
        h->pw_e += 1;
    }
    LD v = 0.0L;
    for (int j = 0; j < J; ++j) v += (j < k->np1 ? (LD)k->m1[j] : (LD)k->m2[j - k->np1]) * h->pw[j];
    return v;
}

static void ld_solve2(LD a11, LD a12, LD a21, LD a22, LD r1, LD r2, LD* x1, LD* x2) {
    const LD det = a11 * a22 - a12 * a21;
    *x1 = (r1 * a22 - a12 * r2) / det;
    *x2 = (a11 * r2 - a21 * r1) / det;
}

static int anchor_steps(const fo_kernel* k1, const fo_kernel* k2, LD a, LD tau, long N, long nm,
                        const LD* lam, const LD* u0, const LD* v0, double* uN, double* vN);

int fo_anchor_ld(const fo_kernel* k1, const fo_kernel* k2, double a_, double tau_, long N, int M,
                 long nm, const int* modes, const double* g1, const double* g2, double* uN,
                 double* vN) {
    if (N < 1 || nm < 1 || M < 1 || k1->sbd != k2->sbd) return FO_EINVAL;
    const LD pi = acosl(-1.0L), Mp1 = (LD)(M + 1);
    LD *lam = malloc(sizeof(LD) * nm), *u0 = malloc(sizeof(LD) * nm), *v0 = malloc(sizeof(LD) * nm);
    for (long q = 0; q < nm; ++q) {
        const int k = modes[q];
        const LD s = sinl((LD)k * pi / (2.0L * Mp1));
        lam[q] = 4.0L * Mp1 * Mp1 * s * s;
        LD c1 = 0.0L, c2 = 0.0L;
        for (int j = 1; j <= M; ++j) {
            const LD sn = sinl((LD)k * (LD)j * pi / Mp1);
            c1 += sn * (LD)g1[j - 1];
            c2 += sn * (LD)g2[j - 1];
        }
        u0[q] = 2.0L / Mp1 * c1;
        v0[q] = 2.0L / Mp1 * c2;
    }
    const int st = anchor_steps(k1, k2, a_, tau_, N, nm, lam, u0, v0, uN, vN);
    free(lam);
    free(u0);
    free(v0);
    return st;
}

/* The same stepping for caller-given modes: eigenvalues lam (e.g. lambda_k + lambda_l of the 2D
 * five-point stencil) and initial coefficients u0 / v0, each given as a (hi, lo) pair of doubles
 * (value = hi + lo, so an extended-precision projection passes through unrounded). */
int fo_anchor_modes_ld(const fo_kernel* k1, const fo_kernel* k2, double a_, double tau_, long N,
                       long nm, const double* lam2, const double* u02, const double* v02,
                       double* uN, double* vN) {
    if (N < 1 || nm < 1 || k1->sbd != k2->sbd) return FO_EINVAL;
    LD *lam = malloc(sizeof(LD) * nm), *u0 = malloc(sizeof(LD) * nm), *v0 = malloc(sizeof(LD) * nm);
    for (long q = 0; q < nm; ++q) {
        lam[q] = (LD)lam2[2 * q] + (LD)lam2[2 * q + 1];
        u0[q] = (LD)u02[2 * q] + (LD)u02[2 * q + 1];
        v0[q] = (LD)v02[2 * q] + (LD)v02[2 * q + 1];
    }
    const int st = anchor_steps(k1, k2, a_, tau_, N, nm, lam, u0, v0, uN, vN);
    free(lam);
    free(u0);
    free(v0);
    return st;
}

static int anchor_steps(const fo_kernel* k1, const fo_kernel* k2, LD a, LD tau, long N, long nm,
                        const LD* lam, const LD* u0, const LD* v0, double* uN, double* vN) {
    const int sbd = k1->sbd;
    LD *s1 = malloc(sizeof(LD) * nm), *s2 = malloc(sizeof(LD) * nm);
    LD *x1 = malloc(sizeof(LD) * nm), *x2 = malloc(sizeof(LD) * nm);
    ld_hist h1, h2;
    int st = ld_init(&h1, k1, nm);
    if (!st) st = ld_init(&h2, k2, nm);
    const LD d10 = k1->head[0], d20 = k2->head[0];
    ld_append(&h1, u0);
    ld_append(&h2, v0);
    for (long n = 1; !st && n <= N; ++n) {
        ld_advance(&h1);
        ld_advance(&h2);
        const LD* u1 = ld_lagged(&h1, 0);
        const LD* v1 = ld_lagged(&h2, 0);
        if (sbd && n == 1) {
            /* 2/3 - 1/3 first step from G0 (fpfp.cpp:293-303) */
            for (long q = 0; q < nm; ++q) {
                const LD al = a + lam[q];
                const LD r1 = u1[q] / tau - (d10 / 3.0L) * al * u1[q] + (a * d20 / 3.0L) * v1[q];
                const LD r2 = v1[q] / tau - (d20 / 3.0L) * al * v1[q] + (a * d10 / 3.0L) * u1[q];
                ld_solve2(1.0L / tau + (2.0L / 3.0L) * d10 * al, -(2.0L / 3.0L) * a * d20,
                          -(2.0L / 3.0L) * a * d10, 1.0L / tau + (2.0L / 3.0L) * d20 * al, r1, r2,
                          &x1[q], &x2[q]);
            }
        } else {
            ld_sum(&h1, s1);
            ld_sum(&h2, s2);
            const LD *u2 = NULL, *v2 = NULL;
            if (!sbd) {
                if (n >= 2)
                    for (long q = 0; q < nm; ++q) {
                        s1[q] += (LD)k1->head[1] * u1[q];
                        s2[q] += (LD)k2->head[1] * v1[q];
                    }
            } else {
                for (int f = 0; f < 2; ++f) {
                    const fo_kernel* kk = f ? k2 : k1;
                    ld_hist* hh = f ? &h2 : &h1;
                    LD* ss = f ? s2 : s1;
                    const long top = (kk->n_head - 1 < n - 1) ? kk->n_head - 1 : n - 1;
                    for (long i = 1; i <= top; ++i) {
                        const LD* u = ld_lagged(hh, i - 1);
                        for (long q = 0; q < nm; ++q) ss[q] += (LD)kk->head[i] * u[q];
                    }
                }
                const LD c1 = (n - 1 < k1->n_head) ? (LD)k1->head[n - 1] : ld_corr(&h1, n - 4);
                const LD c2 = (n - 1 < k2->n_head) ? (LD)k2->head[n - 1] : ld_corr(&h2, n - 4);
                for (long q = 0; q < nm; ++q) {
                    s1[q] += 0.5L * c1 * u0[q];
                    s2[q] += 0.5L * c2 * v0[q];
                }
                u2 = ld_lagged(&h1, 1);
                v2 = ld_lagged(&h2, 1);
            }
            const LD lead = sbd ? 1.5L : 1.0L;
            for (long q = 0; q < nm; ++q) {
                const LD al = a + lam[q];
                const LD l1 = sbd ? (2.0L * u1[q] - 0.5L * u2[q]) / tau : u1[q] / tau;
                const LD l2 = sbd ? (2.0L * v1[q] - 0.5L * v2[q]) / tau : v1[q] / tau;
                const LD r1 = l1 - al * s1[q] + a * s2[q];
                const LD r2 = l2 - al * s2[q] + a * s1[q];
                ld_solve2(lead / tau + d10 * al, -a * d20, -a * d10, lead / tau + d20 * al, r1, r2,
                          &x1[q], &x2[q]);
            }
        }
        ld_append(&h1, x1);
        ld_append(&h2, x2);
    }
    if (!st)
        for (long q = 0; q < nm; ++q) {
            uN[q] = (double)x1[q];
            vN[q] = (double)x2[q];
        }
    ld_free(&h1);
    ld_free(&h2);
    free(s1);
    free(s2);
    free(x1);
    free(x2);
    return st;
}
