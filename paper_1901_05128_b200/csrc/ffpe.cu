// ffpe.cu -- two-state fractional Fokker-Planck steppers on the device (fpfp.cpp:81-381).
//
// Per time level (fast schemes):
//   K5  history advance + node sum + exact head window for both fields of every instance
//       (MODE_FFPE, history.cu) -> s1, s2
//   K6  per instance: RHS assembly (stencil Laplacian of s, BE / BDF2 lead terms, SBD G^0
//       correction from the precomputed K7 sequence), the 2x2-block tridiagonal solve of the
//       interleaved (G1_k, G2_k) system (block_solver.cpp:95-153), and the append of G^n into
//       both lag rings.
// The block system is constant in time, so it is reduced once at setup: block cyclic reduction
// coefficients when grid_m + 1 is a power of two (all BASELINE grids: 255, 1023, 4095), else a
// block-Thomas factorization.  The reference factors a pivoted banded LU once instead
// (block_solver.cpp:38-74); both are direct solves of the same matrix.
//
// Classical schemes (ClassicalStepper, fpfp.cpp:81-175) keep the full solution history on the
// device and evaluate the O(n) direct CQ sums per level (kernel K10).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "history.cuh"

namespace fraqcu {

namespace {

constexpr int kMaxLevels = 20;

struct M2 {  // row-major 2x2
    double a, b, c, d;
};
__host__ __device__ inline M2 mul(const M2& x, const M2& y) {
    return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c,
            x.c * y.b + x.d * y.d};
}
__host__ __device__ inline M2 inv(const M2& x) {
    const double det = x.a * x.d - x.b * x.c;
    return {x.d / det, -x.b / det, -x.c / det, x.a / det};
}
__host__ __device__ inline M2 sub(const M2& x, const M2& y) {
    return {x.a - y.a, x.b - y.b, x.c - y.c, x.d - y.d};
}
__device__ inline double2 mv(const M2& m, double2 v) {
    return make_double2(fma(m.a, v.x, m.b * v.y), fma(m.c, v.x, m.d * v.y));
}

// Per system (instance x {first step, main}) solver data.
struct CRLevel {
    M2 F, G, H;  // F = E D^-1 (forward), G = D^-1, H = D^-1 E (backward)
};
struct SysDev {
    int K;               // CR levels (grid_m = 2^K - 1); 0 -> Thomas
    CRLevel lv[kMaxLevels];
    // Thomas: W[k] = E Delta_{k-1}^{-1}, Dinv[k] = Delta_k^{-1}; E stored below
    M2 E;
    long th_off;         // offset into thomas buffer (2 * grid_m M2 entries)
    // the block system's entries UNROUNDED, as double-double (hi, lo) pairs, for the residual of
    // the refinement step: row of field f reads
    //   diag_f x_f - e_f (x_f,left + x_f,right) - c_f x_other = b_f
    double dh[2], dl[2], eh[2], el[2], ch[2], cl[2];
};

// Block matrices of BlockSystem (block_solver.cpp:95-117), rounded exactly as the reference
// forms them: its Release build contracts the diagonal into fma(d0, fma(2, 1/h^2, a), lead/tau)
// (vfmadd132sd in the -O3 -march build).  These entries are the one place where fp64 rounding
// matters: the block system has cond ~1.4e6 at M = 4095, its diagonal is constant along the
// grid, so a rounding of the diagonal shifts every row the same way and the solution drifts
// systematically (3.8e-9 relative after 256 C3 steps for the reference itself).  Identical
// entries make the B200 solve converge to the reference's fp64 system, not to a neighbour of it.
void blocks(double d01, double d02, double a, double tau, double h, double lead, M2& D, M2& E) {
    const double ih2 = 1.0 / (h * h);
    const double lt = lead / tau;
    const double ad = std::fma(2.0, ih2, a);
    D = {std::fma(d01, ad, lt), -a * d02, -a * d01, std::fma(d02, ad, lt)};
    E = {-d01 * ih2, 0.0, 0.0, -d02 * ih2};
}

int cr_levels(int m) {
    int K = 0;
    while ((1L << K) - 1 < m) ++K;
    return ((1L << K) - 1 == m && K <= kMaxLevels) ? K : 0;
}

// Block cyclic-reduction coefficients of one system, computed in extended precision (x87 long
// double) and rounded once.  With fp64 recursion D_(l+1) = D_l - 2 E_l D_l^-1 E_l, every level's
// rounding is shared by all rows of that level -- a coherent perturbation of the system, like
// the entry rounding above -- and the solution drifted 6.6e-9 from the reference's after 256 C3
// steps; from extended-precision coefficients it stays within 1.2e-11 (profiles/r02/
// physical_bisect.txt).  The per-step reduction and substitution run in fp64 on the device:
// their rounding is not coherent across rows and does not accumulate.
struct M2L {
    long double a, b, c, d;
};
M2L mulL(const M2L& x, const M2L& y) {
    return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c,
            x.c * y.b + x.d * y.d};
}
M2L invL(const M2L& x) {
    const long double det = x.a * x.d - x.b * x.c;
    return {x.d / det, -x.b / det, -x.c / det, x.a / det};
}
M2 rnd(const M2L& x) { return {(double)x.a, (double)x.b, (double)x.c, (double)x.d}; }

void setup_cr(SysDev& S, const M2& D0, const M2& E0) {
    M2L D{D0.a, D0.b, D0.c, D0.d}, E{E0.a, E0.b, E0.c, E0.d};
    for (int l = 0; l < S.K; ++l) {
        const M2L Di = invL(D);
        const M2L F = mulL(E, Di);
        S.lv[l].F = rnd(F);
        S.lv[l].G = rnd(Di);
        S.lv[l].H = rnd(mulL(Di, E));
        const M2L FE = mulL(F, E);
        E = {-FE.a, -FE.b, -FE.c, -FE.d};
        D = {D.a - 2 * FE.a, D.b - 2 * FE.b, D.c - 2 * FE.c, D.d - 2 * FE.d};
    }
}

// ------------------------------------------------------------------ exact entries
// Double-double values (error-free transforms on fp64) of the unrounded block-system entries.
// The fp64 rounding of the constant diagonal lead/tau + d0 (a + 2/h^2) ~ 1e10 is what moves the
// reference's physical-space solution ~1e-6 away from the exact discrete one at C3 (the system's
// smooth modes amplify a diagonal shift by ~1e10 over the run, profiles/r02/physical_bisect.txt).
// One refinement step per level with a residual formed from these entries removes it.
struct DD {
    double hi, lo;
};
DD dd_two_sum(double a, double b) {
    const double s = a + b, bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
DD dd_norm(double hi, double lo) {
    const double s = hi + lo;
    return {s, lo - (s - hi)};
}
DD dd_add(DD x, DD y) {
    const DD s = dd_two_sum(x.hi, y.hi);
    return dd_norm(s.hi, s.lo + x.lo + y.lo);
}
DD dd_mul_d(DD x, double y) {
    const double p = x.hi * y;
    return dd_norm(p, std::fma(x.hi, y, -p) + x.lo * y);
}
DD dd_div_d(DD x, double y) {  // x / y
    const double q = x.hi / y;
    const double r = std::fma(-q, y, x.hi) + x.lo;
    return dd_norm(q, r / y);
}
DD dd_div_dd(double x, DD y) {  // x / y
    const double q = x / y.hi;
    const double r = std::fma(-q, y.hi, x) - q * y.lo;
    return dd_norm(q, r / y.hi);
}

// d0f = d0 * fnum / fden exactly (the SBD first step uses 2/3 d0, fpfp.cpp:224)
void exact_entries(SysDev& S, double d01, double d02, double fnum, double fden, double a,
                   double tau, double h, double lead) {
    const DD h2 = dd_norm(h * h, std::fma(h, h, -h * h));
    const DD ih2 = dd_div_dd(1.0, h2);
    const DD lt = dd_div_d(DD{lead, 0.0}, tau);
    const DD d0[2] = {dd_div_d(dd_mul_d(DD{d01, 0.0}, fnum), fden),
                      dd_div_d(dd_mul_d(DD{d02, 0.0}, fnum), fden)};
    for (int f = 0; f < 2; ++f) {
        const DD e = dd_mul_d(ih2, d0[f].hi);
        const DD e_full = dd_add(e, dd_mul_d(ih2, d0[f].lo));
        const DD da = dd_add(dd_mul_d(d0[f], a), DD{0.0, 0.0});
        const DD diag = dd_add(lt, dd_add(da, dd_mul_d(e_full, 2.0)));
        const DD c = dd_mul_d(d0[1 - f], a);
        S.dh[f] = diag.hi;
        S.dl[f] = diag.lo;
        S.eh[f] = e_full.hi;
        S.el[f] = e_full.lo;
        S.ch[f] = c.hi;
        S.cl[f] = c.lo;
    }
}

__global__ void thomas_setup_kernel(const SysDev* sys, const M2* Dm, int n_sys, int m, M2* buf) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_sys) return;
    const SysDev& S = sys[t];
    if (S.K) return;
    const M2 D = Dm[t], E = S.E;
    M2* W = buf + S.th_off;      // W[k], k >= 1
    M2* Dinv = W + m;            // Delta_k^{-1}
    M2 Delta = D;
    Dinv[0] = inv(Delta);
    W[0] = {0, 0, 0, 0};
    for (int k = 1; k < m; ++k) {
        const M2 Wk = mul(E, Dinv[k - 1]);
        W[k] = Wk;
        Delta = sub(D, mul(Wk, E));
        Dinv[k] = inv(Delta);
    }
}

// ----------------------------------------------------------------------------- per-instance data
struct InstDev {
    double a, tau, h;
    int g1, g2;          // history groups of the two fields
    int sys_main, sys_first;
    long g0_off;         // G^0 copies (2 * m doubles)
    long corr_off1, corr_off2;  // SBD correction sequences (index e)
    int nh1, nh2;        // exact head lengths of the reference kernels (the history groups may
                         // carry folded kernels with longer heads)
};

struct SolveArgs {
    const InstDev* inst;
    const SysDev* sys;
    const M2* thomas;
    const GroupDev* groups;
    double* ring;
    const double* s;      // s1/s2 per group, user layout (group dof0)
    const double* g0;
    const double* corr;   // K7 sequences
    const double* head;   // per group heads (hd_off)
    int m;
    long n;               // level being produced
    int sbd;
    int first;            // SBD first step
    double* out;          // nullable: final state (inst * 2m: g1 then g2)
    int refine;           // refinement step against the unrounded entries (always, except in
                          // the FRAQ_K6_NOREFINE timing experiment)
    int tap1;             // add the newest head tap d_1 G^(n-1) here (K5 ran with first_tap 2)
    const long* n_dev;    // CUDA-graph replays: n = *n_dev + n_off, first step never inside
    int n_off;
    long long* prof;      // nullable: block 0 phase timestamps (FRAQ_K6_PROFILE experiment)
    double* hist_out;     // classical schemes: G^n also into the full history row n
    long hist_total;
};

// Row storage of the on-chip solve: row i at slot i + i/8 + i/64 + i/512.  Cyclic reduction
// touches rows at power-of-two strides; with rows packed densely (16-byte double2) a warp at
// stride 8+ hit one bank group 32 times over (levels 1-2 and their back-substitution took ~2200
// cycles each at M = 4095); the pad slots spread every power-of-two stride over the banks
// (profiles/microbench/mb_cr.cu: one solve 21.9k -> 13.1k cycles).
struct Rows {
    double2* p;
    __device__ __forceinline__ double2& operator[](int i) const {
        return p[i + (i >> 3) + (i >> 6) + (i >> 9)];
    }
};
// slots for rows 0 .. m+1
__host__ __device__ constexpr size_t rows_len(int m) {
    return (size_t)(m + 1) + ((m + 1) >> 3) + ((m + 1) >> 6) + ((m + 1) >> 9) + 1;
}

// The 2x2-block tridiagonal solve of BlockSystem::solve (block_solver.cpp:119-153) on one CTA,
// in place on sb[1..m] (sb[0] = sb[m+1] = 0): block cyclic reduction with the setup
// coefficients (grid_m = 2^K - 1), else block Thomas (one thread; general grid sizes).  The
// levels with at most 32 active rows run on warp 0 alone (__syncwarp between them; -10%).
// Ends with __syncthreads().
template <int THREADS>
__device__ void block_solve_smem(Rows sb, const SysDev& S, const M2* thomas, int m) {
    if (S.K > 0) {
        const int K = S.K;
        const int lw = K > 6 ? K - 6 : 0;  // first level with <= 31 rows
        // forward reduction
        for (int l = 0; l < lw; ++l) {
            const int s = 1 << l;
            const M2 F = S.lv[l].F;
            for (int i = 2 * s * (threadIdx.x + 1); i <= m; i += 2 * s * THREADS) {
                const double2 sum = make_double2(sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y);
                const double2 t = mv(F, sum);
                sb[i] = make_double2(sb[i].x - t.x, sb[i].y - t.y);
            }
            __syncthreads();
        }
        if (threadIdx.x < 32) {
            for (int l = lw; l < K - 1; ++l) {
                const int s = 1 << l;
                const M2 F = S.lv[l].F;
                for (int i = 2 * s * (threadIdx.x + 1); i <= m; i += 64 * s) {
                    const double2 sum =
                        make_double2(sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y);
                    const double2 t = mv(F, sum);
                    sb[i] = make_double2(sb[i].x - t.x, sb[i].y - t.y);
                }
                __syncwarp();
            }
            if (threadIdx.x == 0) {
                const int i = 1 << (K - 1);
                sb[i] = mv(S.lv[K - 1].G, sb[i]);
            }
            __syncwarp();
            for (int l = K - 2; l >= lw; --l) {
                const int s = 1 << l;
                const M2 Gm = S.lv[l].G, H = S.lv[l].H;
                for (int i = s * (2 * (int)threadIdx.x + 1); i <= m; i += 64 * s) {
                    const double2 xb = mv(Gm, sb[i]);
                    const double2 nb =
                        make_double2(sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y);
                    const double2 t = mv(H, nb);
                    sb[i] = make_double2(xb.x - t.x, xb.y - t.y);
                }
                __syncwarp();
            }
        }
        __syncthreads();
        for (int l = lw - 1; l >= 0; --l) {
            const int s = 1 << l;
            const M2 Gm = S.lv[l].G, H = S.lv[l].H;
            for (int i = s * (2 * (int)threadIdx.x + 1); i <= m; i += 2 * s * THREADS) {
                const double2 xb = mv(Gm, sb[i]);
                const double2 nb = make_double2(sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y);
                const double2 t = mv(H, nb);
                sb[i] = make_double2(xb.x - t.x, xb.y - t.y);
            }
            __syncthreads();
        }
    } else if (threadIdx.x == 0) {
        // block Thomas with the setup factors
        const M2* W = thomas + S.th_off;
        const M2* Dinv = W + m;
        for (int k = 1; k < m; ++k) {
            const double2 t = mv(W[k], sb[k]);
            sb[k + 1] = make_double2(sb[k + 1].x - t.x, sb[k + 1].y - t.y);
        }
        sb[m] = mv(Dinv[m - 1], sb[m]);
        for (int k = m - 2; k >= 0; --k) {
            const double2 ex = mv(S.E, sb[k + 2]);
            sb[k + 1] = mv(Dinv[k], make_double2(sb[k + 1].x - ex.x, sb[k + 1].y - ex.y));
        }
    }
    __syncthreads();
}

// One refinement step: sb holds x0 (solve of b), sr holds b.  sr <- b - A x0 with the unrounded
// entries in double-double accumulation, solved in place, and added: sb <- x0 + A^-1 r.  The
// correction is ~1e-10 of x0 (cond ~1e6 x eps), so the approximate reduction suffices for it.
__device__ inline void dd_acc(double& s, double& t, double p) {
    const double u = s + p, bb = u - s;
    t += (s - (u - bb)) + (p - bb);
    s = u;
}
__device__ inline void dd_acc_prod(double& s, double& t, double c, double x) {
    const double p = c * x;
    t += fma(c, x, -p);
    dd_acc(s, t, p);
}
__device__ inline double residual_row(double b, double x, double xl, double xr, double xo,
                                      double dh, double dl, double eh, double el, double ch,
                                      double cl) {
    double s = b, t = 0.0;
    dd_acc_prod(s, t, -dh, x);
    dd_acc_prod(s, t, eh, xl);
    dd_acc_prod(s, t, eh, xr);
    dd_acc_prod(s, t, ch, xo);
    t += el * (xl + xr) + cl * xo - dl * x;
    return s + t;
}
template <int THREADS>
__device__ void refine_smem(Rows sb, Rows sr, const SysDev& S, const M2* thomas, int m) {
    for (int k = threadIdx.x; k < m; k += THREADS) {
        const double2 x = sb[k + 1], l = sb[k], r = sb[k + 2], b = sr[k + 1];
        const double r1 = residual_row(b.x, x.x, l.x, r.x, x.y, S.dh[0], S.dl[0], S.eh[0],
                                       S.el[0], S.ch[0], S.cl[0]);
        const double r2 = residual_row(b.y, x.y, l.y, r.y, x.x, S.dh[1], S.dl[1], S.eh[1],
                                       S.el[1], S.ch[1], S.cl[1]);
        sr[k + 1] = make_double2(r1, r2);
    }
    if (threadIdx.x == 0) {
        sr[0] = make_double2(0.0, 0.0);
        sr[m + 1] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    block_solve_smem<THREADS>(sr, S, thomas, m);
    for (int k = threadIdx.x; k < m; k += THREADS) {
        const double2 x = sb[k + 1], d = sr[k + 1];
        sb[k + 1] = make_double2(x.x + d.x, x.y + d.y);
    }
    __syncthreads();
}

// The system's reduction coefficients into shared memory, one coalesced copy: read from global
// memory level by level, every CR level would first wait for an L1 miss (~700 cycles) -- 2/3 of
// the whole solve at M = 4095 before this (41 -> 25 us per level at C3 with the refinement).
template <int THREADS>
__device__ void stage_sys(SysDev* dst, const SysDev* src) {
    static_assert(sizeof(SysDev) % sizeof(double) == 0, "SysDev is copied as doubles");
    const double* s = reinterpret_cast<const double*>(src);
    double* d = reinterpret_cast<double*>(dst);
    for (int i = threadIdx.x; i < (int)(sizeof(SysDev) / sizeof(double)); i += THREADS) d[i] = s[i];
}

// BlockSystem::solve on its own (block_solver.cpp:119-153): one CTA per system.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) block_solve_kernel(const SysDev* sys, const M2* thomas,
                                                              int m, const double* rhs1,
                                                              const double* rhs2, double* g1,
                                                              double* g2) {
    extern __shared__ double2 smem_rows[];
    const Rows sb{smem_rows};
    const Rows sr{smem_rows + rows_len(m)};  // the right-hand side, kept for the refinement
    __shared__ SysDev S;
    stage_sys<THREADS>(&S, sys);
    for (int k = threadIdx.x; k < m; k += THREADS) {
        sb[k + 1] = make_double2(rhs1[k], rhs2[k]);
        sr[k + 1] = sb[k + 1];
    }
    if (threadIdx.x == 0) {
        sb[0] = make_double2(0.0, 0.0);
        sb[m + 1] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    block_solve_smem<THREADS>(sb, S, thomas, m);
    refine_smem<THREADS>(sb, sr, S, thomas, m);
    for (int k = threadIdx.x; k < m; k += THREADS) {
        g1[k] = sb[k + 1].x;
        g2[k] = sb[k + 1].y;
    }
}

// DiscreteLaplacian::apply (block_solver.cpp:10-19): y = (2 x_i - x_{i-1} - x_{i+1}) / h^2.
__global__ void laplacian_kernel(int m, double ih2, const double* x, double* y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    double v = 2.0 * x[i];
    if (i > 0) v -= x[i - 1];
    if (i + 1 < m) v -= x[i + 1];
    y[i] = v * ih2;
}

// BandedLU (block_solver.cpp:28-93): LAPACK gbtrf band storage ab[(kl+ku+row-col) + col*ldab],
// partial pivoting from the kl rows below the diagonal.  A general-purpose sequential
// factorization; one thread (the FFPE path uses the block solve above instead).
__global__ void banded_factor_kernel(double* ab, int* piv, int n, int kl, int ku, int* status) {
    const int ldab = 2 * kl + ku + 1, kv = kl + ku;
    for (int j = 0; j < n; ++j) {
        const int jmax = min(n - 1, j + kl);
        int p = j;
        double pmax = fabs(ab[(size_t)j * ldab + kv]);
        for (int i = j + 1; i <= jmax; ++i) {
            const double v = fabs(ab[(size_t)j * ldab + kv + (i - j)]);
            if (v > pmax) {
                pmax = v;
                p = i;
            }
        }
        if (pmax == 0.0) {
            *status = 1;
            return;
        }
        piv[j] = p;
        const int cmax = min(n - 1, j + kv);
        if (p != j)
            for (int c = j; c <= cmax; ++c) {
                double* base = ab + (size_t)c * ldab + kv;
                const double t = base[j - c];
                base[j - c] = base[p - c];
                base[p - c] = t;
            }
        const double dinv = 1.0 / ab[(size_t)j * ldab + kv];
        for (int i = j + 1; i <= jmax; ++i) {
            double& lij = ab[(size_t)j * ldab + kv + (i - j)];
            lij *= dinv;
            const double l = lij;
            for (int c = j + 1; c <= cmax; ++c) {
                double* base = ab + (size_t)c * ldab + kv;
                base[i - c] -= l * base[j - c];
            }
        }
    }
    *status = 0;
}

__global__ void banded_solve_kernel(const double* ab, const int* piv, int n, int kl, int ku,
                                    double* rhs) {
    const int ldab = 2 * kl + ku + 1, kv = kl + ku;
    for (int j = 0; j < n; ++j) {
        if (piv[j] != j) {
            const double t = rhs[j];
            rhs[j] = rhs[piv[j]];
            rhs[piv[j]] = t;
        }
        const int imax = min(n - 1, j + kl);
        const double xj = rhs[j];
        for (int i = j + 1; i <= imax; ++i) rhs[i] -= ab[(size_t)j * ldab + kv + (i - j)] * xj;
    }
    for (int j = n - 1; j >= 0; --j) {
        double v = rhs[j];
        for (int c = j + 1; c <= min(n - 1, j + kv); ++c)
            v -= ab[(size_t)c * ldab + kv + (j - c)] * rhs[c];
        rhs[j] = v / ab[(size_t)j * ldab + kv];
    }
}

__device__ inline int m_of(const SolveArgs& A) { return A.m; }

// RHS (fpfp.cpp:277-279, 298-302, 339-344) then the block solve + one refinement step; one CTA
// per instance.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) solve_kernel(SolveArgs A) {
    extern __shared__ double2 smem_rows[];
    const Rows sb{smem_rows};                       // b / x, rows 1..m (rows 0, m+1 are zero)
    const Rows sr{smem_rows + rows_len(m_of(A))};  // b, kept for the refinement residual
    auto stamp = [&](int q) {
        if (A.prof && blockIdx.x == 0 && threadIdx.x == 0) A.prof[q] += clock64();
    };
    stamp(0);
    __shared__ SysDev S;
    const InstDev I = A.inst[blockIdx.x];
    stage_sys<THREADS>(&S, A.sys + (A.sbd && !A.n_dev && A.first ? I.sys_first : I.sys_main));
    const GroupDev G1 = A.groups[I.g1], G2 = A.groups[I.g2];
    const int m = A.m;
    const double a = I.a, tau = I.tau, ih2 = 1.0 / (I.h * I.h);
    // 1/tau once: the reference divides by tau per entry; for the power-of-two steps of every
    // BASELINE config the product is bit-identical, otherwise it differs in the last bit of the
    // RHS, which the refinement step does not care about (fp64 division is ~40 instructions)
    const double itau = 1.0 / tau;
    const long n = A.n_dev ? *A.n_dev + A.n_off : A.n;
    const int first = A.n_dev ? 0 : A.first;
    const double* r1 = A.ring + G1.ring_off;
    const double* r2 = A.ring + G2.ring_off;
    const long ld = G1.ld;
    const double* p1 = r1 + ((n - 1) % G1.L) * ld;  // G^{n-1}
    const double* p2 = r2 + ((n - 1) % G2.L) * ld;
    double c1 = 0.0, c2 = 0.0;
    const double* s1 = A.s + G1.dof0;
    const double* s2 = A.s + G2.dof0;
    const double* q1 = nullptr;
    const double* q2 = nullptr;
    if (A.sbd && !first) {
        q1 = r1 + ((n - 2) % G1.L) * ld;  // G^{n-2}
        q2 = r2 + ((n - 2) % G2.L) * ld;
        if (A.corr) {
            // (1/2) d_{n-1} G^0: exact head inside, reconstructed (running powers) beyond
            c1 = (n - 1 < I.nh1) ? A.head[G1.hd_off + n - 1] : A.corr[I.corr_off1 + (n - 4)];
            c2 = (n - 1 < I.nh2) ? A.head[G2.hd_off + n - 1] : A.corr[I.corr_off2 + (n - 4)];
        }
    }
    const double* g01 = A.g0 + I.g0_off;
    const double* g02 = g01 + m;
    const double d10 = A.head[G1.hd_off], d20 = A.head[G2.hd_off];
    // newest head tap (fpfp.cpp:270-275 BE, 313-324 SBD i = 1), when the history pass left it
    const bool tap = A.tap1 && n >= 2;
    const double d11 = tap ? A.head[G1.hd_off + 1] : 0.0, d21 = tap ? A.head[G2.hd_off + 1] : 0.0;
    for (int k = threadIdx.x; k < m; k += THREADS) {
        double b1, b2;
        if (A.sbd && first) {
            // 2/3-1/3 first step from G^0 (fpfp.cpp:293-303)
            const double u = p1[k], v = p2[k];
            const double au = (2.0 * u - (k > 0 ? p1[k - 1] : 0.0) - (k + 1 < m ? p1[k + 1] : 0.0)) * ih2;
            const double av = (2.0 * v - (k > 0 ? p2[k - 1] : 0.0) - (k + 1 < m ? p2[k + 1] : 0.0)) * ih2;
            b1 = u * itau - (d10 / 3.0) * (a * u + au) + (a * d20 / 3.0) * v;
            b2 = v * itau - (d20 / 3.0) * (a * v + av) + (a * d10 / 3.0) * u;
        } else {
            double x1 = s1[k], x2 = s2[k];
            double l1 = k > 0 ? s1[k - 1] : 0.0, rr1 = k + 1 < m ? s1[k + 1] : 0.0;
            double l2 = k > 0 ? s2[k - 1] : 0.0, rr2 = k + 1 < m ? s2[k + 1] : 0.0;
            if (tap) {
                x1 = fma(d11, p1[k], x1);
                x2 = fma(d21, p2[k], x2);
                if (k > 0) {
                    l1 = fma(d11, p1[k - 1], l1);
                    l2 = fma(d21, p2[k - 1], l2);
                }
                if (k + 1 < m) {
                    rr1 = fma(d11, p1[k + 1], rr1);
                    rr2 = fma(d21, p2[k + 1], rr2);
                }
            }
            if (A.sbd && A.corr) {
                x1 += 0.5 * c1 * g01[k];
                x2 += 0.5 * c2 * g02[k];
                if (k > 0) {
                    l1 += 0.5 * c1 * g01[k - 1];
                    l2 += 0.5 * c2 * g02[k - 1];
                }
                if (k + 1 < m) {
                    rr1 += 0.5 * c1 * g01[k + 1];
                    rr2 += 0.5 * c2 * g02[k + 1];
                }
            }
            const double as1 = (2.0 * x1 - l1 - rr1) * ih2;
            const double as2 = (2.0 * x2 - l2 - rr2) * ih2;
            double lead1, lead2;
            if (A.sbd) {
                lead1 = (2.0 * p1[k] - 0.5 * q1[k]) * itau;
                lead2 = (2.0 * p2[k] - 0.5 * q2[k]) * itau;
            } else {
                lead1 = p1[k] * itau;
                lead2 = p2[k] * itau;
            }
            b1 = lead1 - a * x1 - as1 + a * x2;
            b2 = lead2 - a * x2 - as2 + a * x1;
        }
        sb[k + 1] = make_double2(b1, b2);
        sr[k + 1] = sb[k + 1];
    }
    if (threadIdx.x == 0) {
        sb[0] = make_double2(0.0, 0.0);
        sb[m + 1] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    stamp(1);
    block_solve_smem<THREADS>(sb, S, A.thomas, m);
    stamp(2);
    if (A.refine) refine_smem<THREADS>(sb, sr, S, A.thomas, m);
    stamp(3);
    // append G^n into both rings (slot n % L)
    double* w1 = A.ring + G1.ring_off + (n % G1.L) * ld;
    double* w2 = A.ring + G2.ring_off + (n % G2.L) * ld;
    for (int k = threadIdx.x; k < m; k += THREADS) {
        const double2 x = sb[k + 1];
        w1[k] = x.x;
        w2[k] = x.y;
        if (A.out) {
            A.out[(long)blockIdx.x * 2 * m + k] = x.x;
            A.out[(long)blockIdx.x * 2 * m + m + k] = x.y;
        }
        if (A.hist_out) {
            double* row = A.hist_out + n * A.hist_total;
            row[G1.dof0 + k] = x.x;
            row[G2.dof0 + k] = x.y;
        }
    }
    if (A.prof) {
        __syncthreads();
        stamp(4);
    }
}

// Classical direct sums (fpfp.cpp:114-122, 150-164):
//   s_n[k] = (SBD: 0.5 d_(n-1) G^0[k]) + sum_(i=1)^(n-1) d_i G^(n-i)[k]
// over the full device history hist[t][k] (k = group * m + j; group g = field of an instance,
// weights d of group g at ctab + g * (N + 1)).  Evaluated per block of kCB levels: the levels
// before the block enter once per block as a Toeplitz GEMM on the fp64 tensor cores (K10's tile
// scheme, per-group weights), the levels inside the block per level.  The direct per-level sum
// re-read the whole history every level (O(N^2 M) memory traffic: ~1400 s for C3's shape,
// slower than the reference's CPU loop); blocked, the history is read once per kCB levels.
constexpr int kCB = 64;            // classical block (levels) == GEMM M tile
constexpr int CT_N = 64, CT_K = 16;

__device__ __forceinline__ void cdmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// S_old[r][k] = sum_(q<n0) A_g[r][q] hist[q][k], level n = n0 + r, A_g[r][q] = d_g[n - q] for
// q >= 1, the SBD correction 0.5 d_g[n - 1] for q = 0 (BE: 0).  grid.x = (group, 64-DOF tile).
__global__ void __launch_bounds__(128) classical_old_kernel(const double* __restrict__ hist,
                                                           long total, const double* __restrict__ ctab,
                                                           long d_ld, int m, int tiles_per_group,
                                                           long n0, int rows, int sbd, double* Sold) {
    __shared__ double sA[kCB][CT_K + 1];
    __shared__ double sB[CT_K][CT_N + 1];
    const int grp = blockIdx.x / tiles_per_group, tile = blockIdx.x % tiles_per_group;
    const double* w = ctab + (size_t)grp * d_ld;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int g = lane >> 2, t = lane & 3;
    const long j0c = (long)tile * CT_N;          // first DOF of the tile within the group
    const long k0 = (long)grp * m + j0c;         // history column
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (long q0 = 0; q0 < n0; q0 += CT_K) {
        __syncthreads();
        for (int idx = tid; idx < kCB * CT_K; idx += 128) {
            const int r = idx / CT_K, cq = idx % CT_K;
            const long q = q0 + cq, n = n0 + r;
            double v = 0.0;
            if (r < rows && q < n0) v = q == 0 ? (sbd ? 0.5 * w[n - 1] : 0.0) : w[n - q];
            sA[r][cq] = v;
        }
        for (int idx = tid; idx < CT_K * CT_N; idx += 128) {
            const int r = idx / CT_N, cc = idx % CT_N;
            const long q = q0 + r;
            sB[r][cc] = (q < n0 && j0c + cc < m) ? hist[q * total + k0 + cc] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < CT_K; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = sA[wm + 8 * a + g][kk + t];
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = sB[kk + t][wn + 8 * b + g];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) cdmma(acc[a][b], af[a], bf[b]);
        }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = wm + 8 * a + g;
                const long jj = j0c + wn + 8 * b + 2 * t + e;
                if (r < rows && jj < m) Sold[(long)r * total + (long)grp * m + jj] = acc[a][b][e];
            }
}

// s_n[k] = S_old[n - n0][k] + sum_(q = n0)^(n-1) d[n - q] hist[q][k]  (levels of the block)
__global__ void classical_inblock_kernel(const double* hist, long total, const double* ctab,
                                         long d_ld, int m, long n0, long n, const double* Sold,
                                         double* s) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= total) return;
    const double* w = ctab + (k / m) * d_ld;
    double acc = Sold[(n - n0) * total + k];
    for (long q = n0; q < n; ++q) acc = fma(w[n - q], hist[q * total + k], acc);
    s[k] = acc;
}

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void initial_field(const fraq_spec_t& s, double* g1, double* g2) {
    // fpfp.cpp:40-70
    const int m = s.grid_m;
    const double h = s.length / double(m + 1);
    for (int j = 0; j < m; ++j) {
        const double x = (j + 1) * h;
        switch (s.initial) {
            case FRAQ_POLY_SIN:
                g1[j] = x * (1.0 - x);
                g2[j] = std::sin(x);
                break;
            case FRAQ_INDICATOR:
                g1[j] = x > 0.5 ? 1.0 - x : 0.0;
                g2[j] = x < 0.5 ? x : 0.0;
                break;
            default:
                g1[j] = s.custom_g1[j];
                g2[j] = s.custom_g2[j];
        }
    }
}

}  // namespace

// Kernel tables for both fields of every instance (auto-sized like FastStepper, or fixed
// sizes + certificate), batched over exponents on the device.  fpfp.cpp:185-227.
void build_ffpe_kernels(fraq_ctx c, const std::vector<double>& gam, double tau, long N, bool sbd,
                        const fraq_kconf_t& kc, std::vector<fraq_kernel_t>& ks,
                        std::vector<double>& eps) {
    const int n = (int)gam.size();
    ks.resize(n);
    eps.assign(n, 0.0);
    if (kc.auto_size) {
        std::vector<fraq_budget_t> bud(n);
        for (auto& b : bud) b = fraq_budget_t{N, kc.eps_tol, 256, 256, 0.0};
        build_kernel_auto_dev(c, sbd, n, gam.data(), tau, bud.data(), ks.data());
        for (int t = 0; t < n; ++t) eps[t] = bud[t].achieved_eps;
        return;
    }
    for (int t = 0; t < n; ++t) {
        long am;
        if (sbd) {
            const int hh = kc.sbd_head > 0 ? kc.sbd_head : (gam[t] <= 0.5 ? 15 : 17);
            build_sbd_kernel_dev(c, gam[t], tau, kc.sbd_points_1, kc.sbd_points_2, hh, &ks[t]);
            kernel_error_report_dev(c, &ks[t], N > 8 ? N : 8, nullptr, &eps[t], &am);
        } else {
            build_be_kernel_dev(c, gam[t], tau, kc.be_points, &ks[t]);
            kernel_error_report_dev(c, &ks[t], N > 2 ? N : 2, nullptr, &eps[t], &am);
        }
    }
}

void ffpe_run_modal(fraq_ctx c, const fraq_spec_t* specs, int n_inst, bool sbd,
                    const fraq_kconf_t& kc, double* g1_out, double* g2_out, fraq_run_info_t* info);

// ================================================================================ PhysStepper
// ClassicalStepper / FastStepper (fpfp.cpp:81-349) for a batch of instances in physical space:
// the device state of one or many instances stepped level by level.  Behind ffpe_run (physical
// solver, observer runs) and the stepper handles of the C ABI (fraq_stepper_*).
struct PhysStepper {
    fraq_ctx c = nullptr;
    int n_inst = 0, m = 0;
    int fold_levels[2] = {0, 0};  // head levels the last instance's kernels were folded by
    long N = 0;        // horizon the kernels / classical tables are sized for
    bool sbd = false, fast = false;
    double tau = 0.0;
    std::vector<double> G0, eps, d0;
    std::vector<fraq_kernel_t> ks;
    DevBuf<double> ctab, g0, corr, sbuf, outb, hist, sold;
    DevBuf<SysDev> dsys;
    DevBuf<M2> thomas;
    DevBuf<InstDev> dinst;
    HistDevice hd;
    SolveArgs sa{};
    long level = 0, appended = 1, step_idx = 0, total = 0;
    size_t smem = 0;
    int k6_threads = 512;
    double setup_seconds = 0.0;
    // CUDA graph of kGraphLevels levels of the fast schemes: the history pass of level n+1 (K5,
    // side stream) overlaps the solve of level n (K6, context stream); the level comes from a
    // device counter that the graph's last node advances, so one instantiated graph replays
    // for the whole run.  Built on first use.
    static constexpr int kGraphLevels = 64;
    cudaGraphExec_t gexec = nullptr;
    cudaStream_t s5 = nullptr;
    std::vector<cudaEvent_t> gev;
    DevBuf<long> ndev;
    bool use_graph = true;

    PhysStepper(fraq_ctx c_, const fraq_spec_t* specs, int n_inst_, int scheme,
                const fraq_kconf_t& kc);
    ~PhysStepper();
    StepArgs k5_args(long n) const;
    void launch_k6(long n, bool last, cudaStream_t stream, const long* n_dev, int n_off);
    void build_graph();
    void step(long n_steps, std::vector<cudaEvent_t>* ev = nullptr);  // stream-ordered
    // diagnostics: step n levels with an event pair around every kernel; returns the summed
    // device time of the history kernels (K5 / classical sums) and of the solves (K6)
    void time_split(long n_steps, double* ms_hist, double* ms_solve);
    void state(double* g1, double* g2);  // [n_inst][m] each; synchronizes
};

void validate_specs(const fraq_spec_t* specs, int n_inst, int scheme) {
    if (n_inst < 1) fail(FRAQ_EINVAL, "run: need at least one instance");
    const fraq_spec_t& s0 = specs[0];
    if (s0.grid_m < 1) fail(FRAQ_EINVAL, "run: grid_m must be >= 1");
    if (s0.n_steps < 1) fail(FRAQ_EINVAL, "run: n_steps must be >= 1");
    for (int i = 0; i < n_inst; ++i) {
        const fraq_spec_t& s = specs[i];
        if (s.grid_m != s0.grid_m || s.n_steps != s0.n_steps || s.t_final != s0.t_final ||
            s.length != s0.length)
            fail(FRAQ_EINVAL, "run: batched instances must share grid_m, n_steps, t_final, length");
        if (s.initial == FRAQ_CUSTOM && (!s.custom_g1 || !s.custom_g2))
            fail(FRAQ_EINVAL, "initial_field: custom samples must have grid_m entries");
        if (s.initial < 0 || s.initial > 2) fail(FRAQ_EINVAL, "unknown initial data tag");
    }
    if (scheme < FRAQ_BE || scheme > FRAQ_FASTSBD) fail(FRAQ_EINVAL, "run: unknown scheme");
}

PhysStepper::PhysStepper(fraq_ctx c_, const fraq_spec_t* specs, int n_inst_, int scheme,
                         const fraq_kconf_t& kc)
    : c(c_), n_inst(n_inst_) {
    const double t_setup0 = now_s();
    const fraq_spec_t& s0 = specs[0];
    m = s0.grid_m;
    N = s0.n_steps;
    sbd = scheme == FRAQ_SBD || scheme == FRAQ_FASTSBD;
    fast = scheme == FRAQ_FASTBE || scheme == FRAQ_FASTSBD;
    tau = s0.t_final / double(N);
    const double h = s0.length / double(m + 1);

    // ---------------------------------------------------------------- initial data
    G0.resize((size_t)n_inst * 2 * m);
    for (int i = 0; i < n_inst; ++i)
        initial_field(specs[i], G0.data() + (size_t)i * 2 * m, G0.data() + (size_t)i * 2 * m + m);

    // ---------------------------------------------------------------- kernels / weights
    std::vector<double> gam(2 * n_inst);
    for (int i = 0; i < n_inst; ++i) {
        gam[2 * i] = 1.0 - specs[i].alpha1;
        gam[2 * i + 1] = 1.0 - specs[i].alpha2;
    }
    eps.assign(2 * n_inst, 0.0);
    d0.resize(2 * n_inst);
    if (fast) {
        build_ffpe_kernels(c, gam, tau, N, sbd, kc, ks, eps);
        for (int t = 0; t < 2 * n_inst; ++t) d0[t] = ks[t].head[0];
    } else {
        ctab.alloc((size_t)2 * n_inst * (N + 1));
        for (int t = 0; t < 2 * n_inst; ++t) {
            if (sbd)
                sbd_weights_dev(c, gam[t], tau, N, ctab.p + (size_t)t * (N + 1));
            else
                be_weights_dev(c, gam[t], tau, N, ctab.p + (size_t)t * (N + 1));
            FRAQ_CUDA(cudaMemcpy(&d0[t], ctab.p + (size_t)t * (N + 1), sizeof(double),
                                 cudaMemcpyDeviceToHost));
        }
    }

    // ---------------------------------------------------------------- block systems
    const int K = cr_levels(m);
    const int n_sys = n_inst * (sbd ? 2 : 1);
    std::vector<SysDev> sys(n_sys);
    std::vector<M2> sysD(n_sys);
    std::vector<InstDev> inst(n_inst);
    long th = 0;
    for (int i = 0; i < n_inst; ++i) {
        const double a = specs[i].coupling_a;
        auto mk = [&](int sidx, double f, double lead) {
            M2 D, E;
            // d01 = f * d0 as the reference scales it (2/3 d_0 for the first SBD step)
            blocks(f * d0[2 * i], f * d0[2 * i + 1], a, tau, h, lead, D, E);
            SysDev& S = sys[sidx];
            S.K = K;
            S.E = E;
            exact_entries(S, d0[2 * i], d0[2 * i + 1], f == 1.0 ? 1.0 : 2.0, f == 1.0 ? 1.0 : 3.0,
                          a, tau, h, lead);
            sysD[sidx] = D;
            if (K)
                setup_cr(S, D, E);
            else {
                S.th_off = th;
                th += 2L * m;
            }
        };
        InstDev& I = inst[i];
        I.a = a;
        I.tau = tau;
        I.h = h;
        I.g1 = 2 * i;
        I.g2 = 2 * i + 1;
        I.g0_off = (long)i * 2 * m;
        I.nh1 = fast ? ks[2 * i].n_head : 2;
        I.nh2 = fast ? ks[2 * i + 1].n_head : 2;
        if (sbd) {
            I.sys_main = 2 * i;
            I.sys_first = 2 * i + 1;
            mk(2 * i, 1.0, 1.5);
            mk(2 * i + 1, 2.0 / 3.0, 1.0);
        } else {
            I.sys_main = i;
            I.sys_first = i;
            mk(i, 1.0, 1.0);
        }
    }
    dsys.alloc(n_sys);
    FRAQ_CUDA(cudaMemcpy(dsys.p, sys.data(), sizeof(SysDev) * n_sys, cudaMemcpyHostToDevice));
    thomas.alloc(std::max<long>(1, th));
    if (!K) {
        DevBuf<M2> dD(n_sys);
        FRAQ_CUDA(cudaMemcpy(dD.p, sysD.data(), sizeof(M2) * n_sys, cudaMemcpyHostToDevice));
        thomas_setup_kernel<<<(n_sys + 127) / 128, 128, 0, c->stream>>>(dsys.p, dD.p, n_sys, m,
                                                                       thomas.p);
        FRAQ_LAUNCH_CHECK();
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    }

    // ---------------------------------------------------------------- histories / buffers
    std::vector<long> dims(2 * n_inst, m);
    std::vector<const fraq_kernel_t*> kp(2 * n_inst);
    std::vector<fraq_kernel_t> pseudo;  // classical: a 2-slot lag ring carrier (no nodes)
    std::vector<fraq_kernel_t> folded;  // fast: kernels with the fast-decaying nodes in the head
    if (fast) {
        for (int t = 0; t < 2 * n_inst; ++t) kp[t] = &ks[t];
        // The K5 pass streams every node's state once per level; the nodes that forget within M
        // levels move into the exact head instead (fold_kernel, history_fir.cu: the rewrite
        // K13 and K5e / K5f use), which leaves 16 bytes per kept node + 8 per head tap.
        if (!std::getenv("FRAQ_NO_PHYS_FOLD")) {
            int lcap = 96;
            if (const char* e = std::getenv("FRAQ_PHYS_LCAP")) lcap = std::atoi(e);  // experiment
            folded.resize(2 * n_inst);
            for (int t = 0; t < 2 * n_inst; ++t) {
                fold_levels[t % 2] = 0;
                if (int M = fold_kernel(ks[t], lcap, &folded[t])) {
                    kp[t] = &folded[t];
                    fold_levels[t % 2] = M;
                }
            }
        }
    } else {
        pseudo.resize(2 * n_inst);
        for (int t = 0; t < 2 * n_inst; ++t) {
            std::memset(&pseudo[t], 0, sizeof(fraq_kernel_t));
            pseudo[t].sbd = 0;
            pseudo[t].n_head = 2;
            pseudo[t].head[0] = d0[t];
            kp[t] = &pseudo[t];
        }
    }
    hd.build(c, 2 * n_inst, kp.data(), dims.data());
    dinst.alloc(n_inst);
    g0.alloc((size_t)n_inst * 2 * m);
    FRAQ_CUDA(cudaMemcpy(g0.p, G0.data(), sizeof(double) * G0.size(), cudaMemcpyHostToDevice));
    // append G^0 into ring slot 0 of both fields (FastStepper ctor, fpfp.cpp:229-237)
    for (int i = 0; i < n_inst; ++i)
        for (int f = 0; f < 2; ++f) {
            const GroupDev& G = hd.groups_h[2 * i + f];
            FRAQ_CUDA(cudaMemcpy(hd.ring.p + G.ring_off, G0.data() + (size_t)i * 2 * m + f * m,
                                 sizeof(double) * m, cudaMemcpyHostToDevice));
        }
    // SBD correction sequences: corr[e] for e = 0 .. N (K7)
    corr.alloc(1);
    if (fast && sbd) {
        corr.alloc((size_t)2 * n_inst * (N + 1));
        corr_sequence_batch_dev(c, ks.data(), 2 * n_inst, N, corr.p, N + 1);
        for (int i = 0; i < n_inst; ++i) {
            inst[i].corr_off1 = (long)(2 * i) * (N + 1);
            inst[i].corr_off2 = (long)(2 * i + 1) * (N + 1);
        }
    }
    FRAQ_CUDA(cudaMemcpy(dinst.p, inst.data(), sizeof(InstDev) * n_inst, cudaMemcpyHostToDevice));
    sbuf.alloc((size_t)(fast ? 2 : 1) * 2 * n_inst * m);  // fast: one buffer per level parity
    outb.alloc((size_t)2 * n_inst * m);
    // classical: full history of both fields, [t][2 n_inst m]
    total = (long)2 * n_inst * m;
    if (!fast) {
        hist.alloc((size_t)(N + 1) * total);
        FRAQ_CUDA(cudaMemcpy(hist.p, G0.data(), sizeof(double) * total, cudaMemcpyHostToDevice));
        sold.alloc((size_t)kCB * total);
    }
    smem = 2 * sizeof(double2) * rows_len(m);
    if (smem > 227 * 1024) fail(FRAQ_EINVAL, "run: grid_m too large for the on-chip block solve");
    k6_threads = std::getenv("FRAQ_K6_T1024") ? 1024 : 512;  // experiment switch
    if (smem > 48 * 1024) {
        FRAQ_CUDA(cudaFuncSetAttribute(solve_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        FRAQ_CUDA(cudaFuncSetAttribute(solve_kernel<1024>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    }
    sa.inst = dinst.p;
    sa.sys = dsys.p;
    sa.thomas = thomas.p;
    sa.groups = hd.groups.p;
    sa.ring = hd.ring.p;
    sa.s = sbuf.p;
    sa.g0 = g0.p;
    sa.corr = (fast && sbd) ? corr.p : nullptr;  // classical sums already hold the correction
    sa.head = hd.head.p;
    sa.m = m;
    sa.sbd = sbd;
    sa.out = outb.p;
    sa.refine = std::getenv("FRAQ_K6_NOREFINE") ? 0 : 1;  // experiment switch (timing only)
    sa.tap1 = fast ? 1 : 0;
    sa.hist_out = fast ? nullptr : hist.p;
    sa.hist_total = total;
    use_graph = fast && !std::getenv("FRAQ_PHYS_NOGRAPH");  // experiment switch
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    setup_seconds = now_s() - t_setup0;
}

__global__ void counter_kernel(long* ctr, long value, int add) {
    if (add)
        *ctr += value;
    else
        *ctr = value;
}

PhysStepper::~PhysStepper() {
    if (c && c->stream) cudaStreamSynchronize(c->stream);
    if (gexec) cudaGraphExecDestroy(gexec);
    for (cudaEvent_t e : gev) cudaEventDestroy(e);
    if (s5) cudaStreamDestroy(s5);
}

// History pass (K5, FFPE mode) of level n: advance to n, sum, head taps i >= 2 -> sbuf[n & 1].
StepArgs PhysStepper::k5_args(long n) const {
    StepArgs a{};
    a.groups = hd.groups.p;
    a.tiles = hd.tiles.p;
    a.state = hd.state.p;
    a.ring = hd.ring.p;
    a.cr = hd.cr.p;
    a.cf = hd.cf.p;
    a.head = hd.head.p;
    a.level = n - 1;
    a.appended = n;
    a.lo = 1;
    a.adv = 1;
    a.mode = MODE_FFPE;
    a.first_tap = 2;
    a.out = sbuf.p + (size_t)(n & 1) * total;
    return a;
}

void PhysStepper::launch_k6(long n, bool last, cudaStream_t stream, const long* n_dev, int n_off) {
    SolveArgs a = sa;
    a.n = n;
    a.first = sbd && n == 1;
    a.n_dev = n_dev;
    a.n_off = n_off;
    if (fast) a.s = sbuf.p + (size_t)(n & 1) * total;
    // the last level of a call leaves G^n in outb (state reads, ffpe_run's result); graph
    // replays write it every level
    a.out = (last || n_dev) ? outb.p : nullptr;
    if (k6_threads == 1024)
        solve_kernel<1024><<<n_inst, 1024, smem, stream>>>(a);
    else
        solve_kernel<512><<<n_inst, 512, smem, stream>>>(a);
    FRAQ_LAUNCH_CHECK();
}

void PhysStepper::build_graph() {
    const int G = kGraphLevels;
    FRAQ_CUDA(cudaStreamCreateWithFlags(&s5, cudaStreamNonBlocking));
    gev.resize(2 * G + 1);
    for (auto& e : gev) FRAQ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    ndev.alloc(1);
    cudaStream_t s6 = c->stream;
    cudaGraph_t graph = nullptr;
    FRAQ_CUDA(cudaStreamBeginCapture(s6, cudaStreamCaptureModeThreadLocal));
    try {
        FRAQ_CUDA(cudaEventRecord(gev[2 * G], s6));  // fork
        FRAQ_CUDA(cudaStreamWaitEvent(s5, gev[2 * G], 0));
        // chunk levels n0 + q, n0 even (replays start on even levels): parity of n = q & 1
        for (int q = 0; q < G; ++q) {
            if (q >= 2) FRAQ_CUDA(cudaStreamWaitEvent(s5, gev[G + q - 2], 0));  // K6(n-2) done
            StepArgs a = k5_args(q);  // parity slot of level n0 + q
            a.n_dev = ndev.p;
            a.n_off = q;
            hd.launch_step(c, a, s5);
            FRAQ_CUDA(cudaEventRecord(gev[q], s5));
            FRAQ_CUDA(cudaStreamWaitEvent(s6, gev[q], 0));  // K5(n) done
            launch_k6(q, false, s6, ndev.p, q);
            FRAQ_CUDA(cudaEventRecord(gev[G + q], s6));
        }
        counter_kernel<<<1, 1, 0, s6>>>(ndev.p, G, 1);
        FRAQ_LAUNCH_CHECK();
    } catch (...) {
        cudaStreamEndCapture(s6, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    FRAQ_CUDA(cudaStreamEndCapture(s6, &graph));
    const cudaError_t e = cudaGraphInstantiate(&gexec, graph, 0);
    cudaGraphDestroy(graph);
    FRAQ_CUDA(e);
}

void PhysStepper::step(long n_steps, std::vector<cudaEvent_t>* ev) {
    if (n_steps < 0) fail(FRAQ_EINVAL, "step: negative step count");
    if (step_idx + n_steps > N)
        fail(FRAQ_EINVAL, "step: beyond the horizon the stepper was sized for (spec.n_steps)");
    auto mark = [&](int k) {
        if (ev) FRAQ_CUDA(cudaEventRecord((*ev)[k], c->stream));
    };
    const long end = step_idx + n_steps;
    bool counter_set = false;
    while (step_idx < end) {
        const long n = step_idx + 1;
        // graph replay: whole chunks of levels >= 2 starting on an even level (not under the
        // per-kernel timing of time_split)
        if (use_graph && !ev && n >= 2 && (n & 1) == 0 && end - step_idx >= kGraphLevels) {
            if (!gexec) build_graph();
            if (!counter_set) {
                counter_kernel<<<1, 1, 0, c->stream>>>(ndev.p, n, 0);
                FRAQ_LAUNCH_CHECK();
                counter_set = true;
            }
            FRAQ_CUDA(cudaGraphLaunch(gexec, c->stream));
            step_idx += kGraphLevels;
            level += kGraphLevels;
            appended += kGraphLevels;
            continue;
        }
        counter_set = false;
        ++step_idx;
        const bool first = sbd && n == 1;
        if (ev) {
            for (int k = 0; k < 4; ++k) {
                cudaEvent_t e;
                FRAQ_CUDA(cudaEventCreate(&e));
                ev->push_back(e);
            }
        }
        const int e0 = ev ? (int)ev->size() - 4 : 0;
        mark(e0);
        if (fast) {
            // first SBD step: advance() only decays zero accumulators (no feed: 1 - n_head < 1)
            if (!first) hd.launch_step(c, k5_args(n));
        } else {
            const long n0 = n - (n - 1) % kCB;  // first level of this classical block
            if (n == n0) {  // (also at the first SBD level: the block's later levels need it)
                const int tpg = (m + CT_N - 1) / CT_N;
                const int rows = (int)std::min<long>(kCB, N - n0 + 1);
                classical_old_kernel<<<(unsigned)(tpg * 2 * n_inst), 128, 0, c->stream>>>(
                    hist.p, total, ctab.p, N + 1, m, tpg, n0, rows, sbd, sold.p);
                FRAQ_LAUNCH_CHECK();
            }
            if (!first) {
                classical_inblock_kernel<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(
                    hist.p, total, ctab.p, N + 1, m, n0, n, sold.p, sbuf.p);
                FRAQ_LAUNCH_CHECK();
            }
        }
        mark(e0 + 1);
        mark(e0 + 2);
        launch_k6(n, step_idx == end, c->stream, nullptr, 0);
        mark(e0 + 3);
        level += 1;
        appended += 1;
    }
}

void PhysStepper::time_split(long n_steps, double* ms_hist, double* ms_solve) {
    DevBuf<long long> prof;
    if (std::getenv("FRAQ_K6_PROFILE")) {  // experiment: K6 phase cycles (block 0)
        prof.alloc(8);
        FRAQ_CUDA(cudaMemset(prof.p, 0, 8 * sizeof(long long)));
        sa.prof = prof.p;
    }
    std::vector<cudaEvent_t> ev;
    try {
        step(n_steps, &ev);
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
        double h = 0.0, s = 0.0;
        for (size_t k = 0; k + 3 < ev.size(); k += 4) {
            float a = 0.f, b = 0.f;
            FRAQ_CUDA(cudaEventElapsedTime(&a, ev[k], ev[k + 1]));
            FRAQ_CUDA(cudaEventElapsedTime(&b, ev[k + 2], ev[k + 3]));
            h += a;
            s += b;
        }
        *ms_hist = h;
        *ms_solve = s;
        if (prof.p) {
            long long v[8];
            FRAQ_CUDA(cudaMemcpy(v, prof.p, sizeof(v), cudaMemcpyDeviceToHost));
            std::fprintf(stderr, "K6 phases (cycles per level): rhs %.0f solve %.0f refine %.0f "
                         "store %.0f\n", double(v[1] - v[0]) / n_steps,
                         double(v[2] - v[1]) / n_steps, double(v[3] - v[2]) / n_steps,
                         double(v[4] - v[3]) / n_steps);
            sa.prof = nullptr;
        }
    } catch (...) {
        for (auto e : ev) cudaEventDestroy(e);
        throw;
    }
    for (auto e : ev) cudaEventDestroy(e);
}

void PhysStepper::state(double* g1, double* g2) {
    std::vector<double> outh((size_t)2 * n_inst * m);
    if (step_idx == 0) {
        outh = G0;
    } else {
        // G^n of every instance from the rings (slot n % L)
        for (int t = 0; t < 2 * n_inst; ++t) {
            const GroupDev& G = hd.groups_h[t];
            FRAQ_CUDA(cudaMemcpyAsync(outh.data() + (size_t)t * m,
                                      hd.ring.p + G.ring_off + (step_idx % G.L) * (long)G.ld,
                                      sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
        }
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    }
    for (int i = 0; i < n_inst; ++i) {
        if (g1) std::memcpy(g1 + (size_t)i * m, outh.data() + (size_t)i * 2 * m, sizeof(double) * m);
        if (g2)
            std::memcpy(g2 + (size_t)i * m, outh.data() + (size_t)i * 2 * m + m, sizeof(double) * m);
    }
}

void ffpe_run(fraq_ctx c, const fraq_spec_t* specs, int n_inst, int scheme,
              const fraq_kconf_t* kc_in, double* g1_out, double* g2_out, fraq_run_info_t* info,
              fraq_observer_fn obs, void* user) {
    fraq_kconf_t kc;
    if (kc_in)
        kc = *kc_in;
    else
        fraq_kconf_default(&kc);
    validate_specs(specs, n_inst, scheme);
    const bool sbd = scheme == FRAQ_SBD || scheme == FRAQ_FASTSBD;
    const bool fast = scheme == FRAQ_FASTBE || scheme == FRAQ_FASTSBD;
    if (kc.solver == FRAQ_SOLVER_MODAL) {
        if (!fast) fail(FRAQ_EINVAL, "run: the modal solver needs a fast scheme");
        if (obs) fail(FRAQ_EINVAL, "run: the modal solver does not stream intermediate states");
        ffpe_run_modal(c, specs, n_inst, sbd, kc, g1_out, g2_out, info);
        return;
    }
    if (kc.solver == FRAQ_SOLVER_AUTO && fast && !obs) {
        bool done = false;
        try {
            ffpe_run_modal(c, specs, n_inst, sbd, kc, g1_out, g2_out, info);
            done = true;
        } catch (const Error& e) {
            if (e.code != FRAQ_EINVAL || std::string(e.what()).find("modal run:") != 0) throw;
        }
        if (done) return;
    }
    if (kc.solver < 0 || kc.solver > FRAQ_SOLVER_AUTO) fail(FRAQ_EINVAL, "run: unknown solver");
    PhysStepper st(c, specs, n_inst, scheme, kc);
    const long N = st.N;
    const int m = st.m;

    // ---------------------------------------------------------------- time loop
    cudaEvent_t e0, e1;
    FRAQ_CUDA(cudaEventCreate(&e0));
    FRAQ_CUDA(cudaEventCreate(&e1));
    FRAQ_CUDA(cudaEventRecord(e0, c->stream));
    if (obs) {
        // the observer sees every accepted level (fpfp.cpp:367-375), G^0 first
        std::vector<double> ob1(m), ob2(m);
        obs(0, st.G0.data(), st.G0.data() + m, m, user);
        for (long n = 1; n <= N; ++n) {
            st.step(1);
            st.state(ob1.data(), ob2.data());  // instance 0 (observer runs are single-instance)
            obs(n, ob1.data(), ob2.data(), m, user);
        }
    } else {
        st.step(N);
    }
    FRAQ_CUDA(cudaEventRecord(e1, c->stream));
    FRAQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FRAQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::vector<double> outh((size_t)2 * n_inst * m);
    FRAQ_CUDA(cudaMemcpy(outh.data(), st.outb.p, sizeof(double) * outh.size(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n_inst; ++i) {
        std::memcpy(g1_out + (size_t)i * m, outh.data() + (size_t)i * 2 * m, sizeof(double) * m);
        std::memcpy(g2_out + (size_t)i * m, outh.data() + (size_t)i * 2 * m + m, sizeof(double) * m);
    }
    if (info) {
        info->loop_seconds = ms * 1e-3;
        info->setup_seconds = st.setup_seconds;
        info->kernel_eps1 = st.eps[0];
        info->kernel_eps2 = st.eps[1];
        if (fast) {
            info->np[0] = st.ks[0].np1;
            info->np[1] = st.ks[0].np2;
            info->np[2] = st.ks[1].np1;
            info->np[3] = st.ks[1].np2;
            info->n_head[0] = st.ks[0].n_head;
            info->n_head[1] = st.ks[1].n_head;
        } else {
            for (int q = 0; q < 4; ++q) info->np[q] = 0;
            info->n_head[0] = info->n_head[1] = 0;
        }
    }
}

// ================================================================================ ABI objects
// Stepper handle: ClassicalStepper / FastStepper (fpfp.hpp:96-140), always physical space (the
// reference's algorithm: histories K5 + RHS and block solve K6; classical O(n) sums).
void stepper_create(fraq_ctx c, const fraq_spec_t* spec, int scheme, const fraq_kconf_t* kc_in,
                    PhysStepper** out) {
    fraq_kconf_t kc;
    if (kc_in)
        kc = *kc_in;
    else
        fraq_kconf_default(&kc);
    validate_specs(spec, 1, scheme);
    *out = new PhysStepper(c, spec, 1, scheme, kc);
}
void stepper_step(PhysStepper* st, long n) { st->step(n); }
void stepper_state(PhysStepper* st, double* g1, double* g2, long* step) {
    st->state(g1, g2);
    if (step) *step = st->step_idx;
}
void stepper_time_split(PhysStepper* st, long n, double* ms_hist, double* ms_solve) {
    st->time_split(n, ms_hist, ms_solve);
}
void stepper_eps(PhysStepper* st, double* e1, double* e2) {
    if (e1) *e1 = st->eps[0];
    if (e2) *e2 = st->eps[1];
}
void stepper_destroy(PhysStepper* st) {
    cudaStreamSynchronize(st->c->stream);
    delete st;
}

// BlockSystem (block_solver.hpp:38-58): the factored system of one (d01, d02, a, tau, lead).
struct BlockDev {
    fraq_ctx c;
    int m;
    DevBuf<SysDev> sys;
    DevBuf<M2> thomas;
    DevBuf<double> io;  // rhs1, rhs2, g1, g2 staging for host calls
};
void block_create(fraq_ctx c, double d01, double d02, double a, double tau, int m, double h,
                  double lead, BlockDev** out) {
    if (m < 1) fail(FRAQ_EINVAL, "BlockSystem: grid_m must be >= 1");
    if (!(tau > 0.0) || !(h > 0.0)) fail(FRAQ_EINVAL, "BlockSystem: tau and h must be > 0");
    if (2 * sizeof(double2) * rows_len(m) > 227 * 1024)
        fail(FRAQ_EINVAL, "BlockSystem: grid_m too large for the on-chip block solve");
    auto* b = new BlockDev();
    try {
        b->c = c;
        b->m = m;
        M2 D, E;
        blocks(d01, d02, a, tau, h, lead, D, E);
        SysDev S{};
        S.K = cr_levels(m);
        S.E = E;
        S.th_off = 0;
        exact_entries(S, d01, d02, 1.0, 1.0, a, tau, h, lead);
        if (S.K) setup_cr(S, D, E);
        b->sys.alloc(1);
        FRAQ_CUDA(cudaMemcpy(b->sys.p, &S, sizeof(SysDev), cudaMemcpyHostToDevice));
        b->thomas.alloc(S.K ? 1 : 2L * m);
        if (!S.K) {
            DevBuf<M2> dD(1);
            FRAQ_CUDA(cudaMemcpy(dD.p, &D, sizeof(M2), cudaMemcpyHostToDevice));
            thomas_setup_kernel<<<1, 32, 0, c->stream>>>(b->sys.p, dD.p, 1, m, b->thomas.p);
            FRAQ_LAUNCH_CHECK();
            FRAQ_CUDA(cudaStreamSynchronize(c->stream));
        }
        b->io.alloc(4L * m);
    } catch (...) {
        delete b;
        throw;
    }
    *out = b;
}
void block_solve(BlockDev* b, const double* rhs1, const double* rhs2, double* g1, double* g2,
                 int mem) {
    fraq_ctx c = b->c;
    const int m = b->m;
    const size_t smem = 2 * sizeof(double2) * rows_len(m);
    if (smem > 48 * 1024)
        FRAQ_CUDA(cudaFuncSetAttribute(block_solve_kernel<512>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (mem == FRAQ_DEVICE) {
        block_solve_kernel<512><<<1, 512, smem, c->stream>>>(b->sys.p, b->thomas.p, m, rhs1, rhs2,
                                                            g1, g2);
        FRAQ_LAUNCH_CHECK();
        return;
    }
    double* d = b->io.p;
    FRAQ_CUDA(cudaMemcpyAsync(d, rhs1, 8L * m, cudaMemcpyHostToDevice, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(d + m, rhs2, 8L * m, cudaMemcpyHostToDevice, c->stream));
    block_solve_kernel<512><<<1, 512, smem, c->stream>>>(b->sys.p, b->thomas.p, m, d, d + m,
                                                        d + 2 * m, d + 3 * m);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaMemcpyAsync(g1, d + 2 * m, 8L * m, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(g2, d + 3 * m, 8L * m, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}
void block_destroy(BlockDev* b) {
    cudaStreamSynchronize(b->c->stream);
    delete b;
}

void laplacian_apply(fraq_ctx c, int m, double h, const double* x, double* y, int mem) {
    if (m < 1) fail(FRAQ_EINVAL, "DiscreteLaplacian: grid_m must be >= 1");
    const double ih2 = 1.0 / (h * h);
    if (mem == FRAQ_DEVICE) {
        laplacian_kernel<<<(m + 255) / 256, 256, 0, c->stream>>>(m, ih2, x, y);
        FRAQ_LAUNCH_CHECK();
        return;
    }
    DevBuf<double> d(2L * m);
    FRAQ_CUDA(cudaMemcpyAsync(d.p, x, 8L * m, cudaMemcpyHostToDevice, c->stream));
    laplacian_kernel<<<(m + 255) / 256, 256, 0, c->stream>>>(m, ih2, d.p, d.p + m);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaMemcpyAsync(y, d.p + m, 8L * m, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

// BandedLU (block_solver.hpp:25-36): band storage assembled on the host (at()), factored and
// solved on the device.
struct BandedDev {
    fraq_ctx c;
    int n, kl, ku, ldab;
    bool factored = false;
    std::vector<double> ab_h;
    DevBuf<double> ab, rhs;
    DevBuf<int> piv, status;
};
void banded_create(fraq_ctx c, int n, int kl, int ku, BandedDev** out) {
    if (n < 1 || kl < 0 || ku < 0) fail(FRAQ_EINVAL, "BandedLU: bad shape");
    auto* b = new BandedDev();
    b->c = c;
    b->n = n;
    b->kl = kl;
    b->ku = ku;
    b->ldab = 2 * kl + ku + 1;
    b->ab_h.assign((size_t)b->ldab * n, 0.0);
    *out = b;
}
double* banded_at(BandedDev* b, int row, int col) {
    if (row < 0 || row >= b->n || col < 0 || col >= b->n || col - row > b->ku ||
        row - col > b->kl)
        fail(FRAQ_ERANGE, "BandedLU::at: outside the band");
    return &b->ab_h[(size_t)col * b->ldab + (b->kl + b->ku + row - col)];
}
void banded_assign(BandedDev* b, const double* ab) {
    if (!ab) fail(FRAQ_EINVAL, "BandedLU: null band");
    b->ab_h.assign(ab, ab + b->ab_h.size());
    b->factored = false;
}
void banded_factorize(BandedDev* b) {
    fraq_ctx c = b->c;
    b->ab.alloc(b->ab_h.size());
    b->piv.alloc(b->n);
    b->status.alloc(1);
    FRAQ_CUDA(cudaMemcpyAsync(b->ab.p, b->ab_h.data(), 8 * b->ab_h.size(), cudaMemcpyHostToDevice,
                              c->stream));
    banded_factor_kernel<<<1, 1, 0, c->stream>>>(b->ab.p, b->piv.p, b->n, b->kl, b->ku,
                                                 b->status.p);
    FRAQ_LAUNCH_CHECK();
    int st = 0;
    FRAQ_CUDA(cudaMemcpyAsync(&st, b->status.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    if (st) fail(FRAQ_ERUNTIME, "BandedLU: zero pivot (singular system)");
    b->factored = true;
}
void banded_solve(BandedDev* b, double* rhs, int mem) {
    if (!b->factored) fail(FRAQ_ELOGIC, "BandedLU::solve before factorize");
    fraq_ctx c = b->c;
    if (mem == FRAQ_DEVICE) {
        banded_solve_kernel<<<1, 1, 0, c->stream>>>(b->ab.p, b->piv.p, b->n, b->kl, b->ku, rhs);
        FRAQ_LAUNCH_CHECK();
        return;
    }
    if (!b->rhs.p) b->rhs.alloc(b->n);
    FRAQ_CUDA(cudaMemcpyAsync(b->rhs.p, rhs, 8L * b->n, cudaMemcpyHostToDevice, c->stream));
    banded_solve_kernel<<<1, 1, 0, c->stream>>>(b->ab.p, b->piv.p, b->n, b->kl, b->ku, b->rhs.p);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaMemcpyAsync(rhs, b->rhs.p, 8L * b->n, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}
void banded_destroy(BandedDev* b) {
    cudaStreamSynchronize(b->c->stream);
    delete b;
}

}  // namespace fraqcu
