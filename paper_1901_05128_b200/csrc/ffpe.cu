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
__host__ __device__ inline M2 scal(double s, const M2& x) { return {s * x.a, s * x.b, s * x.c, s * x.d}; }
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
};

// Block matrices of BlockSystem (block_solver.cpp:95-117).
void blocks(double d01, double d02, double a, double tau, double h, double lead, M2& D, M2& E) {
    const double ih2 = 1.0 / (h * h);
    D = {lead / tau + d01 * (a + 2.0 * ih2), -a * d02, -a * d01, lead / tau + d02 * (a + 2.0 * ih2)};
    E = {-d01 * ih2, 0.0, 0.0, -d02 * ih2};
}

int cr_levels(int m) {
    int K = 0;
    while ((1L << K) - 1 < m) ++K;
    return ((1L << K) - 1 == m && K <= kMaxLevels) ? K : 0;
}

// Setup of one system on the host from its scalar description (tiny: O(levels) or O(M) 2x2
// algebra per system; the O(M) Thomas factors are computed by thomas_setup_kernel).
void setup_cr(SysDev& S, const M2& D0, const M2& E0) {
    M2 D = D0, E = E0;
    for (int l = 0; l < S.K; ++l) {
        const M2 Di = inv(D);
        S.lv[l].F = mul(E, Di);
        S.lv[l].G = Di;
        S.lv[l].H = mul(Di, E);
        const M2 FE = mul(S.lv[l].F, E);
        E = scal(-1.0, FE);
        D = sub(D, scal(2.0, FE));
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
};

// RHS (fpfp.cpp:277-279, 298-302, 339-344) then the block solve; one CTA per instance.
template <int THREADS>
__global__ void __launch_bounds__(THREADS) solve_kernel(SolveArgs A) {
    extern __shared__ double2 sb[];  // b / x, rows 1..m (index 0 and m+1 are zero)
    const InstDev I = A.inst[blockIdx.x];
    const GroupDev G1 = A.groups[I.g1], G2 = A.groups[I.g2];
    const int m = A.m;
    const double a = I.a, tau = I.tau, ih2 = 1.0 / (I.h * I.h);
    const long n = A.n;
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
    if (A.sbd && !A.first) {
        q1 = r1 + ((n - 2) % G1.L) * ld;  // G^{n-2}
        q2 = r2 + ((n - 2) % G2.L) * ld;
        if (A.corr) {
            // (1/2) d_{n-1} G^0: exact head inside, reconstructed (running powers) beyond
            c1 = (n - 1 < G1.L) ? A.head[G1.hd_off + n - 1] : A.corr[I.corr_off1 + (n - 4)];
            c2 = (n - 1 < G2.L) ? A.head[G2.hd_off + n - 1] : A.corr[I.corr_off2 + (n - 4)];
        }
    }
    const double* g01 = A.g0 + I.g0_off;
    const double* g02 = g01 + m;
    const double d10 = A.head[G1.hd_off], d20 = A.head[G2.hd_off];
    for (int k = threadIdx.x; k < m; k += THREADS) {
        double b1, b2;
        if (A.sbd && A.first) {
            // 2/3-1/3 first step from G^0 (fpfp.cpp:293-303)
            const double u = p1[k], v = p2[k];
            const double au = (2.0 * u - (k > 0 ? p1[k - 1] : 0.0) - (k + 1 < m ? p1[k + 1] : 0.0)) * ih2;
            const double av = (2.0 * v - (k > 0 ? p2[k - 1] : 0.0) - (k + 1 < m ? p2[k + 1] : 0.0)) * ih2;
            b1 = u / tau - (d10 / 3.0) * (a * u + au) + (a * d20 / 3.0) * v;
            b2 = v / tau - (d20 / 3.0) * (a * v + av) + (a * d10 / 3.0) * u;
        } else {
            double x1 = s1[k], x2 = s2[k];
            double l1 = k > 0 ? s1[k - 1] : 0.0, rr1 = k + 1 < m ? s1[k + 1] : 0.0;
            double l2 = k > 0 ? s2[k - 1] : 0.0, rr2 = k + 1 < m ? s2[k + 1] : 0.0;
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
                lead1 = (2.0 * p1[k] - 0.5 * q1[k]) / tau;
                lead2 = (2.0 * p2[k] - 0.5 * q2[k]) / tau;
            } else {
                lead1 = p1[k] / tau;
                lead2 = p2[k] / tau;
            }
            b1 = lead1 - a * x1 - as1 + a * x2;
            b2 = lead2 - a * x2 - as2 + a * x1;
        }
        sb[k + 1] = make_double2(b1, b2);
    }
    if (threadIdx.x == 0) {
        sb[0] = make_double2(0.0, 0.0);
        sb[m + 1] = make_double2(0.0, 0.0);
    }
    __syncthreads();
    const SysDev& S = A.sys[A.first ? I.sys_first : I.sys_main];
    if (S.K > 0) {
        const int K = S.K;
        // forward reduction
        for (int l = 0; l < K - 1; ++l) {
            const int s = 1 << l;
            const M2 F = S.lv[l].F;
            for (int i = 2 * s * (threadIdx.x + 1); i <= m; i += 2 * s * THREADS) {
                const double2 sum = make_double2(sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y);
                const double2 t = mv(F, sum);
                sb[i] = make_double2(sb[i].x - t.x, sb[i].y - t.y);
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const int i = 1 << (K - 1);
            sb[i] = mv(S.lv[K - 1].G, sb[i]);
        }
        __syncthreads();
        for (int l = K - 2; l >= 0; --l) {
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
        // block Thomas with the setup factors (single thread; general grid sizes)
        const M2* W = A.thomas + S.th_off;
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
    }
}

// Classical direct sums (fpfp.cpp:114-122, 150-164): s[k] = (SBD: 0.5 d_{n-1} G^0) +
// sum_{i=1}^{n-1} d_i G^{n-i}, serial in i like the reference.  Full history hist[t][group dof].
__global__ void classical_sum_kernel(const double* hist, long hist_ld, const double* d, long d_ld,
                                     const int* group_of_dof, long total, long n, int sbd,
                                     double* s) {
    const long k = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (k >= total) return;
    const double* w = d + group_of_dof[k] * d_ld;
    double acc = sbd ? 0.5 * w[n - 1] * hist[k] : 0.0;
    for (long i = 1; i <= n - 1; ++i) acc += w[i] * hist[(n - i) * hist_ld + k];
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

void ffpe_run(fraq_ctx c, const fraq_spec_t* specs, int n_inst, int scheme,
              const fraq_kconf_t* kc_in, double* g1_out, double* g2_out, fraq_run_info_t* info,
              fraq_observer_fn obs, void* user) {
    if (n_inst < 1) fail(FRAQ_EINVAL, "run: need at least one instance");
    fraq_kconf_t kc;
    if (kc_in)
        kc = *kc_in;
    else
        fraq_kconf_default(&kc);
    const fraq_spec_t& s0 = specs[0];
    const int m = s0.grid_m;
    const long N = s0.n_steps;
    if (m < 1) fail(FRAQ_EINVAL, "run: grid_m must be >= 1");
    if (N < 1) fail(FRAQ_EINVAL, "run: n_steps must be >= 1");
    for (int i = 0; i < n_inst; ++i) {
        const fraq_spec_t& s = specs[i];
        if (s.grid_m != m || s.n_steps != N || s.t_final != s0.t_final || s.length != s0.length)
            fail(FRAQ_EINVAL, "run: batched instances must share grid_m, n_steps, t_final, length");
        if (s.initial == FRAQ_CUSTOM && (!s.custom_g1 || !s.custom_g2))
            fail(FRAQ_EINVAL, "initial_field: custom samples must have grid_m entries");
        if (s.initial < 0 || s.initial > 2) fail(FRAQ_EINVAL, "unknown initial data tag");
    }
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
    const double tau = s0.t_final / double(N);
    const double h = s0.length / double(m + 1);
    const double t_setup0 = now_s();

    // ---------------------------------------------------------------- initial data
    std::vector<double> G0((size_t)n_inst * 2 * m);
    for (int i = 0; i < n_inst; ++i)
        initial_field(specs[i], G0.data() + (size_t)i * 2 * m, G0.data() + (size_t)i * 2 * m + m);

    // ---------------------------------------------------------------- kernels / weights
    std::vector<double> gam(2 * n_inst);
    for (int i = 0; i < n_inst; ++i) {
        gam[2 * i] = 1.0 - specs[i].alpha1;
        gam[2 * i + 1] = 1.0 - specs[i].alpha2;
    }
    std::vector<fraq_kernel_t> ks;
    std::vector<double> eps(2 * n_inst, 0.0);
    std::vector<double> d0(2 * n_inst);
    DevBuf<double> ctab;  // classical tables (2 n_inst x (N+1))
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
            blocks(f * d0[2 * i], f * d0[2 * i + 1], a, tau, h, lead, D, E);
            SysDev& S = sys[sidx];
            S.K = K;
            S.E = E;
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
    DevBuf<SysDev> dsys(n_sys);
    FRAQ_CUDA(cudaMemcpy(dsys.p, sys.data(), sizeof(SysDev) * n_sys, cudaMemcpyHostToDevice));
    DevBuf<M2> thomas(std::max<long>(1, th));
    if (!K) {
        DevBuf<M2> dD(n_sys);
        FRAQ_CUDA(cudaMemcpy(dD.p, sysD.data(), sizeof(M2) * n_sys, cudaMemcpyHostToDevice));
        thomas_setup_kernel<<<(n_sys + 127) / 128, 128, 0, c->stream>>>(dsys.p, dD.p, n_sys, m,
                                                                       thomas.p);
        FRAQ_LAUNCH_CHECK();
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    }

    // ---------------------------------------------------------------- histories / buffers
    HistDevice hd;
    std::vector<long> dims(2 * n_inst, m);
    std::vector<const fraq_kernel_t*> kp(2 * n_inst);
    std::vector<fraq_kernel_t> pseudo;  // classical: a 2-slot lag ring carrier (no nodes)
    if (fast) {
        for (int t = 0; t < 2 * n_inst; ++t) kp[t] = &ks[t];
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
    DevBuf<InstDev> dinst(n_inst);
    FRAQ_CUDA(cudaMemcpy(dinst.p, inst.data(), sizeof(InstDev) * n_inst, cudaMemcpyHostToDevice));
    DevBuf<double> g0((size_t)n_inst * 2 * m);
    FRAQ_CUDA(cudaMemcpy(g0.p, G0.data(), sizeof(double) * G0.size(), cudaMemcpyHostToDevice));
    // append G^0 into ring slot 0 of both fields (FastStepper ctor, fpfp.cpp:229-237)
    for (int i = 0; i < n_inst; ++i)
        for (int f = 0; f < 2; ++f) {
            const GroupDev& G = hd.groups_h[2 * i + f];
            FRAQ_CUDA(cudaMemcpy(hd.ring.p + G.ring_off, G0.data() + (size_t)i * 2 * m + f * m,
                                 sizeof(double) * m, cudaMemcpyHostToDevice));
        }
    // SBD correction sequences: corr[e] for e = 0 .. N (K7)
    DevBuf<double> corr(1);
    if (fast && sbd) {
        corr.alloc((size_t)2 * n_inst * (N + 1));
        corr_sequence_batch_dev(c, ks.data(), 2 * n_inst, N, corr.p, N + 1);
        for (int i = 0; i < n_inst; ++i) {
            inst[i].corr_off1 = (long)(2 * i) * (N + 1);
            inst[i].corr_off2 = (long)(2 * i + 1) * (N + 1);
        }
        FRAQ_CUDA(cudaMemcpy(dinst.p, inst.data(), sizeof(InstDev) * n_inst, cudaMemcpyHostToDevice));
    }
    DevBuf<double> sbuf((size_t)2 * n_inst * m);
    DevBuf<double> outb((size_t)2 * n_inst * m);
    // classical: full history of both fields, [t][2 n_inst m]
    DevBuf<double> hist;
    DevBuf<int> gof;
    const long total = (long)2 * n_inst * m;
    if (!fast) {
        hist.alloc((size_t)(N + 1) * total);
        FRAQ_CUDA(cudaMemcpy(hist.p, G0.data(), sizeof(double) * total, cudaMemcpyHostToDevice));
        std::vector<int> go(total);
        for (long k = 0; k < total; ++k) go[k] = (int)(k / m);
        gof.alloc(total);
        FRAQ_CUDA(cudaMemcpy(gof.p, go.data(), sizeof(int) * total, cudaMemcpyHostToDevice));
    }
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    const double t_setup1 = now_s();

    // ---------------------------------------------------------------- time loop
    cudaEvent_t e0, e1;
    FRAQ_CUDA(cudaEventCreate(&e0));
    FRAQ_CUDA(cudaEventCreate(&e1));
    FRAQ_CUDA(cudaEventRecord(e0, c->stream));
    const int threads = 512;
    const size_t smem = sizeof(double2) * (m + 2);
    if (smem > 48 * 1024)
        FRAQ_CUDA(cudaFuncSetAttribute(solve_kernel<512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)std::min<size_t>(smem, 227 * 1024)));
    if (smem > 227 * 1024) fail(FRAQ_EINVAL, "run: grid_m too large for the on-chip block solve");
    SolveArgs sa{};
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
    long level = 0, appended = 1;
    std::vector<double> ob1, ob2;
    if (obs) {
        ob1.resize(m);
        ob2.resize(m);
        obs(0, G0.data(), G0.data() + m, m, user);
    }
    for (long n = 1; n <= N; ++n) {
        const bool first = sbd && n == 1;
        if (fast) {
            if (!first) {
                StepArgs a{};
                a.groups = hd.groups.p;
                a.tiles = hd.tiles.p;
                a.state = hd.state.p;
                a.ring = hd.ring.p;
                a.cr = hd.cr.p;
                a.cf = hd.cf.p;
                a.head = hd.head.p;
                a.level = level;
                a.appended = appended;
                a.lo = 1;
                a.adv = 1;
                a.mode = MODE_FFPE;
                a.out = sbuf.p;
                hd.launch_step(c, a);
            }
            // first SBD step: advance() only decays zero accumulators (no feed: 1 - n_head < 1)
        } else if (!first) {
            classical_sum_kernel<<<(unsigned)((total + 255) / 256), 256, 0, c->stream>>>(
                hist.p, total, ctab.p, N + 1, gof.p, total, n, sbd, sbuf.p);
            FRAQ_LAUNCH_CHECK();
        }
        sa.n = n;
        sa.first = first;
        sa.out = (n == N) ? outb.p : nullptr;
        solve_kernel<512><<<n_inst, threads, smem, c->stream>>>(sa);
        FRAQ_LAUNCH_CHECK();
        if (!fast) {
            // keep the full history: copy G^n rows out of the 2-slot rings
            for (int t = 0; t < 2 * n_inst; ++t) {
                const GroupDev& G = hd.groups_h[t];
                FRAQ_CUDA(cudaMemcpyAsync(hist.p + n * total + (long)t * m,
                                          hd.ring.p + G.ring_off + (n % G.L) * (long)G.ld,
                                          sizeof(double) * m, cudaMemcpyDeviceToDevice, c->stream));
            }
        }
        level += 1;
        appended += 1;
        if (obs) {
            const GroupDev& G1 = hd.groups_h[0];
            const GroupDev& G2 = hd.groups_h[1];
            FRAQ_CUDA(cudaMemcpyAsync(ob1.data(), hd.ring.p + G1.ring_off + (n % G1.L) * (long)G1.ld,
                                      sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
            FRAQ_CUDA(cudaMemcpyAsync(ob2.data(), hd.ring.p + G2.ring_off + (n % G2.L) * (long)G2.ld,
                                      sizeof(double) * m, cudaMemcpyDeviceToHost, c->stream));
            FRAQ_CUDA(cudaStreamSynchronize(c->stream));
            obs(n, ob1.data(), ob2.data(), m, user);
        }
    }
    FRAQ_CUDA(cudaEventRecord(e1, c->stream));
    FRAQ_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    FRAQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    std::vector<double> outh((size_t)2 * n_inst * m);
    FRAQ_CUDA(cudaMemcpy(outh.data(), outb.p, sizeof(double) * outh.size(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n_inst; ++i) {
        std::memcpy(g1_out + (size_t)i * m, outh.data() + (size_t)i * 2 * m, sizeof(double) * m);
        std::memcpy(g2_out + (size_t)i * m, outh.data() + (size_t)i * 2 * m + m, sizeof(double) * m);
    }
    if (info) {
        info->loop_seconds = ms * 1e-3;
        info->setup_seconds = t_setup1 - t_setup0;
        info->kernel_eps1 = eps[0];
        info->kernel_eps2 = eps[1];
        if (fast) {
            info->np[0] = ks[0].np1;
            info->np[1] = ks[0].np2;
            info->np[2] = ks[1].np1;
            info->np[3] = ks[1].np2;
            info->n_head[0] = ks[0].n_head;
            info->n_head[1] = ks[1].n_head;
        } else {
            for (int q = 0; q < 4; ++q) info->np[q] = 0;
            info->n_head[0] = info->n_head[1] = 0;
        }
    }
}

}  // namespace fraqcu
