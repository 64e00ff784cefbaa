// ref_shim.cpp -- extern "C" access to the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// Compiled by oracle/Makefile together with the reference's own sources, read in place from
// /root/reference/proj/src, into oracle/_ref/libfraq_ref.so.  Nothing here re-implements the
// reference: every entry point forwards to the reference API (fraq::*) and copies results into
// caller-owned arrays so ctypes can read them.  Used (a) to pin the C restatement in
// oracle/fraq_oracle.c, (b) to generate golden fixtures, (c) as the CPU baseline
// (bench.py --impl reference and the cpu_baseline leg).
//
// Error codes: 0 ok, -1 invalid_argument, -2 logic_error, -3 out_of_range, -4 runtime_error,
// -5 other.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <thread>
#include <vector>

#include "fraq/fpfp.hpp"
#include "fraq/gauss_jacobi.hpp"

using namespace fraq;

namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    } catch (const std::logic_error& e) {
        // out_of_range derives from logic_error
        if (dynamic_cast<const std::out_of_range*>(&e)) return -3;
        return -2;
    } catch (const std::runtime_error&) {
        return -4;
    } catch (...) {
        return -5;
    }
}

void copy_out(const std::vector<double>& v, double* out) {
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(double));
}

// Kernel descriptor in the shim's flat form: BE uses (m1, r1) and head[2].
struct FlatKernel {
    int sbd, n_head, np1, np2;
    double gamma, tau;
    const double *head, *m1, *r1, *m2, *r2;
};

FastKernelBE to_be(const FlatKernel& f) {
    FastKernelBE k;
    k.alpha = f.gamma;
    k.tau = f.tau;
    k.head[0] = f.head[0];
    k.head[1] = f.head[1];
    k.node_weights.assign(f.m1, f.m1 + f.np1);
    k.ratios.assign(f.r1, f.r1 + f.np1);
    return k;
}

FastKernelSBD to_sbd(const FlatKernel& f) {
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

}  // namespace

extern "C" {

int ref_gauss_jacobi(double a, double b, int n, double* nodes, double* weights) {
    return guard([&] {
        const JacobiRule r = gauss_jacobi(a, b, n);
        copy_out(r.nodes, nodes);
        copy_out(r.weights, weights);
    });
}

double ref_gamma(double x) { return gamma_fn(x); }

int ref_jacobi_moment(double a, double b, int k, double* out) {
    return guard([&] { *out = jacobi_moment(a, b, k); });
}

int ref_be_weights(double g, double tau, long nmax, double* out) {
    return guard([&] { copy_out(be_weights(g, tau, nmax).weights, out); });
}

int ref_sbd_weights(double g, double tau, long nmax, double* out) {
    return guard([&] { copy_out(sbd_weights(g, tau, nmax).weights, out); });
}

int ref_coupling_from_transition(double m, double* out) {
    return guard([&] { *out = coupling_from_transition(m); });
}

int ref_default_sbd_head(double g) { return default_sbd_head(g); }

// BE kernel: out head[2], m[np], r[np]
int ref_build_be_kernel(double g, double tau, int np, double* head, double* m, double* r) {
    return guard([&] {
        const FastKernelBE k = build_be_kernel(g, tau, np);
        head[0] = k.head[0];
        head[1] = k.head[1];
        copy_out(k.node_weights, m);
        copy_out(k.ratios, r);
    });
}

int ref_build_sbd_kernel(double g, double tau, int np1, int np2, int nh, double* head, double* m1,
                         double* r1, double* m2, double* r2) {
    return guard([&] {
        const FastKernelSBD k = build_sbd_kernel(g, tau, np1, np2, nh);
        copy_out(k.head, head);
        copy_out(k.mult1, m1);
        copy_out(k.ratio1, r1);
        copy_out(k.mult2, m2);
        copy_out(k.ratio2, r2);
    });
}

// Auto builders.  sizes[0..2] = (np1, np2, n_head); arrays must hold 256 (head: 256).
int ref_build_be_kernel_auto(double g, double tau, long horizon, double eps_tol, int max_points,
                             int max_head, int* sizes, double* achieved, double* head, double* m,
                             double* r) {
    return guard([&] {
        KernelBudget b;
        b.horizon = horizon;
        b.eps_tol = eps_tol;
        b.max_points = max_points;
        b.max_head = max_head;
        const FastKernelBE k = build_be_kernel_auto(g, tau, b);
        sizes[0] = int(k.n_points());
        sizes[1] = 0;
        sizes[2] = 2;
        *achieved = b.achieved_eps;
        head[0] = k.head[0];
        head[1] = k.head[1];
        copy_out(k.node_weights, m);
        copy_out(k.ratios, r);
    });
}

int ref_build_sbd_kernel_auto(double g, double tau, long horizon, double eps_tol, int max_points,
                              int max_head, int* sizes, double* achieved, double* head, double* m1,
                              double* r1, double* m2, double* r2) {
    return guard([&] {
        KernelBudget b;
        b.horizon = horizon;
        b.eps_tol = eps_tol;
        b.max_points = max_points;
        b.max_head = max_head;
        const FastKernelSBD k = build_sbd_kernel_auto(g, tau, b);
        sizes[0] = int(k.ratio1.size());
        sizes[1] = int(k.ratio2.size());
        sizes[2] = k.n_head;
        *achieved = b.achieved_eps;
        copy_out(k.head, head);
        copy_out(k.mult1, m1);
        copy_out(k.ratio1, r1);
        copy_out(k.mult2, m2);
        copy_out(k.ratio2, r2);
    });
}

int ref_reconstruct(int sbd, double g, double tau, int nh, int np1, int np2, const double* head,
                    const double* m1, const double* r1, const double* m2, const double* r2,
                    long n_idx, const long* idx, double* out) {
    return guard([&] {
        const FlatKernel f{sbd, nh, np1, np2, g, tau, head, m1, r1, m2, r2};
        if (sbd) {
            const FastKernelSBD k = to_sbd(f);
            for (long i = 0; i < n_idx; ++i) out[i] = k.reconstruct(idx[i]);
        } else {
            const FastKernelBE k = to_be(f);
            for (long i = 0; i < n_idx; ++i) out[i] = k.reconstruct(idx[i]);
        }
    });
}

int ref_kernel_error_report(int sbd, double g, double tau, int nh, int np1, int np2,
                            const double* head, const double* m1, const double* r1,
                            const double* m2, const double* r2, long nmax, double* eps,
                            double* max_eps, long* argmax) {
    return guard([&] {
        const FlatKernel f{sbd, nh, np1, np2, g, tau, head, m1, r1, m2, r2};
        const KernelErrorReport rep =
            sbd ? kernel_error_report(to_sbd(f), nmax) : kernel_error_report(to_be(f), nmax);
        copy_out(rep.eps, eps);
        *max_eps = rep.max_eps;
        *argmax = rep.argmax;
    });
}

// Pushes U[n][dim] through the reference history for n = 0..n_steps-1 and stores the
// derivative after each push (NaN when the reference throws "too early").
int ref_hist_run(int sbd, double g, double tau, int nh, int np1, int np2, const double* head,
                 const double* m1, const double* r1, const double* m2, const double* r2,
                 int scheme_variant, long dim, long n_steps, const double* U, double* D) {
    return guard([&] {
        const FlatKernel f{sbd, nh, np1, np2, g, tau, head, m1, r1, m2, r2};
        const HistoryVariant v = scheme_variant ? HistoryVariant::scheme : HistoryVariant::standalone;
        auto drive = [&](auto& h) {
            for (long n = 0; n < n_steps; ++n) {
                h.push(std::span<const double>(U + n * dim, dim));
                std::span<double> o(D + n * dim, dim);
                try {
                    h.derivative(o);
                } catch (const std::logic_error&) {
                    std::fill(o.begin(), o.end(), NAN);
                }
            }
        };
        if (sbd) {
            const FastKernelSBD k = to_sbd(f);
            SbdHistory h(k, v, dim);
            drive(h);
        } else {
            const FastKernelBE k = to_be(f);
            BeHistory h(k, v, dim);
            drive(h);
        }
    });
}

// FFPE run through fraq::run.  scheme: 0 BE, 1 FastBE, 2 SBD, 3 FastSBD.  initial: 0 poly_sin,
// 1 indicator, 2 custom.  kconf = (be_points, sbd_points_1, sbd_points_2, sbd_head, auto_size).
int ref_run(double alpha1, double alpha2, double a, int grid_m, double t_final, long n_steps,
            int initial, const double* cg1, const double* cg2, int scheme, const int* kconf_i,
            double eps_tol, double* g1, double* g2, double* eps1, double* eps2,
            double* loop_seconds) {
    return guard([&] {
        ProblemSpec s;
        s.alpha1 = alpha1;
        s.alpha2 = alpha2;
        s.coupling_a = a;
        s.grid_m = grid_m;
        s.t_final = t_final;
        s.n_steps = n_steps;
        s.initial = initial == 0 ? InitialData::poly_sin
                                 : (initial == 1 ? InitialData::indicator : InitialData::custom);
        if (initial == 2) {
            s.custom_g1.assign(cg1, cg1 + grid_m);
            s.custom_g2.assign(cg2, cg2 + grid_m);
        }
        KernelConfig kc;
        if (kconf_i) {
            kc.be_points = kconf_i[0];
            kc.sbd_points_1 = kconf_i[1];
            kc.sbd_points_2 = kconf_i[2];
            kc.sbd_head = kconf_i[3];
            kc.auto_size = kconf_i[4] != 0;
        }
        kc.eps_tol = eps_tol;
        const RunResult rr = run(s, Scheme(scheme), kc);
        copy_out(rr.final_state.g1, g1);
        copy_out(rr.final_state.g2, g2);
        *eps1 = rr.kernel_eps1;
        *eps2 = rr.kernel_eps2;
        *loop_seconds = rr.loop_seconds;
    });
}

int ref_block_solve(double d01, double d02, double a, double tau, int m, double lead,
                    const double* rhs1, const double* rhs2, double* g1, double* g2) {
    return guard([&] {
        const DiscreteLaplacian lap(m, 1.0);
        solve_block_system(d01, d02, a, tau, lap, std::span<const double>(rhs1, m),
                           std::span<const double>(rhs2, m), std::span<double>(g1, m),
                           std::span<double>(g2, m), lead);
    });
}

// ---------------------------------------------------------------------------------------------
// CPU baseline: the reference SbdHistory/BeHistory pushed over a DOF sample by `threads` worker
// threads, each owning an independent history over its DOF slice (the run_convergence worker
// pattern, bench.cpp:194-223).  Kernel tables per group are passed in flat form; group g covers
// DOFs [g*dofs_per_group, (g+1)*dofs_per_group) of the sample.  Inputs U[n][dofs] are produced
// before timing.  Returns the loop wall time (push + derivative per step), seconds.
int ref_bench_history(int sbd, int n_groups, const double* gammas, double tau, const int* nh,
                      const int* np1, const int* np2, const double* const* heads,
                      const double* const* m1, const double* const* r1,
                      const double* const* m2, const double* const* r2, long dofs,
                      long n_steps, const double* U, double* D_last, int threads,
                      double* seconds) {
    return guard([&] {
        std::vector<FastKernelBE> kbe;
        std::vector<FastKernelSBD> ksbd;
        for (int g = 0; g < n_groups; ++g) {
            const FlatKernel f{sbd, nh[g], np1[g], np2[g], gammas[g], tau, heads[g],
                               m1[g],  r1[g], m2 ? m2[g] : nullptr, r2 ? r2[g] : nullptr};
            if (sbd)
                ksbd.push_back(to_sbd(f));
            else
                kbe.push_back(to_be(f));
        }
        const long per_group = dofs / n_groups;
        // work items: (group, lo, hi) slices, one per thread per group share
        struct Slice {
            int g;
            long lo, hi;
        };
        std::vector<Slice> slices;
        const int T = std::max(1, threads);
        const int per = std::max(1, T / n_groups);
        for (int g = 0; g < n_groups; ++g)
            for (int t = 0; t < per; ++t) {
                const long lo = g * per_group + per_group * t / per;
                const long hi = g * per_group + per_group * (t + 1) / per;
                if (hi > lo) slices.push_back({g, lo, hi});
            }
        std::vector<double> secs(slices.size(), 0.0);
        auto work = [&](std::size_t si) {
            const Slice s = slices[si];
            const long w = s.hi - s.lo;
            std::vector<double> in(w), out(w);
            auto drive = [&](auto& h) {
                const auto t0 = std::chrono::steady_clock::now();
                for (long n = 0; n < n_steps; ++n) {
                    std::memcpy(in.data(), U + n * dofs + s.lo, w * sizeof(double));
                    h.push(in);
                    if (n >= 1) h.derivative(out);
                }
                secs[si] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                if (D_last) std::memcpy(D_last + s.lo, out.data(), w * sizeof(double));
            };
            if (sbd) {
                SbdHistory h(ksbd[s.g], HistoryVariant::standalone, w);
                drive(h);
            } else {
                BeHistory h(kbe[s.g], HistoryVariant::standalone, w);
                drive(h);
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (std::size_t i = 0; i < slices.size(); ++i) pool.emplace_back(work, i);
        for (auto& t : pool) t.join();
        (void)t0;
        *seconds = *std::max_element(secs.begin(), secs.end());
    });
}


// Reference histories over U[n_steps, dofs] (groups of equal width, one kernel each), `threads`
// workers over DOF slices, recording the derivative D at levels n = stride-1, 2 stride-1, ...
// into D_trace[(n + 1) / stride - 1][dofs] (the parity trace of many lanes at a full horizon).
int ref_hist_trace(int sbd, int n_groups, const double* gammas, double tau, const int* nh,
                   const int* np1, const int* np2, const double* const* heads,
                   const double* const* m1, const double* const* r1, const double* const* m2,
                   const double* const* r2, long dofs, long n_steps, const double* U,
                   long stride, double* D_trace, int threads) {
    return guard([&] {
        std::vector<FastKernelBE> kbe;
        std::vector<FastKernelSBD> ksbd;
        for (int g = 0; g < n_groups; ++g) {
            const FlatKernel f{sbd, nh[g], np1[g], np2[g], gammas[g], tau, heads[g],
                               m1[g],  r1[g], m2 ? m2[g] : nullptr, r2 ? r2[g] : nullptr};
            if (sbd)
                ksbd.push_back(to_sbd(f));
            else
                kbe.push_back(to_be(f));
        }
        const long per_group = dofs / n_groups;
        struct Slice {
            int g;
            long lo, hi;
        };
        std::vector<Slice> slices;
        const int T = std::max(1, threads);
        const int per = std::max(1, T / n_groups);
        for (int g = 0; g < n_groups; ++g)
            for (int t = 0; t < per; ++t) {
                const long lo = g * per_group + per_group * t / per;
                const long hi = g * per_group + per_group * (t + 1) / per;
                if (hi > lo) slices.push_back({g, lo, hi});
            }
        auto work = [&](std::size_t si) {
            const Slice s = slices[si];
            const long w = s.hi - s.lo;
            std::vector<double> in(w), out(w);
            auto drive = [&](auto& h) {
                for (long n = 0; n < n_steps; ++n) {
                    std::memcpy(in.data(), U + n * dofs + s.lo, w * sizeof(double));
                    h.push(in);
                    if (n >= 1) h.derivative(out);
                    if ((n + 1) % stride == 0) {
                        double* row = D_trace + ((n + 1) / stride - 1) * dofs + s.lo;
                        if (n >= 1)
                            std::memcpy(row, out.data(), w * sizeof(double));
                        else
                            for (long i = 0; i < w; ++i) row[i] = std::nan("");
                    }
                }
            };
            if (sbd) {
                SbdHistory h(ksbd[s.g], HistoryVariant::standalone, w);
                drive(h);
            } else {
                BeHistory h(kbe[s.g], HistoryVariant::standalone, w);
                drive(h);
            }
        };
        std::vector<std::thread> pool;
        for (std::size_t i = 0; i < slices.size(); ++i) pool.emplace_back(work, i);
        for (auto& t : pool) t.join();
    });
}

// ---------------------------------------------------------------------------------------------
// Mode-space FFPE restatement over the reference's own history lanes: the
// reference's mode-space oracle algebra (test_fpfp.cpp:79-134, mode_be / mode_sbd, solve2x2)
// with the O(n) sums replaced by fraq::BeHistory / SbdHistory (scheme variant, one lane per
// mode), i.e. FastStepper (fpfp.cpp:259-349) with A -> diag(lam).  The SBD correction
// c_n = sum m r^(n-4) uses running powers as CorrPowers does (fpfp.cpp:240-250; restated here,
// it is internal to fpfp.cpp).  `threads` workers each own a contiguous slice of modes.
// Kernel k (0, 1) of field k is given in flat form.  Returns the loop wall time (max over
// workers) in *seconds.
int ref_modal_run(int sbd, const double* gammas, double tau, const int* nh, const int* np1,
                  const int* np2, const double* const* heads, const double* const* m1,
                  const double* const* r1, const double* const* m2, const double* const* r2,
                  double a, long N, long nm, const double* lam, const double* u0,
                  const double* v0, double* uN, double* vN, int threads, double* seconds) {
    return guard([&] {
        FastKernelBE kb[2];
        FastKernelSBD ks[2];
        for (int f = 0; f < 2; ++f) {
            const FlatKernel fk{sbd, nh[f], np1[f], np2[f], gammas[f], tau, heads[f],
                                m1[f],  r1[f], m2 ? m2[f] : nullptr, r2 ? r2[f] : nullptr};
            if (sbd)
                ks[f] = to_sbd(fk);
            else
                kb[f] = to_be(fk);
        }
        const int T = (int)std::max(1L, std::min<long>(threads, nm));
        std::vector<double> secs(T, 0.0);
        auto corr_at = [&](const FastKernelSBD& k, std::vector<double>& p1, std::vector<double>& p2,
                           long& e, long target) {
            while (e < target) {
                for (std::size_t j = 0; j < p1.size(); ++j) p1[j] *= k.ratio1[j];
                for (std::size_t j = 0; j < p2.size(); ++j) p2[j] *= k.ratio2[j];
                ++e;
            }
            double v = 0.0;
            for (std::size_t j = 0; j < p1.size(); ++j) v += k.mult1[j] * p1[j];
            for (std::size_t j = 0; j < p2.size(); ++j) v += k.mult2[j] * p2[j];
            return v;
        };
        auto work = [&](int w) {
            const long lo = nm * w / T, hi = nm * (w + 1) / T, d = hi - lo;
            if (d <= 0) return;
            std::vector<double> s1(d), s2(d), x1(u0 + lo, u0 + hi), x2(v0 + lo, v0 + hi);
            const double d10 = sbd ? ks[0].head[0] : kb[0].head[0];
            const double d20 = sbd ? ks[1].head[0] : kb[1].head[0];
            auto drive = [&](auto& h1, auto& h2) {
                std::vector<double> p11, p12, p21, p22;
                long e1 = 0, e2 = 0;
                if (sbd) {
                    p11.assign(ks[0].ratio1.size(), 1.0);
                    p12.assign(ks[0].ratio2.size(), 1.0);
                    p21.assign(ks[1].ratio1.size(), 1.0);
                    p22.assign(ks[1].ratio2.size(), 1.0);
                }
                const auto t0 = std::chrono::steady_clock::now();
                h1.append(x1);
                h2.append(x2);
                for (long n = 1; n <= N; ++n) {
                    h1.advance();
                    h2.advance();
                    const auto u1 = h1.lagged(0);
                    const auto v1 = h2.lagged(0);
                    if (sbd && n == 1) {
                        for (long k = 0; k < d; ++k) {
                            const double al = a + lam[lo + k];
                            const double r1v = u1[k] / tau - (d10 / 3.0) * al * u1[k] + (a * d20 / 3.0) * v1[k];
                            const double r2v = v1[k] / tau - (d20 / 3.0) * al * v1[k] + (a * d10 / 3.0) * u1[k];
                            const double a11 = 1.0 / tau + (2.0 / 3.0) * d10 * al, a12 = -(2.0 / 3.0) * a * d20;
                            const double a21 = -(2.0 / 3.0) * a * d10, a22 = 1.0 / tau + (2.0 / 3.0) * d20 * al;
                            const double det = a11 * a22 - a12 * a21;
                            x1[k] = (r1v * a22 - a12 * r2v) / det;
                            x2[k] = (a11 * r2v - a21 * r1v) / det;
                        }
                    } else {
                        h1.history_sum(s1);
                        h2.history_sum(s2);
                        std::span<const double> u2, v2;
                        if (!sbd) {
                            if (n >= 2)
                                for (long k = 0; k < d; ++k) {
                                    s1[k] += kb[0].head[1] * u1[k];
                                    s2[k] += kb[1].head[1] * v1[k];
                                }
                        } else {
                            for (int f = 0; f < 2; ++f) {
                                const FastKernelSBD& kk = ks[f];
                                auto& hh = f ? h2 : h1;
                                std::vector<double>& ss = f ? s2 : s1;
                                const long top = std::min<long>(kk.n_head - 1, n - 1);
                                for (long i = 1; i <= top; ++i) {
                                    const auto u = hh.lagged(i - 1);
                                    for (long k = 0; k < d; ++k) ss[k] += kk.head[i] * u[k];
                                }
                            }
                            const double c1 = (n - 1 < ks[0].n_head) ? ks[0].head[n - 1] : corr_at(ks[0], p11, p12, e1, n - 4);
                            const double c2 = (n - 1 < ks[1].n_head) ? ks[1].head[n - 1] : corr_at(ks[1], p21, p22, e2, n - 4);
                            for (long k = 0; k < d; ++k) {
                                s1[k] += 0.5 * c1 * u0[lo + k];
                                s2[k] += 0.5 * c2 * v0[lo + k];
                            }
                            u2 = h1.lagged(1);
                            v2 = h2.lagged(1);
                        }
                        const double lead = sbd ? 1.5 : 1.0;
                        for (long k = 0; k < d; ++k) {
                            const double al = a + lam[lo + k];
                            const double l1 = sbd ? (2.0 * u1[k] - 0.5 * u2[k]) / tau : u1[k] / tau;
                            const double l2 = sbd ? (2.0 * v1[k] - 0.5 * v2[k]) / tau : v1[k] / tau;
                            const double r1v = l1 - al * s1[k] + a * s2[k];
                            const double r2v = l2 - al * s2[k] + a * s1[k];
                            const double a11 = lead / tau + d10 * al, a12 = -a * d20;
                            const double a21 = -a * d10, a22 = lead / tau + d20 * al;
                            const double det = a11 * a22 - a12 * a21;
                            x1[k] = (r1v * a22 - a12 * r2v) / det;
                            x2[k] = (a11 * r2v - a21 * r1v) / det;
                        }
                    }
                    h1.append(x1);
                    h2.append(x2);
                }
                secs[w] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
                std::memcpy(uN + lo, x1.data(), d * sizeof(double));
                std::memcpy(vN + lo, x2.data(), d * sizeof(double));
            };
            if (sbd) {
                SbdHistory h1(ks[0], HistoryVariant::scheme, d), h2(ks[1], HistoryVariant::scheme, d);
                drive(h1, h2);
            } else {
                BeHistory h1(kb[0], HistoryVariant::scheme, d), h2(kb[1], HistoryVariant::scheme, d);
                drive(h1, h2);
            }
        };
        std::vector<std::thread> pool;
        for (int w = 0; w < T; ++w) pool.emplace_back(work, w);
        for (auto& t : pool) t.join();
        *seconds = *std::max_element(secs.begin(), secs.end());
    });
}

}  // extern "C"
