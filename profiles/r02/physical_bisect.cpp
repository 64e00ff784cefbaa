// Throwaway experiment: where does the physical-space FastBE deviation come from?
#include <fraq/fast_kernel.hpp>
#include <fraq/block_solver.hpp>
#include <fraq/fpfp.hpp>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
using namespace fraq;
typedef long double LD;

template <class T>
struct LU {  // reference BandedLU algorithm, templated real type
    int n, kl = 2, ku = 2, ldab = 7; std::vector<T> ab; std::vector<int> piv;
    LU(int n_) : n(n_), ab((size_t)7 * n_, 0), piv(n_) {}
    T& at(int r, int c) { return ab[(size_t)c * ldab + (kl + ku + r - c)]; }
    void factor() {
        const int kv = kl + ku;
        for (int j = 0; j < n; ++j) {
            const int jmax = std::min(n - 1, j + kl);
            int p = j; T pmax = std::abs(ab[(size_t)j * ldab + kv]);
            for (int i = j + 1; i <= jmax; ++i) { T v = std::abs(ab[(size_t)j * ldab + kv + (i - j)]); if (v > pmax) { pmax = v; p = i; } }
            piv[j] = p;
            const int cmax = std::min(n - 1, j + kv);
            if (p != j) for (int c = j; c <= cmax; ++c) { size_t b = (size_t)c * ldab + kv; std::swap(ab[b + (j - c)], ab[b + (p - c)]); }
            const T dinv = T(1) / ab[(size_t)j * ldab + kv];
            for (int i = j + 1; i <= jmax; ++i) {
                T& lij = ab[(size_t)j * ldab + kv + (i - j)]; lij *= dinv; const T l = lij;
                for (int c = j + 1; c <= cmax; ++c) { size_t b = (size_t)c * ldab + kv; ab[b + (i - c)] -= l * ab[b + (j - c)]; }
            }
        }
    }
    template <class S> void solve(std::vector<S>& r) const {
        const int kv = kl + ku;
        for (int j = 0; j < n; ++j) {
            if (piv[j] != j) std::swap(r[j], r[piv[j]]);
            const int imax = std::min(n - 1, j + kl); const S xj = r[j];
            for (int i = j + 1; i <= imax; ++i) r[i] -= S(ab[(size_t)j * ldab + kv + (i - j)]) * xj;
        }
        for (int j = n - 1; j >= 0; --j) {
            S v = r[j];
            for (int c = j + 1; c <= std::min(n - 1, j + kv); ++c) v -= S(ab[(size_t)c * ldab + kv + (j - c)]) * r[c];
            r[j] = v / S(ab[(size_t)j * ldab + kv]);
        }
    }
};

template <class T, class TA = T>
LU<T> make_lu(double d01, double d02, double a, double tau, int m, double h, double lead) {
    LU<T> lu(2 * m);
    typedef TA TT;
    const TA ih2 = TA(1) / (TA(h) * TA(h));
    for (int k = 0; k < m; ++k) {
        int r1 = 2 * k, r2 = 2 * k + 1;
        lu.at(r1, r1) = T(TT(lead) / TT(tau) + TT(d01) * (TT(a) + TT(2) * ih2));
        lu.at(r2, r2) = T(TT(lead) / TT(tau) + TT(d02) * (TT(a) + TT(2) * ih2));
        lu.at(r1, r2) = T(-TT(a) * TT(d02)); lu.at(r2, r1) = T(-TT(a) * TT(d01));
        if (k > 0) { lu.at(r1, r1 - 2) = T(-TT(d01) * ih2); lu.at(r2, r2 - 2) = T(-TT(d02) * ih2); }
        if (k + 1 < m) { lu.at(r1, r1 + 2) = T(-TT(d01) * ih2); lu.at(r2, r2 + 2) = T(-TT(d02) * ih2); }
    }
    lu.factor();
    return lu;
}


struct M2 { double a, b, c, d; };
struct ML { LD a, b, c, d; };
static ML mulL(const ML& x, const ML& y) { return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d}; }
static ML invL(const ML& x) { const LD det = x.a * x.d - x.b * x.c; return {x.d / det, -x.b / det, -x.c / det, x.a / det}; }
static M2 rnd(const ML& x) { return {(double)x.a, (double)x.b, (double)x.c, (double)x.d}; }
static M2 mul(const M2& x, const M2& y) { return {x.a * y.a + x.b * y.c, x.a * y.b + x.b * y.d, x.c * y.a + x.d * y.c, x.c * y.b + x.d * y.d}; }
static M2 inv(const M2& x) { const double det = x.a * x.d - x.b * x.c; return {x.d / det, -x.b / det, -x.c / det, x.a / det}; }
static M2 sub(const M2& x, const M2& y) { return {x.a - y.a, x.b - y.b, x.c - y.c, x.d - y.d}; }
static M2 scal(double s, const M2& x) { return {s * x.a, s * x.b, s * x.c, s * x.d}; }
struct V2 { double x, y; };
static V2 mv(const M2& m, V2 v) { return {std::fma(m.a, v.x, m.b * v.y), std::fma(m.c, v.x, m.d * v.y)}; }
struct CR {
    int K, m; std::vector<M2> F, G, H;
    CR(double d01, double d02, double a, double tau, int m_, double h, double lead, bool fmaent, bool ldsetup = false) : m(m_) {
        K = 0; while ((1 << K) - 1 < m) ++K;
        const double ih2 = 1.0 / (h * h);
        M2 D, E;
        if (fmaent) D = {std::fma(d01, std::fma(2.0, ih2, a), lead / tau), -a * d02, -a * d01, std::fma(d02, std::fma(2.0, ih2, a), lead / tau)};
        else { volatile double t1 = d01 * (a + 2.0 * ih2), t2 = d02 * (a + 2.0 * ih2); D = {lead / tau + t1, -a * d02, -a * d01, lead / tau + t2}; }
        E = {-d01 * ih2, 0, 0, -d02 * ih2};
        F.resize(K); G.resize(K); H.resize(K);
        if (ldsetup) {
            ML DL{D.a, D.b, D.c, D.d}, EL{E.a, E.b, E.c, E.d};
            for (int l = 0; l < K; ++l) { ML Di = invL(DL); ML FL = mulL(EL, Di); F[l] = rnd(FL); G[l] = rnd(Di); H[l] = rnd(mulL(Di, EL)); ML FE = mulL(FL, EL);
                EL = {-FE.a, -FE.b, -FE.c, -FE.d}; DL = {DL.a - 2 * FE.a, DL.b - 2 * FE.b, DL.c - 2 * FE.c, DL.d - 2 * FE.d}; }
            return;
        }
        for (int l = 0; l < K; ++l) { M2 Di = inv(D); F[l] = mul(E, Di); G[l] = Di; H[l] = mul(Di, E); M2 FE = mul(F[l], E); E = scal(-1.0, FE); D = sub(D, scal(2.0, FE)); }
    }
    template <class S> void solve(std::vector<S>& w) const {
        std::vector<V2> sb(m + 2, V2{0, 0});
        for (int k = 0; k < m; ++k) sb[k + 1] = {(double)w[2 * k], (double)w[2 * k + 1]};
        for (int l = 0; l < K - 1; ++l) { int s = 1 << l; for (int i = 2 * s; i <= m; i += 2 * s) { V2 sum{sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y}; V2 t = mv(F[l], sum); sb[i] = {sb[i].x - t.x, sb[i].y - t.y}; } }
        { int i = 1 << (K - 1); sb[i] = mv(G[K - 1], sb[i]); }
        for (int l = K - 2; l >= 0; --l) { int s = 1 << l; for (int i = s; i <= m; i += 2 * s) { V2 xb = mv(G[l], sb[i]); V2 nb{sb[i - s].x + sb[i + s].x, sb[i - s].y + sb[i + s].y}; V2 t = mv(H[l], nb); sb[i] = {xb.x - t.x, xb.y - t.y}; } }
        for (int k = 0; k < m; ++k) { w[2 * k] = sb[k + 1].x; w[2 * k + 1] = sb[k + 1].y; }
    }
};
// TH: history/accumulator type; TR: RHS type; TF: factor type; TS: substitution type
template <class TH, class TR, class TF, class TS, class TA = TF, int SOLVER = 0>
std::vector<LD> run_be(const FastKernelBE& k1, const FastKernelBE& k2, double a, int m, double tau, long N,
                       const std::vector<double>& G1, const std::vector<double>& G2) {
    const double h = 1.0 / (m + 1);
    const int np1 = k1.ratios.size(), np2 = k2.ratios.size();
    std::vector<TH> A1((size_t)np1 * m, 0), A2((size_t)np2 * m, 0);
    std::vector<TR> p1(G1.begin(), G1.end()), p2(G2.begin(), G2.end()), q1(m, 0), q2(m, 0);  // G^{n-1}, G^{n-2}
    LU<TF> lu = make_lu<TF, TA>(k1.head[0], k2.head[0], a, tau, m, h, 1.0);
    CR cr(k1.head[0], k2.head[0], a, tau, m, h, 1.0, SOLVER == 1 || SOLVER == 3, SOLVER == 3);
    std::vector<TR> s1(m), s2(m), r1(m), r2(m);
    std::vector<TS> w(2 * m);
    const TR ih2 = TR(1) / (TR(h) * TR(h));
    for (long n = 1; n <= N; ++n) {
        // advance: feed G^{n-2} if n-2 >= 1
        const bool feed = n - 2 >= 1;
        for (int j = 0; j < np1; ++j) { TH r = k1.ratios[j], ww = k1.node_weights[j]; TH* acc = &A1[(size_t)j * m];
            for (int i = 0; i < m; ++i) acc[i] = feed ? r * acc[i] + ww * TH(q1[i]) : acc[i] * r; }
        for (int j = 0; j < np2; ++j) { TH r = k2.ratios[j], ww = k2.node_weights[j]; TH* acc = &A2[(size_t)j * m];
            for (int i = 0; i < m; ++i) acc[i] = feed ? r * acc[i] + ww * TH(q2[i]) : acc[i] * r; }
        for (int i = 0; i < m; ++i) { TH x = 0, y = 0; for (int j = 0; j < np1; ++j) x += A1[(size_t)j * m + i];
            for (int j = 0; j < np2; ++j) y += A2[(size_t)j * m + i]; s1[i] = TR(x); s2[i] = TR(y); }
        if (n >= 2) for (int i = 0; i < m; ++i) { s1[i] += TR(k1.head[1]) * p1[i]; s2[i] += TR(k2.head[1]) * p2[i]; }
        for (int i = 0; i < m; ++i) {
            TR v1 = TR(2) * s1[i], v2 = TR(2) * s2[i];
            if (i > 0) { v1 -= s1[i - 1]; v2 -= s2[i - 1]; }
            if (i + 1 < m) { v1 -= s1[i + 1]; v2 -= s2[i + 1]; }
            r1[i] = p1[i] / TR(tau) - TR(a) * s1[i] - v1 * ih2 + TR(a) * s2[i];
            r2[i] = p2[i] / TR(tau) - TR(a) * s2[i] - v2 * ih2 + TR(a) * s1[i];
        }
        for (int i = 0; i < m; ++i) { w[2 * i] = TS(r1[i]); w[2 * i + 1] = TS(r2[i]); }
        if (SOLVER == 0) lu.solve(w); else cr.solve(w);
        q1 = p1; q2 = p2;
        for (int i = 0; i < m; ++i) { p1[i] = TR(w[2 * i]); p2[i] = TR(w[2 * i + 1]); }
    }
    std::vector<LD> out(2 * m);
    for (int i = 0; i < m; ++i) { out[i] = p1[i]; out[m + i] = p2[i]; }
    return out;
}

int main(int argc, char** argv) {
    long N = argc > 1 ? atol(argv[1]) : 256;
    const int m = 4095; const double tau = 1.0 / 16384; const double a = (1.0 - 0.45) / (2 * 0.45 - 1);
    KernelBudget b1{16384, 1e-12}, b2{16384, 1e-12};
    FastKernelBE k1 = build_be_kernel_auto(1 - 0.4, tau, b1), k2 = build_be_kernel_auto(1 - 0.8, tau, b2);
    std::vector<double> G1(m), G2(m);
    for (int j = 0; j < m; ++j) { double x = (j + 1) / 4096.0; G1[j] = x < 0.5 ? 1 : 0; G2[j] = x > 0.5 ? 1 : 0; }
    // reference run
    ProblemSpec sp; sp.alpha1 = 0.4; sp.alpha2 = 0.8; sp.coupling_a = a; sp.grid_m = m; sp.t_final = N * tau; sp.n_steps = N;
    sp.initial = InitialData::custom; sp.custom_g1 = G1; sp.custom_g2 = G2;
    KernelConfig kc; kc.auto_size = false; kc.be_points = 256;
    RunResult rr = run(sp, Scheme::FastBE, kc);
    bool full = getenv("FULL") != nullptr;
    auto T = full ? run_be<double, LD, LD, LD>(k1, k2, a, m, tau, N, G1, G2) : run_be<LD, LD, LD, LD>(k1, k2, a, m, tau, N, G1, G2);
    LD mx = 0; for (auto v : T) mx = std::max(mx, std::abs(v));
    auto err = [&](const std::vector<LD>& v) { LD e = 0; for (size_t i = 0; i < v.size(); ++i) e = std::max(e, std::abs(v[i] - T[i])); return (double)(e / mx); };
    std::vector<LD> R(2 * m); for (int i = 0; i < m; ++i) { R[i] = rr.final_state.g1[i]; R[m + i] = rr.final_state.g2[i]; }
    auto vsref = [&](const std::vector<LD>& v) { LD e = 0; for (size_t i = 0; i < v.size(); ++i) e = std::max(e, std::abs(v[i] - R[i])); return (double)(e / mx); };
    if (full) {
        printf("N=%ld max|T|=%.3e\nreference vs truth: %.3e\n", N, (double)mx, err(R));
        { auto V = run_be<double, double, double, double, double, 3>(k1, k2, a, m, tau, N, G1, G2); printf("CR fp64, LD setup vs ref: %.3e  vs truth %.3e\n", vsref(V), err(V)); }
        auto S = run_be<double, LD, LD, LD, double>(k1, k2, a, m, tau, N, G1, G2);  // exact solution of the fp64-entry system
        auto vsS = [&](const std::vector<LD>& v) { LD e = 0; for (size_t i = 0; i < v.size(); ++i) e = std::max(e, std::abs(v[i] - S[i])); return (double)(e / mx); };
        printf("rounded-system truth S vs truth: %.3e   ref vs S: %.3e\n", err(S), vsS(R));
        { auto V = run_be<double, double, double, double, double, 3>(k1, k2, a, m, tau, N, G1, G2); printf("CR fp64, LD setup vs S: %.3e\n", vsS(V)); }
        { auto V = run_be<double, double, LD, LD, double>(k1, k2, a, m, tau, N, G1, G2); printf("fp64 entries + LD elim vs ref: %.3e vs S %.3e\n", vsref(V), vsS(V)); }
        return 0;
    }
    printf("N=%ld  np=%zu/%zu  max|T|=%.3e\n", N, k1.ratios.size(), k2.ratios.size(), (double)mx);
    printf("reference fraq::run       vs truth: %.3e\n", err(R));
    auto V1 = run_be<double, double, double, double>(k1, k2, a, m, tau, N, G1, G2);
    printf("my fp64 replica           vs truth: %.3e   vs ref: %.3e\n", err(V1), [&]{LD e=0; for(size_t i=0;i<V1.size();++i) e=std::max(e,std::abs(V1[i]-R[i])); return (double)(e/mx);}());
    printf("fp64, LD factor+subst      vs truth: %.3e\n", err(run_be<double, double, LD, LD>(k1, k2, a, m, tau, N, G1, G2)));
    printf("fp64, LD subst only        vs truth: %.3e\n", err(run_be<double, double, double, LD>(k1, k2, a, m, tau, N, G1, G2)));
    printf("fp64, LD factor only       vs truth: %.3e\n", err(run_be<double, double, LD, double>(k1, k2, a, m, tau, N, G1, G2)));
    printf("fp64 assembly, LD factor+subst vs truth: %.3e\n", err(run_be<double, double, LD, LD, double>(k1, k2, a, m, tau, N, G1, G2)));
    printf("LD assembly, fp64 factor+subst vs truth: %.3e\n", err(run_be<double, double, double, double, LD>(k1, k2, a, m, tau, N, G1, G2)));
    { auto V = run_be<double, double, LD, LD, double>(k1, k2, a, m, tau, N, G1, G2); printf("fp64 assembly(fma), LD elim   vs ref: %.3e\n", vsref(V)); }
    { auto V = run_be<double, double, double, double, double, 1>(k1, k2, a, m, tau, N, G1, G2); printf("CR fp64, fma entries        vs ref: %.3e  vs truth %.3e\n", vsref(V), err(V)); }
    { auto V = run_be<double, double, double, double, double, 2>(k1, k2, a, m, tau, N, G1, G2); printf("CR fp64, plain entries      vs ref: %.3e  vs truth %.3e\n", vsref(V), err(V)); }
    { auto V = run_be<double, double, double, double, double, 3>(k1, k2, a, m, tau, N, G1, G2); printf("CR fp64, fma entries, LD setup vs ref: %.3e  vs truth %.3e\n", vsref(V), err(V)); }
    printf("fp64 hist, LD rhs+solve    vs truth: %.3e\n", err(run_be<double, LD, LD, LD>(k1, k2, a, m, tau, N, G1, G2)));
    printf("LD hist, fp64 rhs+solve    vs truth: %.3e\n", err(run_be<LD, double, double, double>(k1, k2, a, m, tau, N, G1, G2)));
    printf("LD hist+rhs, fp64 solve    vs truth: %.3e\n", err(run_be<LD, LD, double, double>(k1, k2, a, m, tau, N, G1, G2)));
}
