// setup.cu -- device setup kernels K1-K4 of the fast-CQ path.
//
//   K1  classical CQ weights            (cq_weights.cpp:19-59)
//   K2  Gauss-Jacobi rules              (gauss_jacobi.cpp:108-204)
//   K3  prefactor folding               (fast_kernel.cpp:54-124)
//   K4  reconstruction / error scans    (fast_kernel.cpp:22-34,126-256; fpfp.cpp:240-250)
//
// All fp64.  The weight recurrences run the reference's serial chains one thread per chain, so
// be_weights and the SBD Cauchy product reproduce the reference's rounding; node tables differ
// from the reference's implicit-QL ones by ~1 ulp (bisection + Newton polish here).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace fraqcu {

namespace {

constexpr double kPi = 3.14159265358979323846;

// Lanczos gamma, g = 7, nine published coefficients; reflection below 1/2.
__device__ double dev_gamma(double x) {
    const double c[9] = {0.99999999999980993,  676.5203681218851,     -1259.1392167224028,
                         771.32342877765313,   -176.61502916214059,   12.507343278686905,
                         -0.13857109526572012, 9.9843695780195716e-6, 1.5056327351493116e-7};
    double refl = 1.0;
    if (x < 0.5) {
        refl = kPi / sin(kPi * x);
        x = 1.0 - x;
    }
    const double z = x - 1.0;
    double s = c[0];
    for (int i = 1; i < 9; ++i) s += c[i] / (z + i);
    const double t = z + 7.5;
    const double gv = sqrt(2.0 * kPi) * pow(t, z + 0.5) * exp(-t) * s;
    return refl == 1.0 ? gv : refl / gv;
}

__device__ double dev_mu0(double a, double b) {
    return pow(2.0, a + b + 1.0) * dev_gamma(a + 1.0) * dev_gamma(b + 1.0) / dev_gamma(a + b + 2.0);
}

__device__ double rec_alpha(double a, double b, int k) {
    if (k == 0) return (b - a) / (a + b + 2.0);
    const double s = 2.0 * k + a + b;
    return (b * b - a * a) / (s * (s + 2.0));
}

__device__ double rec_beta(double a, double b, int k) {  // k >= 1
    const double s = 2.0 * k + a + b;
    if (k == 1) return 4.0 * (a + 1.0) * (b + 1.0) / (s * s * (s + 1.0));
    return 4.0 * k * (k + a) * (k + b) * (k + a + b) / (s * s * (s + 1.0) * (s - 1.0));
}

// ------------------------------------------------------------------------------------- K2+K3
// One CTA per rule.  Thread i finds the i-th smallest eigenvalue of the Jacobi matrix by Sturm
// bisection, polishes it with Newton on the monic P_n (the reference's single guarded step,
// gauss_jacobi.cpp:180-187), computes the Christoffel weight (gauss_jacobi.cpp:189-201), then
// folds the node into the requested kernel family (fast_kernel.cpp:54-124).
struct RuleJob {
    double a, b;      // Jacobi exponents
    int n;            // points
    int fold;         // 0: raw rule, 1: BE fold, 2: SBD family 1, 3: SBD family 2, 4: SBD both
    double gamma, tau;
    double* out_x;    // nodes / ratios   (family 1 when fold == 4)
    double* out_w;    // weights / mults
    double* out_x2;   // family 2 (fold == 4)
    double* out_w2;
};

constexpr int kRuleThreads = 512;

__global__ void __launch_bounds__(kRuleThreads) rule_kernel(const RuleJob* jobs) {
    const RuleJob J = jobs[blockIdx.x];
    const int n = J.n;
    const double a = J.a, b = J.b;
    __shared__ double s_al[FRAQ_MAX_POINTS];  // monic alpha_k
    __shared__ double s_be[FRAQ_MAX_POINTS];  // monic beta_k (k>=1), squared off-diagonals
    __shared__ double s_sb[FRAQ_MAX_POINTS];  // sqrt(beta_k)
    __shared__ double s_lo, s_hi, s_mu0;
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        s_al[k] = rec_alpha(a, b, k);
        if (k >= 1) {
            const double bk = rec_beta(a, b, k);
            s_be[k] = bk;
            s_sb[k] = sqrt(bk);
        } else {
            s_be[0] = 0.0;
            s_sb[0] = 0.0;
        }
    }
    if (threadIdx.x == 0) s_mu0 = dev_mu0(a, b);
    __syncthreads();
    if (threadIdx.x == 0) {
        // Gershgorin interval
        double lo = 1e300, hi = -1e300;
        for (int k = 0; k < n; ++k) {
            const double r = (k > 0 ? s_sb[k] : 0.0) + (k + 1 < n ? s_sb[k + 1] : 0.0);
            lo = fmin(lo, s_al[k] - r);
            hi = fmax(hi, s_al[k] + r);
        }
        s_lo = lo - 1e-12;
        s_hi = hi + 1e-12;
    }
    __syncthreads();
    const int i = threadIdx.x;
    if (i >= n) return;
    // Sturm count: number of eigenvalues < x (LDL^T pivots, guarded against zero pivots).
    // (a zero pivot is replaced by -tiny and counted as negative, LAPACK dstebz style)
    auto count_below = [&](double x) {
        double q = s_al[0] - x;
        if (q == 0.0) q = -1e-300;
        int cnt = q < 0.0;
        for (int k = 1; k < n; ++k) {
            q = (s_al[k] - x) - s_be[k] / q;
            if (q == 0.0) q = -1e-300;
            cnt += q < 0.0;
        }
        return cnt;
    };
    double lo = s_lo, hi = s_hi;
    for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        if (mid <= lo || mid >= hi) break;
        if (hi - lo <= 1e-13 * fmax(1.0, fabs(mid))) break;
        if (count_below(mid) >= i + 1)
            hi = mid;
        else
            lo = mid;
    }
    double x = 0.5 * (lo + hi);
    // Newton on the monic P_n; the reference applies one step guarded by |step| < 1e-8 to a
    // QL eigenvalue accurate to ~1e-16; from the 1e-13 bisection bracket two guarded steps land
    // on the same root.
    for (int pass = 0; pass < 2; ++pass) {
        double p = 1.0, dp = 0.0, pm = 0.0, dpm = 0.0;
        for (int k = 0; k < n; ++k) {
            const double al = s_al[k], be = (k == 0) ? 0.0 : s_be[k];
            const double pn = (x - al) * p - be * pm;
            const double dpn = p + (x - al) * dp - be * dpm;
            pm = p;
            dpm = dp;
            p = pn;
            dp = dpn;
        }
        if (dp != 0.0) {
            const double step = p / dp;
            if (fabs(step) < 1e-8) x -= step;
        }
    }
    // Christoffel weight, orthonormal recurrence
    double qm = 0.0, q = 1.0 / sqrt(s_mu0), sum = q * q, bprev = 0.0;
    for (int k = 0; k < n - 1; ++k) {
        const double bk1 = s_sb[k + 1];
        const double qn = ((x - s_al[k]) * q - bprev * qm) / bk1;
        qm = q;
        q = qn;
        bprev = bk1;
        sum += q * q;
    }
    const double w = 1.0 / sum;
    const double s = x, g = J.gamma;
    switch (J.fold) {
        case 0:
            J.out_x[i] = s;
            J.out_w[i] = w;
            break;
        case 1: {  // BE: w -> -(sin(pi g)/pi)/(4 tau^g) w, r = (s+1)/2
            const double pref = -(sin(kPi * g) / kPi) / (4.0 * pow(J.tau, g));
            J.out_w[i] = pref * w;
            J.out_x[i] = 0.5 * (s + 1.0);
            break;
        }
        default: {
            const double igg = sin(kPi * g) / kPi;
            const double ta = pow(J.tau, g);
            if (J.fold == 2 || J.fold == 4) {
                // Re[c1 w q^4], c1 = -2^(2+2g) e^{-i pi g} igg / tau^g
                const double c1re = (-pow(2.0, 2.0 + 2.0 * g)) * cos(-kPi * g) * igg / ta;
                const double qq = 1.0 / (s + 5.0);
                J.out_w[i] = (c1re * w) * (qq * qq * qq * qq);
                J.out_x[i] = (s + 1.0) / (s + 5.0);
            }
            if (J.fold == 3 || J.fold == 4) {
                const double c2 = -pow(2.0, -g - 3.0) * igg / ta;
                const double ww = 1.0 + 3.0 * s;
                const double rp = ww >= 0.0 ? pow(ww, g) : pow(-ww, g) * cos(kPi * g);
                double* ox = J.fold == 4 ? J.out_x2 : J.out_x;
                double* ow = J.fold == 4 ? J.out_w2 : J.out_w;
                ow[i] = c2 * w * rp;
                ox[i] = 0.5 * (s + 1.0);
            }
            break;
        }
    }
}

// ------------------------------------------------------------------------------------- K1
// Binomial chains c_i = c_{i-1} ((i-1-g)/i) x, one thread per chain (cq_weights.cpp:19-25).
struct ChainJob {
    double g, x;
    long n_max;
    double* out;
};
// One CTA per chain: the ratios q_i = (i-1-g)/i do not depend on the chain, so the CTA computes
// them in parallel into the output first (an fp64 division is a ~40-instruction sequence; inside
// the serial loop it set the pace), then one thread runs the product c_i = (c_(i-1) q_i) x in the
// reference's order -- bitwise the reference's chain (cq_weights.cpp:19-25).
__global__ void chain_kernel(const ChainJob* jobs, int n_jobs) {
    const ChainJob J = jobs[blockIdx.x];
    for (long i = 1 + threadIdx.x; i <= J.n_max; i += blockDim.x) J.out[i] = (i - 1 - J.g) / i;
    __syncthreads();
    if (threadIdx.x != 0) return;
    double c = 1.0;
    J.out[0] = c;
    // batches of 16 ratios in registers: the loads of a batch are in flight together
    long i = 1;
    for (; i + 15 <= J.n_max; i += 16) {
        double q[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) q[t] = J.out[i + t];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            c = c * q[t] * J.x;
            J.out[i + t] = c;
        }
    }
    for (; i <= J.n_max; ++i) {
        c = c * J.out[i] * J.x;
        J.out[i] = c;
    }
}

// d_i = c_i * tau^-g for every table of a batch (blockIdx.y = table).  The scales come from the
// host's std::pow, the reference's own call (cq_weights.cpp:36), so d_0 -- which enters the
// FFPE block system's diagonal, where one ulp is amplified by the ~1e6 condition number --
// is bit-identical to the reference's.
__global__ void scale_kernel(double* base, long n, const double* scales) {
    double* v = base + (long)blockIdx.y * n;
    const double sc = scales[blockIdx.y];
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        v[i] *= sc;
}

// SBD Cauchy product out_i = (3/(2 tau))^g sum_{j<=i} c1_j c2_{i-j}, serial j per output index
// (cq_weights.cpp:56-59).  blockIdx.y = table in a batch.
struct CauchyJob {
    double sc;  // (3/(2 tau))^g from the host's std::pow (cq_weights.cpp:54)
    long n_max;
    const double* c1;
    const double* c2;
    double* out;
};
__global__ void cauchy_kernel(const CauchyJob* jobs) {
    const CauchyJob J = jobs[blockIdx.y];
    const double sc = J.sc;
    // process indices from the top so long rows start first
    const long i = J.n_max - (blockIdx.x * (long)blockDim.x + threadIdx.x);
    if (i < 0) return;
    const double* __restrict__ c1 = J.c1;
    const double* __restrict__ c2 = J.c2 + i;
    double acc = 0.0;
    long j = 0;
    for (; j + 4 <= i + 1; j += 4) {
        acc = fma(__ldg(c1 + j), __ldg(c2 - j), acc);
        acc = fma(__ldg(c1 + j + 1), __ldg(c2 - j - 1), acc);
        acc = fma(__ldg(c1 + j + 2), __ldg(c2 - j - 2), acc);
        acc = fma(__ldg(c1 + j + 3), __ldg(c2 - j - 3), acc);
    }
    for (; j <= i; ++j) acc = fma(__ldg(c1 + j), __ldg(c2 - j), acc);
    J.out[i] = sc * acc;
}

// ------------------------------------------------------------------------------------- K4
// Reconstruction scan.  One CTA per kernel; thread j owns node j (family 1 then family 2) and
// walks its power chain p_j *= r_j serially in i exactly like the reference's incremental
// scans; per index the node terms m_j p_j are summed by a warp reduce-scatter + cross-warp pass.
// start_mode 0: p_j starts at 1 at i = i_lo; 1: p_j starts at pow(r_j, i_lo - 3) (SBD).
struct ScanJob {
    int J;                 // nodes (<= 1024)
    const double* m;       // J multipliers (device)
    const double* r;       // J ratios
    int start_mode;
    long i_lo, i_hi;
    const double* table;   // nullable: classical weights, index i
    double* out;           // nullable: rec[i] (table == null) or eps[i] (table != null), index i
    double* out_max;       // nullable, with table: max eps
    long* out_arg;         // argmax (first index attaining the max)
};

constexpr int kScanThreads = 512;
constexpr int kScanChunk = 32;

__global__ void __launch_bounds__(kScanThreads) scan_kernel(const ScanJob* jobs) {
    const ScanJob S = jobs[blockIdx.x];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nwarps = blockDim.x >> 5;
    __shared__ double s_part[kScanThreads / 32][kScanChunk];
    __shared__ double s_max[32];
    __shared__ long s_arg[32];
    // each thread may own up to two nodes (J <= 1024)
    double m0 = 0.0, r0 = 0.0, p0 = 0.0, m1 = 0.0, r1 = 0.0, p1 = 0.0;
    const int j0 = tid, j1 = tid + blockDim.x;
    if (j0 < S.J) {
        m0 = S.m[j0];
        r0 = S.r[j0];
        p0 = S.start_mode ? pow(r0, (double)(S.i_lo - 3)) : 1.0;
    }
    if (j1 < S.J) {
        m1 = S.m[j1];
        r1 = S.r[j1];
        p1 = S.start_mode ? pow(r1, (double)(S.i_lo - 3)) : 1.0;
    }
    double best = -1.0;
    long barg = S.i_lo;
    for (long i0 = S.i_lo; i0 <= S.i_hi; i0 += kScanChunk) {
        double v[kScanChunk];
#pragma unroll
        for (int t = 0; t < kScanChunk; ++t) {
            v[t] = m0 * p0 + m1 * p1;
            p0 *= r0;
            p1 *= r1;
        }
        // warp reduce-scatter: after the 5 levels lane l holds the warp sum for index i0 + l
#pragma unroll
        for (int lvl = 0; lvl < 5; ++lvl) {
            const int half = 16 >> lvl;  // values kept per lane after this level = half
            const bool upper = (lane & half) != 0;
#pragma unroll
            for (int t = 0; t < half; ++t) {
                const double send = upper ? v[t] : v[t + half];
                const double keep = upper ? v[t + half] : v[t];
                v[t] = keep + __shfl_xor_sync(0xffffffffu, send, half);
            }
        }
        // lane l now holds index with bit-reversed-by-level mapping: upper halves kept -> the
        // surviving slot index equals lane (bits taken from lane at each level)
        s_part[warp][lane] = v[0];
        __syncthreads();
        if (warp == 0) {
            double rec = 0.0;
            for (int w = 0; w < nwarps; ++w) rec += s_part[w][lane];
            const long i = i0 + lane;
            if (i <= S.i_hi) {
                if (S.table) {
                    const double e = fabs(rec - S.table[i]);
                    if (S.out) S.out[i] = e;
                    if (e > best) {
                        best = e;
                        barg = i;
                    }
                } else if (S.out) {
                    S.out[i] = rec;
                }
            }
        }
        __syncthreads();
    }
    if (warp == 0 && S.out_max) {
        s_max[lane] = best;
        s_arg[lane] = barg;
        __syncwarp();
        if (lane == 0) {
            double bm = -1.0;
            long ba = S.i_lo;
            for (int l = 0; l < 32; ++l)
                if (s_max[l] > bm || (s_max[l] == bm && s_arg[l] < ba)) {
                    bm = s_max[l];
                    ba = s_arg[l];
                }
            *S.out_max = bm < 0.0 ? 0.0 : bm;
            *S.out_arg = bm <= 0.0 ? S.i_lo : ba;
        }
    }
}

// pow-based reconstruct at arbitrary indices (fast_kernel.cpp:38-52)
__global__ void reconstruct_kernel(const double* m, const double* r, int J, double shift,
                                   const long* idx, long n, double* out) {
    const long t = blockIdx.x * (long)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double e = (double)idx[t] - shift;
    double acc = 0.0;
    for (int j = 0; j < J; ++j) acc += m[j] * pow(r[j], e);
    out[t] = acc;
}

// ------------------------------------------------------------------------------------- host side
template <class T>
DevBuf<T> upload(fraq_ctx c, const std::vector<T>& v) {
    DevBuf<T> d(v.size());
    if (!v.empty())
        FRAQ_CUDA(cudaMemcpyAsync(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice,
                                  c->stream));
    return d;
}

void check_rule_args(double a, double b, int n) {
    if (!(a > -1.0) || !(b > -1.0))
        fail(FRAQ_EINVAL, "jacobi exponents must be > -1, got a=" + std::to_string(a) +
                              " b=" + std::to_string(b));
    if (n < 1) fail(FRAQ_EINVAL, "gauss_jacobi: n_points must be >= 1");
    if (n > FRAQ_MAX_POINTS) fail(FRAQ_EINVAL, "gauss_jacobi: n_points capped at 512");
}

void run_rules(fraq_ctx c, const std::vector<RuleJob>& jobs) {
    if (jobs.empty()) return;
    DevBuf<RuleJob> dj = upload(c, jobs);
    rule_kernel<<<(unsigned)jobs.size(), kRuleThreads, 0, c->stream>>>(dj.p);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

void run_scans(fraq_ctx c, const std::vector<ScanJob>& jobs) {
    if (jobs.empty()) return;
    DevBuf<ScanJob> dj = upload(c, jobs);
    // one node per thread; with J <= 256 the upper 256 threads would only add zeros (dropping
    // them leaves every sum bitwise the same and halves the cross-warp pass)
    int maxJ = 0;
    for (const ScanJob& j : jobs) maxJ = std::max(maxJ, j.J);
    const int threads = maxJ <= 256 ? 256 : kScanThreads;
    scan_kernel<<<(unsigned)jobs.size(), threads, 0, c->stream>>>(dj.p);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

// Classical tables for a batch of exponents, device resident: tables[t] points at n_max+1 values.
void weights_batch(fraq_ctx c, bool sbd, const std::vector<double>& gs, double tau, long n_max,
                   double* base /* gs.size() * (n_max+1) */) {
    const int B = (int)gs.size();
    const long L = n_max + 1;
    if (!sbd) {
        std::vector<ChainJob> cj(B);
        for (int t = 0; t < B; ++t) cj[t] = {gs[t], 1.0, n_max, base + t * L};
        DevBuf<ChainJob> d = upload(c, cj);
        chain_kernel<<<B, 256, 0, c->stream>>>(d.p, B);
        FRAQ_LAUNCH_CHECK();
        std::vector<double> sc(B);
        for (int t = 0; t < B; ++t) sc[t] = std::pow(tau, -gs[t]);
        DevBuf<double> dsc = upload(c, sc);
        dim3 grid((unsigned)std::min<long>(256, (L + 255) / 256), (unsigned)B);
        scale_kernel<<<grid, 256, 0, c->stream>>>(base, L, dsc.p);
        FRAQ_LAUNCH_CHECK();
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    DevBuf<double> cs((size_t)2 * B * L);
    std::vector<ChainJob> cj(2 * B);
    for (int t = 0; t < B; ++t) {
        cj[2 * t] = {gs[t], 1.0, n_max, cs.p + (size_t)(2 * t) * L};
        cj[2 * t + 1] = {gs[t], 1.0 / 3.0, n_max, cs.p + (size_t)(2 * t + 1) * L};
    }
    DevBuf<ChainJob> d = upload(c, cj);
    chain_kernel<<<2 * B, 256, 0, c->stream>>>(d.p, 2 * B);
    FRAQ_LAUNCH_CHECK();
    std::vector<CauchyJob> qj(B);
    for (int t = 0; t < B; ++t)
        qj[t] = {std::pow(1.5 / tau, gs[t]), n_max, cs.p + (size_t)(2 * t) * L, cs.p + (size_t)(2 * t + 1) * L,
                 base + t * L};
    DevBuf<CauchyJob> dq = upload(c, qj);
    dim3 grid((unsigned)((L + 127) / 128), (unsigned)B);
    cauchy_kernel<<<grid, 128, 0, c->stream>>>(dq.p);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

// Host copy of a kernel's flat device tables (J = np1 + np2 nodes: m then r).
struct DevKernel {
    DevBuf<double> m, r;
    int J = 0;
};

DevKernel upload_kernel(fraq_ctx c, const fraq_kernel_t* k) {
    DevKernel d;
    d.J = k->np1 + k->np2;
    std::vector<double> m(d.J), r(d.J);
    for (int j = 0; j < k->np1; ++j) {
        m[j] = k->m1[j];
        r[j] = k->r1[j];
    }
    for (int j = 0; j < k->np2; ++j) {
        m[k->np1 + j] = k->m2[j];
        r[k->np1 + j] = k->r2[j];
    }
    d.m = upload(c, m);
    d.r = upload(c, r);
    return d;
}

void fill_head(fraq_ctx c, bool sbd, double g, double tau, int nh, fraq_kernel_t* k) {
    DevBuf<double> h((size_t)nh);
    std::vector<double> gs{g};
    weights_batch(c, sbd, gs, tau, nh - 1, h.p);
    FRAQ_CUDA(cudaMemcpy(k->head, h.p, sizeof(double) * nh, cudaMemcpyDeviceToHost));
}

}  // namespace

// ============================================================================ public (internal)
void gauss_jacobi_dev(fraq_ctx c, double a, double b, int n, double* nodes_h, double* w_h) {
    check_rule_args(a, b, n);
    DevBuf<double> out(2 * (size_t)n);
    RuleJob j{a, b, n, 0, 0.0, 0.0, out.p, out.p + n, nullptr, nullptr};
    run_rules(c, {j});
    FRAQ_CUDA(cudaMemcpy(nodes_h, out.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(w_h, out.p + n, sizeof(double) * n, cudaMemcpyDeviceToHost));
}

void be_weights_dev(fraq_ctx c, double g, double tau, long n_max, double* out_d) {
    check_weight_args(g, tau);
    if (n_max < 0) fail(FRAQ_EINVAL, "be_weights: n_max must be >= 0");
    weights_batch(c, false, {g}, tau, n_max, out_d);
}

void sbd_weights_dev(fraq_ctx c, double g, double tau, long n_max, double* out_d) {
    check_weight_args(g, tau);
    if (n_max < 0) fail(FRAQ_EINVAL, "sbd_weights: n_max must be >= 0");
    weights_batch(c, true, {g}, tau, n_max, out_d);
}

void build_be_kernel_dev(fraq_ctx c, double g, double tau, int np, fraq_kernel_t* k) {
    check_kernel_gamma(g);
    if (np < 2) fail(FRAQ_EINVAL, "build_be_kernel: n_points must be >= 2");
    check_rule_args(g, 1.0 - g, np);
    std::memset(k, 0, sizeof(*k));
    k->sbd = 0;
    k->gamma = g;
    k->tau = tau;
    k->n_head = 2;
    k->np1 = np;
    k->np2 = 0;
    DevBuf<double> out(2 * (size_t)np);
    run_rules(c, {RuleJob{g, 1.0 - g, np, 1, g, tau, out.p, out.p + np, nullptr, nullptr}});
    FRAQ_CUDA(cudaMemcpy(k->r1, out.p, sizeof(double) * np, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(k->m1, out.p + np, sizeof(double) * np, cudaMemcpyDeviceToHost));
    fill_head(c, false, g, tau, 2, k);
}

void build_sbd_kernel_dev(fraq_ctx c, double g, double tau, int np1, int np2, int nh,
                          fraq_kernel_t* k) {
    check_kernel_gamma(g);
    if (np1 < 1 || np2 < 1) fail(FRAQ_EINVAL, "build_sbd_kernel: point counts must be >= 1");
    if (nh < 3) fail(FRAQ_EINVAL, "build_sbd_kernel: n_head must be >= 3");
    if (nh > FRAQ_MAX_HEAD) fail(FRAQ_EINVAL, "build_sbd_kernel: n_head above 512");
    check_rule_args(g, 2.0 - 2.0 * g, np1);
    check_rule_args(g, 2.0 - 2.0 * g, np2);
    std::memset(k, 0, sizeof(*k));
    k->sbd = 1;
    k->gamma = g;
    k->tau = tau;
    k->n_head = nh;
    k->np1 = np1;
    k->np2 = np2;
    DevBuf<double> out(2 * (size_t)(np1 + np2));
    double* x1 = out.p;
    double* w1 = out.p + np1;
    double* x2 = out.p + 2 * np1;
    double* w2 = out.p + 2 * np1 + np2;
    run_rules(c, {RuleJob{g, 2.0 - 2.0 * g, np1, 2, g, tau, x1, w1, nullptr, nullptr},
                  RuleJob{g, 2.0 - 2.0 * g, np2, 3, g, tau, x2, w2, nullptr, nullptr}});
    FRAQ_CUDA(cudaMemcpy(k->r1, x1, sizeof(double) * np1, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(k->m1, w1, sizeof(double) * np1, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(k->r2, x2, sizeof(double) * np2, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(k->m2, w2, sizeof(double) * np2, cudaMemcpyDeviceToHost));
    fill_head(c, true, g, tau, nh, k);
}

void kernel_error_report_dev(fraq_ctx c, const fraq_kernel_t* k, long n_max, double* eps_h,
                             double* max_eps, long* argmax) {
    if (!k->sbd && n_max < 2) fail(FRAQ_EINVAL, "kernel_error_report: n_max too small");
    if (k->sbd && n_max < k->n_head) fail(FRAQ_EINVAL, "kernel_error_report: n_max below head");
    DevBuf<double> table((size_t)n_max + 1);
    weights_batch(c, k->sbd != 0, {k->gamma}, k->tau, n_max, table.p);
    DevBuf<double> eps((size_t)n_max + 1);
    FRAQ_CUDA(cudaMemsetAsync(eps.p, 0, sizeof(double) * (n_max + 1), c->stream));
    DevBuf<double> mx(1);
    DevBuf<long> am(1);
    DevKernel dk = upload_kernel(c, k);
    const long lo = k->sbd ? k->n_head : 2;
    run_scans(c, {ScanJob{dk.J, dk.m.p, dk.r.p, k->sbd ? 1 : 0, lo, n_max, table.p, eps.p, mx.p,
                          am.p}});
    double m;
    long a;
    FRAQ_CUDA(cudaMemcpy(&m, mx.p, sizeof(double), cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(&a, am.p, sizeof(long), cudaMemcpyDeviceToHost));
    if (eps_h) FRAQ_CUDA(cudaMemcpy(eps_h, eps.p, sizeof(double) * (n_max + 1), cudaMemcpyDeviceToHost));
    *max_eps = m;
    *argmax = m > 0.0 ? a : 0;  // KernelErrorReport defaults (fast_kernel.hpp:49-50)
}

void reconstruct_dev(fraq_ctx c, const fraq_kernel_t* k, long n, const long* idx, double* out_h) {
    if (n <= 0) return;
    DevKernel dk = upload_kernel(c, k);
    DevBuf<long> di((size_t)n);
    FRAQ_CUDA(cudaMemcpyAsync(di.p, idx, sizeof(long) * n, cudaMemcpyHostToDevice, c->stream));
    DevBuf<double> o((size_t)n);
    reconstruct_kernel<<<(unsigned)((n + 127) / 128), 128, 0, c->stream>>>(
        dk.m.p, dk.r.p, dk.J, k->sbd ? 3.0 : 2.0, di.p, n, o.p);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaMemcpyAsync(out_h, o.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

void corr_sequence_dev(fraq_ctx c, const fraq_kernel_t* k, long e_max, double* corr_d) {
    // rec over i = 3 .. e_max + 3 with chains starting at 1 (exponent 0): corr[e] = rec[e + 3]
    DevKernel dk = upload_kernel(c, k);
    run_scans(c, {ScanJob{dk.J, dk.m.p, dk.r.p, 0, 3, e_max + 3, nullptr, corr_d - 3, nullptr,
                          nullptr}});
}

// The same for n kernels in one scan launch (one CTA per kernel): corr of kernel t at
// corr_base + t * stride.  (One launch per kernel cost ~0.9 ms each at N = 16384: 110 ms of setup
// for a 64-instance BDF2 batch.)
void corr_sequence_batch_dev(fraq_ctx c, const fraq_kernel_t* ks, int n, long e_max,
                             double* corr_base, long stride) {
    if (n <= 0) return;
    // every kernel's (m, r) tables packed into one host vector: one allocation, one copy
    std::vector<size_t> off(n);
    size_t total = 0;
    for (int t = 0; t < n; ++t) {
        off[t] = total;
        total += (size_t)(ks[t].np1 + ks[t].np2);
    }
    std::vector<double> m(std::max<size_t>(1, total)), r(std::max<size_t>(1, total));
    for (int t = 0; t < n; ++t) {
        const fraq_kernel_t& k = ks[t];
        double* mt = m.data() + off[t];
        double* rt = r.data() + off[t];
        for (int j = 0; j < k.np1; ++j) mt[j] = k.m1[j], rt[j] = k.r1[j];
        for (int j = 0; j < k.np2; ++j) mt[k.np1 + j] = k.m2[j], rt[k.np1 + j] = k.r2[j];
    }
    DevBuf<double> dm = upload(c, m), dr = upload(c, r);
    std::vector<ScanJob> jobs;
    jobs.reserve(n);
    for (int t = 0; t < n; ++t)
        jobs.push_back(ScanJob{ks[t].np1 + ks[t].np2, dm.p + off[t], dr.p + off[t], 0, 3,
                               e_max + 3, nullptr, corr_base + (size_t)t * stride - 3, nullptr,
                               nullptr});
    run_scans(c, jobs);
}

// Batched auto sizing (fast_kernel.cpp:182-256): point counts 64 (BE) / 41 (SBD) grown by x1.5
// up to max_points until eps <= eps_tol tau^-g; SBD then grows the head by x1.5 while the argmax
// of the error lies below 8 head0.  All exponents of the batch advance together; each round is
// one rule launch + one scan launch over the still-active exponents.
// chosen ladder rung of exponent t -> its table slot (1024 doubles of m and of r)
__global__ void gather_tables_kernel(const double* lm, const double* lr, const long* pick,
                                     double* mt, double* rt) {
    const double* m = lm + (size_t)pick[blockIdx.x] * 1024;
    const double* r = lr + (size_t)pick[blockIdx.x] * 1024;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
        mt[(size_t)blockIdx.x * 1024 + i] = m[i];
        rt[(size_t)blockIdx.x * 1024 + i] = r[i];
    }
}

void build_kernel_auto_dev(fraq_ctx c, bool sbd, int n, const double* gammas, double tau,
                           fraq_budget_t* budgets, fraq_kernel_t* out) {
    if (n <= 0) return;
    long H = 0;
    for (int t = 0; t < n; ++t) {
        check_kernel_gamma(gammas[t]);
        check_weight_args(gammas[t], tau);
        long& h = budgets[t].horizon;
        if (!sbd && h < 4) h = 4;
        if (sbd && h < 8) h = 8;
        H = std::max(H, h);
    }
    // classical tables for every exponent (shared stride L).  They also supply the exact head
    // d_0 .. d_(n_head-1), and the initial SBD head (15 / 17) may exceed a short horizon: the
    // tables reach at least index 17 (heads only grow while below the horizon).
    const long HT = std::max<long>(H, 17);
    const long L = HT + 1;
    DevBuf<double> tables((size_t)n * L);
    {
        std::vector<double> gs(gammas, gammas + n);
        // all horizons padded to the max: the chains are exact prefixes
        weights_batch(c, sbd, gs, tau, HT, tables.p);
    }
    std::vector<int> np(n, sbd ? 41 : 64), done(n, 0), head(n, 0);
    std::vector<double> tol(n);
    for (int t = 0; t < n; ++t) {
        tol[t] = budgets[t].eps_tol * std::pow(tau, -gammas[t]);
        head[t] = sbd ? (gammas[t] <= 0.5 ? 15 : 17) : 2;
    }
    // device node tables per exponent: m[1024], r[1024] (family 1 then family 2)
    DevBuf<double> mt((size_t)n * 1024), rt((size_t)n * 1024);
    DevBuf<double> mx((size_t)n);
    DevBuf<long> am((size_t)n);
    std::vector<double> hmx(n);
    std::vector<long> ham(n);
    auto scan_round = [&](const std::vector<int>& which, const std::vector<long>& from) {
        std::vector<ScanJob> sj;
        for (size_t q = 0; q < which.size(); ++q) {
            const int t = which[q];
            const int J = sbd ? 2 * np[t] : np[t];
            sj.push_back({J, mt.p + (size_t)t * 1024, rt.p + (size_t)t * 1024, sbd ? 1 : 0,
                          from[q], budgets[t].horizon, tables.p + (size_t)t * L, nullptr,
                          mx.p + t, am.p + t});
        }
        run_scans(c, sj);
        FRAQ_CUDA(cudaMemcpy(hmx.data(), mx.p, sizeof(double) * n, cudaMemcpyDeviceToHost));
        FRAQ_CUDA(cudaMemcpy(ham.data(), am.p, sizeof(long) * n, cudaMemcpyDeviceToHost));
    };
    // phase 1: point counts.  The reference grows N_p by x1.5 from 64 (BE) / 41 (SBD) up to the
    // cap, stopping at the first size whose eps meets the tolerance (fast_kernel.cpp:182-235).
    // Every size on that ladder is independent of the others (its own rule, its own scan from
    // the same start index), so all of them are evaluated at once -- one rule launch and one
    // scan launch instead of one round per size -- and the first passing size is picked on the
    // host: the same decisions and tables, bitwise, at the latency of a single round.
    struct Rung {
        int t, p;
    };
    std::vector<Rung> rungs;
    std::vector<int> first_rung(n);
    for (int t = 0; t < n; ++t) {
        first_rung[t] = (int)rungs.size();
        int p = np[t];
        for (;;) {
            p = std::min(p, budgets[t].max_points);
            check_rule_args(gammas[t], sbd ? 2.0 - 2.0 * gammas[t] : 1.0 - gammas[t], p);
            rungs.push_back({t, p});
            if (p >= budgets[t].max_points) break;
            p = p + p / 2;
        }
    }
    const size_t R = rungs.size();
    DevBuf<double> lm(R * 1024), lr(R * 1024), lmx(R);
    DevBuf<long> lam(R);
    {
        std::vector<RuleJob> rj;
        std::vector<ScanJob> sj;
        for (size_t q = 0; q < R; ++q) {
            const int t = rungs[q].t, p = rungs[q].p;
            double* m = lm.p + q * 1024;
            double* r = lr.p + q * 1024;
            if (sbd)
                rj.push_back({gammas[t], 2.0 - 2.0 * gammas[t], p, 4, gammas[t], tau, r, m, r + p,
                              m + p});
            else
                rj.push_back({gammas[t], 1.0 - gammas[t], p, 1, gammas[t], tau, r, m, nullptr,
                              nullptr});
            const long from = sbd ? std::min<long>(budgets[t].horizon, 8L * head[t]) : 2L;
            sj.push_back({sbd ? 2 * p : p, m, r, sbd ? 1 : 0, from, budgets[t].horizon,
                          tables.p + (size_t)t * L, nullptr, lmx.p + q, lam.p + q});
        }
        run_rules(c, rj);
        run_scans(c, sj);
    }
    std::vector<double> rmx(R);
    FRAQ_CUDA(cudaMemcpy(rmx.data(), lmx.p, sizeof(double) * R, cudaMemcpyDeviceToHost));
    std::vector<long> pick(n);
    for (int t = 0; t < n; ++t) {
        size_t q = first_rung[t];
        while (q + 1 < R && rungs[q + 1].t == t && !(rmx[q] <= tol[t])) ++q;
        pick[t] = (long)q;
        np[t] = rungs[q].p;
        if (!sbd) budgets[t].achieved_eps = rmx[q];
    }
    {
        DevBuf<long> dpick = upload(c, pick);
        gather_tables_kernel<<<n, 256, 0, c->stream>>>(lm.p, lr.p, dpick.p, mt.p, rt.p);
        FRAQ_LAUNCH_CHECK();
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
    }
    if (sbd) {
        // phase 2: head growth on the final node tables
        const std::vector<int> head0 = head;
        std::vector<int> act;
        for (int t = 0; t < n; ++t) act.push_back(t);
        std::vector<long> from;
        for (int t : act) from.push_back(head[t]);
        scan_round(act, from);
        std::vector<int> live;
        for (int t = 0; t < n; ++t) live.push_back(t);
        for (;;) {
            std::vector<int> grow;
            for (int t : live) {
                const double w = hmx[t];
                const long a = ham[t];
                if (w > tol[t] && a < 8L * head0[t] && head[t] < budgets[t].max_head &&
                    head[t] < budgets[t].horizon)
                    grow.push_back(t);
                else
                    budgets[t].achieved_eps = w;
            }
            if (grow.empty()) break;
            std::vector<long> fr;
            for (int t : grow) {
                head[t] = (int)std::min<long>(
                    {(long)head[t] + head[t] / 2, (long)budgets[t].max_head, budgets[t].horizon});
                fr.push_back(head[t]);
            }
            scan_round(grow, fr);
            live = grow;
        }
    }
    // download the final tables + heads
    std::vector<double> hm((size_t)n * 1024), hr((size_t)n * 1024);
    FRAQ_CUDA(cudaMemcpy(hm.data(), mt.p, sizeof(double) * n * 1024, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(hr.data(), rt.p, sizeof(double) * n * 1024, cudaMemcpyDeviceToHost));
    // only the heads leave the device (a C5 batch's full tables are 67 MB)
    int HW = 1;
    for (int t = 0; t < n; ++t) HW = std::max(HW, head[t]);
    HW = (int)std::min<long>(HW, L);
    std::vector<double> ht((size_t)n * HW);
    FRAQ_CUDA(cudaMemcpy2D(ht.data(), sizeof(double) * HW, tables.p, sizeof(double) * L,
                           sizeof(double) * HW, n, cudaMemcpyDeviceToHost));
    for (int t = 0; t < n; ++t) {
        fraq_kernel_t* k = out + t;
        std::memset(k, 0, sizeof(*k));
        k->sbd = sbd;
        k->gamma = gammas[t];
        k->tau = tau;
        k->n_head = head[t];
        k->np1 = np[t];
        k->np2 = sbd ? np[t] : 0;
        const double* m = hm.data() + (size_t)t * 1024;
        const double* r = hr.data() + (size_t)t * 1024;
        for (int j = 0; j < np[t]; ++j) {
            k->m1[j] = m[j];
            k->r1[j] = r[j];
        }
        if (sbd)
            for (int j = 0; j < np[t]; ++j) {
                k->m2[j] = m[np[t] + j];
                k->r2[j] = r[np[t] + j];
            }
        // head = classical weights d_0 .. d_{head-1} (prefix of the sizing table)
        for (int i = 0; i < head[t]; ++i) k->head[i] = ht[(size_t)t * HW + i];
    }
}

}  // namespace fraqcu
