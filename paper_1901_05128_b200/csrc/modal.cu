// modal.cu -- mode-space (DST-diagonalised) fast FFPE stepping, 1D and 2D.
//
// With homogeneous Dirichlet data the five-/three-point Laplacian is diagonalised by the type-I
// discrete sine transform, and every operation of FastStepper (fpfp.cpp:259-349) is linear and
// DOF-wise, so the scheme decouples exactly into independent modes: per mode k (eigenvalue
// lambda_k, block_solver.cpp:21-24; 2D: lambda_k + lambda_l) a scalar 2x2 system per level with
// its own fast history for both fields.  This is the reference's own mode-space oracle
// (test_fpfp.cpp:21-180, acceptance crit 5) with the fast histories of fast_kernel.cpp in place of
// the direct sums.  It removes the per-level grid-wide block solve: every mode runs all N levels
// independently.
//
// K11 modal_kernel: one warp per mode; lane l holds node slice l of both fields (z = y / f in
// registers).  Levels are processed in passes of P (P <= lag L: all feeds G^(n-L) of a pass are
// known at its start): one node sweep updates the state for the P levels and accumulates
// P x 2 partial readouts, plus the distributed old part of the exact head window; a warp
// reduce-scatter produces the sums; then the P levels are solved in order (2x2 Cramer, the new part
// of the head window, SBD correction), redundantly in every lane -- no barriers at all.
// K12 dst_kernel: S = sin((k+1)(j+1) pi/(M+1)) applied as a DMMA GEMM (sine generated from an
// integer-indexed table), forward (x 2/(M+1)) and inverse.
#include <cuda_runtime.h>

#include <cstdio>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "history.cuh"

namespace fraqcu {

namespace {

constexpr int MD_CAP = 64;  // max lag (ring of solved levels per mode)

struct ModalField {          // per instance x field
    const double* r;         // node ratios (J)
    const double* f;         // feed coefficients (J)
    const double* head;      // d_0 .. d_{L-1}
    const double* corr;      // SBD correction sequence corr[e] (e = n-4), nullable
    int J, L;
};

struct ModalInst {
    double a, tau;
    ModalField fld[2];
};

struct ModalArgs {
    const ModalInst* inst;
    const double* lam;       // eigenvalue per mode (per instance row: lam[m] shared)
    int n_modes;             // modes per instance
    int n_inst;
    long N;
    int sbd;
    const double* c0;        // initial coefficients [inst][field][mode]
    double* cN;              // final coefficients  [inst][field][mode]
};

// per-warp dynamic shared memory: ring [MD_CAP][2], and (CS) node coefficients [2][2][NPL*32]
template <int NPL, int P, bool CS>
__global__ void __launch_bounds__(128) modal_kernel(ModalArgs A) {
    extern __shared__ double msm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long gw = (long)blockIdx.x * 4 + warp;
    if (gw >= (long)A.n_modes * A.n_inst) return;
    const int inst = (int)(gw / A.n_modes), mode = (int)(gw % A.n_modes);
    const ModalInst I = A.inst[inst];
    constexpr int per_warp = MD_CAP * 2 + (CS ? 4 * NPL * 32 : 0);
    double* wsm = msm + (size_t)warp * per_warp;
    double(*ring)[2] = reinterpret_cast<double(*)[2]>(wsm);
    double* csm = wsm + MD_CAP * 2;  // [field][r|f][NPL*32]
    const double lam = A.lam[mode];
    const double a = I.a, tau = I.tau;
    // coefficients and state: lane holds nodes j = lane + 32 p of each field
    double rr[2][CS ? 1 : NPL], ff[2][CS ? 1 : NPL], z[2][NPL];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
            const int j = lane + 32 * p;
            const bool ok = j < I.fld[f].J;
            const double rv = ok ? I.fld[f].r[j] : 0.0, fv = ok ? I.fld[f].f[j] : 0.0;
            if (CS) {
                csm[(f * 2 + 0) * NPL * 32 + j] = rv;
                csm[(f * 2 + 1) * NPL * 32 + j] = fv;
            } else {
                rr[f][CS ? 0 : p] = rv;
                ff[f][CS ? 0 : p] = fv;
            }
            z[f][p] = 0.0;
        }
    __syncwarp();
    const int L0 = I.fld[0].L, L1 = I.fld[1].L;
    const int Lmin = min(L0, L1);
    const double d10 = I.fld[0].head[0], d20 = I.fld[1].head[0];
    const double g10 = A.c0[((long)inst * 2 + 0) * A.n_modes + mode];
    const double g20 = A.c0[((long)inst * 2 + 1) * A.n_modes + mode];
    // ring[n % CAP] = G^n (both fields); G^0 kept separately for the SBD correction
    if (lane == 0) {
        ring[0][0] = g10;
        ring[0][1] = g20;
    }
    __syncwarp();
    const double al = a + lam;
    // main system (lead 1 for BE, 1.5 for SBD) -- Cramer like the reference's oracle
    const double lead = A.sbd ? 1.5 : 1.0;
    const double m11 = lead / tau + d10 * al, m12 = -a * d20, m21 = -a * d10,
                 m22 = lead / tau + d20 * al;
    const double det = m11 * m22 - m12 * m21;
    double gprev1 = g10, gprev2 = g20, gpp1 = 0.0, gpp2 = 0.0;  // G^{n-1}, G^{n-2}
    long n = 1;
    if (A.sbd) {
        // first step: 2/3 - 1/3 system (fpfp.cpp:293-308), no history contribution
        const double f11 = 1.0 / tau + (2.0 / 3.0) * d10 * al, f12 = -(2.0 / 3.0) * a * d20;
        const double f21 = -(2.0 / 3.0) * a * d10, f22 = 1.0 / tau + (2.0 / 3.0) * d20 * al;
        const double r1 = g10 / tau - (d10 / 3.0) * al * g10 + (a * d20 / 3.0) * g20;
        const double r2 = g20 / tau - (d20 / 3.0) * al * g20 + (a * d10 / 3.0) * g10;
        const double dt = f11 * f22 - f12 * f21;
        const double x1 = (r1 * f22 - f12 * r2) / dt, x2 = (f11 * r2 - f21 * r1) / dt;
        if (lane == 0) {
            ring[1][0] = x1;
            ring[1][1] = x2;
        }
        __syncwarp();
        gpp1 = gprev1;
        gpp2 = gprev2;
        gprev1 = x1;
        gprev2 = x2;
        // level 1 advanced the (zero) accumulators without a feed: nothing to do
        n = 2;
    }
    while (n <= A.N) {
        const int pcount = (int)min((long)P, A.N - n + 1);
        // ---- node sweep for levels n .. n + pcount - 1 (feeds G^(n+k-L), lo = 1)
        double part[P][2];
#pragma unroll
        for (int k = 0; k < P; ++k) part[k][0] = part[k][1] = 0.0;
#pragma unroll
        for (int f = 0; f < 2; ++f) {
            const int L = f ? L1 : L0;
            double v[P];
#pragma unroll
            for (int k = 0; k < P; ++k) {
                const long src = n + k - L;
                v[k] = (k < pcount && src >= 1) ? ring[src % MD_CAP][f] : 0.0;
            }
#pragma unroll
            for (int p = 0; p < NPL; ++p) {
                const double rp = CS ? csm[(f * 2 + 0) * NPL * 32 + lane + 32 * p] : rr[f][CS ? 0 : p];
                const double fp = CS ? csm[(f * 2 + 1) * NPL * 32 + lane + 32 * p] : ff[f][CS ? 0 : p];
                double zz = z[f][p];
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    if (k < pcount) {
                        zz = fma(rp, zz, v[k]);
                        part[k][f] = fma(fp, zz, part[k][f]);
                    }
                }
                z[f][p] = zz;
            }
            // old part of the exact head window: taps i > k (levels solved before this pass);
            // lane handles taps i = lane + 1 (+32)
            const double* hd = I.fld[f].head;
            for (int i = lane + 1; i < L; i += 32) {
                const double h = hd[i];
#pragma unroll
                for (int k = 0; k < P; ++k) {
                    const long src = n + k - i;
                    // BE: only d_1 G^{n-1} for n >= 2 (fpfp.cpp:270-275); SBD: i <= n - 1
                    if (k < pcount && i > k && src >= (A.sbd ? 1 : 1) &&
                        (A.sbd || i == 1))
                        part[k][f] = fma(h, ring[src % MD_CAP][f], part[k][f]);
                }
            }
        }
        // ---- warp all-reduce of the 2P partials (butterfly)
#pragma unroll
        for (int k = 0; k < P; ++k)
#pragma unroll
            for (int f = 0; f < 2; ++f) {
                double s = part[k][f];
#pragma unroll
                for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                part[k][f] = s;
            }
        // ---- sequential solves of the pass
#pragma unroll
        for (int k = 0; k < P; ++k) {
            if (k < pcount) {
                const long nn = n + k;
                double s1 = part[k][0], s2 = part[k][1];
                // new part of the head window: taps i = 1..k (levels solved in this pass)
                for (int i = 1; i <= k; ++i) {
                    const long src = nn - i;
                    if (A.sbd) {
                        if (i < L0 && src >= 1) s1 = fma(I.fld[0].head[i], ring[src % MD_CAP][0], s1);
                        if (i < L1 && src >= 1) s2 = fma(I.fld[1].head[i], ring[src % MD_CAP][1], s2);
                    } else if (i == 1 && src >= 1) {
                        s1 = fma(I.fld[0].head[1], ring[src % MD_CAP][0], s1);
                        s2 = fma(I.fld[1].head[1], ring[src % MD_CAP][1], s2);
                    }
                }
                double r1, r2;
                if (A.sbd) {
                    // (1/2) d_{n-1} G^0 (exact head inside, reconstructed beyond: fpfp.cpp:327-334)
                    const double c1 = (nn - 1 < L0) ? I.fld[0].head[nn - 1] : I.fld[0].corr[nn - 4];
                    const double c2 = (nn - 1 < L1) ? I.fld[1].head[nn - 1] : I.fld[1].corr[nn - 4];
                    s1 = fma(0.5 * c1, g10, s1);
                    s2 = fma(0.5 * c2, g20, s2);
                    r1 = (2.0 * gprev1 - 0.5 * gpp1) / tau - al * s1 + a * s2;
                    r2 = (2.0 * gprev2 - 0.5 * gpp2) / tau - al * s2 + a * s1;
                } else {
                    r1 = gprev1 / tau - al * s1 + a * s2;
                    r2 = gprev2 / tau - al * s2 + a * s1;
                }
                const double x1 = (r1 * m22 - m12 * r2) / det;
                const double x2 = (m11 * r2 - m21 * r1) / det;
                if (lane == 0) {
                    ring[nn % MD_CAP][0] = x1;
                    ring[nn % MD_CAP][1] = x2;
                }
                __syncwarp();
                gpp1 = gprev1;
                gpp2 = gprev2;
                gprev1 = x1;
                gprev2 = x2;
            }
        }
        n += pcount;
    }
    (void)Lmin;
    if (lane == 0) {
        A.cN[((long)inst * 2 + 0) * A.n_modes + mode] = gprev1;
        A.cN[((long)inst * 2 + 1) * A.n_modes + mode] = gprev2;
    }
}

// ------------------------------------------------------------------------------ K12 DST on DMMA
// Out[k][c] = scale * sum_j sin((k+1)(j+1) pi / (M+1)) In[j][c]  (In: M x C row-major, ldc = C)
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

constexpr int ST_M = 64, ST_N = 64, ST_K = 16;

// CTA tile 64 (k) x 64 (c), 4 warps of 32 x 32, K tile 16.  The next K tile's operands (8 sine
// gathers + 8 input loads per thread) are fetched into registers while the tensor pipe works on
// the current one, and land in shared memory behind a single barrier per K tile.
__global__ void __launch_bounds__(128) dst_kernel(const double* __restrict__ sintab, int M,
                                                  const double* __restrict__ In, long ldi,
                                                  long C, double* Out, long ldo, double scale) {
    __shared__ double sA[2][ST_M][ST_K + 1];
    __shared__ double sB[2][ST_K][ST_N + 1];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long k0 = (long)blockIdx.y * ST_M, c0 = (long)blockIdx.x * ST_N;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
    const int g = lane >> 2, t = lane & 3;
    const long period = 2L * (M + 1);
    const unsigned pmask = (period & (period - 1)) == 0 ? (unsigned)period - 1u : 0u;
    const bool small = M < 46340;  // (k+1)(j+1) fits 32 bits
    constexpr int PA = ST_M * ST_K / 128, PB = ST_K * ST_N / 128;  // 8 + 8 per thread
    double ra[PA], rb[PB];
    auto fetch = [&](long j0) {
#pragma unroll
        for (int q = 0; q < PA; ++q) {
            const int idx = tid + 128 * q, r = idx / ST_K, cc = idx % ST_K;
            const long k = k0 + r, j = j0 + cc;
            const long kj = (k + 1) * (j + 1);
            const long ix = small ? (long)(pmask ? ((unsigned)kj & pmask)
                                                 : (unsigned)kj % (unsigned)period)
                                  : kj % period;
            ra[q] = (k < M && j < M) ? __ldg(sintab + ix) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int idx = tid + 128 * q, r = idx / ST_N, cc = idx % ST_N;
            const long j = j0 + r, c = c0 + cc;
            rb[q] = (j < M && c < C) ? __ldg(In + j * ldi + c) : 0.0;
        }
    };
    auto put = [&](int buf) {
#pragma unroll
        for (int q = 0; q < PA; ++q) {
            const int idx = tid + 128 * q;
            sA[buf][idx / ST_K][idx % ST_K] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int idx = tid + 128 * q;
            sB[buf][idx / ST_N][idx % ST_N] = rb[q];
        }
    };
    double acc[4][4][2];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    fetch(0);
    put(0);
    __syncthreads();
    int buf = 0;
    for (long j0 = 0; j0 < M; j0 += ST_K) {
        const bool more = j0 + ST_K < M;
        if (more) fetch(j0 + ST_K);  // in flight during this tile's DMMAs
#pragma unroll
        for (int kk = 0; kk < ST_K; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) af[x] = sA[buf][wm + 8 * x + g][kk + t];
#pragma unroll
            for (int y = 0; y < 4; ++y) bf[y] = sB[buf][kk + t][wn + 8 * y + g];
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
                for (int y = 0; y < 4; ++y) dmma884(acc[x][y], af[x], bf[y]);
        }
        if (more) put(buf ^ 1);  // the other buffer: last read one tile ago, behind a barrier
        __syncthreads();
        buf ^= 1;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long k = k0 + wm + 8 * x + g, c = c0 + wn + 8 * y + 2 * t + e;
                if (k < M && c < C) Out[k * ldo + c] = scale * acc[x][y][e];
            }
}

__global__ void sintab_kernel(double* tab, int M) {
    const long period = 2L * (M + 1);
    const double pi = 3.14159265358979323846;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < period;
         i += (long)gridDim.x * blockDim.x)
        tab[i] = sin(pi * (double)i / (double)(M + 1));
}

// K12s: the same transform for few columns (C <= CT; the 1D instances' two fields): a GEMV with
// the sine gathered from a shared-memory copy of the table.  CTA = 32 outputs (lane = output k) x
// 8 warps splitting the sum over j; the x row is a warp-uniform broadcast load.  The DMMA tile
// kernel above would spend a 64-column tile on 2 columns and run a 4095-long k chain in 64 CTAs
// (0.7 ms per C3 transform, 18% of the C3 run); this one is latency-light (128 CTAs, M/8 terms
// per thread).
template <int CT>
__global__ void __launch_bounds__(256) dst_skinny_kernel(const double* __restrict__ sintab, int M,
                                                         const double* __restrict__ In, long ldi,
                                                         int C, double* Out, long ldo,
                                                         double scale) {
    extern __shared__ double smem[];
    const int period = 2 * (M + 1);
    double* tab = smem;                   // period values
    double* part = smem + period;         // [8][32][CT]
    for (int i = threadIdx.x; i < period; i += 256) tab[i] = sintab[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int k = blockIdx.x * 32 + lane;
    const int kk = k < M ? k + 1 : 0;
    const int per = (M + 7) / 8, j0 = warp * per, j1 = min(M, j0 + per);
    double acc[CT];
#pragma unroll
    for (int c = 0; c < CT; ++c) acc[c] = 0.0;
    // idx = (k+1)(j+1) mod period, advanced by k+1 per j
    int idx = (int)(((long)kk * (j0 + 1)) % period);
#pragma unroll 4
    for (int j = j0; j < j1; ++j) {
        const double sv = tab[idx];
        const double* x = In + (long)j * ldi;
#pragma unroll
        for (int c = 0; c < CT; ++c)
            if (c < C) acc[c] = fma(sv, __ldg(x + c), acc[c]);
        idx += kk;
        if (idx >= period) idx -= period;
    }
#pragma unroll
    for (int c = 0; c < CT; ++c) part[(warp * 32 + lane) * CT + c] = acc[c];
    __syncthreads();
    if (warp == 0 && k < M) {
#pragma unroll
        for (int c = 0; c < CT; ++c) {
            if (c >= C) break;
            double v = 0.0;
            for (int w = 0; w < 8; ++w) v += part[(w * 32 + lane) * CT + c];
            Out[(long)k * ldo + c] = scale * v;
        }
    }
}

__global__ void transpose_kernel(const double* in, long rows, long cols, double* out) {
    __shared__ double tile[32][33];
    const long bx = (long)blockIdx.x * 32, by = (long)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long r = by + i, c = bx + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const long r = bx + i, c = by + threadIdx.x;
        if (r < cols && c < rows) out[r * rows + c] = tile[threadIdx.x][i];
    }
}

template <int NPL, int P, bool CS>
void launch_modal_t(const ModalArgs& a, cudaStream_t s) {
    const long warps = (long)a.n_modes * a.n_inst;
    const size_t smem = sizeof(double) * 4 * (MD_CAP * 2 + (CS ? 4 * NPL * 32 : 0));
    if (smem > 48 * 1024)
        FRAQ_CUDA(cudaFuncSetAttribute(modal_kernel<NPL, P, CS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    modal_kernel<NPL, P, CS><<<(unsigned)((warps + 3) / 4), 128, smem, s>>>(a);
}

void launch_modal(int npl, int P, const ModalArgs& a, cudaStream_t s) {
    if (P == 8) {
        if (npl <= 4) launch_modal_t<4, 8, false>(a, s);
        else if (npl <= 8) launch_modal_t<8, 8, false>(a, s);
        else launch_modal_t<16, 8, true>(a, s);
    } else {
        if (npl <= 4) launch_modal_t<4, 2, false>(a, s);
        else if (npl <= 8) launch_modal_t<8, 2, false>(a, s);
        else launch_modal_t<16, 2, true>(a, s);
    }
    FRAQ_LAUNCH_CHECK();
}

}  // namespace

struct ModalPlan {
    bool use_k13 = false;
    K13Plan k13;
    DevBuf<double> fold;    // K13: node tables with the fast-decaying nodes folded into the head
    int fold_levels = 0;
    DevBuf<ModalInst> dmi;  // K11 instance records
    int n_inst = 0, npl = 0, P = 2;
    bool sbd = false;
};

struct Dst2D {
    int M = 0;
    const double* tab = nullptr;
    DevBuf<double> A, B;
    void init(fraq_ctx c, int m);
    void apply(fraq_ctx c, int n_fields, const double* in, double* out, bool inverse);
};

// Apply the DST along the mode axis: Out (M x C) = scale * S In (M x C).
void dst_apply(fraq_ctx c, int M, const double* sintab, const double* In, long C, double* Out,
               double scale) {
    const size_t skinny_smem = sizeof(double) * (2 * (M + 1) + 8 * 32 * 8);
    if (C <= 8 && skinny_smem <= 227 * 1024) {
        const unsigned grid = (unsigned)((M + 31) / 32);
        if (C <= 2) {
            const size_t sm = sizeof(double) * (2 * (M + 1) + 8 * 32 * 2);
            FRAQ_CUDA(cudaFuncSetAttribute(dst_skinny_kernel<2>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            dst_skinny_kernel<2><<<grid, 256, sm, c->stream>>>(sintab, M, In, C, (int)C, Out, C,
                                                               scale);
        } else {
            FRAQ_CUDA(cudaFuncSetAttribute(dst_skinny_kernel<8>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)skinny_smem));
            dst_skinny_kernel<8><<<grid, 256, skinny_smem, c->stream>>>(sintab, M, In, C, (int)C,
                                                                       Out, C, scale);
        }
        FRAQ_LAUNCH_CHECK();
        return;
    }
    dim3 grid((unsigned)((C + ST_N - 1) / ST_N), (unsigned)((M + ST_M - 1) / ST_M));
    dst_kernel<<<grid, 128, 0, c->stream>>>(sintab, M, In, C, C, Out, C, scale);
    FRAQ_LAUNCH_CHECK();
}

void transpose_dev(fraq_ctx c, const double* in, long rows, long cols, double* out) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    transpose_kernel<<<grid, dim3(32, 8), 0, c->stream>>>(in, rows, cols, out);
    FRAQ_LAUNCH_CHECK();
}

// the context's sine table for grid size M (built on the context's stream on first use)
const double* ctx_sintab(fraq_ctx c, int M) {
    if (c->sintab_m != M || !c->sintab.p) {
        c->sintab.alloc((size_t)2 * (M + 1));
        sintab_kernel<<<64, 256, 0, c->stream>>>(c->sintab.p, M);
        FRAQ_LAUNCH_CHECK();
        c->sintab_m = M;
    }
    return c->sintab.p;
}

// Mode-space stepping of n_inst instances with per-instance kernels (device tables already in
// HistDevice hd: group 2i = field 1, 2i+1 = field 2 of instance i).  c0 / cN: [inst][2][modes].
// modal_plan does the setup (K13 fragment tables, or the K11 instance records); modal_exec
// launches the stepping only.
void modal_plan(fraq_ctx c, const HistDevice& hd, const std::vector<double>& a,
                const std::vector<double>& tau, const double* corr,
                const std::vector<long>& corr_off, int n_inst, bool sbd, ModalPlan& P) {
    std::vector<ModalInst> mi(n_inst);
    int maxJ = 0, minL = 1 << 30, maxL = 0;
    for (int i = 0; i < n_inst; ++i) {
        mi[i].a = a[i];
        mi[i].tau = tau[i];
        for (int f = 0; f < 2; ++f) {
            const GroupDev& G = hd.groups_h[2 * i + f];
            ModalField& F = mi[i].fld[f];
            F.r = hd.cr.p + G.co_off;
            F.f = hd.cf.p + G.co_off;
            F.head = hd.head.p + G.hd_off;
            F.corr = (sbd && corr) ? corr + corr_off[2 * i + f] : nullptr;
            F.J = G.J;
            F.L = G.L;
            maxJ = std::max(maxJ, G.J);
            minL = std::min(minL, G.L);
            maxL = std::max(maxL, G.L);
            if (G.L > MD_CAP - 8) fail(FRAQ_EINVAL, "modal run: head window longer than 56 levels");
        }
    }
    P.n_inst = n_inst;
    P.sbd = sbd;
    P.use_k13 = k13_supported(maxJ, minL, maxL);
    if (P.use_k13) {
        // The fast-decaying nodes folded into the exact head (the rewrite behind K5e,
        // history_fir.cu): a node with |r_j|^M <= 2^-70 contributes only to the lags
        // L <= m < L + M, so the kernel (head d_0..d_(L-1); nodes (r_j, f_j) fed at lag L) equals,
        // to below rounding, the kernel with the head c_0..c_(L+M-1) (c_m = sum_j f_j r_j^(m-L)
        // over ALL nodes for m >= L) and only the slow nodes, fed at lag L + M with f_j r_j^M.
        // K13 then carries a fraction of the nodes through its GEMMs (BE, 256 nodes at
        // tau = 1/16384: 162 left at M = 40) against a longer Toeplitz window in the solver warps.
        // M: the largest multiple of 8 that keeps the head within `lcap` levels.
        // (head caps swept on B200 with the window rows split between GEMM and solver warps,
        // profiles/r02/k13_split2.sh: 80 levels best for C3 / C5-BE / C5-BDF2, 72 for C4 by 1.4%)
        int lcap = 80;
        if (const char* e = std::getenv("FRAQ_K13_LCAP")) lcap = std::atoi(e);  // experiment
        int M = std::max(0, (lcap - maxL) / 8 * 8);
        if (const char* e = std::getenv("FRAQ_K13_FOLD")) M = std::max(0, std::min(M, std::atoi(e) / 8 * 8));
        std::vector<double> ft;            // per group: r'[JL], f'[JL], head'[L + M]
        std::vector<size_t> off(2 * n_inst);
        std::vector<int> JLv(2 * n_inst), Lv(2 * n_inst);
        const long double thr = std::pow(2.0L, -70.0L);
        for (int g2 = 0; g2 < 2 * n_inst && M > 0; ++g2) {
            const GroupDev& G = hd.groups_h[g2];
            const double* r = hd.cr_h.data() + G.co_off;
            const double* f = hd.cf_h.data() + G.co_off;
            const fraq_kernel_t& K = hd.kernels[g2];
            std::vector<long double> rM(G.J);
            std::vector<int> lng;
            long double tail = 0.0L;
            for (int j = 0; j < G.J; ++j) {
                long double a = std::fabs((long double)r[j]), pw = 1.0L;
                for (int q = 0; q < M; ++q) pw *= a;
                rM[j] = pw;
                if (pw > thr)
                    lng.push_back(j);
                else
                    tail += std::fabs((long double)f[j]) * pw / (1.0L - a);
            }
            // (what the fold drops must stay far below rounding of the newest head weight)
            if (!(tail <= std::pow(2.0L, -60.0L) * std::fabs((long double)K.head[0]))) {
                M = 0;
                break;
            }
            off[g2] = ft.size();
            JLv[g2] = (int)lng.size();
            Lv[g2] = G.L + M;
            for (int j : lng) ft.push_back(r[j]);
            for (int j : lng) {
                long double v = (long double)f[j];
                for (int q = 0; q < M; ++q) v *= (long double)r[j];
                ft.push_back((double)v);
            }
            std::vector<long double> cm(M, 0.0L);
            for (int j = 0; j < G.J; ++j) {
                long double pw = (long double)f[j];
                for (int m = 0; m < M; ++m, pw *= (long double)r[j]) cm[m] += pw;
            }
            for (int i = 0; i < G.L; ++i) ft.push_back(i < K.n_head ? K.head[i] : 0.0);
            for (int m = 0; m < M; ++m) ft.push_back((double)cm[m]);
            if (lng.empty()) {  // (K13 wants at least one node per field)
                M = 0;
                break;
            }
        }
        int fJ = 0, fminL = 1 << 30, fmaxL = 0;
        for (int g2 = 0; g2 < 2 * n_inst && M > 0; ++g2) {
            fJ = std::max(fJ, JLv[g2]);
            fminL = std::min(fminL, Lv[g2]);
            fmaxL = std::max(fmaxL, Lv[g2]);
        }
        if (M > 0 && !k13_supported(fJ, fminL, fmaxL)) M = 0;
        P.fold_levels = M;
        if (M > 0) {
            P.fold.alloc(ft.size());
            FRAQ_CUDA(cudaMemcpyAsync(P.fold.p, ft.data(), ft.size() * sizeof(double),
                                      cudaMemcpyHostToDevice, c->stream));
            FRAQ_CUDA(cudaStreamSynchronize(c->stream));  // (ft goes out of scope)
        }
        std::vector<K13Inst> ki(n_inst);
        for (int i = 0; i < n_inst; ++i) {
            ki[i].a = a[i];
            ki[i].tau = tau[i];
            for (int f = 0; f < 2; ++f) {
                ki[i].corr[f] = mi[i].fld[f].corr;
                if (M > 0) {
                    const int g2 = 2 * i + f;
                    const double* base = P.fold.p + off[g2];
                    ki[i].r[f] = base;
                    ki[i].f[f] = base + JLv[g2];
                    ki[i].head[f] = base + 2 * JLv[g2];
                    ki[i].J[f] = JLv[g2];
                    ki[i].L[f] = Lv[g2];
                    continue;
                }
                ki[i].r[f] = mi[i].fld[f].r;
                ki[i].f[f] = mi[i].fld[f].f;
                ki[i].head[f] = mi[i].fld[f].head;
                ki[i].J[f] = mi[i].fld[f].J;
                ki[i].L[f] = mi[i].fld[f].L;
            }
        }
        k13_prepare(c, ki, sbd, P.k13);
        return;
    }
    P.npl = (maxJ + 31) / 32;
    if (P.npl > 16) fail(FRAQ_EINVAL, "modal run: more than 512 nodes per field");
    P.P = minL >= 8 ? 8 : 2;
    P.dmi.alloc(n_inst);
    FRAQ_CUDA(cudaMemcpyAsync(P.dmi.p, mi.data(), sizeof(ModalInst) * n_inst,
                              cudaMemcpyHostToDevice, c->stream));
}

void modal_exec(fraq_ctx c, ModalPlan& P, const double* lam, int n_modes, long N,
                const double* c0, double* cN) {
    if (P.use_k13) {
        k13_exec(c, P.k13, lam, n_modes, N, c0, cN);
        return;
    }
    ModalArgs A{P.dmi.p, lam, n_modes, P.n_inst, N, P.sbd ? 1 : 0, c0, cN};
    launch_modal(P.npl, P.P, A, c->stream);
}

// 2D DST workspace: forward out[f][ky][kx] = (2/(M+1))^2 sum S[ky][y] S[kx][x] in[f][y][x],
// inverse out[f][y][x] = sum S[y][ky] S[x][kx] in[f][ky][kx] (S symmetric); each as two DMMA GEMMs
// along y and x with transposes in between.
void Dst2D::init(fraq_ctx c, int m) {
    M = m;
    tab = ctx_sintab(c, M);
    A.alloc((size_t)M * M);
    B.alloc((size_t)M * M);
}

void Dst2D::apply(fraq_ctx c, int n_fields, const double* in, double* out, bool inverse) {
    const long MM = (long)M * M;
    const double sc = inverse ? 1.0 : 2.0 / (M + 1);
    for (int f = 0; f < n_fields; ++f) {
        dst_apply(c, M, tab, in + f * MM, M, A.p, sc);   // A[k][x]
        transpose_dev(c, A.p, M, M, B.p);                  // B[x][k]
        dst_apply(c, M, tab, B.p, M, A.p, sc);           // A[l][k]
        transpose_dev(c, A.p, M, M, out + f * MM);         // out[k][l]
    }
}

}  // namespace fraqcu

// ============================================================================ host drivers
namespace fraqcu {

void build_ffpe_kernels(fraq_ctx c, const std::vector<double>& gam, double tau, long N, bool sbd,
                        const fraq_kconf_t& kc, std::vector<fraq_kernel_t>& ks,
                        std::vector<double>& eps);

namespace {

double now_s2() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Shared tail of the 1D and 2D drivers: kernel tables, SBD correction sequences, stepping.
// coef0 / coefN: [inst][2][modes] (device).
struct ModalSetup {
    std::vector<fraq_kernel_t> ks;
    std::vector<double> eps;
    HistDevice hd;
    DevBuf<double> corr;
    std::vector<long> corr_off;
    ModalPlan plan;
};

// gam: 2 exponents per instance (field 1, field 2); a: coupling per instance.
void modal_prepare(fraq_ctx c, ModalSetup& S, const std::vector<double>& gam,
                   const std::vector<double>& a, double tau, long N, bool sbd,
                   const fraq_kconf_t& kc) {
    const bool trace = std::getenv("FRAQ_SETUP_TRACE") != nullptr;  // diagnostics
    double tt = now_s2();
    auto lap = [&](const char* what) {
        if (!trace) return;
        cudaStreamSynchronize(c->stream);
        const double t = now_s2();
        std::fprintf(stderr, "setup %-14s %8.2f ms\n", what, 1e3 * (t - tt));
        tt = t;
    };
    build_ffpe_kernels(c, gam, tau, N, sbd, kc, S.ks, S.eps);
    lap("kernels");
    const int ng = (int)gam.size();
    std::vector<const fraq_kernel_t*> kp(ng);
    std::vector<long> dims(ng, 1);
    for (int t = 0; t < ng; ++t) kp[t] = &S.ks[t];
    S.hd.build(c, ng, kp.data(), dims.data(), /*tables_only=*/true);
    lap("hist tables");
    S.corr_off.assign(ng, 0);
    if (sbd) {
        S.corr.alloc((size_t)ng * (N + 1));
        corr_sequence_batch_dev(c, S.ks.data(), ng, N, S.corr.p, N + 1);
        for (int t = 0; t < ng; ++t) S.corr_off[t] = (long)t * (N + 1);
    }
    const int n_inst = ng / 2;
    lap("corr");
    modal_plan(c, S.hd, a, std::vector<double>(n_inst, tau), sbd ? S.corr.p : nullptr, S.corr_off,
               n_inst, sbd, S.plan);
    lap("plan");
}

struct EventTimer {
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    cudaStream_t s;
    explicit EventTimer(cudaStream_t st) : s(st) {
        FRAQ_CUDA(cudaEventCreate(&e0));
        FRAQ_CUDA(cudaEventCreate(&e1));
        FRAQ_CUDA(cudaEventRecord(e0, s));
    }
    double stop() {
        FRAQ_CUDA(cudaEventRecord(e1, s));
        FRAQ_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        FRAQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        return ms * 1e-3;
    }
    ~EventTimer() {
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
};

void fill_info(fraq_run_info_t* info, const ModalSetup& S, double loop_s, double setup_s) {
    if (!info) return;
    info->loop_seconds = loop_s;
    info->setup_seconds = setup_s;
    info->kernel_eps1 = S.eps[0];
    info->kernel_eps2 = S.eps[1];
    info->np[0] = S.ks[0].np1;
    info->np[1] = S.ks[0].np2;
    info->np[2] = S.ks[1].np1;
    info->np[3] = S.ks[1].np2;
    info->n_head[0] = S.ks[0].n_head;
    info->n_head[1] = S.ks[1].n_head;
}

}  // namespace

// 1D: n_inst instances sharing grid_m, n_steps, t_final.
void ffpe_run_modal(fraq_ctx c, const fraq_spec_t* specs, int n_inst, bool sbd,
                    const fraq_kconf_t& kc, double* g1_out, double* g2_out,
                    fraq_run_info_t* info) {
    const double t0 = now_s2();
    const int M = specs[0].grid_m;
    const long N = specs[0].n_steps;
    const double tau = specs[0].t_final / double(N);
    const double h = specs[0].length / double(M + 1);
    const long C = 2L * n_inst;
    // initial data, instance-major rows (row c = 2 inst + field): contiguous host writes; the
    // device transposes to the [grid point][c] layout the DST takes
    std::vector<double> G0((size_t)M * C);
    std::vector<double> gam(C), av(n_inst), tv(n_inst, tau);
    for (int i = 0; i < n_inst; ++i) {
        const fraq_spec_t& s = specs[i];
        double* r1 = G0.data() + (size_t)(2 * i) * M;
        double* r2 = r1 + M;
        if (s.initial == FRAQ_CUSTOM) {
            std::memcpy(r1, s.custom_g1, sizeof(double) * M);
            std::memcpy(r2, s.custom_g2, sizeof(double) * M);
        } else {
            for (int j = 0; j < M; ++j) {
                const double x = (j + 1) * h;
                if (s.initial == FRAQ_POLY_SIN) {
                    r1[j] = x * (1.0 - x);
                    r2[j] = std::sin(x);
                } else {
                    r1[j] = x > 0.5 ? 1.0 - x : 0.0;
                    r2[j] = x < 0.5 ? x : 0.0;
                }
            }
        }
        gam[2 * i] = 1.0 - s.alpha1;
        gam[2 * i + 1] = 1.0 - s.alpha2;
        av[i] = s.coupling_a;
    }
    if (std::getenv("FRAQ_SETUP_TRACE"))
        std::fprintf(stderr, "setup %-14s %8.2f ms\n", "initial data", 1e3 * (now_s2() - t0));
    ModalSetup S;
    modal_prepare(c, S, gam, av, tau, N, sbd, kc);
    // eigenvalues lambda_k = (4/h^2) sin^2(k pi h / (2 L)) (block_solver.cpp:21-24)
    std::vector<double> lam(M);
    for (int k = 0; k < M; ++k) {
        const double sk = std::sin((k + 1) * 3.14159265358979323846 * h / (2.0 * specs[0].length));
        lam[k] = 4.0 / (h * h) * sk * sk;
    }
    DevBuf<double> dlam(M), dG((size_t)M * C), dW((size_t)M * C), dc0((size_t)M * C),
        dcN((size_t)M * C);
    FRAQ_CUDA(cudaMemcpyAsync(dlam.p, lam.data(), sizeof(double) * M, cudaMemcpyHostToDevice, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(dW.p, G0.data(), sizeof(double) * G0.size(), cudaMemcpyHostToDevice,
                              c->stream));
    transpose_dev(c, dW.p, C, M, dG.p);  // [c][grid point] -> [grid point][c]
    const double* tab = ctx_sintab(c, M);
    const double t1 = now_s2();
    if (std::getenv("FRAQ_SETUP_TRACE"))
        std::fprintf(stderr, "setup %-14s %8.2f ms\n", "total", 1e3 * (t1 - t0));
    EventTimer timer(c->stream);
    // forward DST (projection, 2/(M+1) S G): rows = modes; then [C][M] for the stepper
    dst_apply(c, M, tab, dG.p, C, dW.p, 2.0 / (M + 1));
    transpose_dev(c, dW.p, M, C, dc0.p);
    modal_exec(c, S.plan, dlam.p, M, N, dc0.p, dcN.p);
    // inverse: g = S^T c (S symmetric)
    transpose_dev(c, dcN.p, C, M, dW.p);
    dst_apply(c, M, tab, dW.p, C, dG.p, 1.0);
    const double loop_s = timer.stop();
    // back to instance-major rows on the device, then contiguous copies out
    transpose_dev(c, dG.p, M, C, dW.p);
    FRAQ_CUDA(cudaMemcpy(G0.data(), dW.p, sizeof(double) * G0.size(), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n_inst; ++i) {
        std::memcpy(g1_out + (size_t)i * M, G0.data() + (size_t)(2 * i) * M, sizeof(double) * M);
        std::memcpy(g2_out + (size_t)i * M, G0.data() + (size_t)(2 * i + 1) * M,
                    sizeof(double) * M);
    }
    fill_info(info, S, loop_s, t1 - t0);
}

std::vector<double> eig2d(int M) {
    const double h = 1.0 / double(M + 1);
    std::vector<double> lam1(M), lam2((size_t)M * M);
    for (int k = 0; k < M; ++k) {
        const double sk = std::sin((k + 1) * 3.14159265358979323846 * h / 2.0);
        lam1[k] = 4.0 / (h * h) * sk * sk;
    }
    for (int ky = 0; ky < M; ++ky)
        for (int kx = 0; kx < M; ++kx) lam2[(size_t)ky * M + kx] = lam1[ky] + lam1[kx];
    return lam2;
}

fraq_kconf_t kconf_or_default(const fraq_kconf_t* kc_in) {
    fraq_kconf_t kc;
    if (kc_in)
        kc = *kc_in;
    else
        fraq_kconf_default(&kc);
    return kc;
}

// 2D: modes (k, l) with lambda_k + lambda_l; forward transform c = (2/(M+1))^2 S G S, inverse
// g = S c S (S symmetric); data row-major (x fastest): G[y][x], coefficients c[ky][kx].
void ffpe_run_2d(fraq_ctx c, double alpha1, double alpha2, double a, int M, double t_final,
                 long N, int scheme, const fraq_kconf_t* kc_in, const double* g1_0,
                 const double* g2_0, double* g1, double* g2, fraq_run_info_t* info) {
    if (M < 1 || N < 1) fail(FRAQ_EINVAL, "run_2d: grid_m and n_steps must be >= 1");
    if (scheme != FRAQ_FASTBE && scheme != FRAQ_FASTSBD)
        fail(FRAQ_EINVAL, "run_2d: scheme must be FastBE or FastSBD");
    const fraq_kconf_t kc = kconf_or_default(kc_in);
    const bool sbd = scheme == FRAQ_FASTSBD;
    const double t0 = now_s2();
    const double tau = t_final / double(N);
    const long MM = (long)M * M;
    ModalSetup S;
    modal_prepare(c, S, {1.0 - alpha1, 1.0 - alpha2}, {a}, tau, N, sbd, kc);
    const std::vector<double> lam2 = eig2d(M);
    DevBuf<double> dlam(MM), dA(2 * MM), dc0(2 * MM), dcN(2 * MM);
    FRAQ_CUDA(cudaMemcpyAsync(dlam.p, lam2.data(), sizeof(double) * MM, cudaMemcpyHostToDevice,
                              c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(dA.p, g1_0, sizeof(double) * MM, cudaMemcpyHostToDevice, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(dA.p + MM, g2_0, sizeof(double) * MM, cudaMemcpyHostToDevice,
                              c->stream));
    Dst2D dst;
    dst.init(c, M);
    const double t1 = now_s2();
    EventTimer timer(c->stream);
    dst.apply(c, 2, dA.p, dc0.p, false);
    modal_exec(c, S.plan, dlam.p, (int)MM, N, dc0.p, dcN.p);
    dst.apply(c, 2, dcN.p, dA.p, true);
    const double loop_s = timer.stop();
    FRAQ_CUDA(cudaMemcpy(g1, dA.p, sizeof(double) * MM, cudaMemcpyDeviceToHost));
    FRAQ_CUDA(cudaMemcpy(g2, dA.p + MM, sizeof(double) * MM, cudaMemcpyDeviceToHost));
    fill_info(info, S, loop_s, t1 - t0);
}

// 2D DST of n_fields grid_m x grid_m arrays (forward: coefficients [ky][kx] from G[y][x] with the
// (2/(M+1))^2 projection scale; inverse: synthesis).  mem: FRAQ_HOST or FRAQ_DEVICE for in / out.
void dst2d(fraq_ctx c, int M, int n_fields, const double* in, double* out, bool inverse, int mem) {
    if (M < 1 || n_fields < 1) fail(FRAQ_EINVAL, "dst2d: grid_m and n_fields must be >= 1");
    const long n = (long)n_fields * M * M;
    Dst2D dst;
    dst.init(c, M);
    if (mem == FRAQ_DEVICE) {
        dst.apply(c, n_fields, in, out, inverse);
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    DevBuf<double> di(n), dout(n);
    FRAQ_CUDA(cudaMemcpyAsync(di.p, in, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    dst.apply(c, n_fields, di.p, dout.p, inverse);
    FRAQ_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

// 1D DST pass along the leading axis of a grid_m x n_cols array (K12): forward scale 2/(M+1),
// inverse 1.  mem: FRAQ_HOST or FRAQ_DEVICE for in / out.
void dst_cols(fraq_ctx c, int M, long n_cols, const double* in, double* out, bool inverse,
              int mem) {
    if (M < 1 || n_cols < 0) fail(FRAQ_EINVAL, "dst_cols: grid_m must be >= 1, n_cols >= 0");
    if (n_cols == 0) return;
    const long n = (long)M * n_cols;
    const double sc = inverse ? 1.0 : 2.0 / (M + 1);
    const double* tab = ctx_sintab(c, M);
    if (mem == FRAQ_DEVICE) {
        dst_apply(c, M, tab, in, n_cols, out, sc);
        FRAQ_CUDA(cudaStreamSynchronize(c->stream));
        return;
    }
    DevBuf<double> di(n), dout(n);
    FRAQ_CUDA(cudaMemcpyAsync(di.p, in, sizeof(double) * n, cudaMemcpyHostToDevice, c->stream));
    dst_apply(c, M, tab, di.p, n_cols, dout.p, sc);
    FRAQ_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * n, cudaMemcpyDeviceToHost, c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

// One instance stepped over a caller-chosen set of modes (eigenvalues lam[n_modes]); c0 / cN are
// [2][n_modes] (field-major).  The building block of the mode-sharded 2D driver: every rank
// steps its slab of modes.  mem: FRAQ_HOST or FRAQ_DEVICE for lam / c0 / cN.
void modal_run_modes(fraq_ctx c, double alpha1, double alpha2, double a, double t_final, long N,
                     int scheme, const fraq_kconf_t* kc_in, long n_modes, const double* lam,
                     const double* c0, double* cN, int mem, fraq_run_info_t* info) {
    if (N < 1 || n_modes < 1 || n_modes > (1L << 30))
        fail(FRAQ_EINVAL, "modal_run: n_steps and n_modes must be >= 1");
    if (scheme != FRAQ_FASTBE && scheme != FRAQ_FASTSBD)
        fail(FRAQ_EINVAL, "modal_run: scheme must be FastBE or FastSBD");
    const fraq_kconf_t kc = kconf_or_default(kc_in);
    const bool sbd = scheme == FRAQ_FASTSBD;
    const double t0 = now_s2();
    const double tau = t_final / double(N);
    ModalSetup S;
    modal_prepare(c, S, {1.0 - alpha1, 1.0 - alpha2}, {a}, tau, N, sbd, kc);
    DevBuf<double> dl, d0, dN;
    const double *pl = lam, *p0 = c0;
    double* pN = cN;
    if (mem != FRAQ_DEVICE) {
        dl.alloc(n_modes);
        d0.alloc(2 * n_modes);
        dN.alloc(2 * n_modes);
        FRAQ_CUDA(cudaMemcpyAsync(dl.p, lam, sizeof(double) * n_modes, cudaMemcpyHostToDevice, c->stream));
        FRAQ_CUDA(cudaMemcpyAsync(d0.p, c0, sizeof(double) * 2 * n_modes, cudaMemcpyHostToDevice, c->stream));
        pl = dl.p;
        p0 = d0.p;
        pN = dN.p;
    }
    const double t1 = now_s2();
    EventTimer timer(c->stream);
    modal_exec(c, S.plan, pl, (int)n_modes, N, p0, pN);
    const double loop_s = timer.stop();
    if (mem != FRAQ_DEVICE) {
        FRAQ_CUDA(cudaMemcpy(cN, dN.p, sizeof(double) * 2 * n_modes, cudaMemcpyDeviceToHost));
    }
    fill_info(info, S, loop_s, t1 - t0);
}

}  // namespace fraqcu
