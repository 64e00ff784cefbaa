// modal_dmma.cu -- K13: mode-space FFPE stepping on the fp64 tensor cores.
//
// Same scheme as K11 (modal.cu: per mode k a 2x2 system per level with a fast history per field,
// the reference's FastStepper algebra fpfp.cpp:259-349 in the DST eigenbasis), re-blocked the way
// K5d (history_dmma.cu) blocks the standalone history: 8 levels per block, node contractions as
// DMMA GEMMs over a CTA tile of 16 modes x all nodes of both fields.
//
// Per field, with the history state y_j at level n0 - 1 - 8 delta (block start n0):
//
//   s(n0+k) = sum_j r_j^(k+1+8 delta) y_j  +  sum_{m=1}^{k+8 delta+L} c_m G^(n0+k-m)   (G^q, q >= 1)
//
// where c_m are the combined CQ weights of the scheme: the exact head d_m for m < L
// (fpfp.cpp:270-275 BE, 313-324 SBD) and the compressed tail w_(m-L) = sum_j f_j r_j^(m-L) for
// m >= L (the feed G^(n-L) enters y at level n, fast_kernel.cpp:268-289,343-365).  The first term
// is the readout GEMM; the second is a short Toeplitz sum over solved levels.  The state moves
// 8 levels per block: y <- r^8 (.) y + R V (R_ij = f_j r_j^(7-i), V = the block's 8 feeds).
//
// Warp specialisation: nwg GEMM warps (64 nodes of one field each; state in DMMA accumulator
// fragments, as in K5d) and one solver warp.  The GEMM warps run one block ahead of the solver:
// in iteration i they advance the state by block i-1-delta and issue the readout of block i,
// while the solver reduces the partials of block i-1, adds the Toeplitz terms, and solves its 8
// levels in order (one lane per mode, 2x2 Cramer, SBD correction 1/2 c_n G^0 of
// fpfp.cpp:327-334).  delta = 0 when the lag L >= 8 (SBD: every feed of block i-1 is at least
// 9 levels old), delta = 1 otherwise (BE, L = 2): the state then trails the readout by 8 more
// levels, with readout table r^(k+9).  One __syncthreads per block separates the two roles.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <cstdlib>
#include <vector>

#include "history.cuh"

namespace fraqcu {

namespace {

constexpr int K13_CW = 128;  // combined weights c_m, m < 128

struct K13Dev {
    double a, itau;
    const double* corr[2];
    int L[2];
};

struct K13Args {
    const K13Dev* inst;
    const double* tabs;   // per (inst, field): TS doubles
    int TS, Jp, nwf, nwg;
    const double* lam;
    int n_modes, nmb;
    long n_tasks;
    long N;
    int sbd, delta, ring_mask;
    int split;            // GEMM warps take the window rows older than the previous block
    const double* c0;     // [inst][2][modes]
    double* cN;
    int* counter;
};

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct K13TabSrc {
    const double* r;
    const double* f;
    const double* head;
    int J, L;
};

// Tables of one (instance, field), CTA of 256 threads:
//   C  [Jp/8][2][32]  readout B fragments: r_j^(g+1+8 delta), j = 8 nt + 2t + e
//   R  [Jp/8][2][32]  state B fragments: f_j r_j^(7-4h-t), j = 8 nt + g
//   R8 [Jp]           r_j^8 (natural node order == accumulator fragment order)
//   CW [64]           combined weights c_m
__global__ void k13_tables_kernel(const K13TabSrc* src, int Jp, int delta, double* tabs, int TS) {
    const K13TabSrc S = src[blockIdx.x];
    double* T = tabs + (size_t)blockIdx.x * TS;
    auto node_r = [&](int j) { return j < S.J ? S.r[j] : 0.0; };
    auto node_f = [&](int j) { return j < S.J ? S.f[j] : 0.0; };
    for (int idx = threadIdx.x; idx < Jp * 8; idx += blockDim.x) {
        const int nt = idx / 64, e = (idx / 32) % 2, lane = idx % 32, g = lane >> 2, t = lane & 3;
        const int j = 8 * nt + 2 * t + e;
        const double r = node_r(j);
        double p = 1.0;
        for (int q = 0; q < g + 1 + 8 * delta; ++q) p *= r;
        T[idx] = j < S.J ? p : 0.0;
        const int jn = 8 * nt + g, lev = 4 * e + t;
        const double rn = node_r(jn);
        double pn = 1.0;
        for (int q = 0; q < 7 - lev; ++q) pn *= rn;
        T[Jp * 8 + idx] = jn < S.J ? node_f(jn) * pn : 0.0;
    }
    for (int j = threadIdx.x; j < Jp; j += blockDim.x) {
        const double r = node_r(j);
        double p = 1.0;
        for (int q = 0; q < 8; ++q) p *= r;
        T[Jp * 16 + j] = j < S.J ? p : 0.0;
    }
    __shared__ double red[256];
    const int mmax = 7 + 8 * delta + S.L;  // largest m the stepper uses
    for (int m = 0; m < K13_CW; ++m) {
        double v = 0.0;
        if (m >= S.L && m <= mmax) {
            double acc = 0.0;
            for (int j = threadIdx.x; j < S.J; j += blockDim.x) {
                double p = 1.0;
                for (int q = 0; q < m - S.L; ++q) p *= S.r[j];
                acc = fma(S.f[j], p, acc);
            }
            red[threadIdx.x] = acc;
            __syncthreads();
            for (int w = blockDim.x / 2; w > 0; w >>= 1) {
                if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
                __syncthreads();
            }
            v = red[0];
            __syncthreads();
        } else if (m < S.L) {
            v = S.head[m];  // exact head; c_0 = d_0 is the diagonal of the level system
        }
        if (threadIdx.x == 0) T[Jp * 17 + m] = v;
    }
}

// RB: 8-mode row blocks per CTA (modes = 8 RB); NT: 8-node tiles per GEMM warp; MAXT: threads.
// * RB = 2, NT = 8, MAXT = 320 (J <= 192; ~90 KB of shared memory): two CTAs per SM, so one
//   CTA's solver phase overlaps the other's GEMMs and each SM sub-partition runs 4 GEMM warps.
// * RB = 2, NT = 16, MAXT = 384 launched with 192 threads (192 < J <= 256): 2 GEMM warps per
//   field, still two CTAs per SM (2 GEMM warps + 1 solver warp per SM sub-partition).
// * RB = 2, NT = 13 / 16, MAXT = 384 (256 < J <= 416 / <= 512, "wide"): 16 modes x 104 / 128
//   nodes per GEMM warp, 4 GEMM warps per field + 2 solver warps, one CTA per SM (the tables
//   of J = 512 take 140 KB).  16 modes per task double the GEMM work behind each sequential
//   8-level solve; 2 GEMM warps per SM sub-partition beat 3 or 4 narrower ones.  (NT = 8,
//   MAXT = 576, up to 8 GEMM warps per field: FRAQ_K13_NT=8.)
// * RB = 1 (NT = 12..16, MAXT = 320): 8 modes, 4 GEMM warps per field, one CTA per SM (~170
//   registers per thread for the state fragments); kept as the FRAQ_K13_NARROW experiment path.
template <int RB, int NT, int MAXT>
__global__ void __launch_bounds__(MAXT, (MAXT <= 320 && RB == 2) ? 2 : 1) k13_kernel(K13Args A) {
    constexpr int MODES = 8 * RB;
    extern __shared__ double ksm[];
    const int nwg = A.nwg, nwf = A.nwf, TS = A.TS, Jp = A.Jp;
    const int RING = A.ring_mask + 1, mask = A.ring_mask;
    double* tab = ksm;                                   // [2][TS]
    double* part = tab + 2 * TS;                         // [2][nwg][8][MODES]
    double* ring = part + 2 * nwg * 8 * MODES;           // [2][RING][MODES]
    double* sA = ring + 2 * RING * MODES;                // [2][8][MODES]
    double* g0s = sA + 2 * 8 * MODES;                    // [2][MODES]
    __shared__ long s_task;
    __shared__ int s_inst;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    // warps nwg, nwg + 1: solver warps (field 0 / field 1 of the known part); warp nwg also runs
    // the coupled sequential solve
    const bool solver = warp >= nwg;
    const int sf = solver ? warp - nwg : 0;
    const long nb = (A.N + 7) / 8;
    if (tid == 0) s_inst = -1;
    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(A.counter, 1);
        __syncthreads();
        const long task = s_task;
        if (task >= A.n_tasks) return;
        const int inst = (int)(task / A.nmb);
        const int m0 = (int)(task % A.nmb) * MODES;
        if (s_inst != inst) {
            const double* src = A.tabs + (size_t)inst * 2 * TS;
            for (int i = tid; i < 2 * TS; i += blockDim.x) tab[i] = src[i];
        }
        for (int i = tid; i < 2 * RING * MODES; i += blockDim.x) ring[i] = 0.0;
        for (int i = tid; i < 2 * MODES; i += blockDim.x) {
            const int f = i / MODES, d = i % MODES;
            g0s[i] = (m0 + d < A.n_modes) ? A.c0[((long)inst * 2 + f) * A.n_modes + m0 + d] : 0.0;
        }
        __syncthreads();
        if (tid == 0) s_inst = inst;
        const double* cwt[2] = {tab + Jp * 17, tab + TS + Jp * 17};
        if (!solver) {
            // ------------------------------------------------------------ GEMM warps
            const int f = warp / nwf, sl = warp % nwf;
            const int Lf = f ? A.inst[inst].L[1] : A.inst[inst].L[0];
            const double* Tf = tab + f * TS;
            const double* cw = Tf + (size_t)(NT * sl) * 64 + lane;
            const double* rw = Tf + Jp * 8 + (size_t)(NT * sl) * 64 + lane;
            const double* r8p = Tf + Jp * 16 + 8 * NT * sl + 2 * t;
            const double* rg = ring + f * RING * MODES;
            double Y[RB][NT][2];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                for (int q = 0; q < NT; ++q) Y[rb][q][0] = Y[rb][q][1] = 0.0;
            for (long i = 0; i <= nb; ++i) {
                if (i < nb) {
                    const long ib = i - 1 - A.delta;
                    if (ib >= 0) {
                        // ---- state: Y <- r^8 (.) Y + V R, feeds of block ib: G^(nb0 - L + 4h + t)
                        const long nb0 = 1 + 8 * ib;
                        double vf[RB][2];
#pragma unroll
                        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                const long lev = nb0 - Lf + 4 * h + t;
                                vf[rb][h] = lev >= 1 ? rg[(lev & mask) * MODES + 8 * rb + g] : 0.0;
                            }
#pragma unroll
                        for (int q = 0; q < NT; ++q) {
                            const double ra = r8p[q * 8], rbv = r8p[q * 8 + 1];
                            const double b0 = rw[(q * 2) * 32], b1 = rw[(q * 2 + 1) * 32];
#pragma unroll
                            for (int rb = 0; rb < RB; ++rb) {
                                Y[rb][q][0] *= ra;
                                Y[rb][q][1] *= rbv;
                                dmma(Y[rb][q], vf[rb][0], b0);
                                dmma(Y[rb][q], vf[rb][1], b1);
                            }
                        }
                    }
                    // ---- readout of block i: S[mode][k] = sum_j y_j C[j][k]
                    // accumulator chains per row block: one for RB = 2 (no merging DADDs; C5-BE
                    // full horizon +2.7%), four for RB = 1, whose single row block would otherwise
                    // be one chain of 2 NT dependent DMMAs with ~2.5 warps per SMSP (C4 -3.6%)
                    constexpr int NACC = RB == 2 ? 1 : 4;
                    double sacc[RB][NACC][2];
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                        for (int p = 0; p < NACC; ++p) sacc[rb][p][0] = sacc[rb][p][1] = 0.0;
#pragma unroll
                    for (int q = 0; q < NT; ++q)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const double b = cw[(q * 2 + e) * 32];
#pragma unroll
                            for (int rb = 0; rb < RB; ++rb) dmma(sacc[rb][q % NACC], Y[rb][q][e], b);
                        }
                    if (A.split) {
                        // ---- the known part's older rows: the solved levels up to block i - 2
                        // (lags >= 9 from block i's first level) are in the ring by now, so their
                        // Toeplitz terms sum_q c_(n0+k-q) G^q join this readout, shared among the
                        // field's GEMM warps; the solver warp's critical path keeps only the 8
                        // levels of block i - 1.  A[mode g][row t] = G^lev, B[row t][level g] = c
                        const int Lts = 8 * A.delta + Lf, n0 = 1 + 8 * (int)i;
                        const double* CWf = f ? cwt[1] : cwt[0];
#pragma unroll 2
                        for (int j0 = 4 * sl; j0 < Lts - 8; j0 += 4 * nwf) {
                            const int j = j0 + t, lev = n0 - Lts + j;
                            const bool ok = j < Lts - 8;
                            const double bv = ok ? CWf[g + Lts - j] : 0.0;
                            const double* rr = rg + (lev & mask) * MODES + g;
#pragma unroll
                            for (int rb = 0; rb < RB; ++rb)
                                dmma(sacc[rb][0], (ok && lev >= 1) ? rr[8 * rb] : 0.0, bv);
                        }
                    }
                    double* pw = part + ((size_t)(i & 1) * nwg + warp) * 8 * MODES;
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            double v = sacc[rb][0][e];
#pragma unroll
                            for (int p = 1; p < NACC; ++p) v += sacc[rb][p][e];
                            pw[(2 * t + e) * MODES + 8 * rb + g] = v;
                        }
#ifndef K13_SOLVER_REDUCE
                    // the field's nwf partial tiles are summed here, in place into the field's
                    // first tile (each element owned by one thread), so the solver warp's critical
                    // path reads one tile instead of issuing 2 nwf RB DADDs behind the GEMM DMMAs
                    asm volatile("bar.sync %0, %1;" ::"r"(2 + f), "r"(nwf * 32) : "memory");
                    double* pf = part + ((size_t)(i & 1) * nwg + f * nwf) * 8 * MODES;
                    for (int e = sl * 32 + lane; e < 8 * MODES; e += nwf * 32) {
                        double v = pf[e];
                        for (int w = 1; w < nwf; ++w) v += pf[w * 8 * MODES + e];
                        pf[e] = v;
                    }
#endif
                }
                __syncthreads();
            }
        } else {
            // ------------------------------------------------------------ solver warp
            const int d = lane % MODES;
            const bool live = lane < MODES && m0 + d < A.n_modes;
            const K13Dev I = A.inst[inst];
            const double lam = (m0 + d < A.n_modes) ? A.lam[m0 + d] : 0.0;
            const double a = I.a, itau = I.itau, al = a + lam;
            const double h10 = cwt[0][0], h20 = cwt[1][0];  // CW[0] = d_0
            const double lead = A.sbd ? 1.5 : 1.0;
            const double m11 = lead * itau + h10 * al, m12 = -a * h20, m21 = -a * h10,
                         m22 = lead * itau + h20 * al;
            const double idet = 1.0 / (m11 * m22 - m12 * m21);
            const double M11 = m11 * idet, M12 = m12 * idet, M21 = m21 * idet, M22 = m22 * idet;
            // x = M^-1 r with r1 = -al s1 + a s2 + l1, r2 = a s1 - al s2 + l2 (M^-1 = [[M22, -M12],
            // [-M21, M11]]), folded: x = P s + Q l;  l = itau gp (BE), itau (2 gp - gpp / 2) (SBD)
            const double p11 = -fma(al, M22, a * M12), p12 = fma(a, M22, al * M12);
            const double p21 = fma(a, M11, al * M21), p22 = -fma(al, M11, a * M21);
            const double q11 = itau * M22, q12 = -itau * M12, q21 = -itau * M21, q22 = itau * M11;
            // the full-block solve as a two-operation chain: x(k) = z(k) + A1 x(k-1), where
            // A1 = P C(1) + lq Q carries everything level k-1 feeds into level k (lq = 1 BE,
            // 2 SBD), and the older levels enter z off the chain through B_m = P C(m)
            // (m >= 2; SBD: B_2 -= Q/2), C(m) = diag(c1_m, c2_m) the in-block weights
            // (BE in the 192-thread shape -- C3, C5-BE: +6.6% / +3.1%; the SBD chain carries more
            // terms and lost 3% in the wide CTA, and the 96-register shapes would spill)
            constexpr bool kChain2 = MAXT == 192;
            double chA[4], chB[8][4];
            if (kChain2) {
                const double lq = A.sbd ? 2.0 : 1.0;
                const double c11 = cwt[0][1], c21 = cwt[1][1];
                chA[0] = fma(p11, c11, lq * q11);
                chA[1] = fma(p12, c21, lq * q12);
                chA[2] = fma(p21, c11, lq * q21);
                chA[3] = fma(p22, c21, lq * q22);
#pragma unroll
                for (int m = 2; m < 8; ++m) {
                    const double c1m = cwt[0][m], c2m = cwt[1][m];
                    const double sq = (A.sbd && m == 2) ? -0.5 : 0.0;
                    chB[m][0] = fma(sq, q11, p11 * c1m);
                    chB[m][1] = fma(sq, q12, p12 * c2m);
                    chB[m][2] = fma(sq, q21, p21 * c1m);
                    chB[m][3] = fma(sq, q22, p22 * c2m);
                }
            }
            const double g10 = g0s[d], g20 = g0s[MODES + d];
            double gp1 = g10, gp2 = g20, gpp1 = 0.0, gpp2 = 0.0;
            const double* c1 = cwt[0];  // in-block weights c_1..c_7 (shared memory, broadcast)
            const double* c2 = cwt[1];
            // correction prefetch (this warp's field): fragment row k = g (level n0 + g)
            const int Lsf = sf ? I.L[1] : I.L[0];
            const double* corr_f = sf ? I.corr[1] : I.corr[0];
            const double* CWs = sf ? cwt[1] : cwt[0];
            const int Lts = 8 * A.delta + Lsf;
            double cpre = 0.0;
            auto corr_load = [&](int b) {
                const int n = 1 + 8 * b + g;
                cpre = (A.sbd && n >= 2 && n <= A.N && n - 1 >= Lsf) ? corr_f[n - 4] : 0.0;
            };
            corr_load(0);
            for (int i = 0; i <= (int)nb; ++i) {
                if (i >= 1) {
                    const int b = i - 1, n0 = 1 + 8 * b;
                    const int kmax = (int)min(8L, A.N - n0 + 1);
                    const int buf = b & 1;
                    // ---- known part on DMMA: D[k][d] = partial readouts + sum_j c[k+Lt-j] G^(n0-Lt+j)
                    //      (fragment: thread (g, t) holds rows k = g, columns d = 2t, 2t+1 of a tile;
                    //      as A operand it holds A[k = g][j = t], as B operand B[j = t][d = g])
                    double D[RB][2];
#pragma unroll
                    for (int nt = 0; nt < RB; ++nt) {
                        const double* pb = part + ((size_t)buf * nwg + sf * nwf) * 8 * MODES +
                                           g * MODES + 8 * nt + 2 * t;
#ifdef K13_SOLVER_REDUCE
                        double s0 = 0.0, s1 = 0.0;
#pragma unroll
                        for (int w = 0; w < 8; ++w)
                            if (w < nwf) {
                                const double2 v = *reinterpret_cast<const double2*>(pb + w * 8 * MODES);
                                s0 += v.x;
                                s1 += v.y;
                            }
                        D[nt][0] = s0;
                        D[nt][1] = s1;
#else
                        const double2 v = *reinterpret_cast<const double2*>(pb);  // summed tile
                        D[nt][0] = v.x;
                        D[nt][1] = v.y;
#endif
                    }
                    // (with A.split only the previous block's 8 levels are left here)
                    for (int j0 = A.split ? Lts - 8 : 0; j0 < Lts; j0 += 4) {
                        const int j = j0 + t, lev = n0 - Lts + j;
                        const bool ok = j < Lts;
                        const double av = ok ? CWs[g + Lts - j] : 0.0;
                        const double* rg = ring + (sf * RING + (lev & mask)) * MODES + g;
#pragma unroll
                        for (int nt = 0; nt < RB; ++nt) {
                            const double bv = (ok && lev >= 1) ? rg[8 * nt] : 0.0;
                            dmma(D[nt], av, bv);
                        }
                    }
                    {
                        const int n = n0 + g;
                        const double corr_c =
                            (A.sbd && n >= 2) ? 0.5 * ((n - 1 < Lsf) ? CWs[n - 1] : cpre) : 0.0;
#pragma unroll
                        for (int nt = 0; nt < RB; ++nt) {
                            const double* g0f = g0s + sf * MODES + 8 * nt + 2 * t;
                            *reinterpret_cast<double2*>(sA + (sf * 8 + g) * MODES + 8 * nt + 2 * t) =
                                A.sbd ? make_double2(fma(corr_c, g0f[0], D[nt][0]),
                                                     fma(corr_c, g0f[1], D[nt][1]))
                                      : make_double2(D[nt][0], D[nt][1]);
                        }
                    }
                    if (b + 1 < nb) corr_load(b + 1);  // latency hidden by the solve + barrier
                    asm volatile("bar.sync 1, 64;" ::: "memory");  // both fields' known parts ready
                    if (sf == 0 && lane < MODES) {
                        double acc1[8], acc2[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            acc1[k] = sA[k * MODES + d];
                            acc2[k] = sA[(8 + k) * MODES + d];
                        }
                        if (kmax == 8 && !(A.sbd && n0 == 1)) {
                            // full block, no predicates: z(k) = P acc(k) (+ the l terms reaching
                            // back into the previous block), then the chain x(k) = z(k) +
                            // A1 x(k-1) -- two dependent fp64 operations per level instead of four
                            // -- with the older levels folded into z(k2 >= k+2) off the chain
                            auto full_block_chain2 = [&](auto sbd_c) {
                                constexpr bool SBD = decltype(sbd_c)::value;
                                double z1[8], z2[8];
#pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    z1[k] = fma(p11, acc1[k], p12 * acc2[k]);
                                    z2[k] = fma(p21, acc1[k], p22 * acc2[k]);
                                }
                                if constexpr (SBD) {
                                    const double t1 = fma(2.0, gp1, -0.5 * gpp1),
                                                 t2 = fma(2.0, gp2, -0.5 * gpp2);
                                    z1[0] = fma(q11, t1, fma(q12, t2, z1[0]));
                                    z2[0] = fma(q21, t1, fma(q22, t2, z2[0]));
                                    z1[1] = fma(-0.5 * q11, gp1, fma(-0.5 * q12, gp2, z1[1]));
                                    z2[1] = fma(-0.5 * q21, gp1, fma(-0.5 * q22, gp2, z2[1]));
                                } else {
                                    z1[0] = fma(q11, gp1, fma(q12, gp2, z1[0]));
                                    z2[0] = fma(q21, gp1, fma(q22, gp2, z2[0]));
                                }
                                double x1 = z1[0], x2 = z2[0];
#pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    if (k > 0) {
                                        const double y1 = fma(chA[0], x1, fma(chA[1], x2, z1[k]));
                                        const double y2 = fma(chA[2], x1, fma(chA[3], x2, z2[k]));
                                        gpp1 = x1;
                                        gpp2 = x2;
                                        x1 = y1;
                                        x2 = y2;
                                    }
                                    ring[((n0 + k) & mask) * MODES + d] = x1;
                                    ring[(RING + ((n0 + k) & mask)) * MODES + d] = x2;
#pragma unroll
                                    for (int k2 = k + 2; k2 < 8; ++k2) {
                                        z1[k2] = fma(chB[k2 - k][0], x1, fma(chB[k2 - k][1], x2, z1[k2]));
                                        z2[k2] = fma(chB[k2 - k][2], x1, fma(chB[k2 - k][3], x2, z2[k2]));
                                    }
                                }
                                gp1 = x1;
                                gp2 = x2;
                            };
                            // full block, no predicates: x = P acc + (l terms of earlier levels),
                            // coefficients folded per task (8 fp64 ops per level for BE, 12 SBD)
                            auto full_block = [&](auto sbd_c) {
                                constexpr bool SBD = decltype(sbd_c)::value;
#pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    double h1, h2;
                                    if constexpr (SBD) {
                                        const double t1 = fma(2.0, gp1, -0.5 * gpp1),
                                                     t2 = fma(2.0, gp2, -0.5 * gpp2);
                                        h1 = fma(q11, t1, q12 * t2);
                                        h2 = fma(q21, t1, q22 * t2);
                                    } else {
                                        h1 = fma(q11, gp1, q12 * gp2);
                                        h2 = fma(q21, gp1, q22 * gp2);
                                    }
                                    const double x1 = fma(p11, acc1[k], fma(p12, acc2[k], h1));
                                    const double x2 = fma(p21, acc1[k], fma(p22, acc2[k], h2));
                                    ring[((n0 + k) & mask) * MODES + d] = x1;
                                    ring[(RING + ((n0 + k) & mask)) * MODES + d] = x2;
#pragma unroll
                                    for (int k2 = k + 1; k2 < 8; ++k2) {
                                        acc1[k2] = fma(c1[k2 - k], x1, acc1[k2]);
                                        acc2[k2] = fma(c2[k2 - k], x2, acc2[k2]);
                                    }
                                    gpp1 = gp1;
                                    gpp2 = gp2;
                                    gp1 = x1;
                                    gp2 = x2;
                                }
                            };
                            if (A.sbd)
                                full_block(std::true_type{});
                            else if constexpr (kChain2)
                                full_block_chain2(std::false_type{});
                            else
                                full_block(std::false_type{});
                        } else {
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            if (k < kmax) {
                                const long n = n0 + k;
                                double x1, x2;
                                if (A.sbd && n == 1) {
                                    // first step: 2/3 - 1/3 system (fpfp.cpp:293-308)
                                    const double f11 = itau + (2.0 / 3.0) * h10 * al,
                                                 f12 = -(2.0 / 3.0) * a * h20;
                                    const double f21 = -(2.0 / 3.0) * a * h10,
                                                 f22 = itau + (2.0 / 3.0) * h20 * al;
                                    const double r1 = g10 * itau - (h10 / 3.0) * al * g10 +
                                                      (a * h20 / 3.0) * g20;
                                    const double r2 = g20 * itau - (h20 / 3.0) * al * g20 +
                                                      (a * h10 / 3.0) * g10;
                                    const double dt = 1.0 / (f11 * f22 - f12 * f21);
                                    x1 = (r1 * f22 - f12 * r2) * dt;
                                    x2 = (f11 * r2 - f21 * r1) * dt;
                                } else {
                                    const double t1 = A.sbd ? fma(2.0, gp1, -0.5 * gpp1) : gp1;
                                    const double t2 = A.sbd ? fma(2.0, gp2, -0.5 * gpp2) : gp2;
                                    x1 = fma(p11, acc1[k], fma(p12, acc2[k], fma(q11, t1, q12 * t2)));
                                    x2 = fma(p21, acc1[k], fma(p22, acc2[k], fma(q21, t1, q22 * t2)));
                                }
                                ring[(n & mask) * MODES + d] = x1;
                                ring[(RING + (n & mask)) * MODES + d] = x2;
#pragma unroll
                                for (int k2 = k + 1; k2 < 8; ++k2) {
                                    acc1[k2] = fma(c1[k2 - k], x1, acc1[k2]);
                                    acc2[k2] = fma(c2[k2 - k], x2, acc2[k2]);
                                }
                                gpp1 = gp1;
                                gpp2 = gp2;
                                gp1 = x1;
                                gp2 = x2;
                            }
                        }
                        }
                    }
                }
                __syncthreads();
            }
            if (live && sf == 0) {
                A.cN[((long)inst * 2 + 0) * A.n_modes + m0 + d] = gp1;
                A.cN[((long)inst * 2 + 1) * A.n_modes + m0 + d] = gp2;
            }
        }
    }
}

size_t k13_smem(int TS, int nwg, int ring, int modes) {
    return sizeof(double) *
           ((size_t)2 * TS + 2 * nwg * 8 * modes + 2 * ring * modes + 2 * 8 * modes + 2 * modes);
}

template <int RB, int NT, int MAXT>
void k13_launch(const K13Args& a, size_t smem, int num_sms, cudaStream_t s) {
    FRAQ_CUDA(cudaFuncSetAttribute(k13_kernel<RB, NT, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    int per_sm = 1;
    const int threads = a.nwg * 32 + 64;
    FRAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k13_kernel<RB, NT, MAXT>, threads, smem));
    const long grid = std::max(1L, std::min(a.n_tasks, (long)std::max(1, per_sm) * num_sms));
    k13_kernel<RB, NT, MAXT><<<(unsigned)grid, threads, smem, s>>>(a);
    FRAQ_LAUNCH_CHECK();
}

}  // namespace

// Can K13 run these kernels?  (J <= 512 per field, lag windows fit the 128-slot ring)
bool k13_supported(int maxJ, int minL, int maxL) {
    if (std::getenv("FRAQ_MODAL_K11")) return false;
    if (maxJ > 512 || maxJ < 1 || minL < 2) return false;
    const int delta = minL >= 8 ? 0 : 1;
    return 8 + 8 * delta + maxL + 8 <= 128 && 7 + 8 * delta + maxL < K13_CW;
}

void k13_prepare(fraq_ctx c, const std::vector<K13Inst>& in, bool sbd, K13Plan& P) {
    const int n_inst = (int)in.size();
    int maxJ = 0, minL = 1 << 30, maxL = 0;
    for (const K13Inst& I : in)
        for (int f = 0; f < 2; ++f) {
            maxJ = std::max(maxJ, I.J[f]);
            minL = std::min(minL, I.L[f]);
            maxL = std::max(maxL, I.L[f]);
        }
    P.n_inst = n_inst;
    P.sbd = sbd;
    P.delta = minL >= 8 ? 0 : 1;
    // 16 modes x 64 nodes per GEMM warp (J <= 256: two CTAs per SM; J <= 512: the wide CTA with
    // up to 16 GEMM warps).  Experiment path: 8 modes x 8 NT nodes per GEMM warp with the
    // narrowest NT in {12, 13, 14, 16} that covers J in 4 warps (C4: 408 nodes -> NT = 13)
    const char* narrow = std::getenv("FRAQ_K13_NARROW");  // experiment switch: RB = 1 for J > 256
    P.RB = (maxJ <= 256 || !(narrow && *narrow)) ? 2 : 1;
    if (const char* rb1 = std::getenv("FRAQ_K13_RB1"); rb1 && *rb1 && maxJ <= 256)
        P.RB = 1;  // experiment switch: 8-mode tasks for J <= 256
    P.NT = 8;
    // J > 256: four GEMM warps per field of 104 nodes (J <= 416; C4: 408 -> 416) or 128 nodes
    // (J <= 512; C5-BDF2: 512), 10 warps, ~168 registers.  Measured against 64 / 72 / 88-node
    // warps (8 / 6 / 6 per field): C4 K13 loop 1406 (64) -> 1269 (72) -> 1171 ms (104);
    // C5-shaped BDF2 1.112e10 (64) -> 1.144e10 (88) -> 1.234e10 DOF-steps/s (128).  Fewer GEMM
    // warps per SM sub-partition (2 instead of 4) hold the same DMMA work.
    if (P.RB == 2 && maxJ > 256) P.NT = maxJ <= 416 ? 13 : 16;
    // J in (192, 256] (C3, C5-BE): 2 GEMM warps per field of 128 nodes, 6 warps per CTA, two
    // CTAs per SM (168 registers x 192 threads x 2 fit): C5-shaped BE 2.360e10 -> 2.499e10
    if (P.RB == 2 && maxJ > 192 && maxJ <= 256) P.NT = 16;
    // the same 2-GEMM-warps-per-field shape with narrower warps for node counts between 128 and
    // 192 (what the head fold of modal.cu leaves of a 256-node BE kernel: ~162 at M = 40)
    if (P.RB == 2 && maxJ > 128 && maxJ <= 192 && !std::getenv("FRAQ_K13_NOMID"))
        P.NT = maxJ <= 144 ? 9 : maxJ <= 160 ? 10 : maxJ <= 176 ? 11 : 12;
    // and 4 GEMM warps per field of 96 nodes for 256 < J <= 384 (a folded 512-node SBD kernel:
    // 357 at M = 24)
    if (P.RB == 2 && maxJ > 256 && maxJ <= 384 && !std::getenv("FRAQ_K13_NOMID")) P.NT = 12;
    if (const char* ent = std::getenv("FRAQ_K13_NT")) {  // experiment override: 8, 13 or 16
        const int nt = std::atoi(ent);
        if (P.RB == 2 && (nt == 8 || (nt == 13 && maxJ <= 416) || nt == 16 ||
                          (nt >= 9 && nt <= 12 && 2 * 8 * nt >= maxJ) ||
                          (nt == 12 && maxJ <= 384)))
            P.NT = nt;
    }
    if (P.RB == 1) {
        P.NT = 16;
        for (int cand : {12, 13, 14})
            if (4 * 8 * cand >= maxJ) {
                P.NT = cand;
                break;
            }
    }
    const int nodes_w = 8 * P.NT;
    P.nwf = (maxJ + nodes_w - 1) / nodes_w;
    P.Jp = nodes_w * P.nwf;
    P.nwg = 2 * P.nwf;
    P.TS = 17 * P.Jp + K13_CW;
    const int span = 8 + 8 * P.delta + maxL + 8;
    P.ring = span <= 32 ? 32 : span <= 64 ? 64 : 128;
    std::vector<K13TabSrc> src(2 * n_inst);
    std::vector<K13Dev> dv(n_inst);
    for (int i = 0; i < n_inst; ++i) {
        for (int f = 0; f < 2; ++f)
            src[2 * i + f] = {in[i].r[f], in[i].f[f], in[i].head[f], in[i].J[f], in[i].L[f]};
        dv[i].a = in[i].a;
        dv[i].itau = 1.0 / in[i].tau;
        for (int f = 0; f < 2; ++f) {
            dv[i].corr[f] = in[i].corr[f];
            dv[i].L[f] = in[i].L[f];
        }
    }
    DevBuf<K13TabSrc> dsrc(src.size());
    P.inst.alloc(sizeof(K13Dev) * dv.size());
    P.tabs.alloc((size_t)2 * n_inst * P.TS);
    P.counter.alloc(1);
    FRAQ_CUDA(cudaMemcpyAsync(dsrc.p, src.data(), sizeof(K13TabSrc) * src.size(),
                              cudaMemcpyHostToDevice, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(P.inst.p, dv.data(), sizeof(K13Dev) * dv.size(),
                              cudaMemcpyHostToDevice, c->stream));
    k13_tables_kernel<<<2 * n_inst, 256, 0, c->stream>>>(dsrc.p, P.Jp, P.delta, P.tabs.p, P.TS);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

void k13_exec(fraq_ctx c, K13Plan& P, const double* lam, int n_modes, long N, const double* c0,
              double* cN) {
    const int modes = 8 * P.RB;
    K13Args A{};
    A.inst = reinterpret_cast<const K13Dev*>(P.inst.p);
    A.tabs = P.tabs.p;
    A.TS = P.TS;
    A.Jp = P.Jp;
    A.nwf = P.nwf;
    A.nwg = P.nwg;
    A.lam = lam;
    A.n_modes = n_modes;
    A.nmb = (n_modes + modes - 1) / modes;
    A.n_tasks = (long)A.nmb * P.n_inst;
    A.N = N;
    A.sbd = P.sbd ? 1 : 0;
    A.delta = P.delta;
    A.ring_mask = P.ring - 1;
    A.split = std::getenv("FRAQ_K13_NOSPLIT") ? 0 : 1;
    A.c0 = c0;
    A.cN = cN;
    A.counter = P.counter.p;
    FRAQ_CUDA(cudaMemsetAsync(P.counter.p, 0, sizeof(int), c->stream));
    const size_t smem = k13_smem(P.TS, P.nwg, P.ring, modes);
    if (P.RB == 2 && P.NT == 13)
        k13_launch<2, 13, 384>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 12 && P.nwg > 4)
        k13_launch<2, 12, 384>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 12)
        k13_launch<2, 12, 192>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 11)
        k13_launch<2, 11, 192>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 10)
        k13_launch<2, 10, 192>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 9)
        k13_launch<2, 9, 192>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 16 && P.nwg <= 4)  // J <= 256: two CTAs per SM
        k13_launch<2, 16, 192>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.NT == 16)
        k13_launch<2, 16, 384>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.nwg <= 4 && !std::getenv("FRAQ_K13_NOMID"))
        // J <= 128 (what the head fold leaves of most kernels): the 192-thread, 168-register
        // shape (the 96-register instance below spills with the window rows on the GEMM warps)
        k13_launch<2, 8, 192>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2 && P.nwg <= 8)
        k13_launch<2, 8, 320>(A, smem, c->num_sms, c->stream);
    else if (P.RB == 2)
        k13_launch<2, 8, 576>(A, smem, c->num_sms, c->stream);
    else if (P.NT == 12)
        k13_launch<1, 12, 320>(A, smem, c->num_sms, c->stream);
    else if (P.NT == 13)
        k13_launch<1, 13, 320>(A, smem, c->num_sms, c->stream);
    else if (P.NT == 14)
        k13_launch<1, 14, 320>(A, smem, c->num_sms, c->stream);
    else
        k13_launch<1, 16, 320>(A, smem, c->num_sms, c->stream);
}

}  // namespace fraqcu
