// history_fir.cu -- K5e: K5d's block GEMMs with the fast-decaying nodes folded into an exact FIR.
//
// The compressed kernels (fast_kernel.cpp:54-124) spread their nodes over decay rates from
// ~1/T to far above 1/tau: in the reference's own auto-sized C2 tables 361 of the 512 ratios
// satisfy r_j^48 < 1e-21.  Such a node forgets everything older than M levels, so its whole
// recurrence y_j(n) = r_j y_j(n-1) + f_j v(n) (fast_kernel.cpp:268-289, 343-365) and readout
// (fast_kernel.cpp:302-308, 378-388) collapse into a Toeplitz sum over the last M feeds,
//
//   sum_{j short} y_j(n) = sum_{m<M} wS_m v(n-m) + O(2^-70),   wS_m = sum_{j short} f_j r_j^m,
//
// which is shift invariant like the exact head window and joins it in ONE combined window over
// the input rows: taps d_i (i < n_head) on X(n-i) and wS_(i-L) on X(n-i), L <= i < L+M (v(n) =
// X(n-L)).  Only the slow ("long") nodes keep K5d's block form
//
//   S(n0+k)   = sum_{j long} r_j^(k+1) y_j(n0-1) + [window rows] H,
//   y_j(n0+7) = r_j^8 y_j(n0-1) + sum_i f_j r_j^(7-i) v_i,
//
// with the long nodes' in-block Toeplitz part added to the same matrix H (KW x 8, built on the
// host in extended precision).  For C2 this is 188 DMMAs per 16 DOFs x 8 levels instead of 528.
//
// K5e covers the steady state only: full 8-level blocks from a level past L + M + 1, inputs of
// the last KW levels available (the history keeps them in an HBM ring, `xh`).  Everything else
// (first levels, ragged tails, unaligned inputs) stays on K5d.  The short nodes' states in HBM
// are not touched by K5e; short_state_kernel rebuilds them from the last M inputs
// (y_j = sum_{m<M} f_j r_j^m v(n-m), the reference's recurrence started M levels back) before
// any other path reads them.
//
// The same split serves the per-level calls (K5f, step_fir_kernel below: push / derivative /
// history_sum in the steady state; K5 records its appended values in `xh`, so a history pushed
// level by level gets there by itself) and, as a kernel-to-kernel rewrite (fold_kernel), the
// physical FFPE stepper's history pass.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "history.cuh"

namespace fraqcu {

namespace {

#ifndef FRAQ_K5E_TC
#define FRAQ_K5E_TC 32
#endif
constexpr int E_TC = FRAQ_K5E_TC;  // levels per staged chunk (16 or 32)
constexpr int E_KW_CAP = 128 - (2 * E_TC - 8);  // widest window the 128-row shared ring holds
constexpr int E_TB = 8;    // levels per block
constexpr int E_NT = 8;    // node tiles per warp at most (64 long nodes)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_tile(const CUtensorMap* map, void* dst, unsigned long long* m,
                                         int col, int row, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(m)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
        "%3}], [%4];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<unsigned long long>(map)), "r"(col), "r"(row), "r"(smem_u32(m))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* m, unsigned parity) {
    unsigned done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, "
            "0, p; }"
            : "=r"(done)
            : "r"(smem_u32(m)), "r"(parity)
            : "memory");
}

struct Run4Args {
    const GroupDev* groups;
    const FirGroup* fg;
    const int2* tasks;  // (group, first DOF of the 16-DOF task)
    int n_tasks;
    int* counter;
    double* state;
    double* ring;
    long A0;            // values appended before the call
    long n_steps;       // multiple of 8
    const double* U;
    long ldu;
    double* D;          // nullable
    long ldd;
    const double* tabs;
    const int* perm;
    const double* xh;   // input history ring: level n at row n & xh_mask
    long ldx;
    int xh_mask;
    int ring_rows;      // shared-memory input ring (power of two >= kw_max + 56)
    int capC, capH;     // shared-memory table capacities (doubles)
    const CUtensorMap* umap;  // (set by the kernel: its __grid_constant__ parameter)
};

// What a warp needs of its CTA's task (everything uniform per warp).
struct TaskCtx {
    double *X, *Cfr, *Rfr, *Hfr, *part;
    unsigned long long* mbar;
    int2 tk;
    int tid, warp, lane, g, t, nwg, mask;
};

// One task for a warp that owns NT long-node tiles (NT is a template parameter: a guarded
// `if (tile < owned)` inside the unrolled loops compiles to predicated DMMAs, and a DMMA whose
// predicate is off still occupies the tensor pipe for its 16 cycles -- measured on B200).
template <int NT>
__device__ __forceinline__ void run_task(const Run4Args& A, const TaskCtx& c, const GroupDev& G,
                                         const FirGroup* F, unsigned& phases) {
    constexpr int NY = NT > 0 ? NT : 1;
    const int tid = c.tid, warp = c.warp, lane = c.lane, g = c.g, t = c.t, nwg = c.nwg,
              mask = c.mask;
    const int2 tk = c.tk;
    double* X = c.X;
    double* part = c.part;
    unsigned long long* mbar = c.mbar;
    const int L = G.L, KW = F->KW, NTW = F->NTW;
    const long ld = G.ld;
    const int kk0 = F->kk0[warp], kk1 = F->kk0[warp + 1];
    // state fragments Y[rb][ntl][e]: DOF tk.y + 2g + rb, long position 8 tile + 2t + e.  (Row g
    // of row block rb is DOF 2g + rb: a lane's two A operands of an input row are then adjacent
    // -- one 128-bit LDS, each 128-byte row one wavefront -- and so are its partial outputs)
    double Y[2][NY][2];
    const int* pm = A.perm + F->perm_off + 8 * (warp * NTW) + 2 * t;
#pragma unroll
    for (int ntl = 0; ntl < NT; ++ntl)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = pm[8 * ntl + e];
#pragma unroll
            for (int rb = 0; rb < 2; ++rb) {
                const int m = tk.y + 2 * g + rb;
                Y[rb][ntl][e] = (j >= 0 && m < G.dim) ? A.state[G.st_off + j * ld + m] : 0.0;
            }
        }
    // input rows of the KW - 8 levels before the call (call-relative level q at ring row
    // q & mask, so they sit at the top of the ring)
    const int pre = KW - E_TB;
    for (int idx = tid; idx < pre * 16; idx += blockDim.x) {
        const int row = idx >> 4, d = idx & 15, q = row - pre;
        double x = 0.0;
        if (tk.y + d < G.dim)
            x = A.xh[(size_t)((A.A0 + q) & A.xh_mask) * A.ldx + G.dof0 + tk.y + d];
        X[(q & mask) * 16 + d] = x;
    }
    // (ring rows written through the generic proxy here are overwritten by TMA later)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0)
        tma_tile(A.umap, X, &mbar[0], (int)(G.dof0 + tk.y), 0, E_TC * 16 * 8);
    double* Db = A.D ? A.D + G.dof0 + tk.y : nullptr;
    const double* cw = c.Cfr + (size_t)(warp * NTW) * 64 + lane;
    const double* rw = c.Rfr + (size_t)(warp * NTW) * 64 + lane;
    const double* r8w = c.Cfr + (size_t)(warp * NTW) * 64 + 28 + t;  // r^8: readout row g = 7
    const double* Hl = c.Hfr + lane;
    int p_row = 0, p_nb = 0, p_buf = 0;
    auto reduce_pair = [&]() {
#ifdef FRAQ_EXP_NOREDUCE  // (timing experiments only: profiles/r02/k5e_variants.sh)
        return;
#endif
        // one item = two adjacent DOFs of one level: 128-bit loads of the warps' partial tiles, a
        // two-level add tree (every DADD waits behind the DMMAs on the shared fp64 pipe, so the
        // chain depth is what costs), one 128-bit store
        for (int o = tid; o < 2 * E_TB * 8; o += blockDim.x) {
            const int slot = o >> 6, k = (o >> 3) & 7, d = 2 * (o & 7);
            if (slot >= p_nb) continue;
            const double* pb = part + ((size_t)(p_buf * 2 + slot) * nwg) * 128 + k * 16 + d;
            double2 s;
            if (nwg == 4) {
                const double2 a0 = *reinterpret_cast<const double2*>(pb);
                const double2 a1 = *reinterpret_cast<const double2*>(pb + 128);
                const double2 a2 = *reinterpret_cast<const double2*>(pb + 256);
                const double2 a3 = *reinterpret_cast<const double2*>(pb + 384);
                s.x = (a0.x + a1.x) + (a2.x + a3.x);
                s.y = (a0.y + a1.y) + (a2.y + a3.y);
            } else {
                double2 s0 = *reinterpret_cast<const double2*>(pb), s1 = make_double2(0.0, 0.0);
                for (int w = 1; w + 1 < nwg; w += 2) {
                    const double2 a = *reinterpret_cast<const double2*>(pb + w * 128);
                    const double2 b = *reinterpret_cast<const double2*>(pb + (w + 1) * 128);
                    s1.x += a.x;
                    s1.y += a.y;
                    s0.x += b.x;
                    s0.y += b.y;
                }
                if (!(nwg & 1)) {
                    const double2 a = *reinterpret_cast<const double2*>(pb + (nwg - 1) * 128);
                    s1.x += a.x;
                    s1.y += a.y;
                }
                s.x = s0.x + s1.x;
                s.y = s0.y + s1.y;
            }
            if (!Db) continue;
            double* dst = Db + (size_t)(p_row + 8 * slot + k) * A.ldd + d;
            if (tk.y + d + 1 < G.dim)
                *reinterpret_cast<double2*>(dst) = s;  // (D 16-byte aligned, ldd even: fir_eligible)
            else if (tk.y + d < G.dim)
                dst[0] = s.x;
        }
    };
    int buf = 0;
    bool pending = false;
    unsigned ck = 0;
    for (long c0l = 0; c0l < A.n_steps; c0l += E_TC, ++ck) {
        const int c0 = (int)c0l;
        const int tmax = (int)min((long)E_TC, A.n_steps - c0l);
        __syncthreads();  // everyone is done with the rows the next tile overwrites
        if (tid == 0 && c0l + E_TC < A.n_steps)
            tma_tile(A.umap, &X[((c0 + E_TC) & mask) * 16], &mbar[(ck + 1) & 1],
                     (int)(G.dof0 + tk.y), c0 + E_TC, E_TC * 16 * 8);
        mbar_wait(&mbar[ck & 1], (phases >> (ck & 1)) & 1u);
        phases ^= 1u << (ck & 1);
        auto do_block = [&](int t0, int slot, bool mid_reduce) {
            const int q0 = c0 + t0;
            double* pw = part + ((size_t)(buf * 2 + slot) * nwg + warp) * 128;
            // ---- readout: long nodes from the block-start state, then this warp's share of
            // the combined window (head taps, short-node FIR, long nodes' local part)
            double sacc[2][2];
#pragma unroll
            for (int rb = 0; rb < 2; ++rb) sacc[rb][0] = sacc[rb][1] = 0.0;
#pragma unroll
            for (int ntl = 0; ntl < NT; ++ntl)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double b = cw[(ntl * 2 + e) * 32];
#pragma unroll
                    for (int rb = 0; rb < 2; ++rb) dmma(sacc[rb], Y[rb][ntl][e], b);
                }
#ifndef FRAQ_EXP_NOFIR
            {
                const int w0 = q0 + E_TB - KW + t;
#pragma unroll 2
                for (int kk = kk0; kk < kk1; ++kk) {
                    const double b = Hl[kk * 32];
                    const double2 a = *reinterpret_cast<const double2*>(
                        X + ((w0 + 4 * kk) & mask) * 16 + 2 * g);
                    dmma(sacc[0], a.x, b);
                    dmma(sacc[1], a.y, b);
                }
            }
#endif
            double vf[2][2];
            if (NT > 0) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const double2 a = *reinterpret_cast<const double2*>(
                        X + ((q0 + 4 * h + t - L) & mask) * 16 + 2 * g);
                    vf[0][h] = a.x;
                    vf[1][h] = a.y;
                }
            }
            if (mid_reduce) reduce_pair();
            // ---- state: Y <- r^8 (.) Y + V R (rescale DMULs first, as in K5d)
#pragma unroll
            for (int ntl = 0; ntl < NT; ++ntl) {
                const double ra = r8w[(ntl * 2) * 32], rbv = r8w[(ntl * 2 + 1) * 32];
#ifndef FRAQ_EXP_NODMUL
#pragma unroll
                for (int rb = 0; rb < 2; ++rb) {
                    Y[rb][ntl][0] *= ra;
                    Y[rb][ntl][1] *= rbv;
                }
#endif
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int ntl = 0; ntl < NT; ++ntl) {
                    const double b = rw[(ntl * 2 + h) * 32];
#pragma unroll
                    for (int rb = 0; rb < 2; ++rb) dmma(Y[rb][ntl], vf[rb][h], b);
                }
            *reinterpret_cast<double2*>(pw + (2 * t) * 16 + 2 * g) =
                make_double2(sacc[0][0], sacc[1][0]);
            *reinterpret_cast<double2*>(pw + (2 * t + 1) * 16 + 2 * g) =
                make_double2(sacc[0][1], sacc[1][1]);
        };
        for (int t0 = 0; t0 < tmax; t0 += 2 * E_TB) {
            const int nblk = t0 + E_TB < tmax ? 2 : 1;
            do_block(t0, 0, pending);  // reduces the previous pair (p_* still describe it)
            if (nblk == 2) do_block(t0 + E_TB, 1, false);
            p_row = c0 + t0;
            p_nb = nblk;
#ifndef FRAQ_EXP_NOSYNC
            __syncthreads();
#endif
            p_buf = buf;
            pending = true;
            buf ^= 1;
        }
    }
    if (pending) reduce_pair();
    // write back the long states and the lag ring
#pragma unroll
    for (int ntl = 0; ntl < NT; ++ntl)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = pm[8 * ntl + e];
#pragma unroll
            for (int rb = 0; rb < 2; ++rb) {
                const int m = tk.y + 2 * g + rb;
                if (j >= 0 && m < G.dim) A.state[G.st_off + j * ld + m] = Y[rb][ntl][e];
            }
        }
    const long A1 = A.A0 + A.n_steps;
    for (int idx = tid; idx < L * 16; idx += blockDim.x) {
        const int row = idx >> 4, d = idx & 15;
        const long k = A1 - L + row;
        if (tk.y + d < G.dim)
            A.ring[G.ring_off + (k % L) * ld + tk.y + d] =
                X[(((int)A.n_steps - L + row) & mask) * 16 + d];
    }
}

// CTA = one 16-DOF task x the long nodes of its group: nwg warps, warp w owns node tiles
// [w NTW, (w+1) NTW) (state in DMMA accumulator fragments, as in K5d) and the k-steps
// [kk0[w], kk0[w+1]) of the combined window.  Two 8-level blocks per CTA barrier; the
// cross-warp reduction of a pair is issued behind the next block's readout DMMAs.  The warps
// of a CTA run different instances of run_task (by owned tile count) and meet at the same
// CTA barriers.
__global__ void __launch_bounds__(256, 2)
    run4_kernel(Run4Args A, const __grid_constant__ CUtensorMap umap) {
    extern __shared__ __align__(128) double esm[];
    TaskCtx c;
    c.X = esm;  // [ring_rows][16]: TMA lands 16-DOF x 32-level boxes in place
    c.mbar = reinterpret_cast<unsigned long long*>(c.X + A.ring_rows * 16);
    c.Cfr = c.X + A.ring_rows * 16 + 2;
    c.Rfr = c.Cfr + A.capC;
    c.Hfr = c.Rfr + A.capC;
    c.part = c.Hfr + A.capH;  // [2 buffers][2 slots][nwg][8 levels][16 DOFs]
    __shared__ int s_task, s_group;
    c.tid = threadIdx.x;
    c.warp = c.tid >> 5;
    c.lane = c.tid & 31;
    c.g = c.lane >> 2;
    c.t = c.lane & 3;
    c.nwg = blockDim.x >> 5;
    c.mask = A.ring_rows - 1;
    A.umap = &umap;
    const int tid = c.tid;
    // completion barriers of the input tiles: initialised once per CTA; a task's chunk k uses
    // mbar[k & 1], and the phase each barrier is in carries over from task to task
    unsigned phases = 0;
    if (tid == 0) {
        s_group = -1;
        mbar_init(&c.mbar[0]);
        mbar_init(&c.mbar[1]);
    }
    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(A.counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= A.n_tasks) return;
        c.tk = A.tasks[task];
        const GroupDev G = A.groups[c.tk.x];
        const FirGroup* F = A.fg + c.tk.x;
        const int TL = F->TL;
        if (s_group != c.tk.x) {  // (uniform) the group's tables
            const double* src = A.tabs + F->tab_off;
            for (int i = tid; i < TL * 64; i += blockDim.x) {
                c.Cfr[i] = src[i];
                c.Rfr[i] = src[TL * 64 + i];
            }
            for (int i = tid; i < F->nkk * 32; i += blockDim.x) c.Hfr[i] = src[TL * 128 + i];
        }
        __syncthreads();
        if (tid == 0) s_group = c.tk.x;
        const int ntw = max(0, min(F->NTW, TL - c.warp * F->NTW));
        switch (ntw) {
            case 0: run_task<0>(A, c, G, F, phases); break;
            case 1: run_task<1>(A, c, G, F, phases); break;
            case 2: run_task<2>(A, c, G, F, phases); break;
            case 3: run_task<3>(A, c, G, F, phases); break;
            case 4: run_task<4>(A, c, G, F, phases); break;
            case 5: run_task<5>(A, c, G, F, phases); break;
            case 6: run_task<6>(A, c, G, F, phases); break;
            case 7: run_task<7>(A, c, G, F, phases); break;
            default: run_task<8>(A, c, G, F, phases); break;
        }
    }
}

// Short-node states from the last M feeds: y_j = sum_{m<M} f_j r_j^m v(n-m), evaluated as the
// reference's recurrence y <- r y + f v started from zero M levels back (what it leaves out is
// below 2^-70 of a feed).  CTA = 128 DOFs of one group x a slice of the short nodes.
__global__ void __launch_bounds__(128)
    short_state_kernel(const GroupDev* groups, const FirGroup* fg, const int* perm,
                       const double* cr, const double* cf, double* state, const double* xh,
                       long ldx, int xh_mask, long A1, int m_max, int slices) {
    extern __shared__ double xs[];  // [M][128]
    const GroupDev G = groups[blockIdx.y];
    const FirGroup F = fg[blockIdx.y];
    const int m0 = blockIdx.x * 128;
    if (m0 >= G.dim || F.n_short == 0) return;
    const int m = m0 + threadIdx.x;
    const bool live = m < G.dim;
    // feeds v(n - i) = X(n - L - i), n = A1 - 1, i = 0 .. M-1
    for (int i = 0; i < F.M; ++i) {
        const long lev = A1 - 1 - G.L - i;
        xs[i * 128 + threadIdx.x] =
            (live && lev >= 0) ? xh[(size_t)(lev & xh_mask) * ldx + G.dof0 + m] : 0.0;
    }
    (void)m_max;
    if (!live) return;
    const int per = (F.n_short + slices - 1) / slices;
    const int s0 = blockIdx.z * per, s1 = min(F.n_short, s0 + per);
    for (int s = s0; s < s1; ++s) {
        const int j = perm[F.short_off + s];
        const double r = cr[G.co_off + j], f = cf[G.co_off + j];
        double y = 0.0;
        for (int i = F.M - 1; i >= 0; --i) y = fma(r, y, f * xs[i * 128 + threadIdx.x]);
        state[G.st_off + (long)j * G.ld + m] = y;
    }
}

size_t run4_smem(const FirPlan& p) {
    return sizeof(double) *
           ((size_t)p.ring_rows * 16 + 2 + 2 * (size_t)p.capC + p.capH + 2 * 2 * (size_t)p.nwg * 128);
}

}  // namespace

// ---------------------------------------------------------------------------------- planning
// Host side, extended precision: which nodes are short, the permutation, the fragment tables.
void build_fir_plan(fraq_ctx c, HistDevice& d) {
    FirPlan& P = d.fir;
    if (P.built) return;
    P.built = true;
    P.ok = false;
    if (std::getenv("FRAQ_NO_K5E")) return;
    const int ng = (int)d.groups_h.size();
    if (ng == 0 || d.max_L > 32 || d.max_J > 512) return;
    int m_force = -1;
    if (const char* e = std::getenv("FRAQ_K5E_M")) m_force = std::atoi(e);  // experiment override
    std::vector<double> tabs;
    std::vector<int> perm;
    P.groups_h.assign(ng, FirGroup{});
    int units_max = 0;
    const long double thr = std::pow(2.0L, -70.0L);
    for (int gi = 0; gi < ng; ++gi) {
        const GroupDev& G = d.groups_h[gi];
        FirGroup& F = P.groups_h[gi];
        const double* r = d.cr_h.data() + G.co_off;
        const double* f = d.cf_h.data() + G.co_off;
        const double* hd = d.kernels[gi].head;
        const int taps = G.sbd ? G.L : 2;
        // candidate FIR lengths: the DMMA count of a block is 4 per long tile and rb, 1 per
        // window k-step and rb; windows up to 72 rows fit the 128-row shared-memory ring
        // |r|^M for M = 8, 16, ..., 96 by repeated squaring-free products (host, once per history)
        std::vector<long double> r8(G.J);
        for (int j = 0; j < G.J; ++j) {
            long double a = std::fabs((long double)r[j]), p = a;
            for (int q = 1; q < 8; ++q) p *= a;
            r8[j] = p;
        }
        auto rpow = [&](int j, int M) {  // M a multiple of 8
            long double p = 1.0L;
            for (int q = 0; q < M / 8; ++q) p *= r8[j];
            return p;
        };
        auto is_short = [&](int j, int M) { return M > 0 && rpow(j, M) <= thr; };
        auto cost = [&](int M) {
            int jl = 0;
            for (int j = 0; j < G.J; ++j) jl += !is_short(j, M);
            const int kw = (G.L + M + 7 + 3) / 4 * 4;
            return 4 * ((jl + 7) / 8) + kw / 4;
        };
        int M = 0, best = cost(0);
        for (int cand = 8; cand <= 96; cand += 8) {
            if ((G.L + cand + 7 + 3) / 4 * 4 > E_KW_CAP && m_force < 0) break;
            const int cc = cost(cand);
            if (cc < best) best = cc, M = cand;
        }
        if (m_force >= 0) M = std::min(96, m_force / 8 * 8);
        // what the FIR leaves out, against the newest head weight (the output scale): refuse
        // the split when it is not far below rounding
        long double tail = 0.0L;
        for (int j = 0; j < G.J; ++j)
            if (is_short(j, M)) {
                const long double a = std::fabs((long double)r[j]);
                tail += std::fabs((long double)f[j]) * rpow(j, M) / (1.0L - a);
            }
        if (!(tail <= std::pow(2.0L, -60.0L) * std::fabs((long double)hd[0]))) M = 0;
        std::vector<int> lng, sht;
        for (int j = 0; j < G.J; ++j) (is_short(j, M) ? sht : lng).push_back(j);
        F.M = M;
        F.JL = (int)lng.size();
        F.TL = (F.JL + 7) / 8;
        F.KW = (G.L + M + 7 + 3) / 4 * 4;
        F.nkk = F.KW / 4;
        F.perm_off = (int)perm.size();
        for (int p = 0; p < F.TL * 8; ++p) perm.push_back(p < F.JL ? lng[p] : -1);
        for (int p = 0; p < 64; ++p) perm.push_back(-1);  // (a warp's unused tile slots read here)
        F.short_off = (int)perm.size();
        F.n_short = (int)sht.size();
        for (int j : sht) perm.push_back(j);
        units_max = std::max(units_max, 4 * F.TL + F.nkk);
        // ---- tables (fragment order as in K5d's frag_tables_kernel)
        F.tab_off = (long)tabs.size();
        auto rp = [&](int p) { return p < F.JL ? (long double)r[lng[p]] : 0.0L; };
        auto fp = [&](int p) { return p < F.JL ? (long double)f[lng[p]] : 0.0L; };
        std::vector<double> C((size_t)F.TL * 64), R((size_t)F.TL * 64), H((size_t)F.nkk * 32, 0.0);
        for (int idx = 0; idx < F.TL * 64; ++idx) {
            const int nt = idx / 64, e = (idx / 32) % 2, lane = idx % 32, g = lane >> 2, t = lane & 3;
            // readout B: row k = t <-> position 8 nt + 2t + e, column n = g <-> level g: r^(g+1)
            const int p = 8 * nt + 2 * t + e;
            C[idx] = p < F.JL ? (double)std::pow(rp(p), (long double)(g + 1)) : 0.0;
            // state B: half h = e, row k = t <-> level 4h + t, column n = g <-> position 8 nt + g
            const int pn = 8 * nt + g, lev = 4 * e + t;
            R[idx] = pn < F.JL ? (double)(fp(pn) * std::pow(rp(pn), (long double)(7 - lev))) : 0.0;
        }
        // combined window: row jj <-> X(n0 + 8 - KW + jj), column k <-> level n0 + k, lag
        // i = k + KW - 8 - jj.  Head taps d_i (i < taps); short FIR wS_(i-L) (L <= i < L+M);
        // the long nodes' in-block part wL_(i-L) on the rows of this block's own feeds
        // (jj >= KW - 8 - L, i.e. v_i' with i' = jj - (KW - 8 - L) <= k)
        std::vector<long double> wS(std::max(1, M), 0.0L), wL(8, 0.0L);
        for (int j : sht) {
            long double p = (long double)f[j];
            for (int m = 0; m < M; ++m, p *= (long double)r[j]) wS[m] += p;
        }
        for (int j : lng) {
            long double p = (long double)f[j];
            for (int m = 0; m < 8; ++m, p *= (long double)r[j]) wL[m] += p;
        }
        for (int kk = 0; kk < F.nkk; ++kk)
            for (int lane = 0; lane < 32; ++lane) {
                const int gg = lane >> 2, tt = lane & 3, jj = 4 * kk + tt, k = gg;
                const int i = k + F.KW - 8 - jj;
                long double v = 0.0L;
                if (i >= 0 && i < taps) v += (long double)hd[i];
                if (i >= G.L && i < G.L + M) v += wS[i - G.L];
                if (jj >= F.KW - 8 - G.L && i >= G.L && i < G.L + 8) v += wL[i - G.L];
                H[(size_t)kk * 32 + lane] = (double)v;
            }
        tabs.insert(tabs.end(), C.begin(), C.end());
        tabs.insert(tabs.end(), R.begin(), R.end());
        tabs.insert(tabs.end(), H.begin(), H.end());
        while (tabs.size() % 4) tabs.push_back(0.0);
        F.ws_off = (long)tabs.size();
        for (int m = 0; m < M; ++m) tabs.push_back((double)wS[m]);
        tabs.push_back(0.0);
    }
    // warps per CTA: ~24 DMMA pairs per warp and block (C2: 4 warps, 3.46e10 DOF-steps/s; 3 warps
    // 3.33e10, 5 warps 3.18e10), every group's tiles must fit
    int nwg = std::max(1, std::min(E_MAXWG, (units_max + 23) / 24));
    if (const char* e = std::getenv("FRAQ_K5E_NWG")) nwg = std::max(1, std::min(E_MAXWG, std::atoi(e)));
    for (const FirGroup& F : P.groups_h) nwg = std::max(nwg, (F.TL + E_NT - 1) / E_NT);
    P.nwg = nwg;
    P.capC = 64;
    P.capH = 32;
    P.kw_max = 0;
    P.min_level = 0;
    for (int gi = 0; gi < ng; ++gi) {
        FirGroup& F = P.groups_h[gi];
        F.NTW = std::max(1, (F.TL + nwg - 1) / nwg);
        // window k-steps to the least loaded warps (4 units per owned tile, 1 per k-step)
        std::vector<int> load(nwg), nf(nwg, 0);
        for (int w = 0; w < nwg; ++w) load[w] = 4 * std::max(0, std::min(F.NTW, F.TL - w * F.NTW));
        for (int kk = 0; kk < F.nkk; ++kk) {
            int w = 0;
            for (int x = 1; x < nwg; ++x)
                if (load[x] < load[w]) w = x;
            ++load[w];
            ++nf[w];
        }
        F.kk0[0] = 0;
        for (int w = 0; w < E_MAXWG; ++w) F.kk0[w + 1] = F.kk0[w] + (w < nwg ? nf[w] : 0);
        P.capC = std::max(P.capC, F.TL * 64);
        P.capH = std::max(P.capH, F.nkk * 32);
        P.kw_max = std::max(P.kw_max, F.KW);
        P.min_level = std::max(P.min_level, d.groups_h[gi].L + F.M + 2);
    }
    if (std::getenv("FRAQ_K5E_DEBUG"))
        for (int gi = 0; gi < ng; ++gi) {
            const FirGroup& F = P.groups_h[gi];
            std::fprintf(stderr, "K5e group %d: J %d L %d M %d long %d (tiles %d) short %d KW %d "
                         "nwg %d NTW %d kk0", gi, d.groups_h[gi].J, d.groups_h[gi].L, F.M, F.JL,
                         F.TL, F.n_short, F.KW, nwg, F.NTW);
            for (int w = 0; w <= nwg; ++w) std::fprintf(stderr, " %d", F.kk0[w]);
            std::fprintf(stderr, "\n");
        }
    P.ring_rows = 128;
    while (P.ring_rows < P.kw_max + 2 * E_TC - 8) P.ring_rows *= 2;
    P.xh_rows = 128;
    while (P.xh_rows < P.kw_max + 8) P.xh_rows *= 2;
    if (run4_smem(P) > 200 * 1024) return;
    P.groups.alloc(ng);
    P.tabs.alloc(std::max<size_t>(1, tabs.size()));
    P.perm.alloc(std::max<size_t>(1, perm.size()));
    FRAQ_CUDA(cudaMemcpyAsync(P.groups.p, P.groups_h.data(), ng * sizeof(FirGroup),
                              cudaMemcpyHostToDevice, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(P.tabs.p, tabs.data(), tabs.size() * sizeof(double),
                              cudaMemcpyHostToDevice, c->stream));
    FRAQ_CUDA(cudaMemcpyAsync(P.perm.p, perm.data(), perm.size() * sizeof(int),
                              cudaMemcpyHostToDevice, c->stream));
    P.xh.alloc((size_t)P.xh_rows * std::max<long>(1, d.total_dim));
    FRAQ_CUDA(cudaMemsetAsync(P.xh.p, 0, P.xh.n * sizeof(double), c->stream));
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));  // (host vectors go out of scope)
    P.xh_valid = 0;
    P.short_stale = false;
    P.ok = true;
}

namespace {
// rows [n0, n0 + cnt) of U -> the input ring (a kernel, not cudaMemcpy2DAsync: device-to-device
// copies go through the copy engines that the host path's H2D / D2H transfers are using)
__global__ void note_rows_kernel(const double* U, long ldu, long A0, long n0, long cnt, long dim,
                                 double* xh, int xh_mask) {
    const long per = (dim + 1) / 2;  // double2 units per row (dim even: K5e's precondition)
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < cnt * per;
         i += (long)gridDim.x * blockDim.x) {
        const long row = i / per, c = 2 * (i % per), n = n0 + row;
        const double* src = U + (n - A0) * ldu + c;
        double* dst = xh + (size_t)(n & xh_mask) * dim + c;
        if (c + 1 < dim && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
            *reinterpret_cast<double2*>(dst) = *reinterpret_cast<const double2*>(src);
        } else {
            dst[0] = src[0];
            if (c + 1 < dim) dst[1] = src[1];
        }
    }
}
}  // namespace

// Appends the call's last input rows to the HBM input ring (row = level & (xh_rows - 1)).
void fir_note_inputs(fraq_ctx c, HistDevice& d, long A0, const double* U, long ldu, long n_steps) {
    FirPlan& P = d.fir;
    if (!P.ok || n_steps <= 0 || d.total_dim == 0) return;
    const long keep = std::min<long>(n_steps, P.kw_max + 8);
    const long dim = d.total_dim;
    const long n = A0 + n_steps - keep;  // first level copied
    const long units = keep * ((dim + 1) / 2);
    const int grid = (int)std::max<long>(1, std::min<long>((units + 255) / 256, 4L * c->num_sms));
    note_rows_kernel<<<grid, 256, 0, c->stream>>>(U, ldu, A0, n, keep, dim, P.xh.p, P.xh_rows - 1);
    FRAQ_LAUNCH_CHECK();
    // (a longer call leaves only its copied rows valid: the older rows belong to other levels)
    P.xh_valid = n_steps > keep ? keep : std::min<long>(P.xh_rows, P.xh_valid + n_steps);
}

// Can [A0, A0 + n_steps) run on K5e?  (steady state, inputs of the last kw_max levels known)
bool fir_eligible(const HistDevice& d, long A0, const double* U, long ldu, long n_steps,
                  const double* D, long ldd) {
    const FirPlan& P = d.fir;
    if (!P.ok || n_steps < 8 || (n_steps & 7) || n_steps >= (1L << 30)) return false;
    if (A0 < P.min_level || A0 < P.kw_max || P.xh_valid < P.kw_max) return false;
    if (reinterpret_cast<uintptr_t>(U) % 16 != 0 || (ldu % 2) != 0 || ldu < 16 ||
        ldu >= (1L << 31))
        return false;
    // (outputs leave as 128-bit stores)
    if (D && (reinterpret_cast<uintptr_t>(D) % 16 != 0 || (ldd % 2) != 0)) return false;
    return true;
}

void launch_run4(fraq_ctx c, HistDevice& d, const int2* tasks, int n_tasks, int* counter, long A0,
                 const double* U, long ldu, long n_steps, double* D, long ldd) {
    FirPlan& P = d.fir;
    static auto encode = []() -> decltype(&cuTensorMapEncodeTiled) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
    }();
    if (!encode) fail(FRAQ_ECUDA, "K5e: cuTensorMapEncodeTiled not available");
    CUtensorMap umap;
    std::memset(&umap, 0, sizeof(umap));
    const cuuint64_t dims[2] = {(cuuint64_t)ldu, (cuuint64_t)n_steps};
    const cuuint64_t strides[1] = {(cuuint64_t)ldu * 8};
    const cuuint32_t box[2] = {16, (cuuint32_t)E_TC}, estr[2] = {1, 1};
    if (encode(&umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(U), dims, strides,
               box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        fail(FRAQ_ECUDA, "K5e: tensor map encode failed");
    Run4Args a{};
    a.groups = d.groups.p;
    a.fg = P.groups.p;
    a.tasks = tasks;
    a.n_tasks = n_tasks;
    a.counter = counter;
    a.state = d.state.p;
    a.ring = d.ring.p;
    a.A0 = A0;
    a.n_steps = n_steps;
    a.U = U;
    a.ldu = ldu;
    a.D = D;
    a.ldd = ldd;
    a.tabs = P.tabs.p;
    a.perm = P.perm.p;
    a.xh = P.xh.p;
    a.ldx = d.total_dim;
    a.xh_mask = P.xh_rows - 1;
    a.ring_rows = P.ring_rows;
    a.capC = P.capC;
    a.capH = P.capH;
    const size_t smem = run4_smem(P);
    FRAQ_CUDA(cudaFuncSetAttribute(run4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    int per_sm = 1;
    FRAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, run4_kernel, P.nwg * 32, smem));
    if (const char* e = std::getenv("FRAQ_K5E_CTAS")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    const int grid = std::max(1, std::min(n_tasks, std::max(1, per_sm) * c->num_sms));
    run4_kernel<<<grid, P.nwg * 32, smem, c->stream>>>(a, umap);
    FRAQ_LAUNCH_CHECK();
    P.short_stale = true;
}

// Rebuilds the short-node states after K5e calls (A1 = values appended so far).
void fir_materialize(fraq_ctx c, HistDevice& d, long A1) {
    FirPlan& P = d.fir;
    if (!P.ok || !P.short_stale) return;
    P.short_stale = false;
    int m_max = 0;
    long dim_max = 0;
    for (size_t gi = 0; gi < P.groups_h.size(); ++gi) {
        m_max = std::max(m_max, P.groups_h[gi].M);
        dim_max = std::max<long>(dim_max, d.groups_h[gi].dim);
    }
    if (m_max == 0 || dim_max == 0) return;
    const int slices = 8;
    dim3 grid((unsigned)((dim_max + 127) / 128), (unsigned)P.groups_h.size(), slices);
    FRAQ_CUDA(cudaFuncSetAttribute(short_state_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(sizeof(double) * m_max * 128)));
    short_state_kernel<<<grid, 128, sizeof(double) * m_max * 128, c->stream>>>(
        d.groups.p, P.groups.p, P.perm.p, d.cr.p, d.cf.p, d.state.p, P.xh.p, d.total_dim,
        P.xh_rows - 1, A1, m_max, slices);
    FRAQ_LAUNCH_CHECK();
}

// ------------------------------------------------------------------------------------- K5f
// The per-level step (K5's role: one push / advance + append + readout for every DOF,
// fast_kernel.cpp:268-409) in K5e's folded form: only the slow ("long") nodes keep a state in
// HBM -- y_j <- r_j y_j + f_j X(n - L), one 256-bit read and write per node and DOF quad -- and
// the fast-decaying nodes are the exact FIR  sum_{m<M} wS_m X(n - L - m)  over the input ring
// `xh` (L2-resident: 65 rows at C2), next to the exact head taps d_i X(n - i).  For the
// reference's auto-sized C2 tables that is 151 of 512 states per level.  Steady state only
// (step_fir_eligible); everything else stays on K5, after short_state_kernel rebuilt the short
// states it reads.
namespace {

struct F4 {
    double x, y, z, w;
};
__device__ __forceinline__ F4 ldg_stream4(const double* p) {
    F4 v;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void stg_stream4(double* p, const F4& v) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}
// up to 4 consecutive doubles of a user-layout row (any alignment; nv valid)
__device__ __forceinline__ F4 ld_row4(const double* p, int nv) {
    F4 v = {0.0, 0.0, 0.0, 0.0};
    if (nv == 4 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const double2 a = *reinterpret_cast<const double2*>(p);
        const double2 b = *reinterpret_cast<const double2*>(p + 2);
        v = {a.x, a.y, b.x, b.y};
    } else {
        if (nv > 0) v.x = p[0];
        if (nv > 1) v.y = p[1];
        if (nv > 2) v.z = p[2];
        if (nv > 3) v.w = p[3];
    }
    return v;
}
__device__ __forceinline__ void st_row4(double* p, const F4& v, int nv) {
    if (nv == 4 && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        *reinterpret_cast<double2*>(p) = make_double2(v.x, v.y);
        *reinterpret_cast<double2*>(p + 2) = make_double2(v.z, v.w);
    } else {
        if (nv > 0) p[0] = v.x;
        if (nv > 1) p[1] = v.y;
        if (nv > 2) p[2] = v.z;
        if (nv > 3) p[3] = v.w;
    }
}
__device__ __forceinline__ void fma_f4(F4& acc, double c, const F4& x) {
    acc.x = fma(c, x.x, acc.x);
    acc.y = fma(c, x.y, acc.y);
    acc.z = fma(c, x.z, acc.z);
    acc.w = fma(c, x.w, acc.w);
}
__device__ __forceinline__ void add_f4(F4& acc, const F4& x) {
    acc.x += x.x;
    acc.y += x.y;
    acc.z += x.z;
    acc.w += x.w;
}

struct StepFirArgs {
    const GroupDev* groups;
    const FirGroup* fg;
    const int2* tiles;   // K5's tiles: (group, first DOF quad)
    double* state;
    double* ring;
    const double* cr;
    const double* cf;
    const double* head;
    const int* perm;
    const double* tabs;
    double* xh;
    long ldx;
    int xh_mask;
    long appended;       // values appended before this launch
    int push;            // 1: advance + append u (level n = appended); 0: read-only, n = appended - 1
    int mode;            // MODE_NONE / MODE_SUM / MODE_DERIV
    const double* u;     // device, user layout
    double* out;         // device, user layout
};

// CTA = LANES DOF quads x S slices; slice sl takes the long nodes p = sl, sl + S, ... and the
// window taps i = i0 + sl, i0 + sl + S, ...; partial sums meet in shared memory and slice 0
// finishes (lag ring, input ring, output), as in K5.
#ifndef FRAQ_K5F_NB
#define FRAQ_K5F_NB 6
#endif
template <int LANES, int S>
__global__ void __launch_bounds__(LANES* S, 4) step_fir_kernel(StepFirArgs A) {
    const int2 tile = A.tiles[blockIdx.x];
    const GroupDev G = A.groups[tile.x];
    const FirGroup* F = A.fg + tile.x;
    const int lane = threadIdx.x % LANES;
    const int sl = threadIdx.x / LANES;
    const int m = 4 * (tile.y + lane);
    const bool live = m < G.dim;
    const int nv = live ? min(4, G.dim - m) : 0;
    __shared__ F4 s_part[S][LANES];
    // the kept nodes' rows and coefficients, staged once per CTA: the state loads' addresses then
    // hang on a shared-memory read instead of a dependent global load per batch
    __shared__ int s_j[512];
    __shared__ double s_r[512], s_f[512];
    const long n = A.push ? A.appended : A.appended - 1;  // level of the newest value
    const int L = G.L, M = F->M, JL = F->JL;
    const long ld = G.ld;
    {
        const int* pm = A.perm + F->perm_off;
        for (int p = threadIdx.x; p < JL; p += LANES * S) {
            const int j = pm[p];
            s_j[p] = j;
            s_r[p] = A.cr[G.co_off + j];
            s_f[p] = A.cf[G.co_off + j];
        }
    }
    __syncthreads();
    const double* xcol = A.xh + G.dof0 + m;
    F4 acc = {0.0, 0.0, 0.0, 0.0};
    F4 unew = {0.0, 0.0, 0.0, 0.0};
    if (live) {
        if (A.push) unew = ld_row4(A.u + G.dof0 + m, nv);
        double* base = A.state + G.st_off + m;
        if (A.push) {
            // feed of level n: X(n - L)  (steady state: n - L >= lo and still on record)
            const F4 v = ld_row4(xcol + (size_t)((n - L) & A.xh_mask) * A.ldx, nv);
            constexpr int NB = FRAQ_K5F_NB;  // independent 256-bit loads in flight per thread
            // (the last batch is partial: predicated loads, no serial tail)
            for (int p = sl; p < JL; p += NB * S) {
                F4 y[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b)
                    if (p + b * S < JL) y[b] = ldg_stream4(base + s_j[p + b * S] * ld);
#pragma unroll
                for (int b = 0; b < NB; ++b)
                    if (p + b * S < JL) {
                        const double r = s_r[p + b * S], f = s_f[p + b * S];
                        y[b].x = fma(r, y[b].x, f * v.x);
                        y[b].y = fma(r, y[b].y, f * v.y);
                        y[b].z = fma(r, y[b].z, f * v.z);
                        y[b].w = fma(r, y[b].w, f * v.w);
                        stg_stream4(base + s_j[p + b * S] * ld, y[b]);
                        add_f4(acc, y[b]);
                    }
            }
        } else if (A.mode != MODE_NONE) {
#pragma unroll 4
            for (int p = sl; p < JL; p += S) add_f4(acc, ldg_stream4(base + s_j[p] * ld));
        }
        if (A.mode != MODE_NONE) {
            // window: exact head taps d_i (derivative only), then the short nodes' FIR
            const double* hd = A.head + G.hd_off;
            const double* ws = A.tabs + F->ws_off;
            const int i0 = A.mode == MODE_DERIV ? 0 : L;
#pragma unroll 4
            for (int i = i0 + sl; i < L + M; i += S) {
                const double c = i < L ? hd[i] : ws[i - L];
                const F4 x = (i == 0 && A.push)
                                 ? unew
                                 : ld_row4(xcol + (size_t)((n - i) & A.xh_mask) * A.ldx, nv);
                fma_f4(acc, c, x);
            }
        }
    }
    if (A.mode != MODE_NONE && S > 1) {
        s_part[sl][lane] = acc;
        __syncthreads();
        if (sl == 0) {
#pragma unroll
            for (int q = 1; q < S; ++q) add_f4(acc, s_part[q][lane]);
        }
    }
    if (sl != 0 || !live) return;
    if (A.push) {
        // (the feed X(n - L) was read from the input ring, so the lag ring slot n % L -- the
        // one it sat in -- can be overwritten without a barrier)
        double* rg = A.ring + G.ring_off + (n % L) * ld + m;
        *reinterpret_cast<double2*>(rg) = make_double2(unew.x, unew.y);
        *reinterpret_cast<double2*>(rg + 2) = make_double2(unew.z, unew.w);
        st_row4(A.xh + (size_t)(n & A.xh_mask) * A.ldx + G.dof0 + m, unew, nv);
    }
    if (A.mode != MODE_NONE) st_row4(A.out + G.dof0 + m, acc, nv);
}

}  // namespace

// Can the next per-level step run on K5f?  push: a pending push (advance + append) at level
// `appended`; otherwise a read-only output at level appended - 1.
bool step_fir_eligible(const HistDevice& d, long level, long appended, bool push) {
    const FirPlan& P = d.fir;
    if (!P.ok || std::getenv("FRAQ_NO_K5F")) return false;
    if (appended < 1 || level != appended - 1) return false;  // pure push sequence
    const long n = push ? appended : appended - 1;
    if (n < P.min_level || n < P.kw_max || P.xh_valid < P.kw_max) return false;
    return true;
}

void launch_step_fir(fraq_ctx c, HistDevice& d, long appended, int push, int mode, const double* u,
                     double* out) {
    FirPlan& P = d.fir;
    if (d.n_tiles == 0) return;
    StepFirArgs a{};
    a.groups = d.groups.p;
    a.fg = P.groups.p;
    a.tiles = d.tiles.p;
    a.state = d.state.p;
    a.ring = d.ring.p;
    a.cr = d.cr.p;
    a.cf = d.cf.p;
    a.head = d.head.p;
    a.perm = P.perm.p;
    a.tabs = P.tabs.p;
    a.xh = P.xh.p;
    a.ldx = d.total_dim;
    a.xh_mask = P.xh_rows - 1;
    a.appended = appended;
    a.push = push;
    a.mode = mode;
    a.u = u;
    a.out = out;
    // (declaring the input ring a persisting L2 window of the launch made the step slower, 66 us
    // against 36: the window's write-backs doubled the DRAM writes; profiles/r02/k5f_l2.sh ran
    // the experiment on the tree of commit 6e10ee6)
    if (d.lanes == 32)
        step_fir_kernel<32, 4><<<d.n_tiles, 128, 0, c->stream>>>(a);
    else
        step_fir_kernel<8, 16><<<d.n_tiles, 128, 0, c->stream>>>(a);
    FRAQ_LAUNCH_CHECK();
    if (push) {
        P.xh_valid = std::min<long>(P.xh_rows, P.xh_valid + 1);
        P.short_stale = true;  // the short nodes' states in HBM are not advanced
    }
}


// The fold as a kernel rewrite (tests/test_fold_identity.py): head c_0..c_(L+M-1) with c_i = d_i
// for i < L and c_i = sum_{all j} f_j r_j^(i-L) beyond, and only the nodes with |r_j|^M > 2^-70,
// fed at lag L + M with f_j r_j^M.  The result is a kernel in the generic-head (SBD) table
// format, whose feed convention mult * ratio^(n_head - 3) (fast_kernel.cpp:337-340) absorbs r^M:
// SBD families keep their multipliers, BE node weights become m' = w r.  M (a multiple of 8, head
// at most `lcap` levels) minimises the bytes a per-level pass moves, 16 per kept node + 8 per
// head tap.  Returns M (0: `out` untouched).
int fold_kernel(const fraq_kernel_t& k, int lcap, fraq_kernel_t* out) {
    const int L = k.sbd ? std::max(2, k.n_head) : 2;
    const int J = k.np1 + k.np2;
    if (J == 0) return 0;
    std::vector<long double> r(J), f(J);
    for (int j = 0; j < J; ++j) {
        const double rj = j < k.np1 ? k.r1[j] : k.r2[j - k.np1];
        const double mj = j < k.np1 ? k.m1[j] : k.m2[j - k.np1];
        r[j] = rj;
        long double v = mj;
        if (k.sbd) v *= std::pow((long double)rj, (long double)(k.n_head - 3));
        f[j] = v;
    }
    const long double thr = std::pow(2.0L, -70.0L);
    auto n_long = [&](int M) {
        int c = 0;
        for (int j = 0; j < J; ++j) c += !(std::pow(std::fabs(r[j]), (long double)M) <= thr);
        return c;
    };
    int M = 0;
    long best = 16L * J + 8L * L;
    for (int cand = 8; L + cand <= std::min(lcap, FRAQ_MAX_HEAD); cand += 8) {
        const long cost = 16L * n_long(cand) + 8L * (L + cand);
        if (cost < best) best = cost, M = cand;
    }
    if (M == 0) return 0;
    long double tail = 0.0L;
    for (int j = 0; j < J; ++j) {
        const long double a = std::fabs(r[j]), pw = std::pow(a, (long double)M);
        if (pw <= thr) tail += std::fabs(f[j]) * pw / (1.0L - a);
    }
    if (!(tail <= std::pow(2.0L, -60.0L) * std::fabs((long double)k.head[0]))) return 0;
    fraq_kernel_t o;
    std::memset(&o, 0, sizeof(o));
    o.sbd = 1;
    o.gamma = k.gamma;
    o.tau = k.tau;
    o.n_head = L + M;
    for (int i = 0; i < L; ++i) o.head[i] = i < k.n_head ? k.head[i] : 0.0;
    std::vector<long double> pw(f);
    for (int m = 0; m < M; ++m) {
        long double c = 0.0L;
        for (int j = 0; j < J; ++j) {
            c += pw[j];
            pw[j] *= r[j];
        }
        o.head[L + m] = (double)c;
    }
    for (int j = 0; j < J; ++j) {
        if (std::pow(std::fabs(r[j]), (long double)M) <= thr) continue;
        const double rj = (double)r[j];
        const double mj = j < k.np1 ? k.m1[j] : k.m2[j - k.np1];
        const double mo = k.sbd ? mj : mj * rj;  // m' r^(L + M - 3) = f r^M
        if (j < k.np1) {
            o.m1[o.np1] = mo;
            o.r1[o.np1++] = rj;
        } else {
            o.m2[o.np2] = mo;
            o.r2[o.np2++] = rj;
        }
    }
    if (o.np1 + o.np2 == 0) return 0;
    *out = o;
    return M;
}


}  // namespace fraqcu
