// history_dmma.cu -- K5d: temporally blocked history evaluation on the fp64 tensor cores.
//
// The per-node recurrence y_j(n) = r_j y_j(n-1) + f_j v(n) (fast_kernel.cpp:268-289,343-365) and
// the readout S(n) = sum_j y_j(n) (fast_kernel.cpp:302-308,378-388) are evaluated 8 levels at a
// time in closed form, which turns both into small GEMMs (v_k = X(n0 + k - L), block start n0):
//
//   S(n0+k)   = sum_j r_j^(k+1) y_j(n0-1)  +  sum_{i<=k} w_(k-i) v_i,   w_m = sum_j f_j r_j^m
//   y_j(n0+7) = r_j^8 y_j(n0-1)  +  sum_i f_j r_j^(7-i) v_i
//
// Both node contractions run as DMMA (mma.sync m8n8k4 f64).  Layout: a warp owns 16 DOFs x 64
// nodes; the state Y^T (DOF rows x node columns) lives in DMMA accumulator fragments, which are
// used directly as A operands of the readout GEMM by permuting the node order of its constant B
// tables (thread (g,t) holds nodes 2t, 2t+1 of each 8-node tile).  Constant tables (r^(k+1),
// f r^(7-i), r^8) sit in shared memory in fragment order: one contiguous 256-byte LDS per DMMA
// B operand.  A CTA covers 16 DOFs x all nodes (8 warps of 64 nodes), two CTAs per SM; node
// slices meet through shared memory once per 8-level block.  Measured on B200: DMMA alone
// reaches 37 TF/s (latency 26 cycles), whereas DFMA with three distinct register operands is
// capped near 25 TF/s by register-file reads (profiles/microbench/mb_operands.cu).
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

constexpr int D_TC = 32;      // levels per staged chunk
constexpr int D_TB = 8;       // levels per block (one GEMM pair)
constexpr int D_LMAX = 32;    // max lag (longer head windows take K5c)
constexpr int D_RING = D_LMAX + 2 * D_TC;  // input ring: lag chunk, current chunk, next chunk
constexpr int D_NT = 8;       // node tiles (8 nodes) per warp = 64 nodes
constexpr int D_MAXWG = 8;    // max warps per DOF group (512 nodes)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// ---- TMA / mbarrier (input chunk staging)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* m) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(m)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one elected thread: arm the barrier with the byte count, then the 2D tile load that completes it
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

// Fragment tables for one group (one CTA per group, 256 threads).
__global__ void frag_tables_kernel(const GroupDev* groups, const double* cr, const double* cf,
                                   double* frag) {
    const GroupDev G = groups[blockIdx.x];
    double* T = frag + (size_t)blockIdx.x * kFragDoubles;
    auto node_r = [&](int j) { return j < G.J ? cr[G.co_off + j] : 0.0; };
    auto node_f = [&](int j) { return j < G.J ? cf[G.co_off + j] : 0.0; };
    for (int idx = threadIdx.x; idx < 64 * 2 * 32; idx += blockDim.x) {
        const int nt = idx / 64, e = (idx / 32) % 2, lane = idx % 32, g = lane >> 2, t = lane & 3;
        // readout B: row k = t <-> node 8 nt + 2t + e, column n = g <-> level g: r^(g+1)
        const int j = 8 * nt + 2 * t + e;
        const double r = node_r(j);
        double p = r;
        for (int q = 0; q < g; ++q) p *= r;
        T[kFragC + idx] = j < G.J ? p : 0.0;
        // state B: half h = e, row k = t <-> level 4h + t, column n = g <-> node 8 nt + g:
        // f r^(7 - 4h - t)
        const int jn = 8 * nt + g, lev = 4 * e + t;
        const double rn = node_r(jn);
        double pn = 1.0;
        for (int q = 0; q < 7 - lev; ++q) pn *= rn;
        T[kFragR + idx] = jn < G.J ? node_f(jn) * pn : 0.0;
    }
    for (int idx = threadIdx.x; idx < 64 * 4 * 2; idx += blockDim.x) {
        const int nt = idx / 8, t = (idx / 2) % 4, e = idx % 2, j = 8 * nt + 2 * t + e;
        const double r = node_r(j);
        double p = 1.0;
        for (int q = 0; q < 8; ++q) p *= r;
        T[kFragR8 + idx] = j < G.J ? p : 0.0;
        T[kFragRF + 2 * idx] = r;
        T[kFragRF + 2 * idx + 1] = node_f(j);
    }
    // local Toeplitz: w_m = sum_j f_j r_j^m, m = 0..7; B[k = t + 4h][n = g] = w_(g - k) (g >= k)
    __shared__ double wsum[8][256];
    for (int m = 0; m < 8; ++m) {
        double acc = 0.0;
        for (int j = threadIdx.x; j < G.J; j += blockDim.x) {
            double p = 1.0;
            for (int q = 0; q < m; ++q) p *= cr[G.co_off + j];
            acc += cf[G.co_off + j] * p;
        }
        wsum[m][threadIdx.x] = acc;
    }
    __syncthreads();
    if (threadIdx.x < 8) {
        double acc = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) acc += wsum[threadIdx.x][i];
        wsum[threadIdx.x][0] = acc;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 64; idx += blockDim.x) {
        const int h = idx / 32, lane = idx % 32, g = lane >> 2, t = lane & 3, k = t + 4 * h;
        T[kFragW + idx] = g >= k ? wsum[g - k][0] : 0.0;
    }
}

// Input rows live in a ring of three 32-level segments (call-relative level n at row n mod 96):
// the lag chunk, the current chunk and the chunk TMA is landing, so no rows are ever moved.
struct DSmem {
    double X[D_RING][16];         // 128-byte aligned: TMA lands a 16-DOF x 32-level box per segment
    double hd[D_LMAX];
    double hf[16][32];            // head-window Toeplitz as DMMA B fragments (DMMA FIR)
    unsigned long long mbar[2];   // completion barriers, chunk k on mbar[k & 1]
};
__device__ __forceinline__ int xrow(long n) {  // ring row of call-relative level n >= -D_RING
    return (int)((n + D_RING) % D_RING);
}
__device__ __forceinline__ int xwrap(int r) {  // r in [-D_RING, 2 D_RING) -> ring row (32-bit)
    r = r < 0 ? r + D_RING : r;
    return r >= D_RING ? r - D_RING : r;
}

// CTA = one 16-DOF group x all nodes: nwg warps (64 nodes each), 2 CTAs resident per SM so one
// CTA's barrier / reduction phase overlaps the other's DMMA phase.  Within a CTA the cross-warp
// reduction of block b-1 is issued after block b's readout DMMAs (software pipelining), so its
// shared-memory latency hides under the asynchronous tensor pipe.
#ifdef FRAQ_EXP_ONECTA
__global__ void __launch_bounds__(256, 1)
    run3_kernel(RunArgs A, const __grid_constant__ CUtensorMap umap) {
#else
__global__ void __launch_bounds__(256, 2)
    run3_kernel(RunArgs A, const __grid_constant__ CUtensorMap umap) {
#endif
    extern __shared__ __align__(128) double dsm[];
    DSmem& S = *reinterpret_cast<DSmem*>(dsm);
    double* tab = dsm + sizeof(DSmem) / sizeof(double);         // kFragDoubles
    double* part = tab + kFragR8 + 64;  // [2 buffers][2 slots][8 warps][2][8][8]
    __shared__ int s_task, s_group;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    const int nwg = blockDim.x >> 5;  // warps = node slices of 64
    const int sl = warp;
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
    // completion barriers of the input tiles: initialised once per CTA (re-initialising a live
    // barrier per task hung K5e after an odd number of completions); a task's chunk k uses
    // mbar[k & 1] and the phase each barrier is in carries over from task to task
    unsigned phases = 0;
    if (tid == 0) {
        s_group = -1;
        mbar_init(&S.mbar[0]);
        mbar_init(&S.mbar[1]);
    }
    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(A.counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= A.n_tasks) return;
        const int2 tk = A.tasks[task];
        const GroupDev G = A.groups[tk.x];
        const int L = G.L;
        const long ld = G.ld;
        if (s_group != tk.x) {  // (uniform) reload the group's constant tables (C, R, W)
            const double* src = A.frag + (size_t)tk.x * kFragDoubles;
            for (int i = tid; i < kFragR8; i += blockDim.x) tab[i] = src[i];
            for (int i = tid; i < 64; i += blockDim.x) tab[kFragR8 + i] = src[kFragW + i];
        }
        const double* RFg = A.frag + (size_t)tk.x * kFragDoubles + kFragRF;  // partial blocks
        for (int i = tid; i < D_LMAX; i += blockDim.x) S.hd[i] = i < L ? A.head[G.hd_off + i] : 0.0;
        // Exact head window as one more K-segment of the readout GEMM: for a block at n0,
        // FIR^T[d][k] = sum_jj X[js + jj][d] H[jj][k], js = n0 + 8 - KW, H[jj][k] = d_(k+KW-8-jj)
        // (zero outside the taps) -- shift invariant: B fragments per group.
        const int taps = G.sbd ? L : 2;
        const int KW = ((taps + 7) + 3) & ~3;
        for (int i = tid; i < (KW / 4) * 32; i += blockDim.x) {
            const int kk = i >> 5, ln = i & 31, gg = ln >> 2, tt = ln & 3;
            const int ii = gg + KW - 8 - (4 * kk + tt);
            S.hf[kk][ln] = (ii >= 0 && ii < taps) ? A.head[G.hd_off + ii] : 0.0;
        }
        const int nkk = KW / 4;
        // state fragments Y[rb][ntl][e]: DOF tk.y + 8 rb + g, node 64 sl + 8 ntl + 2t + e
        double Y[2][D_NT][2];
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
            const int m = tk.y + 8 * rb + g;
#pragma unroll
            for (int ntl = 0; ntl < D_NT; ++ntl)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 64 * sl + 8 * ntl + 2 * t + e;
                    Y[rb][ntl][e] =
                        (j < G.J && m < G.dim) ? A.state[G.st_off + j * ld + m] : 0.0;
                }
        }
        // lag window X(k), k in [A0 - L, A0 - 1] (negative times read as zero)
        for (int idx = tid; idx < L * 16; idx += blockDim.x) {
            const int row = idx >> 4, d = idx & 15;
            const long k = A.A0 - L + row;
            double x = 0.0;
            if (k >= 0 && tk.y + d < G.dim) x = A.ring[G.ring_off + (k % L) * ld + tk.y + d];
            S.X[D_RING - L + row][d] = x;
        }
        // (segment 2 is written through the generic proxy here and by TMA two chunks later)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0) s_group = tk.x;
        const double* Ub = A.U + G.dof0 + tk.y;
        double* Db = A.D ? A.D + G.dof0 + tk.y : nullptr;
        const double* Cfr = tab + kFragC;
        const double* Rfr = tab + kFragR;
        const double* Wfr = tab + kFragR8;  // (W is stored right after C and R in smem)
        // per-warp table bases: immediate offsets in the unrolled loops
        const double* cw = Cfr + (size_t)(8 * sl) * 64 + lane;
        const double* rw = Rfr + (size_t)(8 * sl) * 64 + lane;
        const double* r8w = Cfr + (size_t)(8 * sl) * 64 + 28 + t;  // r^8: readout row g = 7
        // chunk prefetch: thread covers rows (tid >> 4) + 16 i of the next chunk, DOF tid & 15
        const int prow = tid >> 4, pd = tid & 15;
        const bool plive = tk.y + pd < G.dim;
        double pre[2];
        auto prefetch = [&](long c0) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int row = prow + 16 * i;
                const long tt = c0 + row;
                pre[i] = (row < D_TC && row * 16 < D_TC * 16 && tt < A.n_steps && plive)
                             ? Ub[tt * A.ldu + pd] : 0.0;
            }
        };
        const bool tma = A.use_tma && blockDim.x == 256;
        if (tma) {
            if (tid == 0)
                tma_tile(&umap, &S.X[0][0], &S.mbar[0], (int)(G.dof0 + tk.y), 0, D_TC * 16 * 8);
        } else if (blockDim.x == 256) {
            prefetch(0);
        }
        // reduction of a pair of blocks (node sum over warps + head window -> D): one output
        // (slot, level k, DOF d) per thread, two independent add chains over the warp partials
        long p_row0 = 0, p_row1 = 0, p_n00 = 0, p_n01 = 0;
        int p_kmax0 = 0, p_kmax1 = 0, p_buf = 0;
        bool p_dfir0 = false, p_dfir1 = false;
        auto reduce_pair = [&]() {
#ifdef FRAQ_EXP_NOREDUCE
            return;
#endif
            for (int o = tid; o < 2 * D_TB * 16; o += blockDim.x) {
                const int slot = o >> 7, k = (o >> 4) & 7, d = o & 15;
                const long prow = slot ? p_row1 : p_row0, pn0 = slot ? p_n01 : p_n00;
                if (k >= (slot ? p_kmax1 : p_kmax0)) continue;
                const double* pb = part + ((size_t)(p_buf * 2 + slot) * D_MAXWG) * 128 + k * 16 + d;
                double s0 = 0.0, s1 = 0.0;
                for (int w = 0; w + 1 < nwg; w += 2) {
                    s0 += pb[w * 128];
                    s1 += pb[(w + 1) * 128];
                }
                if (nwg & 1) s0 += pb[(nwg - 1) * 128];
                const double sum = s0 + s1;
                double fir = 0.0;
                if (!(slot ? p_dfir1 : p_dfir0)) {
                    // blocks outside the DMMA head window (early levels, chunk tails): exact
                    // head sum from the staged rows, reference tap rule and order
                    const long n = pn0 + k;
                    const long top = G.sbd ? min((long)L - 1, n - A.lo) : 1;
                    int xr = xrow(prow + k);
                    for (long i = 0; i <= top; ++i) {
                        fir = fma(S.hd[i], S.X[xr][d], fir);
                        xr = xr ? xr - 1 : D_RING - 1;
                    }
                }
                const bool valid = G.sbd ? true : (pn0 + k >= 1);
                if (Db && tk.y + d < G.dim)
                    Db[(prow + k) * A.ldd + d] = valid ? sum + fir : qnan;
            }
        };
        // full blocks whose whole head window is valid take the FIR through DMMA
        auto dfir_block = [&](long n0, int kmax) {
            const bool special = A.lo == 1 && n0 <= L && L < n0 + D_TB;
            const bool ok = G.sbd ? (n0 - (L - 1) >= A.lo) : (n0 >= 1);
            return kmax == D_TB && n0 >= 1 && !special && ok;
        };
        int buf = 0;
        bool pending = false;
        unsigned ck = 0;  // chunk counter (mbarrier slot and phase)
        int seg = 0;      // this chunk's ring segment (first row)
        for (long c0 = 0; c0 < A.n_steps; c0 += D_TC, ++ck, seg = xwrap(seg + D_TC)) {
            const int tmax = (int)min((long)D_TC, A.n_steps - c0);
            // (everyone is done with the previous chunk, whose reduction may read the lag segment)
            __syncthreads();
            if (tma) {
                // next chunk's tile into the segment two chunks back (free after the barrier)
                if (tid == 0 && c0 + D_TC < A.n_steps)
                    tma_tile(&umap, &S.X[xwrap(seg + D_TC)][0], &S.mbar[(ck + 1) & 1],
                             (int)(G.dof0 + tk.y), (int)(c0 + D_TC), D_TC * 16 * 8);
                // this chunk's tile landed (TMA, zero-filled past the ends of U); the mbarrier
                // completion makes it visible to every waiting thread
                mbar_wait(&S.mbar[ck & 1], (phases >> (ck & 1)) & 1u);
                phases ^= 1u << (ck & 1);
            } else {
                if (blockDim.x == 256) {
#pragma unroll
                    for (int i = 0; i < 2; ++i) {
                        const int row = prow + 16 * i;
                        if (row < D_TC) S.X[seg + row][pd] = pre[i];
                    }
                    if (c0 + D_TC < A.n_steps) prefetch(c0 + D_TC);
                } else {  // fewer than 8 warps: direct loads (no prefetch)
                    for (int idx = tid; idx < D_TC * 16; idx += blockDim.x) {
                        const int row = idx >> 4, d = idx & 15;
                        const long tt = c0 + row;
                        S.X[seg + row][d] =
                            (tt < A.n_steps && tk.y + d < G.dim) ? Ub[tt * A.ldu + d] : 0.0;
                    }
                }
                __syncthreads();
            }
            // (head window: DMMA segment of the readout, or per output in reduce_pair)
            auto do_block = [&](int t0, int slot, bool mid_reduce) {
                const long n0 = A.A0 + c0 + t0;
                const int kmax = min(D_TB, tmax - t0);
                double* pw = part + ((size_t)(buf * 2 + slot) * D_MAXWG + warp) * 128;
                const bool special = A.lo == 1 && n0 <= L && L < n0 + D_TB;
                if (kmax == D_TB && n0 >= 1 && !special) {
                    // ---- readout GEMM from the block-start state + local Toeplitz
                    // one accumulator chain per row block: 16+ dependent DMMAs at 26 cycles each
                    // stay well inside a warp's share of the pipe (4+ warps per SMSP)
                    double sacc[2][2];
#pragma unroll
                    for (int rb = 0; rb < 2; ++rb) sacc[rb][0] = sacc[rb][1] = 0.0;
#pragma unroll
                    for (int ntl = 0; ntl < D_NT; ++ntl)
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const double b = cw[(ntl * 2 + e) * 32];
#pragma unroll
                            for (int rb = 0; rb < 2; ++rb) dmma(sacc[rb], Y[rb][ntl][e], b);
                        }
                    double vf[2][2];
#pragma unroll
                    for (int rb = 0; rb < 2; ++rb)
#pragma unroll
                        for (int h = 0; h < 2; ++h)
                            vf[rb][h] = S.X[xwrap(seg + t0 + 4 * h + t - L)][8 * rb + g];
                    // local Toeplitz: 4 DMMAs (rb, h) spread over warps 0..3 of the CTA
                    for (int w4 = sl; w4 < 4; w4 += nwg) {  // (fewer than 4 warps: several each)
                        const int hl = w4 & 1;
                        const double b = Wfr[hl * 32 + lane];
                        if (w4 == 0)
                            dmma(sacc[0], vf[0][0], b);
                        else if (w4 == 1)
                            dmma(sacc[0], vf[0][1], b);
                        else if (w4 == 2)
                            dmma(sacc[1], vf[1][0], b);
                        else
                            dmma(sacc[1], vf[1][1], b);
                    }
                    // head-window FIR: warp w < nkk adds k-step w for both row blocks
                    if (dfir_block(n0, kmax))
                        for (int kk = sl; kk < nkk; kk += nwg) {  // (fewer warps: several each)
                            const double b = S.hf[kk][lane];
                            const int xr = xwrap(seg + t0 + 8 - KW + 4 * kk + t);
                            dmma(sacc[0], S.X[xr][g], b);
                            dmma(sacc[1], S.X[xr][8 + g], b);
                        }
                    // deferred reduction of the previous pair: its LDS / DADD / STG latency
                    // overlaps the readout DMMAs just issued (asynchronous tensor pipe)
                    if (mid_reduce) reduce_pair();
                    // ---- state GEMM: Y <- r^8 (.) Y + V R.  All rescale DMULs first, then the
                    // DMMAs K half by K half: a DMUL queued between DMMAs waits for the shared
                    // fp64 pipe (23% of K5d's stall samples sat on DMULs), and no two
                    // consecutive DMMAs share an accumulator.  +1.1% at C2
                    // (profiles/r02/k5d_variants.sh); every element sees the same operations in
                    // the same order as before
#pragma unroll
                    for (int ntl = 0; ntl < D_NT; ++ntl) {
                        const double ra = r8w[(ntl * 2) * 32], rbv = r8w[(ntl * 2 + 1) * 32];
#pragma unroll
                        for (int rb = 0; rb < 2; ++rb) {
#ifndef FRAQ_EXP_NODMUL
                            Y[rb][ntl][0] *= ra;
                            Y[rb][ntl][1] *= rbv;
#endif
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int ntl = 0; ntl < D_NT; ++ntl) {
                            const double b = rw[(ntl * 2 + h) * 32];
#pragma unroll
                            for (int rb = 0; rb < 2; ++rb) dmma(Y[rb][ntl], vf[rb][h], b);
                        }
                    // partial readout (DOF g, levels 2t, 2t+1) -> shared memory
#pragma unroll
                    for (int rb = 0; rb < 2; ++rb) {
                        // [level][DOF] layout: the reduction reads consecutive DOFs (no conflicts)
                        pw[(2 * t) * 16 + 8 * rb + g] = sacc[rb][0];
                        pw[(2 * t + 1) * 16 + 8 * rb + g] = sacc[rb][1];
                    }
                } else {
                    if (mid_reduce) reduce_pair();
                    // partial block: level by level, elementwise on the fragments
                    for (int k = 0; k < kmax; ++k) {
                        const long n = n0 + k;
                        const bool adv = n >= 1;
                        const bool feed = adv && (n - L >= A.lo);
                        double ps[2] = {0.0, 0.0};
#pragma unroll
                        for (int rb = 0; rb < 2; ++rb) {
                            const double v = feed ? S.X[xwrap(seg + t0 + k - L)][8 * rb + g] : 0.0;
#pragma unroll
                            for (int ntl = 0; ntl < D_NT; ++ntl)
#pragma unroll
                                for (int e = 0; e < 2; ++e) {
                                    const int nt = 8 * sl + ntl;
                                    if (adv) {
                                        const double r = RFg[((nt * 4 + t) * 2 + e) * 2];
                                        const double f = RFg[((nt * 4 + t) * 2 + e) * 2 + 1];
                                        Y[rb][ntl][e] = fma(r, Y[rb][ntl][e], f * v);
                                    }
                                    ps[rb] += Y[rb][ntl][e];
                                }
                        }
#pragma unroll
                        for (int rb = 0; rb < 2; ++rb) {
                            ps[rb] += __shfl_xor_sync(0xffffffffu, ps[rb], 1);
                            ps[rb] += __shfl_xor_sync(0xffffffffu, ps[rb], 2);
                            if (t == 0) pw[k * 16 + 8 * rb + g] = ps[rb];
                        }
                    }
                }
            };
            for (int t0 = 0; t0 < tmax; t0 += 2 * D_TB) {
                // two blocks per barrier: their partials go to slots 0 / 1 of buffer `buf`
                const int nblk = t0 + D_TB < tmax ? 2 : 1;
                do_block(t0, 0, pending);  // reduces the previous pair (p_* still describe it)
                if (nblk == 2) do_block(t0 + D_TB, 1, false);
                p_row0 = c0 + t0;
                p_n00 = A.A0 + c0 + t0;
                p_kmax0 = min(D_TB, tmax - t0);
                p_dfir0 = dfir_block(p_n00, p_kmax0);
                p_kmax1 = 0;
                if (nblk == 2) {
                    p_row1 = c0 + t0 + D_TB;
                    p_n01 = A.A0 + c0 + t0 + D_TB;
                    p_kmax1 = min(D_TB, tmax - t0 - D_TB);
                    p_dfir1 = dfir_block(p_n01, p_kmax1);
                }
#ifndef FRAQ_EXP_NOSYNC
                __syncthreads();
#endif
                p_buf = buf;
                pending = true;
                buf ^= 1;
            }
            // the chunk's last pair: its reduction reads S.X only for blocks outside the DMMA
            // head window; otherwise it is deferred behind the next chunk's first readout DMMAs
            if (pending && !(p_dfir0 && (p_kmax1 == 0 || p_dfir1) && c0 + D_TC < A.n_steps)) {
                reduce_pair();
                pending = false;
            }
        }
        if (pending) reduce_pair();  // (deferred past the last chunk)
        // write back the state and the ring
#pragma unroll
        for (int rb = 0; rb < 2; ++rb) {
            const int m = tk.y + 8 * rb + g;
#pragma unroll
            for (int ntl = 0; ntl < D_NT; ++ntl)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int j = 64 * sl + 8 * ntl + 2 * t + e;
                    if (j < G.J && m < G.dim) A.state[G.st_off + j * ld + m] = Y[rb][ntl][e];
                }
        }
        __syncthreads();
        const long A1 = A.A0 + A.n_steps;
        for (int idx = tid; idx < L * 16; idx += blockDim.x) {
            const int row = idx >> 4, d = idx & 15;
            const long k = A1 - L + row;
            if (k >= 0 && tk.y + d < G.dim)
                A.ring[G.ring_off + (k % L) * ld + tk.y + d] = S.X[xrow(A.n_steps - L + row)][d];
        }
    }
}

size_t run3_smem(int nwg) {
    (void)nwg;
    return sizeof(DSmem) + sizeof(double) * (kFragR8 + 64 + 2 * 2 * D_MAXWG * 128);
}

}  // namespace

void build_frag_tables(fraq_ctx c, HistDevice& d) {
    if (d.frag_built) return;
    d.frag.alloc((size_t)d.groups_h.size() * kFragDoubles);
    frag_tables_kernel<<<(unsigned)d.groups_h.size(), 256, 0, c->stream>>>(d.groups.p, d.cr.p,
                                                                          d.cf.p, d.frag.p);
    FRAQ_LAUNCH_CHECK();
    d.frag_built = true;
}

int run3_max_lag() { return D_LMAX; }

void launch_run3(const RunArgs& a, int nwg, int num_sms, cudaStream_t s, bool allow_tma) {
    const size_t smem = run3_smem(nwg);
    // (per launch: the attribute is per device, and a process may drive several devices)
    FRAQ_CUDA(cudaFuncSetAttribute(run3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)run3_smem(D_MAXWG)));
    int per_sm = 1;
    FRAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, run3_kernel, nwg * 32, smem));
#ifdef FRAQ_EXP_ONECTA
    per_sm = 1;
#endif
    const int grid = std::max(1, std::min(a.n_tasks, std::max(1, per_sm) * num_sms));
    // tensor map over the caller's input rows U[n_steps][ldu] (doubles): 16-DOF x 32-level boxes,
    // zero fill outside -- used when the layout meets the TMA alignment rules
    CUtensorMap umap;
    std::memset(&umap, 0, sizeof(umap));
    RunArgs b = a;
    b.use_tma = 0;
    static auto encode = []() -> decltype(&cuTensorMapEncodeTiled) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
    }();
    const bool aligned = (reinterpret_cast<uintptr_t>(a.U) % 16 == 0) && (a.ldu % 2 == 0) &&
                         a.ldu >= 16 && a.n_steps >= 1 && a.n_steps < (1L << 31) &&
                         a.ldu < (1L << 31) && !std::getenv("FRAQ_NO_TMA");
    // (allow_tma: every group starts at an even DOF, so each box starts 16-byte aligned)
    if (encode && aligned && allow_tma && nwg == D_MAXWG) {
        const cuuint64_t dims[2] = {(cuuint64_t)a.ldu, (cuuint64_t)a.n_steps};
        const cuuint64_t strides[1] = {(cuuint64_t)a.ldu * 8};
        const cuuint32_t box[2] = {16, (cuuint32_t)D_TC}, estr[2] = {1, 1};
        if (encode(&umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(a.U), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
            b.use_tma = 1;
    }
    run3_kernel<<<grid, nwg * 32, smem, s>>>(b, umap);
    FRAQ_LAUNCH_CHECK();
}

}  // namespace fraqcu
