// history.cu -- the fused fast-CQ history kernels and the device history objects.
//
// K5  (step_kernel)    one time level for every DOF: advance (y <- r y + f u_lag) fused with the
//                      append into the lag ring and the readout (node sum + exact head window).
//                      One HBM pass over the state per level.  BeHistory/SbdHistory
//                      advance/append/history_sum/derivative, fast_kernel.cpp:268-409.
// K5c (run2_kernel)    temporally blocked evaluation, lane per DOF, DFMA (head windows over 32
//                      levels); the default blocked paths K5d / K5e (DMMA block GEMMs) are in
//                      history_dmma.cu / history_fir.cu, and so is K5f, the per-level step on
//                      K5e's node split that takes over from K5 in the steady state of a push
//                      sequence (flush() / run_device() below pick per call).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "history.cuh"

namespace fraqcu {

// history_dmma.cu
void build_frag_tables(fraq_ctx c, HistDevice& d);
void launch_run3(const RunArgs& a, int nwg, int num_sms, cudaStream_t s, bool allow_tma);
int run3_max_lag();
// history_fir.cu (K5e)
void build_fir_plan(fraq_ctx c, HistDevice& d);
void fir_note_inputs(fraq_ctx c, HistDevice& d, long A0, const double* U, long ldu, long n_steps);
bool fir_eligible(const HistDevice& d, long A0, const double* U, long ldu, long n_steps,
                  const double* D, long ldd);
void launch_run4(fraq_ctx c, HistDevice& d, const int2* tasks, int n_tasks, int* counter, long A0,
                 const double* U, long ldu, long n_steps, double* D, long ldd);
void fir_materialize(fraq_ctx c, HistDevice& d, long A1);
// history_fir.cu (K5f)
bool step_fir_eligible(const HistDevice& d, long level, long appended, bool push);
void launch_step_fir(fraq_ctx c, HistDevice& d, long appended, int push, int mode, const double* u,
                     double* out);

namespace {

struct d4 {
    double x, y, z, w;
};

// 256-bit streaming access to the history state: L1 bypass, L2 evict-first so the lag rings
// and head windows (touched once per level) stay L2-resident while the state streams.
__device__ __forceinline__ d4 ld_stream(const double* p) {
    d4 v;
    asm volatile("ld.global.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w)
                 : "l"(p));
    return v;
}
__device__ __forceinline__ void st_stream(double* p, const d4& v) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p),
                 "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w)
                 : "memory");
}
__device__ __forceinline__ d4 ld4(const double* p) {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    return {a.x, a.y, b.x, b.y};
}
__device__ __forceinline__ void st4(double* p, const d4& v) {
    *reinterpret_cast<double2*>(p) = make_double2(v.x, v.y);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v.z, v.w);
}
__device__ __forceinline__ void fma4(d4& acc, double h, const d4& x) {
    acc.x = fma(h, x.x, acc.x);
    acc.y = fma(h, x.y, acc.y);
    acc.z = fma(h, x.z, acc.z);
    acc.w = fma(h, x.w, acc.w);
}

// ------------------------------------------------------------------------------------------ K5
// CTA = LANES DOF quads x S node slices.  Thread (slice sl, quad) streams nodes j = sl, sl+S, ..
// of its 4 DOFs with 256-bit loads/stores; slice partial sums meet in shared memory; slice 0
// finishes (append into the ring, exact head window, output).
template <int LANES, int S>
__global__ void __launch_bounds__(LANES* S, 6) step_kernel(StepArgs A) {
    const int2 tile = A.tiles[blockIdx.x];
    const GroupDev G = A.groups[tile.x];
    const int lane = threadIdx.x % LANES;
    const int sl = threadIdx.x / LANES;
    const int m = 4 * (tile.y + lane);  // first DOF of this thread's quad (within the group)
    const bool live = m < G.dim;
    __shared__ d4 s_part[S][LANES];
    long level = A.level, appended = A.appended;
    if (A.n_dev) {
        level = *A.n_dev + A.n_off - 1;
        appended = level + 1;
    }

    // feed value u_{level+1-L} from the ring (read by every slice before the barrier below)
    const long fi = level + 1 - G.L;
    const bool feed = A.adv && fi >= A.lo && fi <= appended - 1;
    const long ld = G.ld;
    d4 v = {0.0, 0.0, 0.0, 0.0};
    if (feed && live) v = ld4(A.ring + G.ring_off + (fi % G.L) * ld + m);

    d4 acc = {0.0, 0.0, 0.0, 0.0};
    if (live && (A.adv || A.mode != MODE_NONE)) {
        const double* __restrict__ cr = A.cr + G.co_off;
        const double* __restrict__ cf = A.cf + G.co_off;
        double* base = A.state + G.st_off + m;
        if (A.adv) {
            // NB independent 256-bit loads in flight per thread before any store (the stores
            // are volatile asm, so loads are batched explicitly rather than left to the scheduler)
            constexpr int NB = 4;
            int j = sl;
            for (; j + (NB - 1) * S < G.J; j += NB * S) {
                d4 y[NB];
#pragma unroll
                for (int b = 0; b < NB; ++b) y[b] = ld_stream(base + (j + b * S) * ld);
#pragma unroll
                for (int b = 0; b < NB; ++b) {
                    const double r = __ldg(cr + j + b * S), f = __ldg(cf + j + b * S);
                    y[b].x = fma(r, y[b].x, f * v.x);
                    y[b].y = fma(r, y[b].y, f * v.y);
                    y[b].z = fma(r, y[b].z, f * v.z);
                    y[b].w = fma(r, y[b].w, f * v.w);
                    st_stream(base + (j + b * S) * ld, y[b]);
                    acc.x += y[b].x;
                    acc.y += y[b].y;
                    acc.z += y[b].z;
                    acc.w += y[b].w;
                }
            }
            for (; j < G.J; j += S) {
                double* p = base + j * ld;
                d4 y = ld_stream(p);
                const double r = __ldg(cr + j), f = __ldg(cf + j);
                y.x = fma(r, y.x, f * v.x);
                y.y = fma(r, y.y, f * v.y);
                y.z = fma(r, y.z, f * v.z);
                y.w = fma(r, y.w, f * v.w);
                st_stream(p, y);
                acc.x += y.x;
                acc.y += y.y;
                acc.z += y.z;
                acc.w += y.w;
            }
        } else {
#pragma unroll 4
            for (int j = sl; j < G.J; j += S) {
                const d4 y = ld_stream(base + j * ld);
                acc.x += y.x;
                acc.y += y.y;
                acc.z += y.z;
                acc.w += y.w;
            }
        }
    }
    if (A.mode == MODE_FFPE && live) {
        // FastStepper: s = history + sum_{i=first}^{top} d_i G^{n-i}, n = appended (G^n not yet
        // in; the solve kernel appends it).  No append in this launch, so the taps are split
        // over the node slices ahead of the barrier (folded kernels carry 60-80 of them).
        const double* hd = A.head + G.hd_off;
        const double* ring = A.ring + G.ring_off + m;
        const long n = appended;
        long top;
        if (!G.sbd)
            top = n >= 2 ? 1 : 0;
        else
            top = min((long)G.L - 1, n - 1);
#pragma unroll 4
        for (long i = (A.first_tap > 1 ? A.first_tap : 1) + sl; i <= top; i += S)
            fma4(acc, hd[i], ld4(ring + ((n - i) % G.L) * ld));
    }
    if (S > 1) {
        s_part[sl][lane] = acc;
        __syncthreads();
        if (sl != 0) return;
#pragma unroll
        for (int q = 1; q < S; ++q) {
            const d4 t = s_part[q][lane];
            acc.x += t.x;
            acc.y += t.y;
            acc.z += t.z;
            acc.w += t.w;
        }
    }
    if (!live) return;
    const int nv = min(4, G.dim - m);  // valid DOFs of this quad
    double* ring = A.ring + G.ring_off + m;
    if (A.app) {
        const double* u = A.u + G.dof0 + m;
        d4 x;
        x.x = u[0];
        x.y = nv > 1 ? u[1] : 0.0;
        x.z = nv > 2 ? u[2] : 0.0;
        x.w = nv > 3 ? u[3] : 0.0;
        st4(ring + (appended % G.L) * ld, x);
        if (A.xh) {
            double* xr = A.xh + (size_t)(appended & A.xh_mask) * A.ldx + G.dof0 + m;
            xr[0] = x.x;
            if (nv > 1) xr[1] = x.y;
            if (nv > 2) xr[2] = x.z;
            if (nv > 3) xr[3] = x.w;
        }
        ++appended;
    }
    if (A.mode == MODE_NONE) return;
    const double* hd = A.head + G.hd_off;
    if (A.mode == MODE_DERIV) {
        const long n = appended - 1;
        long top;
        if (!G.sbd)
            top = 1;
        else {
            const long bound = A.lo == 0 ? n : n - 1;
            top = min((long)G.L - 1, bound);
        }
        for (long i = 0; i <= top; ++i) fma4(acc, hd[i], ld4(ring + ((n - i) % G.L) * ld));
    }
    double* o = A.out + G.dof0 + m;
    o[0] = acc.x;
    if (nv > 1) o[1] = acc.y;
    if (nv > 2) o[2] = acc.z;
    if (nv > 3) o[3] = acc.w;
}

// ----------------------------------------------------------------------------------------- K5c
// Temporally blocked evaluation, B200 mapping: lane = DOF (32 consecutive DOFs per CTA), warp w
// owns nodes j = 32 w + p (p < 32), levels processed in register blocks of 8.  Per node the 8
// levels run back to back on one register (z <- r z + v_k; s_k += f z): 16 DFMA per pair of
// broadcast shared-memory loads (r_j, f_j), no shuffles.  The node sum crosses warps once per
// block through shared memory (double-buffered partials, one barrier per 8 levels).  State is kept
// as z = y / f (two DFMA per node and level); inputs stream through a 32-level chunk window.
constexpr int R2_TC = 32;      // levels per staged chunk
constexpr int R2_TB = 8;       // levels per register block
constexpr int R2_P = 32;       // nodes per warp
constexpr int R2_LMAX = 64;    // max lag on this path
constexpr int R2_MAXW = 16;    // max warps (512 nodes)

__host__ __device__ inline size_t run2_smem_bytes(int nw) {
    return sizeof(double) * ((size_t)(R2_LMAX + R2_TC) * 32 + R2_TC * 32 + 2 * 512 + R2_LMAX +
                             (size_t)2 * nw * R2_TB * 32) + 16;
}

__global__ void __launch_bounds__(R2_MAXW * 32, 1) run2_kernel(RunArgs A) {
    extern __shared__ double sm2[];
    const int nw = blockDim.x >> 5;
    double(*X)[32] = reinterpret_cast<double(*)[32]>(sm2);                  // [LMAX+TC][32]
    double(*F)[32] = reinterpret_cast<double(*)[32]>(sm2 + (R2_LMAX + R2_TC) * 32);  // [TC][32]
    double* cr = sm2 + (R2_LMAX + 2 * R2_TC) * 32;
    double* cf = cr + 512;
    double* hd = cf + 512;
    double* part = hd + R2_LMAX;                                            // [2][nw][TB][32]
    __shared__ int s_task;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const double qnan = __longlong_as_double(0x7ff8000000000000LL);
    const bool fast_red = nw == R2_MAXW;  // 512 threads: one output pair per thread pair
    for (;;) {
        __syncthreads();
        if (tid == 0) s_task = atomicAdd(A.counter, 1);
        __syncthreads();
        const int task = s_task;
        if (task >= A.n_tasks) return;
        const int2 tk = A.tasks[task];
        const GroupDev G = A.groups[tk.x];
        const int m = tk.y + lane;  // this lane's DOF within the group
        const bool live = m < G.dim;
        const int L = G.L, J = G.J;
        const long ld = G.ld;
        for (int j = tid; j < 512; j += blockDim.x) {
            cr[j] = j < J ? A.cr[G.co_off + j] : 0.0;
            cf[j] = j < J ? A.cf[G.co_off + j] : 0.0;
        }
        for (int i = tid; i < R2_LMAX; i += blockDim.x) hd[i] = i < L ? A.head[G.hd_off + i] : 0.0;
        // initial state z = y / f for this warp's nodes
        double z[R2_P];
#pragma unroll
        for (int p = 0; p < R2_P; ++p) {
            const int j = warp * R2_P + p;
            z[p] = 0.0;
            if (j < J && live) z[p] = A.state[G.st_off + j * ld + m] / A.cf[G.co_off + j];
        }
        // lag window: X(k), k in [A0 - L, A0 - 1], rows R2_LMAX - L .. R2_LMAX - 1
        for (int idx = tid; idx < L * 32; idx += blockDim.x) {
            const int row = idx >> 5, d = idx & 31;
            const long k = A.A0 - L + row;
            double x = 0.0;
            if (k >= 0 && tk.y + d < G.dim) x = A.ring[G.ring_off + (k % L) * ld + tk.y + d];
            X[R2_LMAX - L + row][d] = x;  // negative times read as zero
        }
        const double* Ub = A.U + G.dof0 + tk.y;
        double* Db = A.D ? A.D + G.dof0 + tk.y : nullptr;
        // chunk prefetch: rows warp + 16 i (i < 2) of the next chunk, DOF lane
        double pre[2];
        auto load_chunk = [&](long c0) {
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int row = warp + R2_MAXW * i;
                const long t = c0 + row;
                pre[i] = (row < R2_TC && t < A.n_steps && live) ? Ub[t * A.ldu + lane] : 0.0;
            }
        };
        load_chunk(0);
        int buf = 0, last_tmax = 0;
        for (long c0 = 0; c0 < A.n_steps; c0 += R2_TC) {
            const int tmax = (int)min((long)R2_TC, A.n_steps - c0);
            __syncthreads();
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int row = warp + R2_MAXW * i;
                if (row < R2_TC) X[R2_LMAX + row][lane] = pre[i];
            }
            if (nw < R2_MAXW) {  // fewer than 16 warps: remaining rows loaded directly
                for (int row = warp + nw; row < R2_TC; row += nw)
                    if (row >= R2_MAXW * 2 || (row % R2_MAXW) >= nw) {
                        const long t = c0 + row;
                        X[R2_LMAX + row][lane] =
                            (t < A.n_steps && live) ? Ub[t * A.ldu + lane] : 0.0;
                    }
            }
            if (c0 + R2_TC < A.n_steps) load_chunk(c0 + R2_TC);
            __syncthreads();
            // exact head window for the chunk, all threads: F[t][d] = sum_{i<=top} h_i X(n-i)
#ifndef FRAQ_EXP_NOFIR
            for (int idx = tid; idx < R2_TC * 32; idx += blockDim.x) {
                const int t = idx >> 5, d = idx & 31;
                const long n = A.A0 + c0 + t;
                const long top = G.sbd ? min((long)L - 1, n - A.lo) : 1;
                double acc = 0.0;
                for (long i = 0; i <= top; ++i) acc = fma(hd[i], X[R2_LMAX + t - i][d], acc);
                F[t][d] = acc;
            }
            __syncthreads();
#endif
            // reduction of a finished block (partials in buffer pbuf): node sum over warps +
            // head window -> D.  fast path (16 warps, full block): thread pair (2o, 2o+1) sums
            // the two warp halves of output o = (k, d) and combines with one shuffle; straight-
            // line code so it interleaves with the surrounding FMA block.
            auto reduce_block = [&](int bt0, int bk, int pbuf) {
                const double* pr = part + (size_t)pbuf * nw * R2_TB * 32;
#ifdef FRAQ_EXP_NOREDUCE
                return;
#endif
                if (fast_red && bk == R2_TB) {
                    const int o = tid >> 1, h = tid & 1, k = o >> 5, d = o & 31;
                    double sum = 0.0;
#pragma unroll
                    for (int w = 0; w < R2_MAXW / 2; ++w)
                        sum += pr[((h * (R2_MAXW / 2) + w) * R2_TB + k) * 32 + d];
                    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
                    const long n = A.A0 + c0 + bt0 + k;
                    const bool valid = G.sbd ? true : (n >= 1);
                    if (h == 0 && Db && tk.y + d < G.dim)
                        Db[(c0 + bt0 + k) * A.ldd + d] = valid ? sum + F[bt0 + k][d] : qnan;
                } else {
                    for (int idx = tid; idx < bk * 32; idx += blockDim.x) {
                        const int k = idx >> 5, d = idx & 31;
                        double sum = 0.0;
                        for (int w = 0; w < nw; ++w) sum += pr[(w * R2_TB + k) * 32 + d];
                        const long n = A.A0 + c0 + bt0 + k;
                        const bool valid = G.sbd ? true : (n >= 1);
                        if (Db && tk.y + d < G.dim)
                            Db[(c0 + bt0 + k) * A.ldd + d] = valid ? sum + F[bt0 + k][d] : qnan;
                    }
                }
            };
            int prev_t0 = -1, prev_k = 0, prev_buf = 0;
            const double* crw = cr + warp * R2_P;
            const double* cfw = cf + warp * R2_P;
            for (int t0 = 0; t0 < tmax; t0 += R2_TB) {
                const long n0 = A.A0 + c0 + t0;
                const int kmax = min(R2_TB, tmax - t0);
                double* pb = part + (size_t)buf * nw * R2_TB * 32;
                // the scheme variant must not feed G(t_0) (level n = L, lo = 1): partial path
                const bool special = A.lo == 1 && n0 <= L && L < n0 + R2_TB;
                if (kmax == R2_TB && n0 >= 1 && !special) {
                    // full block: every level advances; feeds X(n - L) (negative times are zero)
                    double v[R2_TB], sacc[R2_TB];
#pragma unroll
                    for (int k = 0; k < R2_TB; ++k) {
                        v[k] = X[R2_LMAX + t0 + k - L][lane];
                        sacc[k] = 0.0;
                    }
#pragma unroll
                    for (int p0 = 0; p0 < R2_P / 2; p0 += 4) {
                        double rr[4], ff[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            rr[i] = crw[p0 + i];
                            ff[i] = cfw[p0 + i];
                        }
#pragma unroll
                        for (int k = 0; k < R2_TB; ++k)
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                z[p0 + i] = fma(rr[i], z[p0 + i], v[k]);
                                sacc[k] = fma(ff[i], z[p0 + i], sacc[k]);
                            }
                    }
                    if (prev_t0 >= 0) reduce_block(prev_t0, prev_k, prev_buf);
#pragma unroll
                    for (int p0 = R2_P / 2; p0 < R2_P; p0 += 4) {
                        double rr[4], ff[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            rr[i] = crw[p0 + i];
                            ff[i] = cfw[p0 + i];
                        }
#pragma unroll
                        for (int k = 0; k < R2_TB; ++k)
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                z[p0 + i] = fma(rr[i], z[p0 + i], v[k]);
                                sacc[k] = fma(ff[i], z[p0 + i], sacc[k]);
                            }
                    }
#pragma unroll
                    for (int k = 0; k < R2_TB; ++k) pb[(warp * R2_TB + k) * 32 + lane] = sacc[k];
                } else {
                    if (prev_t0 >= 0) reduce_block(prev_t0, prev_k, prev_buf);
                    // partial block (chunk tail, level 0 of a fresh history, scheme level L)
                    for (int k = 0; k < kmax; ++k) {
                        const long n = n0 + k;
                        double sk = 0.0;  // (partial path)
                        if (n >= 1) {
                            const double vk = (n - L >= A.lo) ? X[R2_LMAX + t0 + k - L][lane] : 0.0;
#pragma unroll
                            for (int p = 0; p < R2_P; ++p) {
                                z[p] = fma(crw[p], z[p], vk);
                                sk = fma(cfw[p], z[p], sk);
                            }
                        } else {
#pragma unroll
                            for (int p = 0; p < R2_P; ++p) sk = fma(cfw[p], z[p], sk);
                        }
                        pb[(warp * R2_TB + k) * 32 + lane] = sk;
                    }
                }
#ifndef FRAQ_EXP_NOSYNC
                __syncthreads();
#endif
                prev_t0 = t0;
                prev_k = kmax;
                prev_buf = buf;
                buf ^= 1;
            }
            if (prev_t0 >= 0) reduce_block(prev_t0, prev_k, prev_buf);
            last_tmax = tmax;
            if (c0 + R2_TC < A.n_steps) {
                // slide (full chunk, tmax = 32): rows R2_LMAX + 32 - L .. -> R2_LMAX - L .., in
                // 32-row phases so sources are read before they are overwritten (L <= 64)
                for (int base = 0; base < L; base += R2_TC) {
                    __syncthreads();
                    for (int idx = tid; idx < R2_TC * 32; idx += blockDim.x) {
                        const int r = base + (idx >> 5);
                        if (r < L) X[R2_LMAX - L + r][idx & 31] = X[R2_LMAX - L + r + R2_TC][idx & 31];
                    }
                }
            }
        }
        // write back y = f z
#pragma unroll
        for (int p = 0; p < R2_P; ++p) {
            const int j = warp * R2_P + p;
            if (j < J && live) A.state[G.st_off + j * ld + m] = cf[j] * z[p];
        }
        __syncthreads();
        // ring <- last L inputs: time A1 - L + row sits in row R2_LMAX + last_tmax - L + row of
        // the final (unslid) chunk window
        const long A1 = A.A0 + A.n_steps;
        for (int idx = tid; idx < L * 32; idx += blockDim.x) {
            const int row = idx >> 5, d = idx & 31;
            const long k = A1 - L + row;
            if (k >= 0 && tk.y + d < G.dim)
                A.ring[G.ring_off + (k % L) * ld + tk.y + d] = X[R2_LMAX + last_tmax - L + row][d];
        }
    }
}

void launch_run2(const RunArgs& a, int nw, int num_sms, cudaStream_t s) {
    const size_t smem = run2_smem_bytes(nw);
    // (per launch: the attribute is per device, and a process may drive several devices)
    FRAQ_CUDA(cudaFuncSetAttribute(run2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)run2_smem_bytes(R2_MAXW)));
    int per_sm = 1;
    FRAQ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, run2_kernel, nw * 32, smem));
    const int grid = std::max(1, std::min(a.n_tasks, std::max(1, per_sm) * num_sms));
    run2_kernel<<<grid, nw * 32, smem, s>>>(a);
    FRAQ_LAUNCH_CHECK();
}

}  // namespace

// ------------------------------------------------------------------------------ HistDevice
void HistDevice::build(fraq_ctx c, int n_groups, const fraq_kernel_t* const* ks, const long* dims,
                       bool tables_only) {
    groups_h.clear();
    tiles_h.clear();
    kernels.assign(n_groups, fraq_kernel_t{});
    long st = 0, rg = 0, dof = 0;
    int co = 0, hd = 0;
    std::vector<double> hr, hf, hh;
    max_J = 0;
    max_L = 0;
    ztrick_ok = true;
    long max_dim = 0;
    for (int g = 0; g < n_groups; ++g) {
        const fraq_kernel_t& k = *ks[g];
        kernels[g] = k;
        GroupDev G{};
        G.dof0 = dof;
        G.dim = (int)dims[g];
        G.ld = (int)((dims[g] + 3) / 4 * 4);
        G.J = k.np1 + k.np2;
        G.L = k.sbd ? std::max(2, k.n_head) : 2;
        G.sbd = k.sbd;
        G.st_off = st;
        G.ring_off = rg;
        G.co_off = co;
        G.hd_off = hd;
        // feed coefficients: BE node weights; SBD mult * ratio^(n_head-3) (fast_kernel.cpp:337-340)
        for (int j = 0; j < k.np1; ++j) {
            hr.push_back(k.r1[j]);
            hf.push_back(k.sbd ? k.m1[j] * std::pow(k.r1[j], double(k.n_head - 3)) : k.m1[j]);
        }
        for (int j = 0; j < k.np2; ++j) {
            hr.push_back(k.r2[j]);
            hf.push_back(k.m2[j] * std::pow(k.r2[j], double(k.n_head - 3)));
        }
        for (int i = 0; i < G.L; ++i) hh.push_back(i < k.n_head ? k.head[i] : 0.0);
        for (int j = co; j < (int)hf.size(); ++j)
            if (hf[j] == 0.0 || !std::isfinite(1.0 / hf[j])) ztrick_ok = false;
        co += G.J;
        hd += G.L;
        st += (long)G.J * G.ld;
        rg += (long)G.L * G.ld;
        dof += dims[g];
        max_J = std::max(max_J, G.J);
        max_L = std::max(max_L, G.L);
        max_dim = std::max(max_dim, dims[g]);
        groups_h.push_back(G);
    }
    total_dim = dof;
    // K5 tile shape: wide DOF tiles when groups are large, more node slices when small
    // (large groups: 128-thread CTAs, 6 resident per SM -> the C2 grid (512 CTAs) is one wave)
    if (max_dim >= 8192) {
        lanes = 32;
        slices = 4;
    } else {
        lanes = 8;
        slices = 16;
    }
    for (int g = 0; g < n_groups; ++g) {
        const int quads = (groups_h[g].dim + 3) / 4;
        for (int q0 = 0; q0 < quads; q0 += lanes) tiles_h.push_back(make_int2(g, q0));
    }
    n_tiles = (int)tiles_h.size();
    groups.alloc(groups_h.size());
    tiles.alloc(tiles_h.size());
    cr.alloc(std::max<size_t>(1, hr.size()));
    cf.alloc(std::max<size_t>(1, hf.size()));
    head.alloc(std::max<size_t>(1, hh.size()));
    state.alloc(tables_only ? 1 : std::max<long>(1, st));
    ring.alloc(tables_only ? 1 : std::max<long>(1, rg));
    auto up = [&](void* d, const void* h, size_t bytes) {
        if (bytes) FRAQ_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, c->stream));
    };
    up(groups.p, groups_h.data(), groups_h.size() * sizeof(GroupDev));
    up(tiles.p, tiles_h.data(), tiles_h.size() * sizeof(int2));
    up(cr.p, hr.data(), hr.size() * sizeof(double));
    up(cf.p, hf.data(), hf.size() * sizeof(double));
    cr_h = hr;
    cf_h = hf;
    up(head.p, hh.data(), hh.size() * sizeof(double));
    zero(c);
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

void HistDevice::zero(fraq_ctx c) {
    FRAQ_CUDA(cudaMemsetAsync(state.p, 0, state.n * sizeof(double), c->stream));
    FRAQ_CUDA(cudaMemsetAsync(ring.p, 0, ring.n * sizeof(double), c->stream));
}

void HistDevice::launch_step(fraq_ctx c, const StepArgs& a) { launch_step(c, a, c->stream); }

void HistDevice::launch_step(fraq_ctx, const StepArgs& a, cudaStream_t stream) {
    if (n_tiles == 0) return;
    if (lanes == 32)
        step_kernel<32, 4><<<n_tiles, 128, 0, stream>>>(a);
    else
        step_kernel<8, 16><<<n_tiles, 128, 0, stream>>>(a);
    FRAQ_LAUNCH_CHECK();
}

}  // namespace fraqcu

// ================================================================================ fraq_hist_s
using namespace fraqcu;

struct fraq_hist_s {
    fraq_ctx ctx = nullptr;
    HistDevice d;
    int variant = 0;
    long lo = 0;
    long level = 0, appended = 0;
    bool pending = false;
    DevBuf<double> stage;   // pending push value (device)
    DevBuf<double> outbuf;  // device output for host reads
    DevBuf<int> counter;
    DevBuf<int2> run2_tasks;   // (group, first DOF of a 32-DOF tile) for K5c
    int n_run2_tasks = 0;
    DevBuf<int2> run3_tasks;   // (group, first DOF of a 16-DOF tile) for K5d
    int n_run3_tasks = 0;
    int last_path = 0;
    long launches[6] = {0, 0, 0, 0, 0, 0};  // by path (1: short-state rebuilds, 5: K5f)
    // chunk staging for host-memory runs
    static constexpr int kMaxStages = 4;
    DevBuf<double> ubuf[kMaxStages], dbuf[kMaxStages];
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_u[kMaxStages] = {}, ev_c[kMaxStages] = {}, ev_d[kMaxStages] = {};
    ~fraq_hist_s() {
        if (s_h2d) cudaStreamDestroy(s_h2d);
        if (s_d2h) cudaStreamDestroy(s_d2h);
        for (int i = 0; i < kMaxStages; ++i) {
            if (ev_u[i]) cudaEventDestroy(ev_u[i]);
            if (ev_c[i]) cudaEventDestroy(ev_c[i]);
            if (ev_d[i]) cudaEventDestroy(ev_d[i]);
        }
    }
};

namespace fraqcu {

namespace {

StepArgs base_args(fraq_hist h) {
    StepArgs a{};
    a.groups = h->d.groups.p;
    a.tiles = h->d.tiles.p;
    a.state = h->d.state.p;
    a.ring = h->d.ring.p;
    a.cr = h->d.cr.p;
    a.cf = h->d.cf.p;
    a.head = h->d.head.p;
    a.level = h->level;
    a.appended = h->appended;
    a.lo = (int)h->lo;
    return a;
}

// reference sequencing checks (fast_kernel.cpp:268-273, 343-347)
void check_advance(fraq_hist h) {
    for (const GroupDev& G : h->d.groups_h) {
        const long fi = h->level + 1 - G.L;
        if (fi >= h->lo && fi < h->appended - G.L)
            fail(FRAQ_ELOGIC, G.sbd ? "SbdHistory::advance: feed value already evicted"
                                    : "BeHistory::advance: feed value already evicted");
    }
}

void copy_in(fraq_hist h, double* dst, const double* src, int mem) {
    const size_t bytes = sizeof(double) * h->d.total_dim;
    FRAQ_CUDA(cudaMemcpyAsync(dst, src, bytes,
                              mem == FRAQ_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                              h->ctx->stream));
}

void copy_out(fraq_hist h, double* dst, const double* src, int mem) {
    const size_t bytes = sizeof(double) * h->d.total_dim;
    FRAQ_CUDA(cudaMemcpyAsync(dst, src, bytes,
                              mem == FRAQ_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                              h->ctx->stream));
    if (mem != FRAQ_DEVICE) FRAQ_CUDA(cudaStreamSynchronize(h->ctx->stream));
}

// A K5 launch that appends a value at level h->appended (before the counters move): in a pure
// push sequence (`pure`) the kernel also records the value in K5e's / K5f's input ring; anything
// else invalidates the ring.
void record_append(fraq_hist h, StepArgs& a, bool pure) {
    FirPlan& P = h->d.fir;
    if (pure && P.ok) {
        a.xh = P.xh.p;
        a.ldx = h->d.total_dim;
        a.xh_mask = P.xh_rows - 1;
        P.xh_valid = std::min<long>(P.xh_rows, P.xh_valid + 1);
    } else {
        P.xh_valid = 0;
    }
}
bool pure_push(fraq_hist h) {
    return h->appended == 0 ? h->level == 0 : h->level == h->appended - 1;
}

// Run a pending push (advance + append from the stage) fused with `mode` output into out_d.
void flush(fraq_hist h, int mode, double* out_d) {
    StepArgs a = base_args(h);
    if (h->pending) {
        a.adv = h->appended > 0;
        a.app = 1;
        a.u = h->stage.p;
    }
    a.mode = mode;
    a.out = out_d;
    if (!a.adv && !a.app && mode == MODE_NONE) return;
    if (step_fir_eligible(h->d, h->level, h->appended, h->pending)) {
        // K5f: the folded per-level step (steady state of a pure push sequence)
        launch_step_fir(h->ctx, h->d, h->appended, h->pending ? 1 : 0, mode, h->stage.p, out_d);
        ++h->launches[5];
    } else {
        fir_materialize(h->ctx, h->d, h->appended);  // K5 reads every node's state
        if (h->pending) record_append(h, a, pure_push(h));
        h->d.launch_step(h->ctx, a);
        ++h->launches[0];
    }
    if (h->pending) {
        if (h->appended > 0) h->level += 1;
        h->appended += 1;
        h->pending = false;
    }
}

}  // namespace

void hist_create(fraq_ctx c, int n_groups, const fraq_kernel_t* const* ks, const long* dims,
                 int variant, fraq_hist* out) {
    check_ctx(c);
    if (n_groups < 1) fail(FRAQ_EINVAL, "history: need at least one group");
    for (int g = 0; g < n_groups; ++g) {
        if (!ks[g]) fail(FRAQ_EINVAL, "history: null kernel");
        if (dims[g] < 0) fail(FRAQ_EINVAL, "history: negative dim");
        const fraq_kernel_t& k = *ks[g];
        if (k.np1 < 0 || k.np2 < 0 || k.np1 + k.np2 > 2 * FRAQ_MAX_POINTS || k.n_head < 2 ||
            k.n_head > FRAQ_MAX_HEAD)
            fail(FRAQ_EINVAL, "history: malformed kernel tables");
    }
    auto* h = new fraq_hist_s();
    try {
        h->ctx = c;
        h->variant = variant;
        h->lo = variant == FRAQ_STANDALONE ? 0 : 1;
        h->d.build(c, n_groups, ks, dims);
        h->stage.alloc(std::max<long>(1, h->d.total_dim));
        h->outbuf.alloc(std::max<long>(1, h->d.total_dim));
        h->counter.alloc(1);
        std::vector<int2> t2;
        for (int g = 0; g < n_groups; ++g)
            for (int m0 = 0; m0 < h->d.groups_h[g].dim; m0 += 32) t2.push_back(make_int2(g, m0));
        std::vector<int2> t3;
        for (int g = 0; g < n_groups; ++g)
            for (int m0 = 0; m0 < h->d.groups_h[g].dim; m0 += 16) t3.push_back(make_int2(g, m0));
        h->n_run3_tasks = (int)t3.size();
        h->run3_tasks.alloc(std::max<size_t>(1, t3.size()));
        if (!t3.empty())
            FRAQ_CUDA(cudaMemcpy(h->run3_tasks.p, t3.data(), t3.size() * sizeof(int2),
                                 cudaMemcpyHostToDevice));
        // K5e plan (host tables, input ring) with the history, not inside its first run
        if (h->d.max_L <= run3_max_lag() && !std::getenv("FRAQ_K5C")) build_fir_plan(c, h->d);
        h->n_run2_tasks = (int)t2.size();
        h->run2_tasks.alloc(std::max<size_t>(1, t2.size()));
        if (!t2.empty())
            FRAQ_CUDA(cudaMemcpy(h->run2_tasks.p, t2.data(), t2.size() * sizeof(int2),
                                 cudaMemcpyHostToDevice));
    } catch (...) {
        delete h;
        throw;
    }
    *out = h;
}

void hist_destroy(fraq_hist h) {
    if (!h) return;
    cudaStreamSynchronize(h->ctx->stream);
    delete h;
}

void hist_info(fraq_hist h, long* level, long* appended, long* dim) {
    // a pending push is already reflected in the reference counters
    if (level) *level = h->level + ((h->pending && h->appended > 0) ? 1 : 0);
    if (appended) *appended = h->appended + (h->pending ? 1 : 0);
    if (dim) *dim = h->d.total_dim;
}

void hist_push(fraq_hist h, const double* v, int mem) {
    check_ctx(h->ctx);
    if (h->pending) flush(h, MODE_NONE, nullptr);
    if (h->appended > 0) check_advance(h);
    copy_in(h, h->stage.p, v, mem);
    h->pending = true;
}

void hist_advance(fraq_hist h) {
    check_ctx(h->ctx);
    if (h->pending) flush(h, MODE_NONE, nullptr);
    check_advance(h);
    StepArgs a = base_args(h);
    a.adv = 1;
    fir_materialize(h->ctx, h->d, h->appended);
    h->d.launch_step(h->ctx, a);
    h->level += 1;
}

void hist_append(fraq_hist h, const double* v, int mem) {
    check_ctx(h->ctx);
    if (h->pending) flush(h, MODE_NONE, nullptr);
    copy_in(h, h->stage.p, v, mem);
    StepArgs a = base_args(h);
    a.app = 1;
    a.u = h->stage.p;
    // advance() then append() is a push: the input ring stays current (K5e / K5f can follow)
    record_append(h, a, h->appended == 0 ? h->level == 0 : h->level == h->appended);
    h->d.launch_step(h->ctx, a);
    ++h->launches[0];
    h->appended += 1;
}

void hist_output(fraq_hist h, int mode, double* out, int mem) {
    check_ctx(h->ctx);
    if (mode == MODE_DERIV) {
        const long app = h->appended + (h->pending ? 1 : 0);
        for (const GroupDev& G : h->d.groups_h) {
            if (!G.sbd && app < 2)
                fail(FRAQ_ELOGIC, "BeHistory::derivative: need at least two pushed values");
            if (G.sbd && app < 1) fail(FRAQ_ELOGIC, "SbdHistory::derivative: no values pushed");
        }
    }
    double* dst = mem == FRAQ_DEVICE ? out : h->outbuf.p;
    if (mem == FRAQ_DEVICE && h->d.total_dim == 0) return;
    flush(h, mode, dst);
    if (!h->pending && mode != MODE_NONE && h->d.total_dim > 0) {
        // flush() launched the fused kernel only if there was pending work; otherwise read-only
    }
    if (mem != FRAQ_DEVICE) copy_out(h, out, h->outbuf.p, FRAQ_HOST);
}

void hist_lagged(fraq_hist h, long depth, double* out, int mem) {
    check_ctx(h->ctx);
    if (h->pending) flush(h, MODE_NONE, nullptr);
    const long idx = h->appended - 1 - depth;
    for (const GroupDev& G : h->d.groups_h)
        if (idx < 0 || depth < 0 || depth >= G.L)
            fail(FRAQ_ERANGE, G.sbd ? "SbdHistory::lagged: value not retained"
                                    : "BeHistory::lagged: value not retained");
    for (const GroupDev& G : h->d.groups_h) {
        const double* src = h->d.ring.p + G.ring_off + (idx % G.L) * (long)G.ld;
        FRAQ_CUDA(cudaMemcpyAsync((mem == FRAQ_DEVICE ? out : h->outbuf.p) + G.dof0, src,
                                  sizeof(double) * G.dim, cudaMemcpyDeviceToDevice, h->ctx->stream));
    }
    if (mem != FRAQ_DEVICE) copy_out(h, out, h->outbuf.p, FRAQ_HOST);
}

namespace {

bool blocked_ok(fraq_hist h) {
    if (!h->d.ztrick_ok) return false;
    if (h->d.max_L > R2_LMAX || h->d.max_J > 32 * 16) return false;
    // pure push sequence: level == appended - 1 (or fresh)
    if (h->appended == 0) return h->level == 0;
    return h->level == h->appended - 1;
}

void run_device(fraq_hist h, const double* U, long ldu, long n_steps, double* D, long ldd) {
    if (n_steps <= 0) return;
    if (blocked_ok(h) && n_steps >= 4) {
        RunArgs a{};
        a.groups = h->d.groups.p;
        a.counter = h->counter.p;
        a.state = h->d.state.p;
        a.ring = h->d.ring.p;
        a.cr = h->d.cr.p;
        a.cf = h->d.cf.p;
        a.head = h->d.head.p;
        a.lo = (int)h->lo;
        a.ldu = ldu;
        a.ldd = ldd;
        const int P = (h->d.max_J + 31) / 32;
        static const bool k5c = std::getenv("FRAQ_K5C") != nullptr;
        const bool k5d = !k5c && h->d.max_L <= run3_max_lag();
        if (k5d) build_fir_plan(h->ctx, h->d);
        // TMA boxes start at a group's first DOF + 16 i: 16-byte aligned only for even starts
        bool even_groups = true;
        for (const GroupDev& G : h->d.groups_h) even_groups = even_groups && (G.dof0 % 2 == 0);
        const FirPlan& fp = h->d.fir;
        // The call runs as up to three launches: K5d until the steady-state form is valid (the
        // first levels of a history), K5e on whole 8-level blocks, K5d on a ragged tail.
        for (long done = 0; done < n_steps;) {
            const long A0 = h->appended, rest = n_steps - done;
            const double* Uc = U + done * ldu;
            double* Dc = D ? D + done * ldd : nullptr;
            long m = rest;
            FRAQ_CUDA(cudaMemsetAsync(h->counter.p, 0, sizeof(int), h->ctx->stream));
            if (k5d && even_groups && fir_eligible(h->d, A0, Uc, ldu, rest & ~7L, Dc, ldd)) {
                // K5e: short nodes as an exact FIR, long nodes in K5d's block form
                m = rest & ~7L;
                h->last_path = 4;
                ++h->launches[4];
                launch_run4(h->ctx, h->d, h->run3_tasks.p, h->n_run3_tasks, h->counter.p, A0, Uc,
                            ldu, m, Dc, ldd);
            } else {
                if (k5d && fp.ok) {
                    // K5d up to the level K5e can take over from: past min_level, with the last
                    // kw_max input rows on record
                    const long s = std::max<long>(std::max(fp.min_level, fp.kw_max),
                                                  A0 + (fp.xh_valid >= fp.kw_max ? 0 : fp.kw_max));
                    const long pre = (s - A0 + 31) / 32 * 32;
                    if (pre > 0 && pre + 64 <= rest) m = pre;
                }
                if (h->d.fir.short_stale) ++h->launches[1];
                fir_materialize(h->ctx, h->d, A0);
                a.A0 = A0;
                a.n_steps = m;
                a.U = Uc;
                a.D = Dc;
                if (k5d) {
                    // K5d (DMMA block formulation)
                    h->last_path = 3;
                    ++h->launches[3];
                    build_frag_tables(h->ctx, h->d);
                    a.tasks = h->run3_tasks.p;
                    a.n_tasks = h->n_run3_tasks;
                    a.frag = h->d.frag.p;
                    launch_run3(a, std::max(1, (h->d.max_J + 63) / 64), h->ctx->num_sms,
                                h->ctx->stream, even_groups);
                } else {
                    h->last_path = 2;
                    ++h->launches[2];
                    a.tasks = h->run2_tasks.p;
                    a.n_tasks = h->n_run2_tasks;
                    launch_run2(a, std::max(1, P), h->ctx->num_sms, h->ctx->stream);
                }
            }
            fir_note_inputs(h->ctx, h->d, A0, Uc, ldu, m);
            h->appended += m;
            h->level = h->appended - 1;
            done += m;
        }
        return;
    }
    h->last_path = 0;
    for (long n = 0; n < n_steps; ++n) {
        if (h->appended > 0) check_advance(h);
        StepArgs a = base_args(h);
        a.adv = h->appended > 0;
        a.app = 1;
        a.u = U + n * ldu;
        bool ok = true;
        for (const GroupDev& G : h->d.groups_h)
            if (!G.sbd && h->appended + 1 < 2) ok = false;
        a.mode = (D && ok) ? MODE_DERIV : MODE_NONE;
        a.out = D ? D + n * ldd : nullptr;
        if (step_fir_eligible(h->d, h->level, h->appended, true)) {
            launch_step_fir(h->ctx, h->d, h->appended, 1, a.mode, a.u, a.out);
            ++h->launches[5];
        } else {
            fir_materialize(h->ctx, h->d, h->appended);
            record_append(h, a, pure_push(h));
            h->d.launch_step(h->ctx, a);
            ++h->launches[0];
        }
        if (D && !ok) {
            // derivative undefined on the first BE push: NaN row (the reference throws)
            std::vector<double> nan(h->d.total_dim, NAN);
            FRAQ_CUDA(cudaMemcpyAsync(D + n * ldd, nan.data(), sizeof(double) * nan.size(),
                                      cudaMemcpyHostToDevice, h->ctx->stream));
            FRAQ_CUDA(cudaStreamSynchronize(h->ctx->stream));
        }
        if (h->appended > 0) h->level += 1;
        h->appended += 1;
    }
}

}  // namespace

void hist_run(fraq_hist h, const double* U, long ldu, long n_steps, double* D, long ldd, int mem) {
    check_ctx(h->ctx);
    if (n_steps < 0) fail(FRAQ_EINVAL, "hist_run: negative n_steps");
    if (ldu < h->d.total_dim || (D && ldd < h->d.total_dim))
        fail(FRAQ_EINVAL, "hist_run: leading dimension below dim");
    if (h->pending) flush(h, MODE_NONE, nullptr);
    if (mem == FRAQ_DEVICE) {
        run_device(h, U, ldu, n_steps, D, ldd);
        return;
    }
    // host buffers: chunks of rows through two device staging buffers.  Copies run on their
    // own streams so the H2D of chunk i+1 and the D2H of chunk i-1 overlap the kernel on chunk
    // i (the kernels themselves are sequential: each chunk continues the history state).
    // Pinned host memory gives full overlap; pageable memory still works (staged copies).
    const long dim = std::max<long>(1, h->d.total_dim);
    // chunk height: ~1/16 of the call in multiples of the kernel's 32-level staging chunk, at most
    // ~32 MB per chunk (but 32 levels at least), with shorter chunks at both ends (below) so the
    // pipeline fill (first H2D) and drain (last D2H) stay short.  (C2, 65536 DOFs, K5e, e2e in 1e9
    // DOF-steps/s: uniform 32 / 64-level chunks 4.74 / 4.77; ramped 32 / 64 / 128: 4.68 / 5.02 /
    // 4.91 -- profiles/r02/e2e_ramp.sh.)
    const long cap = std::max<long>(32, ((32L << 20) / (8 * dim)) / 32 * 32);
    long rows = std::min<long>(cap, std::max<long>(32, ((n_steps / 16 + 31) / 32) * 32));
    const char* ce = std::getenv("FRAQ_HOST_CHUNK");  // experiment override (levels per chunk)
    if (ce && *ce) rows = std::max<long>(1, std::atol(ce));
    rows = std::max<long>(1, std::min<long>(rows, std::max<long>(1, n_steps)));
    // a remainder under 32 rows joins the last chunk (keeps it on the blocked kernels)
    const long cap_rows = rows + 31;
    // staging depth: copies may run up to ns - 1 chunks ahead of / behind the kernel
    int ns = 2;
    if (const char* es = std::getenv("FRAQ_HOST_STAGES"))  // experiment override
        if (*es) ns = std::max(2, std::min(fraq_hist_s::kMaxStages, std::atoi(es)));
    for (int i = 0; i < ns; ++i) {
        if ((long)h->ubuf[i].n < cap_rows * dim) h->ubuf[i].alloc(cap_rows * dim);
        if (D && (long)h->dbuf[i].n < cap_rows * dim) h->dbuf[i].alloc(cap_rows * dim);
        if (!h->ev_u[i]) {
            FRAQ_CUDA(cudaEventCreateWithFlags(&h->ev_u[i], cudaEventDisableTiming));
            FRAQ_CUDA(cudaEventCreateWithFlags(&h->ev_c[i], cudaEventDisableTiming));
            FRAQ_CUDA(cudaEventCreateWithFlags(&h->ev_d[i], cudaEventDisableTiming));
        }
    }
    if (!h->s_h2d) {
        FRAQ_CUDA(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
        FRAQ_CUDA(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    }
    cudaStream_t sc = h->ctx->stream;
    // copies may only start after earlier work on the compute stream (state + buffers)
    for (int j = 0; j < ns; ++j) {
        FRAQ_CUDA(cudaEventRecord(h->ev_c[j], sc));
        FRAQ_CUDA(cudaEventRecord(h->ev_d[j], sc));
    }
    // chunk schedule: `rows` per chunk, with shorter chunks at both ends of a long call (rows/4,
    // rows/2, ..., rows/2, rows/4; multiples of 8, so they stay on K5e) -- the first H2D and the
    // last D2H are the only copies nothing overlaps
    std::vector<long> sched;
    {
        static const bool ramp_on = !std::getenv("FRAQ_HOST_NORAMP");
        const long r4 = rows / 4 / 8 * 8, r2 = rows / 2 / 8 * 8;
        long left = n_steps;
        const bool ramp = ramp_on && r4 >= 8 && n_steps >= 6 * rows;
        if (ramp) {
            sched.push_back(r4);
            sched.push_back(r2);
            left -= r4 + r2 + r2 + r4;
        }
        while (left > 0) {
            const long nr = (left - rows < 32) ? left : rows;
            sched.push_back(nr);
            left -= nr;
        }
        if (ramp) {
            sched.push_back(r2);
            sched.push_back(r4);
        }
    }
    long i = 0;
    for (long n0 = 0, nr = 0; n0 < n_steps; n0 += nr, ++i) {
        const int b = (int)(i % ns);
        nr = sched[i];
        // H2D into ubuf[b] once the kernel that last read it (chunk i - ns) finished
        FRAQ_CUDA(cudaStreamWaitEvent(h->s_h2d, h->ev_c[b], 0));
        if (ldu == dim)  // contiguous rows: one linear copy
            FRAQ_CUDA(cudaMemcpyAsync(h->ubuf[b].p, U + n0 * ldu, (size_t)nr * dim * 8,
                                      cudaMemcpyHostToDevice, h->s_h2d));
        else
            FRAQ_CUDA(cudaMemcpy2DAsync(h->ubuf[b].p, dim * 8, U + n0 * ldu, ldu * 8,
                                        h->d.total_dim * 8, nr, cudaMemcpyHostToDevice, h->s_h2d));
        FRAQ_CUDA(cudaEventRecord(h->ev_u[b], h->s_h2d));
        // kernel on chunk i: needs its inputs and dbuf[b] drained by the D2H of chunk i - ns
        FRAQ_CUDA(cudaStreamWaitEvent(sc, h->ev_u[b], 0));
        if (D) FRAQ_CUDA(cudaStreamWaitEvent(sc, h->ev_d[b], 0));
        run_device(h, h->ubuf[b].p, dim, nr, D ? h->dbuf[b].p : nullptr, dim);
        FRAQ_CUDA(cudaEventRecord(h->ev_c[b], sc));
        if (D) {
            FRAQ_CUDA(cudaStreamWaitEvent(h->s_d2h, h->ev_c[b], 0));
            if (ldd == dim)
                FRAQ_CUDA(cudaMemcpyAsync(D + n0 * ldd, h->dbuf[b].p, (size_t)nr * dim * 8,
                                          cudaMemcpyDeviceToHost, h->s_d2h));
            else
                FRAQ_CUDA(cudaMemcpy2DAsync(D + n0 * ldd, ldd * 8, h->dbuf[b].p, dim * 8,
                                            h->d.total_dim * 8, nr, cudaMemcpyDeviceToHost,
                                            h->s_d2h));
            FRAQ_CUDA(cudaEventRecord(h->ev_d[b], h->s_d2h));
        }
    }
    FRAQ_CUDA(cudaStreamSynchronize(h->s_h2d));
    FRAQ_CUDA(cudaStreamSynchronize(sc));
    FRAQ_CUDA(cudaStreamSynchronize(h->s_d2h));
}

int hist_last_path(fraq_hist h) { return h->last_path; }
void hist_path_info(fraq_hist h, long* launches, int n_groups, int* fir) {
    if (launches)
        for (int i = 0; i < 6; ++i) launches[i] = h->launches[i];
    if (fir)
        for (int g = 0; g < n_groups; ++g) {
            const bool have = h->d.fir.ok && g < (int)h->d.fir.groups_h.size();
            fir[3 * g + 0] = have ? h->d.fir.groups_h[g].M : 0;
            fir[3 * g + 1] = have ? h->d.fir.groups_h[g].JL : 0;
            fir[3 * g + 2] = have ? h->d.fir.groups_h[g].KW : 0;
        }
}
fraq_ctx hist_ctx(fraq_hist h) { return h->ctx; }

}  // namespace fraqcu
