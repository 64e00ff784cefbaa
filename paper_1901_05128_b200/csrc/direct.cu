// direct.cu -- K10: direct O(N^2) convolution quadrature on the fp64 tensor cores.
//
// D[n][m] = sum_{i=0}^{n} d_i U[n-i][m] with the classical weights d (be_weights/sbd_weights,
// cq_weights.cpp:29-59): the reference's direct sum (test_fast_kernel.cpp:27-41,
// acceptance_main.cpp:158-159; a20 in SURVEY.md §8a), i.e. a lower-triangular Toeplitz matrix
// T[n][j] = d_{n-j} times the signal matrix U[j][m].  It is a GEMM, so it runs on DMMA
// (mma.sync m8n8k4 f64 -> DMMA.8x8x4): CTA tile 64 (levels) x 64 (DOFs), 4 warps of 32 x 32,
// K-tiles of 16 source levels staged in shared memory (Toeplitz tile generated from d), only
// K-tiles on or below the diagonal visited.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.cuh"

namespace fraqcu {
namespace {

constexpr int DT_M = 64;   // levels per CTA tile
constexpr int DT_N = 64;   // DOFs per CTA tile
constexpr int DT_K = 16;   // source levels per K-tile

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// grid: (ceil(dim/64), ceil(n_steps/64)); block 128 threads (4 warps, 2 x 2 of 32 x 32)
__global__ void __launch_bounds__(128) toeplitz_kernel(const double* __restrict__ w,
                                                       const double* __restrict__ U, long ldu,
                                                       long n_steps, long dim, double* D,
                                                       long ldd) {
    __shared__ double sA[2][DT_M][DT_K + 1];  // Toeplitz tile A[n][j] = w[n - j] (0 above diag)
    __shared__ double sB[2][DT_K][DT_N + 1];  // signal tile B[j][m]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const long n0 = (long)blockIdx.y * DT_M, m0 = (long)blockIdx.x * DT_N;
    const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;  // warp sub-tile origin
    const int g = lane >> 2, t = lane & 3;
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    // the next K-tile's operands are fetched into registers while the current tile's DMMAs run
    // (as K12 does); one barrier per K-tile
    constexpr int PA = DT_M * DT_K / 128, PB = DT_K * DT_N / 128;
    double ra[PA], rb[PB];
    auto fetch = [&](long j0) {
#pragma unroll
        for (int q = 0; q < PA; ++q) {
            const int idx = tid + 128 * q, r = idx / DT_K, c = idx % DT_K;
            const long n = n0 + r, j = j0 + c;
            ra[q] = (j <= n && n < n_steps) ? __ldg(w + (n - j)) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int idx = tid + 128 * q, r = idx / DT_N, c = idx % DT_N;
            const long j = j0 + r, m = m0 + c;
            rb[q] = (j < n_steps && m < dim) ? __ldg(U + j * ldu + m) : 0.0;
        }
    };
    auto put = [&](int buf) {
#pragma unroll
        for (int q = 0; q < PA; ++q) {
            const int idx = tid + 128 * q;
            sA[buf][idx / DT_K][idx % DT_K] = ra[q];
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) {
            const int idx = tid + 128 * q;
            sB[buf][idx / DT_N][idx % DT_N] = rb[q];
        }
    };
    const long kend = min(n0 + DT_M, n_steps);  // source levels j < kend (lower triangle)
    fetch(0);
    put(0);
    __syncthreads();
    int buf = 0;
    for (long j0 = 0; j0 < kend; j0 += DT_K) {
        const bool more = j0 + DT_K < kend;
        if (more) fetch(j0 + DT_K);
#pragma unroll
        for (int kk = 0; kk < DT_K; kk += 4) {
            double af[4], bf[4];
#pragma unroll
            for (int a = 0; a < 4; ++a) af[a] = sA[buf][wm + 8 * a + g][kk + t];  // A: row g, col t
#pragma unroll
            for (int b = 0; b < 4; ++b) bf[b] = sB[buf][kk + t][wn + 8 * b + g];  // B: row t, col g
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int b = 0; b < 4; ++b) dmma884(acc[a][b], af[a], bf[b]);
        }
        if (more) put(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    // C/D fragment: row g, cols 2t, 2t+1
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const long n = n0 + wm + 8 * a + g, m = m0 + wn + 8 * b + 2 * t + e;
                if (n < n_steps && m < dim) D[n * ldd + m] = acc[a][b][e];
            }
}

}  // namespace

void direct_cq_dev(fraq_ctx c, int sbd, double g, double tau, const double* U, long ldu,
                   long n_steps, long dim, double* D, long ldd) {
    if (n_steps <= 0 || dim <= 0) return;
    DevBuf<double> w((size_t)n_steps);
    if (sbd)
        sbd_weights_dev(c, g, tau, n_steps - 1, w.p);
    else
        be_weights_dev(c, g, tau, n_steps - 1, w.p);
    dim3 grid((unsigned)((dim + DT_N - 1) / DT_N), (unsigned)((n_steps + DT_M - 1) / DT_M));
    toeplitz_kernel<<<grid, 128, 0, c->stream>>>(w.p, U, ldu, n_steps, dim, D, ldd);
    FRAQ_LAUNCH_CHECK();
    FRAQ_CUDA(cudaStreamSynchronize(c->stream));
}

}  // namespace fraqcu
