// Microbenchmark (not part of the library): which ingredient of K5d's block loop costs the fp64
// tensor pipe its last 25%?  The kernel replays K5d's per-warp instruction mix (readout GEMM from
// accumulator fragments, state GEMM, r^8 rescale, B fragments from shared memory, partial tiles,
// pair barrier, cross-warp reduction) with each ingredient behind a template flag.
//   RB    row blocks (8 DOFs each) per warp            (K5d: 2)
//   NT    node tiles (8 nodes each) per warp           (K5d: 8)
//   WARPS warps per CTA, CPS CTAs per SM               (K5d: 8, 2)
// Prints DMMA TFLOP/s per variant (512 flops per DMMA).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_k5dmix mb_k5dmix.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

enum { F_LDSB = 1, F_DMUL = 2, F_SYNC = 4, F_PART = 8, F_VF = 16, F_R8LDS = 32 };

template <int RB, int NT, int WARPS, int CPS, int FLAGS>
__global__ void __launch_bounds__(WARPS * 32, CPS) mix(double* out, int iters) {
    extern __shared__ __align__(128) double sm[];
    constexpr int TILES = WARPS * NT;
    double* tabC = sm;                      // [TILES][2][32]
    double* tabR = tabC + TILES * 64;       // [TILES][2][32]
    double* X = tabR + TILES * 64;          // [96][8 RB]
    double* part = X + 96 * 8 * RB;         // [2][2][WARPS][RB*64]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
    for (int i = tid; i < TILES * 64; i += WARPS * 32) {
        tabC[i] = 0.5 + 1e-4 * (i & 63);
        tabR[i] = 1e-3 * ((i & 31) + 1);
    }
    for (int i = tid; i < 96 * 8 * RB; i += WARPS * 32) X[i] = 1e-3 * (i & 127);
    __syncthreads();
    double Y[RB][NT][2];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
        for (int n = 0; n < NT; ++n) Y[rb][n][0] = Y[rb][n][1] = 1e-3 * (lane + n + rb);
    const double* cw = tabC + warp * NT * 64 + lane;
    const double* rw = tabR + warp * NT * 64 + lane;
    const double* r8w = tabC + warp * NT * 64 + 28 + t;
    double breg = 0.5 + 1e-6 * lane, r8reg = 0.75;
    double tot = 0.0;
    int buf = 0, xr = 0;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
#pragma unroll 1
        for (int blk = 0; blk < 2; ++blk) {
            xr = xr >= 88 ? 0 : xr + 8;
            double sacc[RB][2];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) sacc[rb][0] = sacc[rb][1] = 0.0;
#pragma unroll
            for (int n = 0; n < NT; ++n)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const double b = (FLAGS & F_LDSB) ? cw[(n * 2 + e) * 32] : breg;
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb) dmma(sacc[rb], Y[rb][n][e], b);
                }
            double vf[RB][2];
#pragma unroll
            for (int rb = 0; rb < RB; ++rb)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    vf[rb][h] = (FLAGS & F_VF)
                                    ? X[(xr + 4 * h + t) * 8 * RB + 8 * rb + g]
                                    : 1e-3 * (rb + h + 1);
            if (FLAGS & F_DMUL) {
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const double ra = (FLAGS & F_R8LDS) ? r8w[(n * 2) * 32] : r8reg;
                    const double rbv = (FLAGS & F_R8LDS) ? r8w[(n * 2 + 1) * 32] : r8reg;
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb) {
                        Y[rb][n][0] *= ra;
                        Y[rb][n][1] *= rbv;
                    }
                }
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    const double b = (FLAGS & F_LDSB) ? rw[(n * 2 + h) * 32] : breg;
#pragma unroll
                    for (int rb = 0; rb < RB; ++rb) dmma(Y[rb][n], vf[rb][h], b);
                }
            if (FLAGS & F_PART) {
                double* pw = part + ((size_t)(buf * 2 + blk) * WARPS + warp) * (RB * 64);
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) {
                    pw[(2 * t) * 8 * RB + 8 * rb + g] = sacc[rb][0];
                    pw[(2 * t + 1) * 8 * RB + 8 * rb + g] = sacc[rb][1];
                }
            } else {
#pragma unroll
                for (int rb = 0; rb < RB; ++rb) tot += sacc[rb][0] + sacc[rb][1];
            }
        }
        if (FLAGS & F_SYNC) __syncthreads();
        if (FLAGS & F_PART) {
            // reduction of the pair just finished (K5d defers it behind the next readout; the
            // order matters little here because the other CTA / warps fill the pipe)
            for (int o = tid; o < 2 * 8 * 8 * RB; o += WARPS * 32) {
                const int slot = o / (64 * RB), r = o % (64 * RB);
                const double* pb = part + ((size_t)(buf * 2 + slot) * WARPS) * (RB * 64) + r;
                double s0 = 0.0, s1 = 0.0;
#pragma unroll
                for (int w = 0; w < WARPS; w += 2) {
                    s0 += pb[w * RB * 64];
                    s1 += pb[(w + 1) * RB * 64];
                }
                tot += s0 + s1;
            }
            buf ^= 1;
        }
    }
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
        for (int n = 0; n < NT; ++n) tot += Y[rb][n][0] + Y[rb][n][1];
    if (tot == 1.2345) out[tid] = tot;
}

template <int RB, int NT, int WARPS, int CPS, int FLAGS>
void run(const char* name, double* out) {
    constexpr int TILES = WARPS * NT;
    const size_t smem = sizeof(double) * (TILES * 128 + 96 * 8 * RB + 4 * WARPS * RB * 64);
    auto kern = mix<RB, NT, WARPS, CPS, FLAGS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem);
    const int grid = 148 * CPS, iters = 4000;
    kern<<<grid, WARPS * 32, smem>>>(out, 50);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<grid, WARPS * 32, smem>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = (double)grid * WARPS * iters * 2.0 * (2.0 * RB * NT * 2) * 512.0;
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    printf("%-44s RB%d NT%d W%2d x%d regs %3d occ %d smem %6zu: %6.2f TFLOP/s  (%s)\n", name, RB, NT,
           WARPS, CPS, fa.numRegs, per_sm, smem, fl / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    cudaMalloc(&out, 1 << 16);
    constexpr int ALL = F_LDSB | F_DMUL | F_SYNC | F_PART | F_VF | F_R8LDS;
    run<2, 8, 8, 2, 0>("pure DMMA, B in a register", out);
    run<2, 8, 8, 2, F_LDSB>("+ B fragments from LDS", out);
    run<2, 8, 8, 2, F_LDSB | F_VF>("+ B LDS + vf LDS", out);
    run<2, 8, 8, 2, F_DMUL>("DMUL only (reg operands)", out);
    run<2, 8, 8, 2, F_LDSB | F_DMUL | F_R8LDS>("B LDS + DMUL (r8 from LDS)", out);
    run<2, 8, 8, 2, F_SYNC>("pair barrier only", out);
    run<2, 8, 8, 2, F_LDSB | F_SYNC>("B LDS + pair barrier", out);
    run<2, 8, 8, 2, F_LDSB | F_SYNC | F_PART>("B LDS + barrier + partial/reduce", out);
    run<2, 8, 8, 2, ALL>("all (K5d mix)", out);
    run<2, 8, 8, 2, ALL & ~F_SYNC>("all without the barrier", out);
    run<2, 8, 8, 2, ALL & ~(F_DMUL | F_R8LDS)>("all without DMUL", out);
    // one 16-warp CTA per SM, same per-warp shape
    run<2, 8, 16, 1, 0>("16-warp CTA: pure", out);
    run<2, 8, 16, 1, F_LDSB>("16-warp CTA: B LDS", out);
    run<2, 8, 16, 1, ALL>("16-warp CTA: all", out);
    // 32 DOFs x 32 nodes per warp: one B fragment feeds four row blocks
    run<4, 4, 16, 1, 0>("RB4 NT4: pure", out);
    run<4, 4, 16, 1, F_LDSB>("RB4 NT4: B LDS", out);
    run<4, 4, 16, 1, F_LDSB | F_DMUL | F_R8LDS>("RB4 NT4: B LDS + DMUL", out);
    run<4, 4, 16, 1, ALL>("RB4 NT4: all", out);
    run<4, 4, 8, 2, F_LDSB>("RB4 NT4 8 warps x2: B LDS", out);
    run<4, 4, 8, 2, ALL>("RB4 NT4 8 warps x2: all", out);
    // fewer, fatter warps: 4 warps x 2 CTAs (K13's lever), 128 nodes per warp
    run<2, 16, 4, 2, F_LDSB>("RB2 NT16 4 warps x2: B LDS", out);
    run<2, 16, 4, 2, ALL>("RB2 NT16 4 warps x2: all", out);
    run<2, 8, 4, 4, F_LDSB>("RB2 NT8 4 warps x4: B LDS", out);
    run<2, 8, 4, 4, ALL>("RB2 NT8 4 warps x4: all", out);
    run<2, 8, 4, 3, ALL>("RB2 NT8 4 warps x3: all", out);
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
