// Microbenchmark (not part of the library): throughput of the K5c inner block on B200.
//   variant 0: the K5c block (z = fma(r, z, v_k); s_k = fma(f, z, s_k)), 32 nodes x 8 levels,
//              r/f from shared memory (broadcast), no barriers
//   variant 1: variant 0 + __syncthreads() after every block
//   variant 2: variant 0 with r/f held in registers (no LDS)
//   variant 3: z-chain only (z = fma(r, z, v_k)), no readout
//   variant 4: 16 levels per block (half the LDS per DFMA)
// Prints DFMA TFLOP/s (2 flops per DFMA) per variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_block mb_block.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int VAR, int TB>
__global__ void __launch_bounds__(512, 1) blk(double* out, int iters) {
    __shared__ double cr[512], cf[512], X[64][32];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int j = tid; j < 512; j += 512) {
        cr[j] = 0.999 - 1e-4 * j;
        cf[j] = 1e-3 * (j + 1);
    }
    for (int i = tid; i < 64 * 32; i += 512) X[i / 32][i % 32] = 1e-3 * i;
    __syncthreads();
    double z[32];
#pragma unroll
    for (int p = 0; p < 32; ++p) z[p] = p * 1e-3;
    double rreg[32], freg[32];
    if (VAR == 2) {
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            rreg[p] = cr[warp * 32 + p];
            freg[p] = cf[warp * 32 + p];
        }
    }
    double tot = 0.0;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        double v[TB], s[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) {
            v[k] = X[(it + k) & 63][lane];
            s[k] = 0.0;
        }
#pragma unroll
        for (int p0 = 0; p0 < 32; p0 += 4) {
            double rr[4], ff[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                rr[i] = VAR == 2 ? rreg[p0 + i] : cr[warp * 32 + p0 + i];
                ff[i] = VAR == 2 ? freg[p0 + i] : cf[warp * 32 + p0 + i];
            }
#pragma unroll
            for (int k = 0; k < TB; ++k)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    z[p0 + i] = fma(rr[i], z[p0 + i], v[k]);
                    if (VAR != 3) s[k] = fma(ff[i], z[p0 + i], s[k]);
                }
        }
#pragma unroll
        for (int k = 0; k < TB; ++k) tot += s[k];
        if (VAR == 1) __syncthreads();
    }
#pragma unroll
    for (int p = 0; p < 32; ++p) tot += z[p];
    if (tot == 1.2345) out[tid] = tot;
}

template <int VAR, int TB>
void run(const char* name, double* out) {
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    blk<VAR, TB><<<148, 512>>>(out, 10);
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0);
        blk<VAR, TB><<<148, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    const double dfma = 148.0 * 512 * iters * 32 * TB * (VAR == 3 ? 1 : 2);
    printf("%-40s %8.3f ms  %6.2f TFLOP/s\n", name, best, 2 * dfma / (best * 1e-3) / 1e12);
}

int main() {
    double* out;
    cudaMalloc(&out, 512 * sizeof(double));
    run<0, 8>("v0 K5c block (smem r/f, TB=8)", out);
    run<1, 8>("v1 + barrier per block", out);
    run<2, 8>("v2 r/f in registers", out);
    run<3, 8>("v3 z-chain only", out);
    run<0, 16>("v4 TB=16", out);
    cudaError_t e = cudaGetLastError();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
