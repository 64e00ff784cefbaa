// Which SM sub-partition does each warp of a 320-thread CTA land on when two CTAs share an SM
// (K13's shape: 8 GEMM warps + 2 solver warps)?  Records %smid and %warpid (slot; SMSP =
// slot % 4) per warp; prints the solver warps' SMSPs per co-resident CTA pair.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(320, 2) probe(int* out, long long spin) {
    unsigned sm, ws;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(ws));
    extern __shared__ double pad[];
    long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
    if ((threadIdx.x & 31) == 0) {
        const int w = threadIdx.x >> 5;
        out[(blockIdx.x * 10 + w) * 2 + 0] = (int)sm;
        out[(blockIdx.x * 10 + w) * 2 + 1] = (int)ws;
    }
    if (threadIdx.x == 0) pad[0] = 0.0;
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int grid = 2 * nsm;
    const size_t smem = 90 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int* d;
    cudaMalloc(&d, grid * 10 * 2 * sizeof(int));
    probe<<<grid, 320, smem>>>(d, 2000000);
    int* h = new int[grid * 10 * 2];
    cudaMemcpy(h, d, grid * 10 * 2 * sizeof(int), cudaMemcpyDeviceToHost);
    // histogram: per SM, per SMSP, number of GEMM warps (0..7) and solver warps (8, 9)
    int gemm[256][4] = {}, solv[256][4] = {};
    for (int b = 0; b < grid; ++b)
        for (int w = 0; w < 10; ++w) {
            const int sm = h[(b * 10 + w) * 2], sp = h[(b * 10 + w) * 2 + 1] % 4;
            (w < 8 ? gemm : solv)[sm][sp]++;
        }
    int pattern[5][5][5][5] = {};
    for (int s = 0; s < nsm; ++s) pattern[solv[s][0]][solv[s][1]][solv[s][2]][solv[s][3]]++;
    printf("solver-warp SMSP histograms over %d SMs (count of SMs per [s0 s1 s2 s3]):\n", nsm);
    for (int a = 0; a < 5; ++a)
        for (int b = 0; b < 5; ++b)
            for (int c = 0; c < 5; ++c)
                for (int e = 0; e < 5; ++e)
                    if (pattern[a][b][c][e]) printf("  [%d %d %d %d]: %d\n", a, b, c, e, pattern[a][b][c][e]);
    printf("SM0 gemm per SMSP: %d %d %d %d\n", gemm[0][0], gemm[0][1], gemm[0][2], gemm[0][3]);
    for (int b = 0; b < 4; ++b) {
        printf("block %d:", b);
        for (int w = 0; w < 10; ++w) printf(" (%d,%d)", h[(b * 10 + w) * 2], h[(b * 10 + w) * 2 + 1]);
        printf("\n");
    }
    return 0;
}
