// DMMA (m8n8k4 f64) dependent-chain latency and throughput vs independent accumulators/warps.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int C>
__global__ void k(double* out, int iters, long long* cyc) {
    double acc[C][2];
    for (int c = 0; c < C; ++c) acc[c][0] = acc[c][1] = threadIdx.x + c;
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < C; ++c) dmma(acc[c], a, b);
    long long t1 = clock64();
    double s = 0; for (int c = 0; c < C; ++c) s += acc[c][0] + acc[c][1];
    if (s == 1.2345) out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C> void run(int wps, double* out, long long* cyc) {
    int iters = 2048; cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<C><<<148, 32 * wps>>>(out, 8, cyc);
    cudaEventRecord(e0); k<C><<<148, 32 * wps>>>(out, iters, cyc); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    double fl = 148.0 * wps * iters * 8 * C * 512.0;
    printf("acc/warp %2d warps/SM %2d: %6.2f TFLOP/s, cycles per DMMA per chain %.1f\n", C, wps, fl / (ms * 1e-3) / 1e12, (double)c / (iters * 8));
}
int main() {
    double* out; long long* cyc; cudaMalloc(&out, 8192); cudaMalloc(&cyc, 8);
    run<1>(1, out, cyc); run<1>(4, out, cyc); run<1>(16, out, cyc); run<2>(16, out, cyc);
    run<4>(4, out, cyc); run<4>(8, out, cyc); run<4>(16, out, cyc); run<8>(16, out, cyc);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
