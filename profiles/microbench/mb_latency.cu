// Microbenchmark (not part of the library): DFMA dependent latency and the number of independent
// chains x warps needed to saturate the B200 FP64 pipe.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_latency mb_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void chains(double* out, long iters, double a, double b, long long* cyc) {
    double x[C];
#pragma unroll
    for (int c = 0; c < C; ++c) x[c] = threadIdx.x * 1e-3 + c;
    const long long t0 = clock64();
#pragma unroll 1
    for (long i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < C; ++c) x[c] = fma(x[c], a, b);
    }
    const long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int c = 0; c < C; ++c) s += x[c];
    if (s == 1.2345) out[threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps_per_sm, double* out, long long* cyc) {
    const long iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    chains<C><<<148, 32 * warps_per_sm>>>(out, 16, 0.9999, 1e-9, cyc);
    cudaEventRecord(e0);
    chains<C><<<148, 32 * warps_per_sm>>>(out, iters, 0.9999, 1e-9, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c;
    cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
    const double dfma = 148.0 * 32 * warps_per_sm * iters * 8 * C;
    printf("chains/thread %2d warps/SM %2d: %7.2f TFLOP/s  cycles per DFMA per chain %.2f\n", C,
           warps_per_sm, 2 * dfma / (ms * 1e-3) / 1e12, (double)c / (iters * 8));
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMalloc(&cyc, sizeof(long long));
    run<1>(1, out, cyc);
    run<1>(4, out, cyc);
    run<1>(16, out, cyc);
    run<2>(16, out, cyc);
    run<4>(4, out, cyc);
    run<4>(8, out, cyc);
    run<4>(16, out, cyc);
    run<8>(8, out, cyc);
    run<8>(16, out, cyc);
    run<16>(16, out, cyc);
    run<8>(32, out, cyc);
    printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
}
