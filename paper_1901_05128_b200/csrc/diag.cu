// diag.cu -- roofline denominators measured on the running GPU (diagnostics, not the hot path).
//
// fraq_diag_fp64_peak: dependent-chain-free DFMA stream on every SM (8 independent chains per
// thread, all SMs, enough warps to saturate the FP64 pipe) -> achieved fp64 TFLOP/s (2 flops per
// DFMA).  The fp64-bound blocked history kernel K5b is reported against this number.
#include <cuda_runtime.h>

#include "internal.cuh"

namespace fraqcu {
namespace {

__global__ void __launch_bounds__(256) dfma_kernel(double* sink, int iters, double a, double b) {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
           x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x0 = fma(x0, a, b);
            x1 = fma(x1, a, b);
            x2 = fma(x2, a, b);
            x3 = fma(x3, a, b);
            x4 = fma(x4, a, b);
            x5 = fma(x5, a, b);
            x6 = fma(x6, a, b);
            x7 = fma(x7, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
    if (s == 12345.678) sink[threadIdx.x] = s;  // keep the chains alive
}

// DMMA (fp64 tensor, mma.sync m8n8k4 -> DMMA.8x8x4) stream; mode 1 interleaves an equal number
// of DFMA so the two pipes' concurrency can be measured.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) dmma_kernel(double* sink, int iters, int mode, double a,
                                                   double b) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
    double x0 = 1.0, x1 = 2.0, x2 = 3.0, x3 = 4.0, x4 = 5.0, x5 = 6.0, x6 = 7.0, x7 = 8.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma(acc[i], a, b);
            if (mode) {
#pragma unroll
                for (int v = 0; v < 8; ++v) {
                    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
                }
            }
        }
    }
    double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) sink[threadIdx.x] = s;
}

}  // namespace
}  // namespace fraqcu

using namespace fraqcu;

// tflops[0] = DMMA alone, tflops[1] = DMMA + DFMA interleaved (total fp64 flops of both pipes)
extern "C" int fraq_diag_dmma_peak(fraq_ctx c, double* tflops) {
    return guarded(c, [&] {
        check_ctx(c);
        DevBuf<double> sink(256);
        const int blocks = c->num_sms * 8, iters = 1024;
        cudaEvent_t e0, e1;
        FRAQ_CUDA(cudaEventCreate(&e0));
        FRAQ_CUDA(cudaEventCreate(&e1));
        for (int mode = 0; mode < 2; ++mode) {
            dmma_kernel<<<blocks, 256, 0, c->stream>>>(sink.p, 8, mode, 0.999999, 1e-9);
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                FRAQ_CUDA(cudaEventRecord(e0, c->stream));
                dmma_kernel<<<blocks, 256, 0, c->stream>>>(sink.p, iters, mode, 0.999999, 1e-9);
                FRAQ_CUDA(cudaEventRecord(e1, c->stream));
                FRAQ_CUDA(cudaEventSynchronize(e1));
                float ms;
                FRAQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
                best = ms < best ? ms : best;
            }
            const double warps = (double)blocks * 8;
            const double mma_flops = warps * iters * 4 * 8 * (2.0 * 8 * 8 * 4);
            const double fma_flops = mode ? (double)blocks * 256 * iters * 4 * 8 * 8 * 2.0 : 0.0;
            tflops[mode] = (mma_flops + fma_flops) / (best * 1e-3) / 1e12;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
}

extern "C" int fraq_diag_fp64_peak(fraq_ctx c, double* tflops) {
    return guarded(c, [&] {
        check_ctx(c);
        DevBuf<double> sink(256);
        const int blocks = c->num_sms * 8, iters = 4096;
        dfma_kernel<<<blocks, 256, 0, c->stream>>>(sink.p, 16, 0.999999, 1e-9);  // warm
        cudaEvent_t e0, e1;
        FRAQ_CUDA(cudaEventCreate(&e0));
        FRAQ_CUDA(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            FRAQ_CUDA(cudaEventRecord(e0, c->stream));
            dfma_kernel<<<blocks, 256, 0, c->stream>>>(sink.p, iters, 0.999999, 1e-9);
            FRAQ_CUDA(cudaEventRecord(e1, c->stream));
            FRAQ_CUDA(cudaEventSynchronize(e1));
            float ms;
            FRAQ_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const double dfma = (double)blocks * 256 * iters * 16 * 8;
        *tflops = 2.0 * dfma / (best * 1e-3) / 1e12;
    });
}
