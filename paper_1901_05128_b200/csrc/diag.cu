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

}  // namespace
}  // namespace fraqcu

using namespace fraqcu;

extern "C" int fraq_diag_fp64_peak(fraq_ctx c, double* tflops) {
    return guarded([&] {
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
