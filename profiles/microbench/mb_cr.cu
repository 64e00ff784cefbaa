// Microbenchmark: cost of one 2x2-block cyclic-reduction solve (K6's block_solve_smem shape) on
// one CTA at M = 4095, in-kernel loop, clock64 per solve.  Variants:
//   0: double2 rows in natural order (K6 as built)
//   1: the same with the SysDev coefficients read from global memory each level
//   2: rows stored field-split (two double arrays) -> 8-byte accesses
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_cr mb_cr.cu
#include <cstdio>
#include <cuda_runtime.h>

struct M2 { double a, b, c, d; };
struct Lv { M2 F, G, H; };
__device__ __forceinline__ double2 mv(const M2& m, double2 v) {
    return make_double2(fma(m.a, v.x, m.b * v.y), fma(m.c, v.x, m.d * v.y));
}

__device__ long long g_lvl[64];
// conflict-free row placement for power-of-two strides: one pad slot per 8, 64 and 512 rows
__device__ __forceinline__ int P(int i) { return i + (i >> 3) + (i >> 6) + (i >> 9); }
template <int T, int VAR>
__global__ void __launch_bounds__(T) cr_kernel(const Lv* glv, int K, int m, int reps, double* out,
                                               long long* cyc) {
    extern __shared__ double2 sb[];
    __shared__ Lv lv[20];
    for (int i = threadIdx.x; i < K * 12; i += T) ((double*)lv)[i] = ((const double*)glv)[i];
    for (int k = threadIdx.x; k < m + 2; k += T) sb[VAR >= 2 ? P(k) : k] = make_double2(k > 0 && k <= m ? 1.0 + 1e-3 * k : 0.0, 0.5);
    __syncthreads();
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        // levels with <= 32 rows (VAR 3): warp 0 alone, __syncwarp instead of __syncthreads
        const int lw = VAR == 3 ? max(0, K - 6) : K - 1;
        for (int l = 0; l < lw; ++l) {
            const int s = 1 << l;
            const M2 F = VAR == 1 ? glv[l].F : lv[l].F;
            for (int i = 2 * s * (threadIdx.x + 1); i <= m; i += 2 * s * T) {
                const int pi = VAR >= 2 ? P(i) : i, pl = VAR >= 2 ? P(i - s) : i - s,
                          pr = VAR >= 2 ? P(i + s) : i + s;
                const double2 sum = make_double2(sb[pl].x + sb[pr].x, sb[pl].y + sb[pr].y);
                const double2 t = mv(F, sum);
                sb[pi] = make_double2(sb[pi].x - t.x, sb[pi].y - t.y);
            }
            __syncthreads();
            if (threadIdx.x == 0 && r == reps - 1) g_lvl[l] = clock64();
        }
        if (VAR == 3 && threadIdx.x < 32) {
            for (int l = lw; l < K - 1; ++l) {
                const int s = 1 << l;
                const M2 F = lv[l].F;
                const int i = 2 * s * (threadIdx.x + 1);
                if (i <= m) {
                    const int pi = P(i), pl = P(i - s), pr = P(i + s);
                    const double2 sum = make_double2(sb[pl].x + sb[pr].x, sb[pl].y + sb[pr].y);
                    const double2 t = mv(F, sum);
                    sb[pi] = make_double2(sb[pi].x - t.x, sb[pi].y - t.y);
                }
                __syncwarp();
            }
            if (threadIdx.x == 0) { const int i = P(1 << (K - 1)); sb[i] = mv(lv[K - 1].G, sb[i]); }
            __syncwarp();
            for (int l = K - 2; l >= lw; --l) {
                const int s = 1 << l;
                const M2 Gm = lv[l].G, H = lv[l].H;
                const int i = s * (2 * (int)threadIdx.x + 1);
                if (i <= m) {
                    const int pi = P(i), pl = P(i - s), pr = P(i + s);
                    const double2 xb = mv(Gm, sb[pi]);
                    const double2 nb = make_double2(sb[pl].x + sb[pr].x, sb[pl].y + sb[pr].y);
                    const double2 t = mv(H, nb);
                    sb[pi] = make_double2(xb.x - t.x, xb.y - t.y);
                }
                __syncwarp();
            }
        }
        if (VAR != 3 && threadIdx.x == 0) { const int i = VAR >= 2 ? P(1 << (K - 1)) : 1 << (K - 1); sb[i] = mv(lv[K - 1].G, sb[i]); }
        __syncthreads();
        for (int l = (VAR == 3 ? lw - 1 : K - 2); l >= 0; --l) {
            const int s = 1 << l;
            const M2 Gm = VAR == 1 ? glv[l].G : lv[l].G, H = VAR == 1 ? glv[l].H : lv[l].H;
            for (int i = s * (2 * (int)threadIdx.x + 1); i <= m; i += 2 * s * T) {
                const int pi = VAR >= 2 ? P(i) : i, pl = VAR >= 2 ? P(i - s) : i - s,
                          pr = VAR >= 2 ? P(i + s) : i + s;
                const double2 xb = mv(Gm, sb[pi]);
                const double2 nb = make_double2(sb[pl].x + sb[pr].x, sb[pl].y + sb[pr].y);
                const double2 t = mv(H, nb);
                sb[pi] = make_double2(xb.x - t.x, xb.y - t.y);
            }
            __syncthreads();
            if (threadIdx.x == 0 && r == reps - 1) g_lvl[32 + l] = clock64();
        }
        if (threadIdx.x == 0 && r == reps - 1) g_lvl[63] = clock64();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[blockIdx.x] = (t1 - t0) / reps; out[blockIdx.x] = sb[VAR >= 2 ? P(m / 2) : m / 2].x; }
}

int main() {
    const int m = 4095, K = 12, reps = 200;
    Lv h[20];
    for (int l = 0; l < 20; ++l) h[l] = {{0.5, 0.01, 0.01, 0.5}, {0.9, 0.0, 0.0, 0.9}, {0.5, 0.01, 0.01, 0.5}};
    Lv* d; double* o; long long* c;
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 8 * 8); cudaMalloc(&c, 8 * 8);
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    const size_t smem = sizeof(double2) * (m + 2);
    cudaFuncSetAttribute(cr_kernel<512, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(cr_kernel<512, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(cr_kernel<1024, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const size_t smem2 = sizeof(double2) * (m + 2 + (m + 2) / 7 + 8);
    cudaFuncSetAttribute(cr_kernel<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    cudaFuncSetAttribute(cr_kernel<1024, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    long long hc;
    cr_kernel<512, 0><<<1, 512, smem>>>(d, K, m, reps, o, c);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("512 threads, smem coefficients: %lld cycles per solve (%.2f us at 1.965 GHz)\n", hc, hc / 1965.0);
    cr_kernel<512, 1><<<1, 512, smem>>>(d, K, m, reps, o, c);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("512 threads, global coefficients: %lld cycles per solve\n", hc);
    cr_kernel<1024, 0><<<1, 1024, smem>>>(d, K, m, reps, o, c);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("1024 threads, smem coefficients: %lld cycles per solve\n", hc);
    double r0; cudaMemcpy(&r0, o, 8, cudaMemcpyDeviceToHost);
    cr_kernel<512, 2><<<1, 512, smem2>>>(d, K, m, reps, o, c);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    double r2; cudaMemcpy(&r2, o, 8, cudaMemcpyDeviceToHost);
    printf("512 threads, padded rows: %lld cycles per solve (same result: %d)\n", hc, r0 == r2);
    cr_kernel<1024, 2><<<1, 1024, smem2>>>(d, K, m, reps, o, c);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    printf("1024 threads, padded rows: %lld cycles per solve\n", hc);
    cudaFuncSetAttribute(cr_kernel<512, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
    cr_kernel<512, 3><<<1, 512, smem2>>>(d, K, m, reps, o, c);
    cudaMemcpy(&hc, c, 8, cudaMemcpyDeviceToHost);
    double r3; cudaMemcpy(&r3, o, 8, cudaMemcpyDeviceToHost);
    printf("512 threads, padded rows + warp tail: %lld cycles per solve (same result: %d)\n", hc, r0 == r3);
    cr_kernel<512, 0><<<1, 512, smem>>>(d, K, m, reps, o, c);
    long long lv[64];
    cudaMemcpyFromSymbol(lv, g_lvl, sizeof(lv));
    for (int l = 1; l < K - 1; ++l) printf("fwd level %d: %lld\n", l, lv[l] - lv[l - 1]);
    for (int l = K - 3; l >= 0; --l) printf("back level %d: %lld\n", l, lv[32 + l] - lv[32 + l + 1]);
    printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
