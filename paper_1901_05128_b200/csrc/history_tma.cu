// history_tma.cu -- K5t: the per-level fused history step (K5's job, fast_kernel.cpp:261-409)
// streamed through shared memory by TMA.
//
// One warp owns 32 DOFs of one group and all its nodes.  Lane 0 streams the state y[j][m]
// (node rows j, DOF-contiguous, leading dimension ld) as 2D tensor-map boxes of 32 DOFs x 16 nodes
// through a 3-stage shared-memory ring: TMA loads complete on per-stage mbarriers, the 32 lanes
// update their DOF in place (y <- r_j y + f_j u_lag) and accumulate the node sum in a register --
// one DOF per lane, so no cross-thread reduction -- and lane 0 writes the box back with a TMA
// store (after a generic->async proxy fence).  Warps are independent pipelines (no CTA barriers).
// The epilogue (append into the lag ring, exact head window, output) is K5's, per DOF.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "history.cuh"

namespace fraqcu {

namespace {

constexpr int T_CJ = 16;      // nodes per box
constexpr int T_STAGES = 3;   // boxes in flight per warp
constexpr int T_WARPS = 4;    // warps (independent 32-DOF tiles) per CTA
constexpr int T_MAXG = 8;     // groups with their own tensor map

struct K5tMaps {
    CUtensorMap m[T_MAXG];
};

__device__ __forceinline__ unsigned s32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(T_WARPS * 32) step_tma_kernel(StepArgs A, const int2* tiles,
                                                                int n_tiles,
                                                                const __grid_constant__ K5tMaps maps) {
    extern __shared__ __align__(128) double tsm[];  // [T_WARPS][T_STAGES][T_CJ][32] boxes
    double(*box)[T_STAGES][T_CJ][32] = reinterpret_cast<double(*)[T_STAGES][T_CJ][32]>(tsm);
    __shared__ __align__(8) unsigned long long full[T_WARPS][T_STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ti = blockIdx.x * T_WARPS + warp;
    if (ti >= n_tiles) return;  // whole warp: no CTA-wide synchronisation below
    const int2 tile = tiles[ti];
    const GroupDev G = A.groups[tile.x];
    const int m = tile.y + lane;
    const bool live = m < G.dim;
    const long ld = G.ld;
    const CUtensorMap* map = &maps.m[tile.x];

    // feed value u_{level+1-L} from the lag ring (read before this launch's append)
    const long fi = A.level + 1 - G.L;
    const bool feed = A.adv && fi >= A.lo && fi <= A.appended - 1;
    const double v = (feed && live) ? A.ring[G.ring_off + (fi % G.L) * ld + m] : 0.0;

    double acc = 0.0;
    if (A.adv || A.mode != MODE_NONE) {
        const int nch = (G.J + T_CJ - 1) / T_CJ;
        const double* cr = A.cr + G.co_off;
        const double* cf = A.cf + G.co_off;
        constexpr unsigned bytes = T_CJ * 32 * 8;
        if (lane == 0) {
            for (int s = 0; s < T_STAGES; ++s)
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&full[warp][s])) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        auto load = [&](int c) {  // lane 0
            const int s = c % T_STAGES;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                             s32(&full[warp][s])),
                         "r"(bytes)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], "
                "[%1, {%2, %3}], [%4];" ::"r"(s32(&box[warp][s][0][0])),
                "l"(reinterpret_cast<unsigned long long>(map)), "r"(tile.y), "r"(c * T_CJ),
                "r"(s32(&full[warp][s]))
                : "memory");
        };
        if (lane == 0)
            for (int c = 0; c < min(nch, T_STAGES); ++c) load(c);
        for (int c = 0; c < nch; ++c) {
            const int s = c % T_STAGES;
            const unsigned par = (unsigned)((c / T_STAGES) & 1);
            unsigned done = 0;
            while (!done)
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 "
                    "%0, 1, 0, p; }"
                    : "=r"(done)
                    : "r"(s32(&full[warp][s])), "r"(par)
                    : "memory");
            double* b = &box[warp][s][0][lane];
            const int j0 = c * T_CJ;
            const int jn = min(T_CJ, G.J - j0);
            if (A.adv) {
#pragma unroll 4
                for (int jj = 0; jj < jn; ++jj) {
                    const double y = fma(__ldg(cr + j0 + jj), b[jj * 32], __ldg(cf + j0 + jj) * v);
                    b[jj * 32] = y;
                    acc += y;
                }
                // make the generic-proxy writes visible to the TMA store, then write the box back
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], "
                        "[%3];" ::"l"(reinterpret_cast<unsigned long long>(map)),
                        "r"(tile.y), "r"(j0), "r"(s32(&box[warp][s][0][0]))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                }
            } else {
#pragma unroll 4
                for (int jj = 0; jj < jn; ++jj) acc += b[jj * 32];
                __syncwarp();
            }
            if (lane == 0 && c + T_STAGES < nch) {
                // the stage is reused: its store must have finished reading shared memory
                if (A.adv) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                load(c + T_STAGES);
            }
        }
        if (lane == 0 && A.adv) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        __syncwarp();
    }
    if (!live) return;
    double* ring = A.ring + G.ring_off + m;
    long appended = A.appended;
    if (A.app) {
        ring[(appended % G.L) * ld] = A.u[G.dof0 + m];
        ++appended;
    }
    if (A.mode == MODE_NONE) return;
    const double* hd = A.head + G.hd_off;
    if (A.mode == MODE_DERIV) {
        const long n = appended - 1;
        long top;
        if (!G.sbd)
            top = 1;
        else
            top = min((long)G.L - 1, A.lo == 0 ? n : n - 1);
        for (long i = 0; i <= top; ++i) acc = fma(hd[i], ring[((n - i) % G.L) * ld], acc);
    } else if (A.mode == MODE_FFPE) {
        const long n = appended;
        const long top = G.sbd ? min((long)G.L - 1, n - 1) : (n >= 2 ? 1 : 0);
        for (long i = 1; i <= top; ++i) acc = fma(hd[i], ring[((n - i) % G.L) * ld], acc);
    }
    A.out[G.dof0 + m] = acc;
}

}  // namespace

// Builds one tensor map per group over its state rows (y[j][0..ld), j < J), box 32 x T_CJ.
bool k5t_prepare(HistDevice& d) {
    d.k5t_ok = false;
    if (std::getenv("FRAQ_NO_K5T")) return false;
    const int ng = (int)d.groups_h.size();
    if (ng < 1 || ng > T_MAXG) return false;
    static auto encode = []() -> decltype(&cuTensorMapEncodeTiled) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
                cudaSuccess || q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<decltype(&cuTensorMapEncodeTiled)>(fn);
    }();
    if (!encode) return false;
    d.k5t_maps.assign(ng, CUtensorMap{});
    std::vector<int2> tiles;
    for (int g = 0; g < ng; ++g) {
        const GroupDev& G = d.groups_h[g];
        double* base = d.state.p + G.st_off;
        if (reinterpret_cast<uintptr_t>(base) % 16 || (G.ld * 8) % 16 || G.J < 1) return false;
        const cuuint64_t dims[2] = {(cuuint64_t)G.ld, (cuuint64_t)G.J};
        const cuuint64_t strides[1] = {(cuuint64_t)G.ld * 8};
        const cuuint32_t boxd[2] = {32, T_CJ}, estr[2] = {1, 1};
        if (encode(&d.k5t_maps[g], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, boxd, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
        for (int m0 = 0; m0 < G.dim; m0 += 32) tiles.push_back(make_int2(g, m0));
    }
    d.k5t_tiles.alloc(tiles.size());
    FRAQ_CUDA(cudaMemcpy(d.k5t_tiles.p, tiles.data(), tiles.size() * sizeof(int2),
                         cudaMemcpyHostToDevice));
    d.n_k5t_tiles = (int)tiles.size();
    d.k5t_ok = true;
    return true;
}

void k5t_launch(fraq_ctx c, const HistDevice& d, const StepArgs& a) {
    K5tMaps mp;
    std::memset(&mp, 0, sizeof(mp));
    for (size_t g = 0; g < d.k5t_maps.size(); ++g) mp.m[g] = d.k5t_maps[g];
    const int grid = (d.n_k5t_tiles + T_WARPS - 1) / T_WARPS;
    constexpr size_t smem = sizeof(double) * T_WARPS * T_STAGES * T_CJ * 32;
    static bool attr = false;
    if (!attr) {
        FRAQ_CUDA(cudaFuncSetAttribute(step_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
        attr = true;
    }
    step_tma_kernel<<<grid, T_WARPS * 32, smem, c->stream>>>(a, d.k5t_tiles.p, d.n_k5t_tiles, mp);
    FRAQ_LAUNCH_CHECK();
}

}  // namespace fraqcu
