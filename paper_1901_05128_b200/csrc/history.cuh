// history.cuh -- device history state shared by the history API (history.cu) and the FFPE
// stepper (ffpe.cu).
#pragma once

#include <cuda.h>

#include "internal.cuh"

namespace fraqcu {

// One DOF group: a contiguous slice of the user's DOF vector with its own compressed kernel.
// State y[node][dof] and lag ring [slot][dof] are DOF-contiguous with padded leading dim ld.
struct GroupDev {
    long dof0;     // first DOF of the group in the user's vector
    int dim;       // DOFs in the group
    int ld;        // padded leading dimension (multiple of 4)
    long st_off;   // state + st_off + j*ld + m
    long ring_off; // ring + ring_off + slot*ld + m
    int J;         // nodes (np1 + np2)
    int L;         // lag == ring capacity: 2 (BE) or n_head (SBD)
    int co_off;    // ratios cr[co_off + j], feeds cf[co_off + j]
    int hd_off;    // head[hd_off + i], i < L
    int sbd;
};

// Arguments of one fused step launch (K5).
struct StepArgs {
    const GroupDev* groups;
    const int2* tiles;   // (group, first DOF pair)
    double* state;
    double* ring;
    const double* cr;
    const double* cf;
    const double* head;
    long level;      // level before this launch's advance
    long appended;   // values appended before this launch's append
    int lo;          // 0 standalone, 1 scheme
    int adv;         // run advance()
    int app;         // run append(u)
    int mode;        // 0: none, 1: history_sum, 2: derivative, 3: FFPE history term
    const double* u; // append input (device, user layout dof0-relative)
    double* out;     // output (device, user layout)
    // FFPE stepper extras (zero = off): the level from a device counter (CUDA-graph replays:
    // level = *n_dev + n_off - 1, appended = level + 1), and the first head tap of MODE_FFPE
    // (2: tap 1 -- the newest level, d_1 G^(n-1) -- is left to the solve kernel, so the
    // history pass of level n+1 can overlap the solve of level n)
    const long* n_dev;
    int n_off;
    int first_tap;
    // K5e / K5f input ring (null = off): the appended value is also recorded in row
    // appended & xh_mask (leading dimension ldx, user layout)
    double* xh;
    long ldx;
    int xh_mask;
};

enum { MODE_NONE = 0, MODE_SUM = 1, MODE_DERIV = 2, MODE_FFPE = 3 };

// Arguments of the temporally blocked kernels (K5b/K5c/K5d).
struct RunArgs {
    const GroupDev* groups;
    const int2* tasks;      // (group, first DOF of the 4-DOF task)
    int n_tasks;
    int* counter;           // dynamic task counter (zeroed before launch)
    double* state;
    double* ring;
    const double* cr;
    const double* cf;
    const double* head;
    long A0;                // values appended before the call (pure push sequence)
    int lo;
    long n_steps;
    const double* U;        // device, row n at U + n*ldu, group-relative dof0 offsets
    long ldu;
    double* D;              // nullable
    long ldd;
    const double* frag;     // K5d fragment tables (per group kFragDoubles)
    int use_tma;            // K5d: stage input chunks with TMA (tensor map over U)
};

// K5d fragment tables per group (history_dmma.cu): C (64 node tiles x 2 x 32), R (64 x 2 x 32),
// r^8 (64 x 4 x 2), raw r and f per node pair (64 x 4 x 2 x 2), local Toeplitz W (2 x 32).
constexpr int kFragC = 0, kFragR = 4096, kFragR8 = 8192, kFragRF = 8704, kFragW = 9728;
constexpr int kFragDoubles = 9792;

// K5e (history_fir.cu): the blocked evaluation with the fast-decaying nodes folded into an exact
// FIR over the last M inputs.  Per group: the slow ("long") nodes keep their state recurrence;
// a node j is "short" when |r_j|^M <= 2^-70, so everything it remembers lies within M levels
// and its contribution is the Toeplitz sum  sum_{m<M} (sum_j f_j r_j^m) v(n-m).
constexpr int E_MAXWG = 8;   // warps per CTA (node slices of up to 64 long nodes)
struct FirGroup {
    int JL, TL;              // long nodes, their 8-node tiles
    int M;                   // FIR length of the short nodes (0: none)
    int KW, nkk;             // combined window over the input rows (multiple of 4), k-steps
    int NTW;                 // tiles per warp (warp w owns tiles [w NTW, (w+1) NTW))
    int kk0[E_MAXWG + 1];    // FIR k-steps of warp w: [kk0[w], kk0[w+1])
    long tab_off;            // tables: C[TL*64], R[TL*64], H[nkk*32] (doubles)
    int perm_off;            // original node index of long position p (-1: padding)
    int short_off, n_short;  // original node indices of the short nodes
    long ws_off;             // tables: the short nodes' FIR taps wS_m = sum_j f_j r_j^m, m < M (K5f)
};
struct FirPlan {
    bool built = false, ok = false;
    std::vector<FirGroup> groups_h;
    DevBuf<FirGroup> groups;
    DevBuf<double> tabs;
    DevBuf<int> perm;        // long positions, then short lists
    int nwg = 1;             // warps per CTA
    int capC = 64, capH = 32;  // shared-memory table capacities (doubles)
    int kw_max = 0;          // input rows a call needs from before its first level
    int min_level = 0;       // first level index the steady-state form is valid from
    int ring_rows = 128;     // shared-memory input ring (power of two)
    // input history ring in HBM (rows = level & (xh_rows - 1)), valid trailing rows
    DevBuf<double> xh;
    int xh_rows = 0;
    long xh_valid = 0;
    bool short_stale = false;  // short-node states in `state` lag behind (rebuilt on demand)
};

// history_fir.cu: the fold as a kernel rewrite (longer exact head, only the slow nodes); returns
// the number of head levels added (0: `out` untouched).
int fold_kernel(const fraq_kernel_t& k, int lcap, fraq_kernel_t* out);

// Device-resident tables + state of a set of groups.
struct HistDevice {
    std::vector<GroupDev> groups_h;
    std::vector<int2> tiles_h;
    std::vector<int> tile_lanes;  // LANES per tile config (all tiles same)
    DevBuf<GroupDev> groups;
    DevBuf<int2> tiles;
    DevBuf<double> state, ring, cr, cf, head;
    long total_dim = 0;
    int n_tiles = 0;
    int slices = 4;       // node slices per CTA (K5)
    int lanes = 32;       // DOF quads per CTA (K5)
    bool ztrick_ok = true;
    int max_J = 0, max_L = 0;
    std::vector<fraq_kernel_t> kernels;  // host copies

    // DMMA fragment tables for K5d (built on first use): per group kFragDoubles doubles
    DevBuf<double> frag;
    bool frag_built = false;
    // host copies of the per-node ratios / feeds (cr, cf) for the K5e table builder
    std::vector<double> cr_h, cf_h;
    // K5e plan (history_fir.cu; built on first use)
    FirPlan fir;

    void build(fraq_ctx c, int n_groups, const fraq_kernel_t* const* ks, const long* dims,
               bool tables_only = false);
    void launch_step(fraq_ctx c, const StepArgs& a);
    void launch_step(fraq_ctx c, const StepArgs& a, cudaStream_t stream);
    // reset state/ring to zero
    void zero(fraq_ctx c);
};

// K13 (modal_dmma.cu): mode-space FFPE stepping on DMMA; one entry per instance (device pointers).
struct K13Inst {
    double a, tau;
    const double* r[2];
    const double* f[2];
    const double* head[2];
    const double* corr[2];  // SBD correction sequence corr[n-4], nullable for BE
    int J[2], L[2];
};
bool k13_supported(int maxJ, int minL, int maxL);
// Setup (node fragment tables, combined weights) and launch are split so that the loop timers
// see only the stepping.
struct K13Plan {
    DevBuf<double> tabs;
    DevBuf<unsigned char> inst;  // per-instance device records
    DevBuf<int> counter;
    int n_inst = 0, RB = 2, NT = 8, nwf = 1, Jp = 64, nwg = 2, TS = 0, ring = 32, delta = 0;
    bool sbd = false;
};
void k13_prepare(fraq_ctx c, const std::vector<K13Inst>& in, bool sbd, K13Plan& plan);
void k13_exec(fraq_ctx c, K13Plan& plan, const double* lam, int n_modes, long N, const double* c0,
              double* cN);

}  // namespace fraqcu
