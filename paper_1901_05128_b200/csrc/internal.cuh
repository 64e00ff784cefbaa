// internal.cuh -- shared internals of libfraqcu (context, errors, device math helpers).
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <mutex>
#include <string>
#include <vector>

#include "fraqcu.h"

namespace fraqcu {

// ------------------------------------------------------------------ errors
struct Error : std::exception {
    int code;
    std::string msg;
    Error(int c, std::string m) : code(c), msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

void set_last_error(const std::string& m);

#define FRAQ_CUDA(call)                                                                      \
    do {                                                                                     \
        cudaError_t e_ = (call);                                                             \
        if (e_ != cudaSuccess)                                                               \
            ::fraqcu::fail(e_ == cudaErrorMemoryAllocation ? FRAQ_ENOMEM : FRAQ_ECUDA,       \
                           std::string(#call) + ": " + cudaGetErrorString(e_));              \
    } while (0)

#define FRAQ_LAUNCH_CHECK() FRAQ_CUDA(cudaGetLastError())

// Error mapping of every ABI entry point: exceptions -> return code + thread-local message.
template <class F>
int guarded_nolock(F&& f) {
    try {
        f();
        return FRAQ_OK;
    } catch (const Error& e) {
        set_last_error(e.msg);
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("host allocation failed");
        return FRAQ_ENOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return FRAQ_ERUNTIME;
    }
}

// Context-free entry points (host math, context creation): no shared state, no lock.
template <class F>
int guarded(F&& f) {
    return guarded_nolock(f);
}

// ------------------------------------------------------------------ device buffers
// ------------------------------------------------------------------ device buffers
template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) {
        o.p = nullptr;
        o.n = 0;
    }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            n = o.n;
            o.p = nullptr;
            o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t count) {
        release();
        if (count) FRAQ_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    T* get() const { return p; }
};

// ------------------------------------------------------------------ context
}  // namespace fraqcu

struct fraq_ctx_s {
    // Calls on one context share its stream and setup scratch buffers, so concurrent callers of
    // the SAME context take turns (the reference's run() is reentrant and releases the GIL; its
    // harness runs solves in worker threads).  Different contexts -- one per GPU, INTEGRATION.md
    // section 5 -- never contend.  Recursive: an observer callback may call back into the API.
    std::recursive_mutex mu;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    // scratch reused by setup kernels
    fraqcu::DevBuf<double> scratch_d;
    fraqcu::DevBuf<long> scratch_l;
    // DST sine table of the last grid size (modal.cu ctx_sintab): built once per M, so DST calls
    // inside a caller's timed region do no cudaMalloc / cudaFree
    fraqcu::DevBuf<double> sintab;
    int sintab_m = 0;
    double* scratch(size_t n) {
        if (scratch_d.n < n) scratch_d.alloc(n);
        return scratch_d.p;
    }
};

namespace fraqcu {

// Entry points bound to a context: serialised per context (see fraq_ctx_s::mu).
template <class F>
int guarded(fraq_ctx c, F&& f) {
    if (!c) return guarded_nolock([] { fail(FRAQ_EINVAL, "null fraq_ctx"); });
    std::lock_guard<std::recursive_mutex> lock(c->mu);
    return guarded_nolock(f);
}

inline void check_ctx(fraq_ctx c) {
    if (!c) fail(FRAQ_EINVAL, "null fraq_ctx");
    FRAQ_CUDA(cudaSetDevice(c->device));
}

// ------------------------------------------------------------------ setup API (setup.cu)
// Device-side builders; all write host-visible fraq_kernel_t results.
void gauss_jacobi_dev(fraq_ctx c, double a, double b, int n, double* nodes_h, double* w_h);
// weights into a device buffer (n_max+1 values)
void be_weights_dev(fraq_ctx c, double g, double tau, long n_max, double* out_d);
void sbd_weights_dev(fraq_ctx c, double g, double tau, long n_max, double* out_d);
void build_be_kernel_dev(fraq_ctx c, double g, double tau, int np, fraq_kernel_t* k);
void build_sbd_kernel_dev(fraq_ctx c, double g, double tau, int np1, int np2, int nh,
                          fraq_kernel_t* k);
void build_kernel_auto_dev(fraq_ctx c, bool sbd, int n, const double* gammas, double tau,
                           fraq_budget_t* budgets, fraq_kernel_t* out);
void kernel_error_report_dev(fraq_ctx c, const fraq_kernel_t* k, long n_max, double* eps_h,
                             double* max_eps, long* argmax);
void reconstruct_dev(fraq_ctx c, const fraq_kernel_t* k, long n, const long* idx, double* out_h);
// corr_d[e] = sum_j m_j p_j(e) with p_j(e) = r_j multiplied e times from 1 (fpfp.cpp:240-250),
// for e = 0..e_max.  Device buffer out.
void corr_sequence_dev(fraq_ctx c, const fraq_kernel_t* k, long e_max, double* corr_d);
void corr_sequence_batch_dev(fraq_ctx c, const fraq_kernel_t* ks, int n, long e_max,
                             double* corr_base, long stride);
// direct.cu: classical O(N^2) CQ on DMMA (device pointers)
void direct_cq_dev(fraq_ctx c, int sbd, double g, double tau, const double* U, long ldu,
                   long n_steps, long dim, double* D, long ldd);

// ------------------------------------------------------------------ host checks (reference)
inline void check_kernel_gamma(double g) {
    if (!(g > 0.0) || !(g < 1.0)) fail(FRAQ_EINVAL, "fast kernel: alpha must be in (0,1)");
}
inline void check_weight_args(double g, double tau) {
    if (!(g > 0.0) || !(g <= 1.0))
        fail(FRAQ_EINVAL, "cq_weights: alpha must be in (0,1], got " + std::to_string(g));
    if (!(tau > 0.0)) fail(FRAQ_EINVAL, "cq_weights: tau must be > 0");
}

}  // namespace fraqcu
