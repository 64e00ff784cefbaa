"""GPU: two contexts driven from two host threads on one GPU (one fraq_ctx per
GPU or per worker).  Calls on different contexts hold different locks (fraq_ctx_s::mu), so a
long call on context A does not block a short call on context B, and both results are right.
Through the raw C ABI (ctypes releases the GIL during each call)."""
import ctypes as C
import os
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class Kernel(C.Structure):  # fraq_kernel_t
    _fields_ = [("sbd", C.c_int), ("gamma", C.c_double), ("tau", C.c_double),
                ("n_head", C.c_int), ("np1", C.c_int), ("np2", C.c_int),
                ("head", C.c_double * 512), ("m1", C.c_double * 512), ("r1", C.c_double * 512),
                ("m2", C.c_double * 512), ("r2", C.c_double * 512)]


class Budget(C.Structure):  # fraq_budget_t
    _fields_ = [("horizon", C.c_long), ("eps_tol", C.c_double), ("max_points", C.c_int),
                ("max_head", C.c_int), ("achieved_eps", C.c_double)]


class Spec(C.Structure):  # fraq_spec_t
    _fields_ = [("alpha1", C.c_double), ("alpha2", C.c_double), ("coupling_a", C.c_double),
                ("length", C.c_double), ("t_final", C.c_double), ("grid_m", C.c_int),
                ("n_steps", C.c_long), ("initial", C.c_int),
                ("custom_g1", C.POINTER(C.c_double)), ("custom_g2", C.POINTER(C.c_double))]


class KConf(C.Structure):  # fraq_kconf_t
    _fields_ = [("be_points", C.c_int), ("sbd_points_1", C.c_int), ("sbd_points_2", C.c_int),
                ("sbd_head", C.c_int), ("eps_tol", C.c_double), ("auto_size", C.c_int),
                ("solver", C.c_int)]


DP = C.POINTER(C.c_double)


def _history(lib, ctx, dim):
    k = Kernel()
    b = Budget(65536, 1e-12, 256, 256, 0.0)
    assert lib.fraq_build_sbd_kernel_auto(ctx, C.c_double(0.7), C.c_double(1 / 65536),
                                          C.byref(b), C.byref(k)) == 0
    h = C.c_void_p()
    kp = (C.POINTER(Kernel) * 1)(C.pointer(k))
    dims = (C.c_long * 1)(dim)
    assert lib.fraq_hist_create(ctx, 1, kp, dims, 0, C.byref(h)) == 0
    return k, h


def test_two_contexts_two_threads_do_not_serialise(fraq):
    lib = C.CDLL(os.path.join(ROOT, "paper_1901_05128_b200", "libfraqcu.so"))
    ctx = [C.c_void_p(), C.c_void_p()]
    for c in ctx:
        assert lib.fraq_ctx_create(0, None, C.byref(c)) == 0
    rng = np.random.default_rng(11)
    # A: a long call -- the physical C3-grid stepper over 8192 levels (~0.4 s), which holds A's
    # lock while it waits on A's stream
    spec = Spec(0.4, 0.8, -5.5, 1.0, 0.5, 4095, 8192, 0, None, None)  # poly_sin
    kc = KConf(64, 41, 41, 0, 1e-12, 1, 0)                             # FRAQ_SOLVER_PHYSICAL
    g1, g2 = np.empty(4095), np.empty(4095)
    # B: short calls on the second context
    _, hb = _history(lib, ctx[1], 64)
    UB = rng.uniform(-1, 1, (64, 64))
    DB = np.empty_like(UB)
    done = {}

    def run_a():
        t0 = time.perf_counter()
        done["a_rc"] = lib.fraq_run(ctx[0], C.byref(spec), 1, 1, C.byref(kc),
                                    g1.ctypes.data_as(DP), g2.ctypes.data_as(DP), None)
        done["a"] = (t0, time.perf_counter())

    ta = threading.Thread(target=run_a)
    ta.start()
    time.sleep(0.1)  # A is inside its call
    t0 = time.perf_counter()
    rc = lib.fraq_hist_run(hb, UB.ctypes.data_as(DP), C.c_long(64), C.c_long(64),
                           DB.ctypes.data_as(DP), C.c_long(64), 0)
    t_b = time.perf_counter()
    ta.join()
    assert rc == 0 and done["a_rc"] == 0
    # B finished while A was still running: no process-wide lock
    assert t_b < done["a"][1], (t_b - t0, done["a"][1] - done["a"][0])
    # both results equal the package's single-context evaluation
    b = fraq.KernelBudget(horizon=65536, eps_tol=1e-12)
    k = fraq.build_sbd_kernel_auto(0.7, 1 / 65536, b)
    ref = np.array(fraq.SbdHistory(k, fraq.HistoryVariant.standalone, 64).run(UB))
    ok = ~np.isnan(ref)
    assert np.max(np.abs(DB[ok] - ref[ok])) <= 1e-12 * np.max(np.abs(ref[ok]))
    kp = fraq.KernelConfig()
    kp.solver = fraq.SOLVER_PHYSICAL
    rr = fraq.run(fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=4095,
                                   t_final=0.5, n_steps=8192), fraq.Scheme.FastBE, kp)
    assert np.array_equal(rr.final_state.g1, g1) and np.array_equal(rr.final_state.g2, g2)
    lib.fraq_hist_destroy(hb)
    for c in ctx:
        lib.fraq_ctx_destroy(c)
