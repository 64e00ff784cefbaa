"""GPU parity: the B200 path (through the C ABI, via the `_fraq` module) against the CPU oracle.

The oracle is the reference itself compiled from its own sources (oracle/_ref) when present,
else the C restatement (oracle/liboracle.so), which tests/test_oracle_pin.py pins bitwise to the
reference.  Tolerances follow BASELINE.json's north_star (1e-10 relative, fp64) unless stated.
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def kernel_from_oracle(fraq, k):
    if k.sbd:
        return fraq.make_sbd_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1),
                                    list(k.m2), list(k.r2))
    return fraq.make_be_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1))


def rel_linf(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den > 0 else 1.0)


# ------------------------------------------------------------------ L0 / L1
@pytest.mark.parametrize("a,b,n", [(0.0, 0.0, 2), (0.5, 0.5, 20), (0.3, 0.7, 64), (0.7, 0.6, 256),
                                   (0.2, 1.6, 204), (0.9, 0.2, 512), (-0.5, 2.5, 33)])
def test_gauss_jacobi_matches_oracle(fraq, orc, a, b, n):
    r = fraq.gauss_jacobi(a, b, n)
    x, w = orc.gauss_jacobi(a, b, n)
    assert np.max(np.abs(np.array(r.nodes) - x)) <= 4e-16 * max(1, n / 16)
    assert np.max(np.abs(np.array(r.weights) - w) / w) <= 1e-11


def test_gauss_jacobi_errors(fraq):
    for args in [(-1.0, 0.0, 4), (0.0, -1.5, 4), (0.0, 0.0, 0), (0.0, 0.0, 1000)]:
        with pytest.raises(ValueError):
            fraq.gauss_jacobi(*args)


@pytest.mark.parametrize("g,tau,n", [(0.5, 1.0, 3), (0.3, 1e-3, 2000), (0.999, 0.01, 500),
                                     (0.7, 1 / 65536, 65536)])
def test_weights_match_oracle(fraq, orc, g, tau, n):
    be = np.array(fraq.be_weights(g, tau, n).weights)
    assert rel_linf(be, orc.be_weights(g, tau, n)) <= 1e-15
    # (the 65536-long C2 table too: the device Cauchy product measured 2.9e-16 relative per
    # entry against the reference's serial product, profiles/r02/sbdw_probe.py)
    sbd = np.array(fraq.sbd_weights(g, tau, n).weights)
    ref = orc.sbd_weights(g, tau, n)
    assert np.max(np.abs(sbd - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-12


def test_weights_examples(fraq):
    assert fraq.be_weights(0.5, 1.0, 3).weights == pytest.approx([1.0, -0.5, -0.125, -0.0625], rel=1e-14)
    assert fraq.sbd_weights(1.0, 1.0, 2).weights == pytest.approx([1.5, -2.0, 0.5], rel=1e-13)
    with pytest.raises(ValueError):
        fraq.be_weights(0.0, 1.0, 4)
    with pytest.raises(ValueError):
        fraq.sbd_weights(0.5, -1.0, 4)


# ------------------------------------------------------------------ L2 kernels
@pytest.mark.parametrize("g,tau,np_", [(0.5, 1.0, 32), (0.2, 1e-3, 16), (0.8, 1e-3, 64),
                                       (0.6, 1 / 16384, 256)])
def test_be_kernel_matches_oracle(fraq, orc, g, tau, np_):
    k = fraq.build_be_kernel(g, tau, np_)
    o = orc.build_be_kernel(g, tau, np_)
    assert np.allclose(k.head, o.head, rtol=1e-15, atol=0)
    assert np.max(np.abs(np.array(k.ratios) - o.r1)) <= 1e-15
    assert rel_linf(k.node_weights, o.m1) <= 1e-11


def test_be_kernel_window_and_sum(fraq):
    # exactness window 2 <= i <= 2 np + 1 (test_fast_kernel.cpp:45-67)
    for g in (0.2, 0.5, 0.8):
        tau = 1e-3
        for np_ in (16, 64):
            k = fraq.build_be_kernel(g, tau, np_)
            d = fraq.be_weights(g, tau, 2 * np_ + 1).weights
            tol = 1e-14 * tau ** (-g)
            for i in range(2, 2 * np_ + 2, 7):
                assert abs(k.reconstruct(i) - d[i]) <= tol
    k = fraq.build_be_kernel(0.5, 1.0, 32)
    assert sum(k.node_weights) == pytest.approx(-0.125, rel=1e-13)


@pytest.mark.parametrize("g,np1,np2,nh", [(0.3, 31, 31, 15), (0.8, 41, 41, 17), (0.45, 20, 27, 8),
                                          (0.7, 256, 256, 17)])
def test_sbd_kernel_matches_oracle(fraq, orc, g, np1, np2, nh):
    tau = 1e-3
    k = fraq.build_sbd_kernel(g, tau, np1, np2, nh)
    o = orc.build_sbd_kernel(g, tau, np1, np2, nh)
    assert np.max(np.abs(np.array(k.head) - o.head) / np.abs(o.head)) <= 1e-13
    assert np.max(np.abs(np.array(k.ratio1) - o.r1)) <= 1e-15
    assert np.max(np.abs(np.array(k.ratio2) - o.r2)) <= 1e-15
    assert rel_linf(k.mult1, o.m1) <= 1e-11
    assert rel_linf(k.mult2, o.m2) <= 1e-11


def test_error_report_frozen_goldens(fraq):
    # test_fast_kernel.cpp:105-116 / acceptance crit 3 frozen values
    s1 = fraq.build_sbd_kernel(0.3, 1e-3, 31, 31, 15)
    r1 = fraq.kernel_error_report(s1, 1000)
    assert all(e == 0.0 for e in r1.eps[:15])
    assert r1.max_eps == pytest.approx(3.950380e-5, rel=1e-2)
    assert r1.argmax == 1000
    s2 = fraq.build_sbd_kernel(0.8, 1e-3, 41, 41, 17)
    assert fraq.kernel_error_report(s2, 1000).max_eps == pytest.approx(6.389989e-6, rel=1e-2)
    bk = fraq.build_be_kernel(0.5, 1e-3, 16)
    br = fraq.kernel_error_report(bk, 33)
    assert br.eps[0] == 0.0 and br.eps[1] == 0.0
    assert br.max_eps <= 1e-14 * 1e-3 ** -0.5


def test_error_report_matches_oracle(fraq, orc):
    k = fraq.build_sbd_kernel(0.6, 1e-3, 40, 44, 12)
    ok = orc.build_sbd_kernel(0.6, 1e-3, 40, 44, 12)
    rep = fraq.kernel_error_report(k, 3000)
    eps, mx, am = orc.kernel_error_report(ok, 3000)
    assert rep.max_eps == pytest.approx(mx, rel=1e-6)
    assert rep.argmax == am
    e = np.array(rep.eps)
    big = eps > 1e-3 * mx
    assert np.max(np.abs(e[big] - eps[big]) / eps[big]) <= 1e-5


# reference auto-sizer decisions at the BASELINE configurations
AUTO_CASES = [
    (False, 0.5, 1 / 4096, 4096),       # C1 -> 144
    (False, 0.7, 1e-3, 2000),
    (False, 0.6, 1 / 16384, 16384),     # C3 field 1
    (False, 0.2, 1 / 16384, 16384),     # C3 field 2
    (False, 0.9, 1 / 16384, 16384),     # C5 borderline (eps/tol = 1.00 at 216 points)
    (True, 0.7, 1e-3, 2000),
    (True, 0.7, 1 / 8192, 8192),        # C4 field 1
    (True, 0.4, 1 / 8192, 8192),        # C4 field 2
]


@pytest.mark.parametrize("sbd,g,tau,H", AUTO_CASES)
def test_auto_sizing_matches_oracle(fraq, orc, sbd, g, tau, H):
    b = fraq.KernelBudget(horizon=H, eps_tol=1e-12)
    k = (fraq.build_sbd_kernel_auto if sbd else fraq.build_be_kernel_auto)(g, tau, b)
    o = orc.build_kernel_auto(sbd, g, tau, H)
    if sbd:
        assert (len(k.ratio1), len(k.ratio2), k.n_head) == (o.np1, o.np2, o.n_head)
    else:
        assert len(k.ratios) == o.np1
    assert b.achieved_eps == pytest.approx(o.achieved_eps, rel=1e-4)


# ------------------------------------------------------------------ L2 histories
def test_history_spec_traces(fraq):
    k = fraq.build_be_kernel(0.4, 1.0, 8)
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 1)
    h.push([0.7])
    h.push([-0.3])
    assert h.derivative()[0] == pytest.approx(k.head[0] * -0.3 + k.head[1] * 0.7, rel=1e-15)
    hs = fraq.BeHistory(k, fraq.HistoryVariant.scheme, 1)
    g = [0.3, -0.9, 0.45, 0.11]
    for v in g[:3]:
        hs.push([v])
    assert hs.history_sum()[0] == 0.0
    hs.push([g[3]])
    assert hs.history_sum()[0] == pytest.approx(sum(k.node_weights) * g[1], rel=1e-14)
    ks = fraq.build_sbd_kernel(0.4, 1.0, 16, 16, 15)
    h2 = fraq.SbdHistory(ks, fraq.HistoryVariant.scheme, 1)
    rng = np.random.default_rng(3)
    for _ in range(16):
        h2.push([rng.uniform(-1, 1)])
        assert h2.history_sum()[0] == 0.0
    h2.push([rng.uniform(-1, 1)])
    assert h2.history_sum()[0] != 0.0
    h3 = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 1)
    h3.push([1.0])
    with pytest.raises(RuntimeError):
        h3.derivative()
    with pytest.raises(IndexError):
        h3.lagged(2)
    assert h3.lagged(0) == [1.0]


def test_history_constant_input(fraq):
    k = fraq.build_be_kernel(0.5, 1.0, 16)
    d = fraq.be_weights(0.5, 1.0, 10).weights
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 1)
    for _ in range(11):
        h.push([1.0])
    assert h.derivative()[0] == pytest.approx(sum(d), rel=1e-13)


def test_history_state_is_fixed_size(fraq):
    k = fraq.build_sbd_kernel(0.5, 0.01, 16, 16, 9)
    h = fraq.SbdHistory(k, fraq.HistoryVariant.standalone, 4)
    U = np.full((5000, 4), 0.25)
    h.run(U, False)
    assert h.appended == 5000 and h.level == 4999


def test_eviction_is_a_logic_error(fraq):
    k = fraq.build_be_kernel(0.4, 1.0, 8)
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 2)
    for _ in range(3):
        h.append([1.0, 2.0])
    h.advance()  # feed index -1: nothing to feed, no error (fast_kernel.cpp:269-274)
    with pytest.raises(RuntimeError):
        h.advance()  # feed index 0 evicted by the third append


@pytest.mark.parametrize("sbd", [False, True])
@pytest.mark.parametrize("variant", ["standalone", "scheme"])
@pytest.mark.parametrize("dim", [1, 3, 8, 37])
def test_history_push_matches_oracle(fraq, orc, sbd, variant, dim):
    rng = np.random.default_rng(100 + dim + 7 * sbd)
    g, tau = rng.uniform(0.1, 0.9), 10 ** (-2 * rng.uniform(0, 1))
    o = (orc.build_sbd_kernel(g, tau, 12, 15, 7) if sbd else orc.build_be_kernel(g, tau, 14))
    k = kernel_from_oracle(fraq, o)
    V = getattr(fraq.HistoryVariant, variant)
    h = (fraq.SbdHistory if sbd else fraq.BeHistory)(k, V, dim)
    U = rng.uniform(-1, 1, (60, dim))
    D_ref = orc.hist_run(o, U, variant == "scheme")
    scale = max(1.0, tau ** (-g))
    for n in range(60):
        h.push(list(U[n]))
        if np.isnan(D_ref[n]).any():
            with pytest.raises(RuntimeError):
                h.derivative()
            continue
        d = np.array(h.derivative())
        assert np.max(np.abs(d - D_ref[n])) <= 1e-13 * scale * max(1.0, np.max(np.abs(D_ref[n])))


@pytest.mark.parametrize("np_", [5, 30, 33, 100, 144, 256, 300, 512])
@pytest.mark.parametrize("sbd", [False, True])
def test_run_blocked_matches_oracle(fraq, orc, np_, sbd):
    rng = np.random.default_rng(np_ + 1000 * sbd)
    g, tau = 0.35 + 0.3 * rng.uniform(), 1e-3
    if sbd:
        o = orc.build_sbd_kernel(g, tau, np_ // 2 + 1, np_ - np_ // 2, 11)
    else:
        o = orc.build_be_kernel(g, tau, np_)
    k = kernel_from_oracle(fraq, o)
    dim, n = 13, 300
    U = rng.uniform(-1, 1, (n, dim))
    D_ref = orc.hist_run(o, U)
    h = (fraq.SbdHistory if sbd else fraq.BeHistory)(k, fraq.HistoryVariant.standalone, dim)
    # first a few single pushes, then one blocked run for the rest, then single pushes again
    out = []
    for t in range(5):
        h.push(list(U[t]))
        out.append(h.derivative() if (sbd or t >= 1) else [math.nan] * dim)
    D_mid = h.run(U[5:290])
    J = len(o.r1) + len(o.r2)
    assert (h.last_path >= 1) == (J <= 512)  # blocked kernels hold <= 512 nodes; K5 beyond
    out.extend(D_mid)
    for t in range(290, n):
        h.push(list(U[t]))
        out.append(h.derivative())
    D = np.array(out, dtype=float)
    assert np.array_equal(np.isnan(D), np.isnan(D_ref))
    ok = ~np.isnan(D_ref)
    scale = np.maximum(np.abs(D_ref), tau ** (-g))
    assert np.max(np.abs(D[ok] - D_ref[ok]) / scale[ok]) <= 1e-12


def test_multi_group_history(fraq, orc):
    o1 = orc.build_sbd_kernel(0.7, 1e-3, 20, 20, 17)
    o2 = orc.build_sbd_kernel(0.3, 1e-3, 24, 18, 15)
    k1, k2 = kernel_from_oracle(fraq, o1), kernel_from_oracle(fraq, o2)
    rng = np.random.default_rng(5)
    U = rng.uniform(-1, 1, (200, 11))
    h = fraq.MultiHistory([k1, k2], [5, 6])
    D = h.run(U)
    D1 = orc.hist_run(o1, U[:, :5])
    D2 = orc.hist_run(o2, U[:, 5:])
    assert rel_linf(D, np.concatenate([D1, D2], axis=1)) <= 1e-12


@pytest.mark.parametrize("sbd", [False, True])
def test_blocked_input_staging_tma_and_registers(fraq, orc, sbd, monkeypatch):
    """K5d input staging: TMA tiles into the three-segment ring (even leading dimension, 512-node
    groups) and the register-staged fallback (FRAQ_NO_TMA) give identical results, equal to the
    reference history.  Two groups of 20 and 28 DOFs: 16-DOF tiles straddle the group boundary
    (neighbour columns are loaded but never reach live outputs) and the end of U (zero fill).
    Calls of 300, 37 and 95 levels cover partial chunks and the ring wrap."""
    rng = np.random.default_rng(41 + sbd)
    if sbd:
        o1 = orc.build_sbd_kernel(0.7, 1e-3, 256, 256, 17)
        o2 = orc.build_sbd_kernel(0.3, 1e-3, 250, 256, 15)
    else:
        o1 = orc.build_be_kernel(0.7, 1e-3, 512)
        o2 = orc.build_be_kernel(0.3, 1e-3, 480)
    k1, k2 = kernel_from_oracle(fraq, o1), kernel_from_oracle(fraq, o2)
    U = rng.uniform(-1, 1, (432, 48))
    ref = np.concatenate([orc.hist_run(o1, U[:, :20]), orc.hist_run(o2, U[:, 20:])], axis=1)
    outs = []
    for no_tma in (False, True):
        if no_tma:
            monkeypatch.setenv("FRAQ_NO_TMA", "1")
        else:
            monkeypatch.delenv("FRAQ_NO_TMA", raising=False)
        h = fraq.MultiHistory([k1, k2], [20, 28])
        D = np.concatenate([h.run(U[:300]), h.run(U[300:337]), h.run(U[337:])])
        assert h.last_path in (3, 4)  # K5d, or K5e once past the first levels
        outs.append(D)
    assert np.array_equal(outs[0], outs[1], equal_nan=True)
    assert np.array_equal(np.isnan(outs[0]), np.isnan(ref))
    ok = ~np.isnan(ref)
    scale = np.maximum(np.abs(ref[ok]), 1e-3 ** -0.7)
    assert np.max(np.abs(outs[0][ok] - ref[ok]) / scale) <= 1e-12


# ------------------------------------------------------------------ L4 FFPE
@pytest.mark.parametrize("solver", ["SOLVER_PHYSICAL", "SOLVER_AUTO"])
@pytest.mark.parametrize("scheme", ["BE", "FastBE", "SBD", "FastSBD"])
@pytest.mark.parametrize("grid_m,a", [(31, -1.0), (31, 2.0), (50, 0.5), (63, -5.5)])
def test_ffpe_matches_oracle(fraq, orc, scheme, grid_m, a, solver):
    kconf = dict(auto_size=False, be_points=24, sbd_points_1=24, sbd_points_2=24, sbd_head=9)
    g1, g2, e1, e2 = orc.run(0.3, 0.65, a, grid_m, 0.5, 64, scheme, "indicator", kconf=kconf)
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.65, coupling_a=a, grid_m=grid_m, t_final=0.5,
                            n_steps=64, initial="indicator")
    kc = fraq.KernelConfig()
    kc.auto_size = False
    kc.be_points = 24
    kc.sbd_points_1 = kc.sbd_points_2 = 24
    kc.sbd_head = 9
    kc.solver = getattr(fraq, solver)
    rr = fraq.run(spec, getattr(fraq.Scheme, scheme), kc)
    assert rel_linf(rr.final_state.g1, g1) <= 1e-10
    assert rel_linf(rr.final_state.g2, g2) <= 1e-10


@pytest.mark.parametrize("solver", ["SOLVER_PHYSICAL", "SOLVER_AUTO"])
@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
def test_ffpe_auto_kernels_match_oracle(fraq, orc, scheme, solver):
    g1, g2, e1, e2 = orc.run(0.3, 0.6, 2.0, 63, 1.0, 200, scheme, "poly_sin")
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.6, coupling_a=2.0, grid_m=63, t_final=1.0,
                            n_steps=200)
    kc = fraq.KernelConfig()
    kc.solver = getattr(fraq, solver)
    rr = fraq.run(spec, getattr(fraq.Scheme, scheme), kc)
    assert rel_linf(rr.final_state.g1, g1) <= 1e-10
    assert rel_linf(rr.final_state.g2, g2) <= 1e-10
    assert rr.kernel_eps1 == pytest.approx(e1, rel=1e-3)


def test_ffpe_observer_and_batch(fraq):
    spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.7, coupling_a=-1.0, grid_m=15, t_final=0.1,
                            n_steps=12)
    seen = []
    rr = fraq.run(spec, fraq.Scheme.FastBE, fraq.KernelConfig(), lambda n, f: seen.append((n, f.g1[3])))
    assert [s[0] for s in seen] == list(range(13))
    assert seen[-1][1] == rr.final_state.g1[3]
    specs = [fraq.ProblemSpec(alpha1=0.2 + 0.1 * i, alpha2=0.5, coupling_a=1.0, grid_m=15,
                              t_final=0.1, n_steps=12) for i in range(3)]
    for solver in (fraq.SOLVER_PHYSICAL, fraq.SOLVER_AUTO):
        kc = fraq.KernelConfig()
        kc.solver = solver
        outs = fraq.run_batch(specs, fraq.Scheme.FastSBD, kc)
        for s, o in zip(specs, outs):
            single = fraq.run(s, fraq.Scheme.FastSBD, kc)
            assert rel_linf(o.final_state.g1, single.final_state.g1) <= 1e-14


def test_ffpe_zero_stays_zero(fraq):
    spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.7, coupling_a=-1.0, grid_m=15, t_final=0.1,
                            n_steps=12, initial="custom", custom_g1=[0.0] * 15,
                            custom_g2=[0.0] * 15)
    for s in ("BE", "FastBE", "SBD", "FastSBD"):
        for solver in (fraq.SOLVER_PHYSICAL, fraq.SOLVER_AUTO):
            kc = fraq.KernelConfig()
            kc.solver = solver
            rr = fraq.run(spec, getattr(fraq.Scheme, s), kc)
            assert all(v == 0.0 for v in rr.final_state.g1 + rr.final_state.g2)


@pytest.mark.parametrize("nh", [31, 32, 33, 40, 60])
@pytest.mark.parametrize("variant", ["standalone", "scheme"])
def test_run_blocked_long_heads(fraq, orc, nh, variant):
    """Head windows around the K5d lag limit (32): L <= 32 takes K5d (path 3), longer heads the
    K5c kernel (path 2); both equal the reference history."""
    rng = np.random.default_rng(nh)
    o = orc.build_sbd_kernel(0.55, 2e-3, 60, 70, nh)
    k = kernel_from_oracle(fraq, o)
    dim, n = 19, 260
    U = rng.uniform(-1, 1, (n, dim))
    D_ref = orc.hist_run(o, U, variant == "scheme")
    h = fraq.SbdHistory(k, getattr(fraq.HistoryVariant, variant), dim)
    D = np.array(h.run(U), dtype=float)
    assert h.last_path == (3 if nh <= 32 else 2)
    ok = ~np.isnan(D_ref)
    assert np.array_equal(np.isnan(D), np.isnan(D_ref))
    scale = np.maximum(np.abs(D_ref[ok]), 2e-3 ** -0.55)
    assert np.max(np.abs(D[ok] - D_ref[ok]) / scale) <= 1e-12


def test_run_zero_steps_and_continuation(fraq, orc):
    o = orc.build_be_kernel(0.5, 1e-3, 40)
    k = kernel_from_oracle(fraq, o)
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 5)
    U = np.random.default_rng(0).uniform(-1, 1, (50, 5))
    assert len(h.run(U[:0])) == 0 and h.appended == 0
    D1 = np.array(h.run(U[:20]), dtype=float)
    assert len(h.run(U[20:20])) == 0 and h.appended == 20
    D2 = np.array(h.run(U[20:]), dtype=float)
    D_ref = orc.hist_run(o, U)
    D = np.concatenate([D1, D2])
    ok = ~np.isnan(D_ref)
    assert np.max(np.abs(D[ok] - D_ref[ok])) <= 1e-12 * np.max(np.abs(D_ref[ok]))


@pytest.mark.parametrize("nh", [5, 9, 45, 60])
def test_ffpe_sbd_head_lengths_all_solver_paths(fraq, orc, nh):
    """SBD head windows that select every modal path: K13 with state lag delta = 1 (L < 8) and
    0 (L >= 8), K11 (40 < L <= 56), and beyond 56 the AUTO solver's physical fallback (the
    explicit MODAL solver must refuse)."""
    kconf = dict(auto_size=False, sbd_points_1=24, sbd_points_2=24, sbd_head=nh)
    g1, g2, _, _ = orc.run(0.3, 0.65, -1.5, 31, 0.5, 120, "FastSBD", "indicator", kconf=kconf)
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.65, coupling_a=-1.5, grid_m=31, t_final=0.5,
                            n_steps=120, initial="indicator")
    for solver in ("SOLVER_AUTO", "SOLVER_MODAL", "SOLVER_PHYSICAL"):
        kc = fraq.KernelConfig()
        kc.auto_size = False
        kc.sbd_points_1 = kc.sbd_points_2 = 24
        kc.sbd_head = nh
        kc.solver = getattr(fraq, solver)
        if solver == "SOLVER_MODAL" and nh > 56:
            with pytest.raises(ValueError):
                fraq.run(spec, fraq.Scheme.FastSBD, kc)
            continue
        rr = fraq.run(spec, fraq.Scheme.FastSBD, kc)
        assert rel_linf(rr.final_state.g1, g1) <= 1e-10
        assert rel_linf(rr.final_state.g2, g2) <= 1e-10


@pytest.mark.parametrize("sbd", [False, True])
@pytest.mark.parametrize("np_", [7, 64, 256])
def test_run_blocked_scheme_variant(fraq, orc, sbd, np_):
    """Blocked runs in the scheme variant (lo = 1: G^0 never fed, SBD head taps i <= n-1), split
    over calls so the DMMA head window meets block starts near the lag boundary."""
    rng = np.random.default_rng(np_ + 7 * sbd)
    g, tau = 0.45, 1e-3
    o = orc.build_sbd_kernel(g, tau, np_ // 2 + 1, np_ - np_ // 2, 13) if sbd else orc.build_be_kernel(g, tau, np_)
    k = kernel_from_oracle(fraq, o)
    dim, n = 21, 301
    U = rng.uniform(-1, 1, (n, dim))
    D_ref = orc.hist_run(o, U, True)
    h = (fraq.SbdHistory if sbd else fraq.BeHistory)(k, fraq.HistoryVariant.scheme, dim)
    parts = [h.run(U[a:b]) for a, b in ((0, 9), (9, 40), (40, 173), (173, n))]
    D = np.concatenate([np.array(p, dtype=float).reshape(-1, dim) for p in parts])
    assert np.array_equal(np.isnan(D), np.isnan(D_ref))
    ok = ~np.isnan(D_ref)
    scale = np.maximum(np.abs(D_ref[ok]), tau ** (-g))
    assert np.max(np.abs(D[ok] - D_ref[ok]) / scale) <= 1e-12


def test_multi_history_many_ragged_groups(fraq, orc):
    """Many DOF groups of ragged sizes (1, 3, 16, 17, 33, ...) with different kernels (BE sizes
    differ per group) in one device state: K5d tasks straddle no group boundary, leading
    dimensions are padded, and every group equals its own reference history."""
    rng = np.random.default_rng(77)
    dims = [1, 3, 16, 17, 33, 5, 64, 2]
    os_ = [orc.build_be_kernel(0.2 + 0.08 * i, 1e-3, 20 + 13 * i) for i in range(len(dims))]
    ks = [kernel_from_oracle(fraq, o) for o in os_]
    h = fraq.MultiHistory(ks, dims)
    n = 150
    U = rng.uniform(-1, 1, (n, sum(dims)))
    D = np.array(h.run(U), dtype=float)
    assert h.last_path == 3
    c = 0
    for o, dm in zip(os_, dims):
        D_ref = orc.hist_run(o, U[:, c:c + dm])
        Dg = D[:, c:c + dm]
        ok = ~np.isnan(D_ref)
        assert np.array_equal(np.isnan(Dg), ~ok)
        assert np.max(np.abs(Dg[ok] - D_ref[ok])) <= 1e-12 * max(1.0, np.max(np.abs(D_ref[ok])))
        c += dm


@pytest.mark.parametrize("H", [8, 12, 16])
def test_auto_sbd_head_longer_than_horizon(fraq, orc, H):
    """Short horizons: the initial SBD head (15 / 17) exceeds horizon + 1, and every head entry
    must still be the exact weight d_i (the reference builds the head from sbd_weights up to
    n_head - 1, fast_kernel.cpp:78-124, whatever the horizon).  Regression: the batched device
    sizer used to take the head from the horizon-long sizing tables."""
    tau = 1.0 / 4096
    for g in (0.3, 0.5, 0.7):
        b = fraq.KernelBudget(horizon=H, eps_tol=1e-12)
        k = fraq.build_sbd_kernel_auto(g, tau, b)
        o = orc.build_kernel_auto(True, g, tau, H)
        assert k.n_head == o.n_head
        assert np.allclose(np.array(k.head), np.array(o.head), rtol=1e-15, atol=0)
    # the batched path (several exponents in one sizing pass), as the FFPE steppers use it
    specs = [fraq.ProblemSpec(alpha1=0.2 + 0.1 * i, alpha2=0.5, coupling_a=1.0, grid_m=15,
                              t_final=0.1, n_steps=H) for i in range(3)]
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_MODAL
    outs = fraq.run_batch(specs, fraq.Scheme.FastSBD, kc)
    for s, o in zip(specs, outs):
        g1, g2, _, _ = orc.run(s.alpha1, s.alpha2, 1.0, 15, 0.1, H, "FastSBD", "poly_sin")
        assert rel_linf(o.final_state.g1, g1) <= 1e-10
        assert rel_linf(o.final_state.g2, g2) <= 1e-10


def test_concurrent_runs_from_threads(fraq):
    """fraq.run releases the GIL (as the reference's binding does); solves issued from several
    Python threads at once are serialised by the library and equal the sequential results."""
    import threading
    specs = [fraq.ProblemSpec(alpha1=0.2 + 0.15 * i, alpha2=0.6, coupling_a=1.0 - i,
                              grid_m=63, t_final=0.5, n_steps=96) for i in range(4)]
    seq = [fraq.run(s, fraq.Scheme.FastSBD) for s in specs]
    out = [None] * 4

    def work(i):
        for _ in range(3):
            out[i] = fraq.run(specs[i], fraq.Scheme.FastSBD)
    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for a, b in zip(out, seq):
        assert list(a.final_state.g1) == list(b.final_state.g1)


@pytest.mark.parametrize("sbd", [False, True])
@pytest.mark.parametrize("n,dim", [(1, 1), (17, 3), (65, 67), (130, 5), (200, 129)])
def test_direct_cq_ragged_matches_oracle(fraq, orc, sbd, n, dim):
    """K10 (direct CQ, Toeplitz GEMM on DMMA) on ragged shapes -- partial level and DOF tiles,
    single level / single lane -- against the oracle's direct sum (test_fast_kernel.cpp:27-41)."""
    rng = np.random.default_rng(n * 1000 + dim)
    U = rng.uniform(-1, 1, (n, dim))
    D = fraq.direct_cq(sbd, 0.37, 0.01, U)
    Dr = orc.direct_cq(sbd, 0.37, 0.01, U)
    assert np.max(np.abs(D - Dr)) <= 1e-12 * max(np.max(np.abs(Dr)), 1e-300)
