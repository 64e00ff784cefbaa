"""GPU: the single-step API (FastStepper / ClassicalStepper, fpfp.hpp:80-140), the block_solver.hpp
types (DiscreteLaplacian, BandedLU, BlockSystem, solve_block_system) and the reference's FFPE
property tests (test_fpfp.cpp:313-528) restated on the B200 path, plus the reference's Python
smoke checks (proj/tests/python/test_smoke.py:22-60) restated against this package.

Everything below runs through the C ABI (libfraqcu) via the package; the oracle is the
unmodified reference (oracle/_ref) or its bitwise-pinned C restatement."""
import math
import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SCHEMES = ["BE", "FastBE", "SBD", "FastSBD"]


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def spec_of(fraq, alpha1, alpha2, a, m, t_final, n_steps, initial="poly_sin", g1=None, g2=None):
    s = fraq.ProblemSpec(alpha1=alpha1, alpha2=alpha2, coupling_a=a, grid_m=m, t_final=t_final,
                         n_steps=n_steps)
    s.initial = initial
    if initial == "custom":
        s.custom_g1 = list(g1)
        s.custom_g2 = list(g2)
    return s


def kc_of(fraq, solver=None, auto=True, be_points=64):
    kc = fraq.KernelConfig()
    kc.auto_size = auto
    kc.be_points = be_points
    if solver is not None:
        kc.solver = solver
    return kc


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# ------------------------------------------------------------------ steppers
@pytest.mark.parametrize("sbd", [False, True])
def test_fast_stepper_equals_run_physical(fraq, sbd):
    """N single steps == one run() with the physical solver (same kernels, same order: bitwise)."""
    spec = spec_of(fraq, 0.35, 0.7, -1.5, 63, 0.4, 48)
    st = fraq.FastStepper(spec, sbd, kc_of(fraq))
    assert st.step_index() == 0
    s0 = st.state()
    f0 = fraq.initial_field(spec)
    assert np.array_equal(s0.g1, f0.g1) and np.array_equal(s0.g2, f0.g2)
    for n in range(48):
        st.step()
    assert st.step_index() == 48 and st.state().step == 48
    rr = fraq.run(spec, fraq.Scheme.FastSBD if sbd else fraq.Scheme.FastBE,
                  kc_of(fraq, fraq.SOLVER_PHYSICAL))
    assert np.array_equal(st.state().g1, rr.final_state.g1)
    assert np.array_equal(st.state().g2, rr.final_state.g2)
    assert st.kernel_eps1() == rr.kernel_eps1 and st.kernel_eps2() == rr.kernel_eps2


@pytest.mark.parametrize("sbd", [False, True])
def test_graph_replays_equal_single_steps(fraq, sbd):
    """run() steps the physical scheme through the 64-level CUDA graph (K5 of level n+1 on a side
    stream overlapping K6 of level n, device level counter); single steps launch eagerly.  Both
    must give the same bits, including the eager remainder after the last whole graph chunk."""
    N = 64 * 3 + 13
    spec = spec_of(fraq, 0.45, 0.65, 1.3, 127, 0.3, N, "indicator")
    st = fraq.FastStepper(spec, sbd, kc_of(fraq))
    for n in range(N):
        st.step()
    rr = fraq.run(spec, fraq.Scheme.FastSBD if sbd else fraq.Scheme.FastBE,
                  kc_of(fraq, fraq.SOLVER_PHYSICAL))
    assert np.array_equal(st.state().g1, rr.final_state.g1)
    assert np.array_equal(st.state().g2, rr.final_state.g2)
    # a stepper that mixes both: graph chunks inside step_n, eager steps around them
    st2 = fraq.FastStepper(spec, sbd, kc_of(fraq))
    st2.step()
    st2.step_n(150)
    st2.step_n(N - 151)
    assert np.array_equal(st2.state().g1, rr.final_state.g1)
    assert np.array_equal(st2.state().g2, rr.final_state.g2)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_stepper_trajectory_matches_reference(fraq, orc, scheme):
    """State after every k steps vs the reference's run() to level k (fixed-size kernels, so the
    tables do not depend on the horizon)."""
    sbd = "SBD" in scheme
    fast = scheme.startswith("Fast")
    N, m, tau = 24, 31, 0.25 / 24
    spec = spec_of(fraq, 0.3, 0.6, 2.0, m, N * tau, N)
    if fast:
        st = fraq.FastStepper(spec, sbd, kc_of(fraq, auto=False))
    else:
        st = fraq.ClassicalStepper(spec, sbd)
    kconf = dict(auto_size=False, be_points=64, sbd_points_1=41, sbd_points_2=41, sbd_head=0)
    # the reference's fixed-size FastSBD run needs n_steps >= n_head (its kernel_error_report
    # rejects n_max below the head, fast_kernel.cpp:152)
    ks = (17, 20, 24) if scheme == "FastSBD" else (1, 2, 3, 7, 16, 24)
    for k in ks:
        while st.step_index() < k:
            st.step()
        g1, g2, _, _ = orc.run(0.3, 0.6, 2.0, m, k * tau, k, scheme, "poly_sin", kconf=kconf)
        s = st.state()
        assert rel(s.g1, g1) <= 1e-10, (k, rel(s.g1, g1))
        assert rel(s.g2, g2) <= 1e-10, (k, rel(s.g2, g2))


def test_stepper_errors(fraq):
    spec = spec_of(fraq, 0.3, 0.6, 2.0, 15, 0.1, 4)
    st = fraq.FastStepper(spec, False, kc_of(fraq))
    st.step_n(4)
    with pytest.raises(ValueError):
        st.step()  # beyond the horizon the kernels were sized for
    bad = spec_of(fraq, 0.3, 0.6, 2.0, 15, 0.1, 4, "custom", [0.0] * 3, [0.0] * 3)
    with pytest.raises(ValueError):
        fraq.FastStepper(bad, True, kc_of(fraq))


# ------------------------------------------------------------------ block_solver types
def heat_step(b, c, h):
    """(I + c A) x = b with A the Dirichlet stencil (dense numpy; test_fpfp.cpp heat_step)."""
    m = len(b)
    A = (np.diag(np.full(m, 2.0)) - np.diag(np.ones(m - 1), 1) - np.diag(np.ones(m - 1), -1)) / h**2
    return np.linalg.solve(np.eye(m) + c * A, b)


def test_laplacian_apply(fraq):
    lap = fraq.DiscreteLaplacian(21, 1.0)
    x = np.sin(0.37 * np.arange(21)) + 0.2
    y = np.array(lap.apply(list(x)))
    h = 1.0 / 22
    want = (2 * x - np.r_[0.0, x[:-1]] - np.r_[x[1:], 0.0]) / h**2
    assert rel(y, want) <= 1e-14
    assert lap.eigenvalue(3, 1.0) == pytest.approx(4 / h**2 * math.sin(3 * math.pi * h / 2) ** 2,
                                                   rel=1e-15)


@pytest.mark.parametrize("m", [21, 31, 255])  # Thomas and cyclic-reduction grids
def test_block_system_subcases(fraq, m):
    """test_fpfp.cpp:454-528: a = 0 -> two heat solves; multiply-then-solve roundtrip; an
    eigenmode right-hand side equals the scalar 2x2 solve."""
    lap = fraq.DiscreteLaplacian(m, 1.0)
    h = lap.h
    j = np.arange(m)
    b1, b2 = np.sin(0.3 * j) + 0.1, np.cos(0.2 * j)
    tau, d01, d02 = 0.01, 2.2, 0.9
    g1, g2 = fraq.solve_block_system(d01, d02, 0.0, tau, lap, list(b1), list(b2))
    assert rel(g1, heat_step(tau * b1, tau * d01, h)) < 1e-12
    assert rel(g2, heat_step(tau * b2, tau * d02, h)) < 1e-12

    rng = np.random.default_rng(17)
    x1, x2 = rng.uniform(-1, 1, m), rng.uniform(-1, 1, m)
    d01, d02, a, tau, lead = 1.7, 0.4, -1.3, 0.02, 1.5
    ax1, ax2 = np.array(lap.apply(list(x1))), np.array(lap.apply(list(x2)))
    r1 = lead / tau * x1 + d01 * (a * x1 + ax1) - a * d02 * x2
    r2 = lead / tau * x2 + d02 * (a * x2 + ax2) - a * d01 * x1
    sys_ = fraq.BlockSystem(d01, d02, a, tau, lap, lead)
    y1, y2 = sys_.solve(list(r1), list(r2))
    assert rel(y1, x1) < 1e-12 and rel(y2, x2) < 1e-12

    k = 5
    vk = np.sqrt(2.0 / (m + 1)) * np.sin((k + 1) * (j + 1) * math.pi / (m + 1))
    lam = lap.eigenvalue(k + 1, 1.0)
    d01, d02, a, tau = 0.8, 1.1, 2.0, 0.05
    g1, g2 = fraq.solve_block_system(d01, d02, a, tau, lap, list(vk), [0.0] * m)
    M = np.array([[1 / tau + d01 * (a + lam), -a * d02], [-a * d01, 1 / tau + d02 * (a + lam)]])
    x = np.linalg.solve(M, [1.0, 0.0])
    assert np.max(np.abs(np.array(g1) - x[0] * vk)) <= 1e-11 * np.max(np.abs(x[0] * vk))
    assert np.max(np.abs(np.array(g2) - x[1] * vk)) <= 1e-11 * np.max(np.abs(x[1] * vk))


def test_block_system_matches_reference(fraq, orc):
    """The device block solve equals the reference BlockSystem (pivoted banded LU) on the C3
    grid with the C3 diagonal (the ill-conditioned case, cond ~1.4e6)."""
    m, tau = 4095, 1 / 16384
    d01, d02, a = 16384 ** 0.6, 16384 ** 0.2, -5.5
    rng = np.random.default_rng(3)
    r1, r2 = rng.uniform(-1, 1, m) * 1e4, rng.uniform(-1, 1, m) * 1e4
    lap = fraq.DiscreteLaplacian(m, 1.0)
    g1, g2 = fraq.BlockSystem(d01, d02, a, tau, lap, 1.0).solve(list(r1), list(r2))
    o1, o2 = orc.block_solve(d01, d02, a, tau, m, 1.0, r1, r2)
    assert rel(g1, o1) <= 1e-10 and rel(g2, o2) <= 1e-10


def test_banded_lu(fraq):
    rng = np.random.default_rng(5)
    n, kl, ku = 40, 2, 3
    A = np.zeros((n, n))
    lu = fraq.BandedLU(n, kl, ku)
    for r in range(n):
        for c in range(max(0, r - kl), min(n, r + ku + 1)):
            v = rng.uniform(-1, 1) + (3.0 if r == c and r % 7 else 0.0)
            A[r, c] = v
            lu.set(r, c, v)
    assert lu.get(4, 5) == A[4, 5]
    with pytest.raises(IndexError):
        lu.set(0, 5, 1.0)  # outside the band (std::out_of_range)
    with pytest.raises(RuntimeError):
        lu.solve([0.0] * n)  # before factorize (std::logic_error)
    lu.factorize()
    b = rng.uniform(-1, 1, n)
    x = np.array(lu.solve(list(b)))
    assert rel(A @ x, b) <= 1e-12
    z = fraq.BandedLU(3, 1, 1)
    with pytest.raises(RuntimeError):
        z.factorize()  # zero pivot


# ------------------------------------------------------------------ FFPE properties
@pytest.mark.parametrize("solver", ["SOLVER_AUTO", "SOLVER_PHYSICAL"])
@pytest.mark.parametrize("scheme", SCHEMES)
def test_linearity_and_determinism(fraq, scheme, solver):
    """test_fpfp.cpp:313-345: repeated runs are bitwise identical; scaling G0 by -3.5 scales the
    result to 1e-12."""
    spec = spec_of(fraq, 0.3, 0.6, 2.0, 31, 0.25, 32)
    kc = kc_of(fraq, getattr(fraq, solver))
    sch = getattr(fraq.Scheme, scheme)
    base = fraq.run(spec, sch, kc)
    again = fraq.run(spec, sch, kc)
    assert np.array_equal(base.final_state.g1, again.final_state.g1)
    assert np.array_equal(base.final_state.g2, again.final_state.g2)
    f0 = fraq.initial_field(spec)
    sc = spec_of(fraq, 0.3, 0.6, 2.0, 31, 0.25, 32, "custom", -3.5 * np.array(f0.g1),
                 -3.5 * np.array(f0.g2))
    r = fraq.run(sc, sch, kc)
    for got, want in ((r.final_state.g1, base.final_state.g1),
                      (r.final_state.g2, base.final_state.g2)):
        got, want = np.array(got), -3.5 * np.array(want)
        assert np.all(np.abs(got - want) <= 1e-12 * np.abs(want) + 1e-300)


@pytest.mark.parametrize("scheme", SCHEMES)
def test_zero_stays_zero(fraq, scheme):
    """test_fpfp.cpp:347-365."""
    spec = spec_of(fraq, 0.4, 0.7, -1.0, 15, 0.1, 12, "custom", [0.0] * 15, [0.0] * 15)
    r = fraq.run(spec, getattr(fraq.Scheme, scheme))
    assert not np.any(r.final_state.g1) and not np.any(r.final_state.g2)


def test_be_vs_fastbe_trajectories(fraq):
    """test_fpfp.cpp:378-393: max-over-time discrete L2 difference of BE and FastBE <= 1e-10
    (observer runs: every accepted step)."""
    spec = spec_of(fraq, 0.3, 0.6, 2.0, 63, 1.0, 200)
    h = 1.0 / 64
    cls = []
    fraq.run(spec, fraq.Scheme.BE, fraq.KernelConfig(), lambda n, f: cls.append((n, f.g1, f.g2)))
    worst = 0.0
    seen = []

    def obs(n, f):
        seen.append(n)
        _, c1, c2 = cls[n]
        nonlocal worst
        worst = max(worst, fraq.l2_norm(list(np.array(f.g1) - c1), h),
                    fraq.l2_norm(list(np.array(f.g2) - c2), h))
    fraq.run(spec, fraq.Scheme.FastBE, fraq.KernelConfig(), obs)
    assert seen == list(range(201)) and len(cls) == 201
    assert worst <= 1e-10


def test_fastsbd_equals_sbd_inside_head(fraq):
    """test_fpfp.cpp:395-401: with n <= n_head FastSBD is the classical SBD scheme (both in
    physical space, as in the reference: 1e-13).  The mode-space solver steps the same scheme
    without the stencil solve; against the physical classical run it differs by that solve's
    rounding (measured 3.9e-13 on this grid)."""
    spec = spec_of(fraq, 0.3, 0.6, 2.0, 63, 1.0, 10)
    cls = fraq.run(spec, fraq.Scheme.SBD)
    for solver, tol in ((fraq.SOLVER_PHYSICAL, 1e-13), (fraq.SOLVER_AUTO, 2e-12)):
        fst = fraq.run(spec, fraq.Scheme.FastSBD, kc_of(fraq, solver))
        assert rel(fst.final_state.g1, cls.final_state.g1) < tol
        assert rel(fst.final_state.g2, cls.final_state.g2) < tol


@pytest.mark.parametrize("initial", ["poly_sin", "indicator"])
def test_temporal_order_bands(fraq, initial):
    """test_fpfp.cpp:404-432: convergence rates in (0.9, 1.35) for BE / FastBE and (1.8, 2.45)
    for SBD / FastSBD, through the harness driver run_convergence."""
    cfg = fraq.ExperimentConfig()
    cfg.alpha1, cfg.alpha2, cfg.coupling_a, cfg.grid_m, cfg.t_final = 0.3, 0.6, 2.0, 63, 1.0
    cfg.taus = [1 / 40, 1 / 80, 1 / 160]
    cfg.ref_tau = 1 / 1280
    cfg.initial = initial
    for schemes, lo, hi in (([fraq.Scheme.BE, fraq.Scheme.FastBE], 0.9, 1.35),
                            ([fraq.Scheme.SBD, fraq.Scheme.FastSBD], 1.8, 2.45)):
        cfg.schemes = schemes
        reps = fraq.run_convergence(cfg)
        assert len(reps) == 2
        for rep in reps:
            for row in rep.rows[1:]:
                assert lo < row.rate1 < hi and lo < row.rate2 < hi, (rep.scheme, row.rate1,
                                                                      row.rate2)


def test_a0_decouples_fields(fraq):
    """test_fpfp.cpp:434-452: with a = 0 the first field ignores the second."""
    spec = spec_of(fraq, 0.45, 0.75, 0.0, 31, 0.2, 40)
    f0 = fraq.initial_field(spec)
    for solver in (fraq.SOLVER_AUTO, fraq.SOLVER_PHYSICAL):
        kc = kc_of(fraq, solver)
        base = fraq.run(spec, fraq.Scheme.FastBE, kc)
        other = spec_of(fraq, 0.45, 0.75, 0.0, 31, 0.2, 40, "custom", f0.g1, [0.0] * 31)
        r = fraq.run(other, fraq.Scheme.FastBE, kc)
        g, b = np.array(r.final_state.g1), np.array(base.final_state.g1)
        assert np.all(np.abs(g - b) <= 1e-13 * np.abs(b) + 1e-300)


# ------------------------------------------------------------------ reference Python smoke suite
def test_smoke_gauss_jacobi_legendre(fraq):
    """proj/tests/python/test_smoke.py:22-26."""
    rule = fraq.gauss_jacobi(0.0, 0.0, 2)
    assert rule.nodes[0] == pytest.approx(-1.0 / math.sqrt(3.0), abs=1e-14)
    assert rule.weights == pytest.approx([1.0, 1.0], abs=1e-14)
    assert fraq.jacobi_moment(0.0, 0.0, 2) == pytest.approx(2.0 / 3.0, rel=1e-13)


def test_smoke_weight_tables(fraq):
    """test_smoke.py:29-36."""
    assert fraq.be_weights(0.5, 1.0, 3).weights == pytest.approx([1.0, -0.5, -0.125, -0.0625],
                                                                 rel=1e-14)
    assert fraq.sbd_weights(1.0, 1.0, 2).weights == pytest.approx([1.5, -2.0, 0.5], rel=1e-13)
    assert fraq.coupling_from_transition(0.75) == pytest.approx(0.5)
    with pytest.raises(ValueError):
        fraq.coupling_from_transition(0.5)


def test_smoke_reconstruction_window(fraq):
    """test_smoke.py:39-45."""
    k = fraq.build_be_kernel(0.5, 1.0, 16)
    d = fraq.be_weights(0.5, 1.0, 33).weights
    for i in range(2, 34):
        assert k.reconstruct(i) == pytest.approx(d[i], abs=1e-14)
    assert fraq.kernel_error_report(k, 33).max_eps <= 1e-14


def test_smoke_history_direct_sum(fraq):
    """test_smoke.py:48-60: the SBD history's derivative equals the direct sum over the exact
    head and the reconstructed tail."""
    k = fraq.build_sbd_kernel(0.4, 0.05, 20, 20, 8)
    h = fraq.SbdHistory(k, fraq.HistoryVariant.standalone, 1)
    rng = random.Random(7)
    g = []
    for n in range(40):
        g.append(rng.uniform(-1, 1))
        h.push([g[-1]])
        direct = sum(k.head[i] * g[n - i] for i in range(min(k.n_head - 1, n) + 1))
        direct += sum(k.reconstruct(i) * g[n - i] for i in range(k.n_head, n + 1))
        assert h.derivative()[0] == pytest.approx(direct, rel=1e-12, abs=1e-12)
