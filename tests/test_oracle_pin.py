"""Pins the CPU oracle (C restatement, oracle/fraq_oracle.c) before it is trusted as the checker:

1. against the reference itself, compiled from its own sources (oracle/_ref): bitwise equality
   on weights, rules, kernels, histories and FFPE runs;
2. against the golden values frozen in the reference's tests (test_fast_kernel.cpp,
   test_cq_weights.cpp, test_gauss_jacobi.cpp, acceptance_main.cpp) -- restated here;
3. against the committed fixtures in tests/golden/ (generated from oracle/_ref by
   tests/golden/make_golden.py).
"""
import math
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def series_pow(p, alpha, n_max):
    # J.C.P. Miller recurrence (test_cq_weights.cpp:18-28)
    q = [0.0] * (n_max + 1)
    q[0] = p[0] ** alpha
    for n in range(1, n_max + 1):
        s = 0.0
        for k in range(1, min(n, len(p) - 1) + 1):
            s += (alpha * k - (n - k)) * p[k] * q[n - k]
        q[n] = s / (n * p[0])
    return q


# ------------------------------------------------------------------ 1. port == reference
@pytest.mark.parametrize("a,b,n", [(0.3, 0.7, 64), (0.7, 0.6, 256), (0.2, 1.6, 200),
                                   (0.5, 0.5, 8), (0.9, 0.2, 512)])
def test_port_rules_bitwise(port, ref, a, b, n):
    x1, w1 = port.gauss_jacobi(a, b, n)
    x2, w2 = ref.gauss_jacobi(a, b, n)
    assert np.array_equal(x1, x2) and np.array_equal(w1, w2)


def test_port_weights_bitwise(port, ref):
    for g, tau, n in [(0.3, 1e-3, 1000), (0.7, 1 / 4096, 4096), (0.999, 0.5, 50)]:
        assert np.array_equal(port.be_weights(g, tau, n), ref.be_weights(g, tau, n))
        assert np.array_equal(port.sbd_weights(g, tau, n), ref.sbd_weights(g, tau, n))


def test_port_kernels_and_reports_bitwise(port, ref):
    for make in (lambda o: o.build_be_kernel(0.45, 1e-2, 40),
                 lambda o: o.build_sbd_kernel(0.3, 1e-3, 31, 31, 15),
                 lambda o: o.build_sbd_kernel(0.8, 1e-3, 41, 37, 17)):
        k1, k2 = make(port), make(ref)
        for f in ("head", "m1", "r1", "m2", "r2"):
            assert np.array_equal(getattr(k1, f), getattr(k2, f)), f
        e1 = port.kernel_error_report(k1, 1200)
        e2 = ref.kernel_error_report(k2, 1200)
        assert np.array_equal(e1[0], e2[0]) and e1[1:] == e2[1:]


@pytest.mark.parametrize("sbd,g,tau,H", [(False, 0.5, 1 / 4096, 4096), (True, 0.7, 1e-3, 2000),
                                         (False, 0.9, 1 / 2048, 2048)])
def test_port_auto_bitwise(port, ref, sbd, g, tau, H):
    k1 = port.build_kernel_auto(sbd, g, tau, H)
    k2 = ref.build_kernel_auto(sbd, g, tau, H)
    assert (k1.np1, k1.np2, k1.n_head) == (k2.np1, k2.np2, k2.n_head)
    assert k1.achieved_eps == k2.achieved_eps
    assert np.array_equal(k1.m1, k2.m1)


@pytest.mark.parametrize("sbd", [False, True])
@pytest.mark.parametrize("scheme_variant", [False, True])
def test_port_history_bitwise(port, ref, sbd, scheme_variant):
    rng = np.random.default_rng(11)
    U = rng.uniform(-1, 1, (150, 5))
    k = port.build_sbd_kernel(0.4, 0.05, 20, 23, 8) if sbd else port.build_be_kernel(0.4, 0.05, 20)
    assert np.array_equal(port.hist_run(k, U, scheme_variant), ref.hist_run(k, U, scheme_variant),
                          equal_nan=True)


@pytest.mark.parametrize("scheme", ["BE", "FastBE", "SBD", "FastSBD"])
def test_port_ffpe_bitwise(port, ref, scheme):
    for init in ("poly_sin", "indicator"):
        a = port.run(0.3, 0.6, 2.0, 31, 0.25, 40, scheme, init)
        b = ref.run(0.3, 0.6, 2.0, 31, 0.25, 40, scheme, init)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert a[2] == b[2] and a[3] == b[3]


# ------------------------------------------------------------------ 2. frozen reference goldens
def test_gamma_and_moments(port):
    assert port.gamma_fn(1.0) == pytest.approx(1.0, rel=1e-14)
    assert port.gamma_fn(0.5) == pytest.approx(math.sqrt(math.pi), rel=1e-13)
    assert port.gamma_fn(5.0) == pytest.approx(24.0, rel=1e-13)
    assert port.gamma_fn(1.3) == pytest.approx(0.89747069630627718, rel=1e-13)
    assert port.gamma_fn(1.7) == pytest.approx(0.90863873285329044, rel=1e-13)
    assert port.jacobi_moment(0.0, 0.0, 6) == pytest.approx(2.0 / 7.0, rel=1e-13)
    x, w = port.gauss_jacobi(0.0, 0.0, 2)
    assert x[0] == pytest.approx(-1 / math.sqrt(3), abs=1e-14)
    assert w == pytest.approx([1.0, 1.0], abs=1e-14)


def test_rule_exactness_against_moments(port):
    # test_gauss_jacobi.cpp:54-81
    rng = np.random.default_rng(20240811)
    for _ in range(40):
        a, b, n = rng.uniform(-0.999, 2.0), rng.uniform(-0.999, 3.0), int(rng.integers(1, 41))
        x, w = port.gauss_jacobi(a, b, n)
        mu0 = port.jacobi_moment(a, b, 0)
        assert np.all(np.diff(x) > 0) and np.all(w > 0)
        assert abs(w.sum() - mu0) <= 1e-13 * mu0
        for k in range(2 * n):
            assert abs(np.sum(w * x ** k) - port.jacobi_moment(a, b, k)) <= 1e-12 * mu0


def test_weights_examples_and_miller(port):
    assert port.be_weights(1.0, 0.5, 3)[:2] == pytest.approx([2.0, -2.0])
    assert port.sbd_weights(1.0, 1.0, 4)[:3] == pytest.approx([1.5, -2.0, 0.5], rel=1e-14)
    t2 = port.sbd_weights(0.4, 1.0, 6)
    assert t2 == pytest.approx(series_pow([1.5, -2.0, 0.5], 0.4, 6), rel=1e-13)
    # acceptance crit 1: Miller oracle over 20 random (alpha, tau), i <= 500
    rng = np.random.default_rng(101)
    worst = 0.0
    for _ in range(5):
        g, tau = rng.uniform(0.02, 0.999), 10 ** rng.uniform(-3.5, 0.5)
        sc = tau ** (-g)
        be = port.be_weights(g, tau, 200)
        sbd = port.sbd_weights(g, tau, 200)
        obe = np.array(series_pow([1.0, -1.0], g, 200))
        osbd = np.array(series_pow([1.5, -2.0, 0.5], g, 200))
        worst = max(worst, np.max(np.abs(be - sc * obe) / np.maximum(sc * np.abs(obe), 1e-300)),
                    np.max(np.abs(sbd - sc * osbd) / np.maximum(sc * np.abs(osbd), 1e-300)))
    assert worst <= 1e-12


def test_frozen_eps_curves(port):
    k = port.build_sbd_kernel(0.3, 1e-3, 31, 31, 15)
    eps, mx, am = port.kernel_error_report(k, 1000)
    assert mx == pytest.approx(3.950380e-5, rel=1e-2) and am == 1000
    assert np.all(eps[:15] == 0.0)
    k2 = port.build_sbd_kernel(0.8, 1e-3, 41, 41, 17)
    assert port.kernel_error_report(k2, 1000)[1] == pytest.approx(6.389989e-6, rel=1e-2)


def test_recursion_fidelity(port):
    # acceptance crit 4 (acceptance_main.cpp:136-188): fast vs compressed direct <= 1e-13
    rng = np.random.default_rng(404)
    worst = 0.0
    for trial in range(20):
        g = rng.uniform(0.05, 0.95)
        tau = 10 ** (-3 * rng.uniform(0.05, 0.95))
        n = 20 + int(100 * rng.uniform())
        sbd = trial % 2 == 1
        npts = 8 + int(24 * rng.uniform())
        k = (port.build_sbd_kernel(g, tau, npts, npts + 3, 3 + int(12 * rng.uniform())) if sbd
             else port.build_be_kernel(g, tau, npts))
        u = rng.uniform(-1, 1, n)
        D = port.hist_run(k, u[:, None])[:, 0]
        rec = np.zeros(n + 1)
        lo = k.n_head if sbd else 2
        rec[lo:] = port.reconstruct(k, np.arange(lo, n + 1))
        w = np.concatenate([k.head, rec[len(k.head):]])
        for t in range(1 if not sbd else 0, n):
            direct = sum(w[i] * u[t - i] for i in range(t + 1))
            worst = max(worst, abs(D[t] - direct) / max(abs(direct), tau ** (-g)))
    assert worst <= 1e-13


def test_mode_space_oracle(port):
    # test_fpfp.cpp:287-311: physical-space steppers == per-mode scalar recursion (<= 1e-10)
    m, N, tau = 31, 64, 0.5 / 64
    h = 1.0 / (m + 1)
    j = np.arange(1, m + 1)
    kk = np.arange(1, m + 1)
    V = np.sin(np.outer(kk, j) * math.pi * h)
    lam = 4.0 / h ** 2 * np.sin(kk * math.pi * h / 2.0) ** 2
    x = j * h
    g1 = np.where(x > 0.5, 1.0 - x, 0.0)
    g2 = np.where(x < 0.5, x, 0.0)
    c1, c2 = 2.0 / (m + 1) * V @ g1, 2.0 / (m + 1) * V @ g2
    a, al1, al2 = -1.0, 0.35, 0.72
    o1, o2 = 1 - al1, 1 - al2
    kconf = dict(auto_size=False, be_points=24)
    d1 = port.be_weights(o1, tau, N)
    d2 = port.be_weights(o2, tau, N)
    k1, k2 = port.build_be_kernel(o1, tau, 24), port.build_be_kernel(o2, tau, 24)
    d1[2:] = port.reconstruct(k1, np.arange(2, N + 1))
    d2[2:] = port.reconstruct(k2, np.arange(2, N + 1))
    U = np.zeros((N + 1, m))
    W = np.zeros((N + 1, m))
    U[0], W[0] = c1, c2
    for n in range(1, N + 1):
        s1 = sum(d1[i] * U[n - i] for i in range(1, n)) if n > 1 else np.zeros(m)
        s2 = sum(d2[i] * W[n - i] for i in range(1, n)) if n > 1 else np.zeros(m)
        r1 = U[n - 1] / tau - (a + lam) * s1 + a * s2
        r2 = W[n - 1] / tau - (a + lam) * s2 + a * s1
        a11, a12 = 1 / tau + d1[0] * (a + lam), -a * d2[0]
        a21, a22 = -a * d1[0], 1 / tau + d2[0] * (a + lam)
        det = a11 * a22 - a12 * a21
        U[n] = (r1 * a22 - a12 * r2) / det
        W[n] = (a11 * r2 - a21 * r1) / det
    o1g = V.T @ U[N]
    run = port.run(al1, al2, a, m, 0.5, N, "FastBE", "indicator", kconf=kconf)
    assert np.max(np.abs(run[0] - o1g)) / np.max(np.abs(o1g)) <= 1e-10


# ------------------------------------------------------------------ 3. committed fixtures
def test_golden_fixtures(port):
    path = os.path.join(GOLDEN, "golden.npz")
    if not os.path.exists(path):
        pytest.skip("fixtures not generated")
    z = np.load(path)
    # C1 sample: reference fast derivative on 4 DOFs of the C1 workload
    k = port.build_kernel_auto(False, 0.5, 1 / 4096, 4096)
    assert k.np1 == int(z["c1_np"])
    assert np.array_equal(k.m1, z["c1_m"])
    D = port.hist_run(k, z["c1_U"])
    assert np.array_equal(D[1:], z["c1_D"][1:])
    # SBD tables and eps at the C4 exponents
    for name in ("c4a", "c4b"):
        g, tau, H = z[name + "_cfg"]
        kk = port.build_kernel_auto(True, g, tau, int(H))
        assert (kk.np1, kk.n_head) == tuple(z[name + "_sizes"])
        assert kk.achieved_eps == z[name + "_eps"]
    # FFPE runs
    for i in range(int(z["ffpe_n"])):
        cfg = z[f"ffpe{i}_cfg"]
        scheme = str(z[f"ffpe{i}_scheme"])
        g1, g2, _, _ = port.run(cfg[0], cfg[1], cfg[2], int(cfg[3]), cfg[4], int(cfg[5]), scheme,
                                "poly_sin")
        assert np.array_equal(g1, z[f"ffpe{i}_g1"]) and np.array_equal(g2, z[f"ffpe{i}_g2"])
