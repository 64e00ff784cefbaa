"""The extended-precision anchor of the 1D FFPE fast schemes (oracle/fraq_anchor_ld.c) and the
reference's own deviation from it (CPU).

The reference's physical-space stepper solves a 2x2-block system with cond ~1.4e6 at M = 4095
whose diagonal lead/tau + d0 (a + 2/h^2) is the same on every row; the fp64 rounding of that one
entry shifts the whole solution coherently (block_solver.cpp:103-114; the bisection is
profiles/r02/physical_bisect.cpp, results in profiles/r02/physical_bisect.txt).  The anchor
evaluates the same discrete scheme on sampled DST modes in long double.  Here:
  * the anchor is pinned: the fp64 mode-space restatement (fo_modal_run, itself pinned to the
    reference's own history lanes in test_modal_oracle.py) agrees with it to 1e-13;
  * the reference's own deviation from the anchor is recorded at the C3 grid (N = 256 levels of
    the C3 run): ~5.6e-9 of the largest coefficient, in the smoothest mode.
The GPU solvers are measured against the same anchor in test_gpu_anchor.py."""
import numpy as np
import pytest

from oracle.oracle import Oracle, ref_available
from workloads import c3_instance

MODES = np.array([1, 2, 3, 4, 5, 8, 13, 32, 64, 256, 1024, 2048, 4095])


def project_ld(g, modes, M):
    """DST coefficients 2/(M+1) sum_j sin(k j pi/(M+1)) g_j in long double."""
    dt = np.longdouble
    j = np.arange(1, M + 1, dtype=dt)
    V = np.sin(np.outer(np.asarray(modes, dt), j) * np.arccos(dt(-1)) / (M + 1))
    return (2 / dt(M + 1) * (V @ np.asarray(g, dt))).astype(float)


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return Oracle("reference")


def c3_kernels(orc, sbd, N=16384):
    inst = c3_instance()
    tau = 1 / 16384
    return inst, [orc.build_kernel_auto(sbd, 1 - al, tau, N) for al in (inst.alpha1, inst.alpha2)]


@pytest.mark.parametrize("sbd", [False, True])
def test_anchor_pinned_to_fp64_mode_space(port, sbd):
    inst, ks = c3_kernels(port, sbd)
    M, N, tau = 4095, 256, 1 / 16384
    uN, vN = port.anchor_ld(ks[0], ks[1], inst.coupling_a, tau, N, M, MODES, inst.g1, inst.g2)
    h = 1 / (M + 1)
    lam = 4 / h ** 2 * np.sin(MODES * np.pi * h / 2) ** 2
    u0, v0 = project_ld(inst.g1, MODES, M), project_ld(inst.g2, MODES, M)
    a, b, _ = port.modal_run(ks[0], ks[1], inst.coupling_a, tau, N, lam, u0, v0)
    sc = max(np.abs(uN).max(), np.abs(vN).max())
    assert max(np.abs(a - uN).max(), np.abs(b - vN).max()) <= 1e-13 * sc


def test_reference_physical_deviation_recorded(ref, port):
    """The reference's physical FastBE at the C3 grid after 256 levels deviates from the exact
    discrete solution by ~5.6e-9 of the largest coefficient, concentrated in the smoothest
    modes -- the systematic effect of the rounded block-system diagonal."""
    inst, ks = c3_kernels(ref, False)
    M, N, tau = 4095, 256, 1 / 16384
    g1, g2, _, _ = ref.run(inst.alpha1, inst.alpha2, inst.coupling_a, M, N * tau, N, "FastBE",
                           "custom", inst.g1, inst.g2, kconf=dict(auto_size=False, be_points=256))
    uN, vN = port.anchor_ld(ks[0], ks[1], inst.coupling_a, tau, N, M, MODES, inst.g1, inst.g2)
    sc = max(np.abs(uN).max(), np.abs(vN).max())
    d1 = np.abs(project_ld(g1, MODES, M) - uN) / sc
    d2 = np.abs(project_ld(g2, MODES, M) - vN) / sc
    dev = max(d1.max(), d2.max())
    assert 1e-9 < dev < 2e-8, dev
    assert np.argmax(d1) <= 2  # the smoothest modes carry it
    assert d1[-3:].max() < 1e-13  # high modes: the stencil is well conditioned there
