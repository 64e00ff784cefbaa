"""CPU: the mode-space FFPE restatement (oracle fo_modal_run / ref_modal_run) pinned against the
reference.  (1) The C port equals the restatement over the reference's own BeHistory/SbdHistory
lanes; (2) DST -> modal stepping -> inverse DST equals the reference's physical-space FastStepper
(fraq::run) to 1e-10, the reference's own mode-space equivalence criterion
(test_fpfp.cpp:287-311, acceptance crit 5).  This is the oracle the C4 (2D) checks and the C4 CPU
baseline use."""
import numpy as np
import pytest

from oracle.oracle import Oracle, ref_available


def dst_basis(M):
    k = np.arange(1, M + 1)
    return np.sin(np.outer(k, k) * np.pi / (M + 1))


def eig1d(M, length=1.0):
    h = length / (M + 1)
    k = np.arange(1, M + 1)
    return 4.0 / h ** 2 * np.sin(k * np.pi * h / (2 * length)) ** 2


@pytest.fixture(scope="module")
def port():
    return Oracle("port")


@pytest.fixture(scope="module")
def ref():
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    return Oracle("reference")


@pytest.mark.parametrize("sbd", [False, True])
def test_port_equals_reference_lanes(port, ref, sbd):
    rng = np.random.default_rng(5)
    tau, N, nm = 1.0 / 512, 300, 37
    k1 = port.build_kernel_auto(sbd, 0.65, tau, N)
    k2 = port.build_kernel_auto(sbd, 0.3, tau, N)
    lam = np.sort(rng.uniform(0, 4e4, nm))
    u0, v0 = rng.standard_normal(nm), rng.standard_normal(nm)
    a1, b1, _ = port.modal_run(k1, k2, -2.5, tau, N, lam, u0, v0)
    a2, b2, _ = ref.modal_run(k1, k2, -2.5, tau, N, lam, u0, v0, threads=3)
    s = max(np.abs(a2).max(), np.abs(b2).max())
    assert max(np.abs(a1 - a2).max(), np.abs(b1 - b2).max()) <= 1e-13 * s


@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
@pytest.mark.parametrize("M,a,init", [(31, -1.5, "indicator"), (47, 2.0, "poly_sin")])
def test_modal_restatement_matches_reference_physical(ref, scheme, M, a, init):
    sbd = scheme == "FastSBD"
    T, N, al1, al2 = 0.5, 160, 0.35, 0.7
    tau = T / N
    g1, g2, _, _ = ref.run(al1, al2, a, M, T, N, scheme, init)
    x = np.arange(1, M + 1) / (M + 1)
    if init == "indicator":
        u, v = np.where(x > 0.5, 1 - x, 0.0), np.where(x < 0.5, x, 0.0)
    else:
        u, v = x * (1 - x), np.sin(x)
    S = dst_basis(M)
    k1 = ref.build_kernel_auto(sbd, 1 - al1, tau, N)
    k2 = ref.build_kernel_auto(sbd, 1 - al2, tau, N)
    cu, cv, _ = ref.modal_run(k1, k2, a, tau, N, eig1d(M), 2 / (M + 1) * S @ u,
                              2 / (M + 1) * S @ v)
    r1, r2 = S @ cu, S @ cv
    assert np.abs(r1 - g1).max() <= 1e-10 * np.abs(g1).max()
    assert np.abs(r2 - g2).max() <= 1e-10 * np.abs(g2).max()
