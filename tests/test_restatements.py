"""CPU: the numpy FFPE restatement (tests/ffpe_refs.py) used as the 2D oracle reproduces the
reference's own 1D FastStepper (oracle/_ref, else the pinned port)."""
import numpy as np
import pytest

from ffpe_refs import fast_stepper_nd


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def test_1d_restatement_is_the_reference(orc):
    """The numpy restatement used for 2D reproduces the reference's 1D FastStepper."""
    for sbd, scheme in ((False, "FastBE"), (True, "FastSBD")):
        g1r, g2r, _, _ = orc.run(0.35, 0.7, -1.0, 15, 0.3, 40, scheme, "poly_sin")
        x = (np.arange(15) + 1) / 16
        g1, g2 = fast_stepper_nd(orc, 0.35, 0.7, -1.0, 15, 1, 0.3, 40, sbd, x * (1 - x), np.sin(x))
        assert rel(g1, g1r) <= 1e-11 and rel(g2, g2r) <= 1e-11
