"""Shared test setup.

Markers: ``gpu`` -- needs a CUDA device (B200); run with ``-m gpu``.  Everything else runs on CPU.
The CPU oracle (oracle/, test infrastructure) is built on demand from the committed Makefile.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref (reference built from its sources) not present")
    return Oracle("reference")


@pytest.fixture(scope="session")
def fraq():
    """The product package; must load its CUDA extension (no fallback)."""
    import paper_1901_05128_b200 as f
    return f
