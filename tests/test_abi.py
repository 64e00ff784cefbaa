"""C-ABI boundary checks that need no GPU: libfraqcu.so loads, exports every symbol include/fraqcu.h
declares, host-only entry points behave like the reference, and compute entry points fail loudly
(FRAQ_ECUDA) instead of falling back to the CPU when no device is present."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1901_05128_b200", "libfraqcu.so")
HDR = os.path.join(ROOT, "include", "fraqcu.h")


def declared_symbols():
    text = open(HDR).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = set(re.findall(r"\b(fraq_[a-z0-9_]+)\s*\(", text))
    return sorted(n for n in names if not n.endswith("_fn"))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        import __graft_entry__
        __graft_entry__.build()
    return C.CDLL(LIB)


def test_library_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_host_entry_points(lib):
    lib.fraq_gamma.restype = C.c_double
    lib.fraq_gamma.argtypes = [C.c_double]
    assert lib.fraq_gamma(5.0) == pytest.approx(24.0, rel=1e-13)
    assert lib.fraq_gamma(1.3) == pytest.approx(0.89747069630627718, rel=1e-13)
    out = C.c_double()
    assert lib.fraq_coupling_from_transition(C.c_double(0.75), C.byref(out)) == 0
    assert out.value == pytest.approx(0.5)
    assert lib.fraq_coupling_from_transition(C.c_double(0.5), C.byref(out)) == -1  # invalid_argument
    lib.fraq_default_sbd_head.argtypes = [C.c_double]
    assert lib.fraq_default_sbd_head(0.3) == 15 and lib.fraq_default_sbd_head(0.7) == 17
    assert lib.fraq_jacobi_moment(C.c_double(0.0), C.c_double(0.0), C.c_int(2), C.byref(out)) == 0
    assert out.value == pytest.approx(2.0 / 3.0, rel=1e-13)
    assert lib.fraq_jacobi_moment(C.c_double(-1.2), C.c_double(0.0), C.c_int(3), C.byref(out)) == -1


def test_no_cpu_fallback_without_device(lib):
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    ctx = C.c_void_p()
    st = lib.fraq_ctx_create(0, None, C.byref(ctx))
    assert st == -5  # FRAQ_ECUDA: loud failure, no CPU path
    buf = C.create_string_buffer(256)
    lib.fraq_last_error(buf, 256)
    assert b"CUDA" in buf.value


def test_python_package_fails_loudly_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except Exception:
        pass
    import paper_1901_05128_b200 as fraq
    with pytest.raises(RuntimeError):
        fraq.be_weights(0.5, 1.0, 3)
    # host-only harness helpers mirror the reference (bench.cpp:42-57,140-153)
    assert fraq.parse_fraction("1/3200") == 1.0 / 3200.0
    assert fraq.compute_rates([(0.5, 4.0), (0.25, 1.0)])[0] == pytest.approx(2.0, abs=1e-12)
    with pytest.raises(ValueError):
        fraq.compute_rates([(0.5, 4.0), (0.2, 1.0)])


def test_reference_all_is_exported():
    import paper_1901_05128_b200 as fraq
    ref_all = ["BeHistory", "FastKernelBE", "FastKernelSBD", "HistoryVariant", "JacobiRule",
               "KernelConfig", "KernelErrorReport", "ProblemSpec", "RunResult", "SbdHistory",
               "Scheme", "StateField", "WeightTable", "be_weights", "build_be_kernel",
               "build_sbd_kernel", "compute_rates", "coupling_from_transition",
               "default_sbd_head", "gauss_jacobi", "initial_field", "jacobi_moment",
               "kernel_error_report", "l2_norm", "parse_fraction", "run", "sbd_weights"]
    for name in ref_all:
        assert hasattr(fraq, name), name
