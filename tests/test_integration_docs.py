"""INTEGRATION.md's code is live: the C++ call-site sample compiles and links against the C++
mirror (CPU), and the ctypes stub over the raw C ABI runs on the GPU and agrees with the package."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1901_05128_b200")


def _blocks(lang):
    txt = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    return re.findall(r"```" + lang + r"\n(.*?)```", txt, re.S)


@pytest.mark.parametrize("block", [0, 1])
def test_cpp_call_sites_compile_and_link(tmp_path, block):
    """Block 0: histories / run / batches; block 1: the single-step API and the block-solver
    types (a test_fpfp.cpp-style call site)."""
    body = _blocks("cpp")[block]
    include = [l for l in body.splitlines() if l.startswith("#include")]
    code = "\n".join(l for l in body.splitlines() if not l.startswith("#include"))
    src = "\n".join(include) + """
#include <vector>
// the sample's free variables, as a caller of the reference API would have them
void example(long dim, long N, const std::vector<std::vector<double>>& u,
             std::vector<std::vector<double>>& d, const double* U, double* D,
             const fraq::ProblemSpec& spec, const std::vector<fraq::ProblemSpec>& specs,
             const std::vector<double>& g1, const std::vector<double>& g2) {
""" + code + "\n}\n"
    cpp = tmp_path / "sample.cpp"
    cpp.write_text(src)
    out = tmp_path / "libsample.so"
    r = subprocess.run(["g++", "-std=c++20", "-fPIC", "-shared", f"-I{ROOT}/include",
                        f"-I{PKG}/csrc", str(cpp), "-o", str(out), f"-L{PKG}", "-lfraq",
                        "-lfraqcu", f"-Wl,-rpath,{PKG}", "-Wl,--no-undefined"],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.gpu
def test_ctypes_stub_runs(monkeypatch):
    code = [b for b in _blocks("python") if "ctypes" in b][0]
    monkeypatch.chdir(ROOT)
    ns = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)  # the stub asserts its own status codes
    U, D = ns["U"], ns["D"]
    import paper_1901_05128_b200 as fraq
    b = fraq.KernelBudget(horizon=65536, eps_tol=1e-12)
    k = fraq.build_sbd_kernel_auto(0.7, 1 / 65536, b)
    h = fraq.SbdHistory(k, fraq.HistoryVariant.standalone, U.shape[1])
    ref = np.array(h.run(U), dtype=float)
    ok = ~np.isnan(ref)
    assert np.array_equal(np.isnan(D), ~ok)
    assert np.max(np.abs(D[ok] - ref[ok])) <= 1e-12 * np.max(np.abs(ref[ok]))
