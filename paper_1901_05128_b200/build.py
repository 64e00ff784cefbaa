"""In-tree build of the B200 extension (sm_100a only).

Products (next to this file, so they travel with the repo snapshot):
  libfraqcu.so  -- CUDA kernels + the C ABI (include/fraqcu.h)
  libfraq.so    -- C++ mirror of the reference headers (csrc/fraq.hpp) over the C ABI
  _fraq*.so     -- pybind11 module with the reference binding's surface

Run ``python -m paper_1901_05128_b200.build`` (or ``__graft_entry__.build()``).
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(ROOT, "include")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_HOME = os.path.dirname(os.path.dirname(NVCC))
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CLI = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fraq")
CU_SOURCES = ["setup.cu", "history.cu", "history_dmma.cu", "history_fir.cu", "ffpe.cu", "modal.cu", "modal_dmma.cu", "direct.cu",
              "capi.cu", "diag.cu"]

CUDA_LIB = os.path.join(HERE, "libfraqcu.so")
CXX_LIB = os.path.join(HERE, "libfraq.so")
EXT = os.path.join(HERE, "_fraq" + sysconfig.get_config_var("EXT_SUFFIX"))


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> None:
    objdir = os.path.join(HERE, "_obj")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp"))]
    headers.append(os.path.join(INC, "fraqcu.h"))
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(objdir, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                   f"-I{INC}", "-c", s, "-o", o]
            if verbose_ptxas:
                cmd += ["-Xptxas", "-v"]
            cmd += os.environ.get("FRAQ_NVCC_FLAGS", "").split()  # experiment switches only
            _run(cmd)
    if force or _stale(CUDA_LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", CUDA_LIB, *objs, "-lcudart"])
    cxx = os.environ.get("CXX", "g++")
    cxx_srcs = [os.path.join(CSRC, f) for f in ("fraq.cpp", "fraq_bench.cpp")]
    if force or _stale(CXX_LIB, cxx_srcs + [CUDA_LIB] + headers):
        _run([cxx, "-O2", "-std=c++20", "-fPIC", "-shared", f"-I{INC}", f"-I{CSRC}", *cxx_srcs,
              "-o", CXX_LIB, f"-L{HERE}", "-lfraqcu", "-Wl,-rpath,$ORIGIN"])
    # the `fraq` command line (reference: tools/fraq_main.cpp)
    cli_cpp = os.path.join(CSRC, "fraq_cli.cpp")
    if force or _stale(CLI, [cli_cpp, CXX_LIB] + headers):
        _run([cxx, "-O2", "-std=c++20", f"-I{INC}", f"-I{CSRC}", cli_cpp, "-o", CLI,
              f"-L{HERE}", "-lfraq", "-lfraqcu", "-Wl,-rpath,$ORIGIN"])
    py_cpp = os.path.join(CSRC, "fraq_py.cpp")
    if force or _stale(EXT, [py_cpp, CXX_LIB] + headers):
        import pybind11
        _run([cxx, "-O2", "-std=c++20", "-fPIC", "-shared", f"-I{INC}", f"-I{CSRC}",
              f"-I{pybind11.get_include()}", f"-I{sysconfig.get_paths()['include']}", py_cpp,
              "-o", EXT, f"-L{HERE}", "-lfraq", "-lfraqcu", "-Wl,-rpath,$ORIGIN"])


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
