"""ctypes front end to the CPU oracle (TEST INFRASTRUCTURE ONLY).

Two libraries are exposed with one numpy-friendly interface:

* ``Oracle("port")``      -- oracle/liboracle.so, the C restatement (oracle/fraq_oracle.c);
* ``Oracle("reference")`` -- oracle/_ref/libfraq_ref.so, the UNMODIFIED reference sources
  compiled by oracle/Makefile with the forwarding shim oracle/ref_shim.cpp.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import this module.  The
product package (paper_1901_05128_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfraq_ref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_lp = C.POINTER(C.c_long)

ERRORS = {-1: ValueError, -2: RuntimeError, -3: IndexError, -4: ArithmeticError, -5: Exception}


class OracleError(Exception):
    pass


def _raise(code: int, what: str):
    if code:
        exc = ERRORS.get(code, OracleError)
        raise exc(f"{what}: oracle error {code}")


def ensure_built() -> None:
    """Builds liboracle.so (and _ref when /root/reference is present) with the committed Makefile."""
    need = not os.path.exists(PORT_SO) or (
        os.path.isdir("/root/reference/proj/src") and not os.path.exists(REF_SO))
    if need:
        subprocess.run(["make", "-s", "-f", os.path.join(HERE, "Makefile")], check=True,
                       cwd=os.path.dirname(HERE))


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


@dataclass
class Kernel:
    """Flat kernel tables (FastKernelBE when sbd is False: m1 = node_weights, r1 = ratios)."""
    sbd: bool
    gamma: float
    tau: float
    head: np.ndarray
    m1: np.ndarray
    r1: np.ndarray
    m2: np.ndarray = field(default_factory=lambda: np.zeros(0))
    r2: np.ndarray = field(default_factory=lambda: np.zeros(0))
    achieved_eps: float = 0.0

    @property
    def n_head(self) -> int:
        return len(self.head)

    @property
    def np1(self) -> int:
        return len(self.r1)

    @property
    def np2(self) -> int:
        return len(self.r2)


class _FoKernel(C.Structure):
    _fields_ = [("sbd", C.c_int), ("gamma", C.c_double), ("tau", C.c_double),
                ("n_head", C.c_int), ("head", C.c_double * 512), ("np1", C.c_int),
                ("np2", C.c_int), ("m1", C.c_double * 512), ("r1", C.c_double * 512),
                ("m2", C.c_double * 512), ("r2", C.c_double * 512)]


def _from_fo(k: _FoKernel, eps: float = 0.0) -> Kernel:
    return Kernel(bool(k.sbd), k.gamma, k.tau, np.array(k.head[:k.n_head]),
                  np.array(k.m1[:k.np1]), np.array(k.r1[:k.np1]),
                  np.array(k.m2[:k.np2]), np.array(k.r2[:k.np2]), eps)


def _to_fo(k: Kernel) -> _FoKernel:
    f = _FoKernel()
    f.sbd = int(k.sbd)
    f.gamma = k.gamma
    f.tau = k.tau
    f.n_head = k.n_head
    f.head[:k.n_head] = list(k.head)
    f.np1 = k.np1
    f.np2 = k.np2
    f.m1[:k.np1] = list(k.m1)
    f.r1[:k.np1] = list(k.r1)
    if k.np2:
        f.m2[:k.np2] = list(k.m2)
        f.r2[:k.np2] = list(k.r2)
    return f


SCHEMES = {"BE": 0, "FastBE": 1, "SBD": 2, "FastSBD": 3}
INITIAL = {"poly_sin": 0, "indicator": 1, "custom": 2}


class Oracle:
    def __init__(self, kind: str = "port"):
        ensure_built()
        self.kind = kind
        if kind == "port":
            self.lib = C.CDLL(PORT_SO)
        elif kind == "reference":
            if not ref_available():
                raise FileNotFoundError(REF_SO)
            self.lib = C.CDLL(REF_SO)
        else:
            raise ValueError(kind)
        L = self.lib
        if kind == "port":
            L.fo_gamma.restype = C.c_double
            L.fo_gamma.argtypes = [C.c_double]
            L.fo_reconstruct.restype = C.c_double
            L.fo_reconstruct.argtypes = [C.POINTER(_FoKernel), C.c_long]
            L.fo_laplacian_eigenvalue.restype = C.c_double
            L.fo_l2_norm.restype = C.c_double
        else:
            L.ref_gamma.restype = C.c_double
            L.ref_gamma.argtypes = [C.c_double]

    # ------------------------------------------------------------------ L0
    def gamma_fn(self, x: float) -> float:
        return (self.lib.fo_gamma if self.kind == "port" else self.lib.ref_gamma)(x)

    def gauss_jacobi(self, a: float, b: float, n: int):
        nodes = np.zeros(max(n, 1))
        w = np.zeros(max(n, 1))
        f = self.lib.fo_gauss_jacobi if self.kind == "port" else self.lib.ref_gauss_jacobi
        _raise(f(C.c_double(a), C.c_double(b), C.c_int(n), _p(nodes), _p(w)), "gauss_jacobi")
        return nodes[:n], w[:n]

    def jacobi_moment(self, a: float, b: float, k: int) -> float:
        out = C.c_double()
        f = self.lib.fo_jacobi_moment if self.kind == "port" else self.lib.ref_jacobi_moment
        _raise(f(C.c_double(a), C.c_double(b), C.c_int(k), C.byref(out)), "jacobi_moment")
        return out.value

    # ------------------------------------------------------------------ L1
    def be_weights(self, g: float, tau: float, nmax: int) -> np.ndarray:
        out = np.zeros(max(nmax, 0) + 1)
        f = self.lib.fo_be_weights if self.kind == "port" else self.lib.ref_be_weights
        _raise(f(C.c_double(g), C.c_double(tau), C.c_long(nmax), _p(out)), "be_weights")
        return out

    def sbd_weights(self, g: float, tau: float, nmax: int) -> np.ndarray:
        out = np.zeros(max(nmax, 0) + 1)
        f = self.lib.fo_sbd_weights if self.kind == "port" else self.lib.ref_sbd_weights
        _raise(f(C.c_double(g), C.c_double(tau), C.c_long(nmax), _p(out)), "sbd_weights")
        return out

    def coupling_from_transition(self, m: float) -> float:
        out = C.c_double()
        f = (self.lib.fo_coupling_from_transition if self.kind == "port"
             else self.lib.ref_coupling_from_transition)
        _raise(f(C.c_double(m), C.byref(out)), "coupling_from_transition")
        return out.value

    def default_sbd_head(self, g: float) -> int:
        f = self.lib.fo_default_sbd_head if self.kind == "port" else self.lib.ref_default_sbd_head
        f.argtypes = [C.c_double]
        return f(g)

    # ------------------------------------------------------------------ L2 kernels
    def build_be_kernel(self, g: float, tau: float, np_: int) -> Kernel:
        if self.kind == "port":
            k = _FoKernel()
            _raise(self.lib.fo_build_be_kernel(C.c_double(g), C.c_double(tau), C.c_int(np_),
                                               C.byref(k)), "build_be_kernel")
            return _from_fo(k)
        head = np.zeros(2)
        m = np.zeros(max(np_, 1))
        r = np.zeros(max(np_, 1))
        _raise(self.lib.ref_build_be_kernel(C.c_double(g), C.c_double(tau), C.c_int(np_),
                                            _p(head), _p(m), _p(r)), "build_be_kernel")
        return Kernel(False, g, tau, head, m[:np_], r[:np_])

    def build_sbd_kernel(self, g: float, tau: float, np1: int, np2: int, nh: int) -> Kernel:
        if self.kind == "port":
            k = _FoKernel()
            _raise(self.lib.fo_build_sbd_kernel(C.c_double(g), C.c_double(tau), C.c_int(np1),
                                                C.c_int(np2), C.c_int(nh), C.byref(k)),
                   "build_sbd_kernel")
            return _from_fo(k)
        head = np.zeros(max(nh, 1))
        m1, r1 = np.zeros(max(np1, 1)), np.zeros(max(np1, 1))
        m2, r2 = np.zeros(max(np2, 1)), np.zeros(max(np2, 1))
        _raise(self.lib.ref_build_sbd_kernel(C.c_double(g), C.c_double(tau), C.c_int(np1),
                                             C.c_int(np2), C.c_int(nh), _p(head), _p(m1),
                                             _p(r1), _p(m2), _p(r2)), "build_sbd_kernel")
        return Kernel(True, g, tau, head[:nh], m1[:np1], r1[:np1], m2[:np2], r2[:np2])

    def build_kernel_auto(self, sbd: bool, g: float, tau: float, horizon: int,
                          eps_tol: float = 1e-12, max_points: int = 256,
                          max_head: int = 256) -> Kernel:
        if self.kind == "port":
            k = _FoKernel()
            h = C.c_long(horizon)
            ach = C.c_double()
            f = self.lib.fo_build_sbd_kernel_auto if sbd else self.lib.fo_build_be_kernel_auto
            _raise(f(C.c_double(g), C.c_double(tau), C.byref(h), C.c_double(eps_tol),
                     C.c_int(max_points), C.c_int(max_head), C.byref(k), C.byref(ach)),
                   "build_kernel_auto")
            return _from_fo(k, ach.value)
        sizes = (C.c_int * 3)()
        ach = C.c_double()
        head = np.zeros(512)
        m1, r1, m2, r2 = (np.zeros(512) for _ in range(4))
        if sbd:
            _raise(self.lib.ref_build_sbd_kernel_auto(
                C.c_double(g), C.c_double(tau), C.c_long(horizon), C.c_double(eps_tol),
                C.c_int(max_points), C.c_int(max_head), sizes, C.byref(ach), _p(head), _p(m1),
                _p(r1), _p(m2), _p(r2)), "build_sbd_kernel_auto")
        else:
            _raise(self.lib.ref_build_be_kernel_auto(
                C.c_double(g), C.c_double(tau), C.c_long(horizon), C.c_double(eps_tol),
                C.c_int(max_points), C.c_int(max_head), sizes, C.byref(ach), _p(head), _p(m1),
                _p(r1)), "build_be_kernel_auto")
        n1, n2, nh = sizes[0], sizes[1], sizes[2]
        return Kernel(sbd, g, tau, head[:nh].copy(), m1[:n1].copy(), r1[:n1].copy(),
                      m2[:n2].copy(), r2[:n2].copy(), ach.value)

    def _flat(self, k: Kernel):
        head, m1, r1 = _arr(k.head), _arr(k.m1), _arr(k.r1)
        m2 = _arr(k.m2) if k.np2 else np.zeros(1)
        r2 = _arr(k.r2) if k.np2 else np.zeros(1)
        keep = (head, m1, r1, m2, r2)
        args = [C.c_int(int(k.sbd)), C.c_double(k.gamma), C.c_double(k.tau), C.c_int(k.n_head),
                C.c_int(k.np1), C.c_int(k.np2), _p(head), _p(m1), _p(r1), _p(m2), _p(r2)]
        return keep, args

    def reconstruct(self, k: Kernel, idx) -> np.ndarray:
        idx = np.ascontiguousarray(np.atleast_1d(np.asarray(idx, dtype=np.int64)))
        out = np.zeros(len(idx))
        if self.kind == "port":
            fk = _to_fo(k)
            for t, i in enumerate(idx):
                out[t] = self.lib.fo_reconstruct(C.byref(fk), C.c_long(int(i)))
            return out
        keep, args = self._flat(k)
        _raise(self.lib.ref_reconstruct(*args, C.c_long(len(idx)), idx.ctypes.data_as(_lp),
                                        _p(out)), "reconstruct")
        return out

    def kernel_error_report(self, k: Kernel, nmax: int):
        eps = np.zeros(nmax + 1)
        mx = C.c_double()
        am = C.c_long()
        if self.kind == "port":
            fk = _to_fo(k)
            _raise(self.lib.fo_kernel_error_report(C.byref(fk), C.c_long(nmax), _p(eps),
                                                   C.byref(mx), C.byref(am)),
                   "kernel_error_report")
        else:
            keep, args = self._flat(k)
            _raise(self.lib.ref_kernel_error_report(*args, C.c_long(nmax), _p(eps), C.byref(mx),
                                                    C.byref(am)), "kernel_error_report")
        return eps, mx.value, am.value

    # ------------------------------------------------------------------ L2 histories
    def hist_run(self, k: Kernel, U: np.ndarray, scheme_variant: bool = False) -> np.ndarray:
        """U[n_steps, dim] pushed in order; returns D[n_steps, dim] (NaN where undefined)."""
        U = _arr(U)
        n, dim = U.shape
        D = np.zeros_like(U)
        if self.kind == "port":
            fk = _to_fo(k)
            _raise(self.lib.fo_hist_run(C.byref(fk), C.c_int(int(scheme_variant)), C.c_long(dim),
                                        C.c_long(n), _p(U), _p(D)), "hist_run")
        else:
            keep, args = self._flat(k)
            _raise(self.lib.ref_hist_run(*args, C.c_int(int(scheme_variant)), C.c_long(dim),
                                         C.c_long(n), _p(U), _p(D)), "hist_run")
        return D

    def direct_cq(self, sbd: bool, g: float, tau: float, U: np.ndarray) -> np.ndarray:
        """Classical O(N^2) sum_{i<=n} d_i u_{n-i} with the exact table (port only)."""
        U = _arr(U)
        n, dim = U.shape
        D = np.zeros_like(U)
        lib = Oracle("port").lib if self.kind != "port" else self.lib
        _raise(lib.fo_direct_cq(C.c_int(int(sbd)), C.c_double(g), C.c_double(tau),
                                C.c_long(dim), C.c_long(n), _p(U), _p(D)), "direct_cq")
        return D

    # ------------------------------------------------------------------ L4 FFPE
    def run(self, alpha1, alpha2, a, grid_m, t_final, n_steps, scheme="FastBE",
            initial="poly_sin", custom_g1=None, custom_g2=None, kconf=None, eps_tol=1e-12):
        """fraq::run restated (port) or forwarded (reference).  kconf = dict with be_points,
        sbd_points_1, sbd_points_2, sbd_head, auto_size.  Returns (g1, g2, eps1, eps2)."""
        kc = dict(be_points=64, sbd_points_1=41, sbd_points_2=41, sbd_head=0, auto_size=True)
        if kconf:
            kc.update(kconf)
        g1 = np.zeros(grid_m)
        g2 = np.zeros(grid_m)
        e1, e2 = C.c_double(), C.c_double()
        cg1 = _arr(custom_g1) if custom_g1 is not None else np.zeros(grid_m)
        cg2 = _arr(custom_g2) if custom_g2 is not None else np.zeros(grid_m)
        if self.kind == "port":
            class Spec(C.Structure):
                _fields_ = [("alpha1", C.c_double), ("alpha2", C.c_double), ("a", C.c_double),
                            ("length", C.c_double), ("t_final", C.c_double), ("grid_m", C.c_int),
                            ("n_steps", C.c_long), ("initial", C.c_int), ("custom_g1", _dp),
                            ("custom_g2", _dp)]

            class KC(C.Structure):
                _fields_ = [("be_points", C.c_int), ("sbd_points_1", C.c_int),
                            ("sbd_points_2", C.c_int), ("sbd_head", C.c_int),
                            ("eps_tol", C.c_double), ("auto_size", C.c_int)]
            s = Spec(alpha1, alpha2, a, 1.0, t_final, grid_m, n_steps, INITIAL[initial],
                     _p(cg1), _p(cg2))
            kk = KC(kc["be_points"], kc["sbd_points_1"], kc["sbd_points_2"], kc["sbd_head"],
                    eps_tol, int(kc["auto_size"]))
            _raise(self.lib.fo_run(C.byref(s), C.c_int(SCHEMES[scheme]), C.byref(kk), _p(g1),
                                   _p(g2), C.byref(e1), C.byref(e2), None, None), "run")
        else:
            ki = (C.c_int * 5)(kc["be_points"], kc["sbd_points_1"], kc["sbd_points_2"],
                               kc["sbd_head"], int(kc["auto_size"]))
            loop = C.c_double()
            _raise(self.lib.ref_run(C.c_double(alpha1), C.c_double(alpha2), C.c_double(a),
                                    C.c_int(grid_m), C.c_double(t_final), C.c_long(n_steps),
                                    C.c_int(INITIAL[initial]), _p(cg1), _p(cg2),
                                    C.c_int(SCHEMES[scheme]), ki, C.c_double(eps_tol), _p(g1),
                                    _p(g2), C.byref(e1), C.byref(e2), C.byref(loop)), "run")
            self.last_loop_seconds = loop.value  # fraq::run's own loop timer (fpfp.cpp:361-366)
        return g1, g2, e1.value, e2.value

    def block_solve(self, d01, d02, a, tau, m, lead, rhs1, rhs2):
        rhs1, rhs2 = _arr(rhs1), _arr(rhs2)
        g1, g2 = np.zeros(m), np.zeros(m)
        if self.kind == "port":
            class Blk(C.Structure):
                _fields_ = [("m", C.c_int), ("n", C.c_int), ("kl", C.c_int), ("ku", C.c_int),
                            ("ldab", C.c_int), ("ab", _dp), ("piv", _ip), ("d01", C.c_double),
                            ("d02", C.c_double), ("a", C.c_double), ("lead_tau", C.c_double),
                            ("ih2", C.c_double)]
            b = Blk()
            _raise(self.lib.fo_block_init(C.byref(b), C.c_double(d01), C.c_double(d02),
                                          C.c_double(a), C.c_double(tau), C.c_int(m),
                                          C.c_double(1.0 / (m + 1)), C.c_double(lead)),
                   "block_init")
            self.lib.fo_block_solve(C.byref(b), _p(rhs1), _p(rhs2), _p(g1), _p(g2))
            self.lib.fo_block_free(C.byref(b))
        else:
            _raise(self.lib.ref_block_solve(C.c_double(d01), C.c_double(d02), C.c_double(a),
                                            C.c_double(tau), C.c_int(m), C.c_double(lead),
                                            _p(rhs1), _p(rhs2), _p(g1), _p(g2)), "block_solve")
        return g1, g2

    # ------------------------------------------------------------------ CPU baseline
    def bench_history(self, kernels, U: np.ndarray, threads: int):
        """Times reference histories over U[n_steps, dofs] split evenly into len(kernels) groups,
        `threads` worker threads.  Returns (seconds, D at the last step)."""
        assert self.kind == "reference"
        U = _arr(U)
        n_steps, dofs = U.shape
        G = len(kernels)
        sbd = kernels[0].sbd
        keep = []

        def ptrs(name):
            arrs = [_arr(getattr(k, name)) if len(getattr(k, name)) else np.zeros(1)
                    for k in kernels]
            keep.extend(arrs)
            return (_dp * G)(*[_p(a) for a in arrs])
        gam = (C.c_double * G)(*[k.gamma for k in kernels])
        nh = (C.c_int * G)(*[k.n_head for k in kernels])
        n1 = (C.c_int * G)(*[k.np1 for k in kernels])
        n2 = (C.c_int * G)(*[k.np2 for k in kernels])
        D = np.zeros(dofs)
        secs = C.c_double()
        _raise(self.lib.ref_bench_history(
            C.c_int(int(sbd)), C.c_int(G), gam, C.c_double(kernels[0].tau), nh, n1, n2,
            ptrs("head"), ptrs("m1"), ptrs("r1"), ptrs("m2"), ptrs("r2"), C.c_long(dofs),
            C.c_long(n_steps), _p(U), _p(D), C.c_int(threads), C.byref(secs)), "bench_history")
        return secs.value, D

    def anchor_ld(self, k1: Kernel, k2: Kernel, a: float, tau: float, N: int, M: int, modes,
                  g1, g2):
        """Extended-precision mode-space evaluation of the 1D fast scheme on sampled DST modes
        (oracle/fraq_anchor_ld.c; liboracle.so for either oracle kind).  modes are 1-based.
        Returns the coefficients (uN, vN) after N levels."""
        lib = self.lib if self.kind == "port" else C.CDLL(PORT_SO)
        modes = np.ascontiguousarray(np.asarray(modes, dtype=np.int32))
        g1, g2 = _arr(g1), _arr(g2)
        nm = len(modes)
        uN, vN = np.zeros(nm), np.zeros(nm)
        f1, f2 = _to_fo(k1), _to_fo(k2)
        _raise(lib.fo_anchor_ld(C.byref(f1), C.byref(f2), C.c_double(a), C.c_double(tau),
                                C.c_long(N), C.c_int(M), C.c_long(nm),
                                modes.ctypes.data_as(_ip), _p(g1), _p(g2), _p(uN), _p(vN)),
               "anchor_ld")
        return uN, vN

    def anchor_modes_ld(self, k1: Kernel, k2: Kernel, a: float, tau: float, N: int, lam, u0, v0):
        """anchor_ld for caller-given modes: lam, u0, v0 as numpy longdouble (or float) arrays,
        passed through unrounded as (hi, lo) double pairs.  Returns (uN, vN)."""
        lib = self.lib if self.kind == "port" else C.CDLL(PORT_SO)

        def split(x):
            x = np.asarray(x, dtype=np.longdouble)
            hi = x.astype(np.float64)
            lo = (x - hi.astype(np.longdouble)).astype(np.float64)
            return np.ascontiguousarray(np.stack([hi, lo], axis=1).ravel())
        L2, U2, V2 = split(lam), split(u0), split(v0)
        nm = len(L2) // 2
        uN, vN = np.zeros(nm), np.zeros(nm)
        f1, f2 = _to_fo(k1), _to_fo(k2)
        _raise(lib.fo_anchor_modes_ld(C.byref(f1), C.byref(f2), C.c_double(a), C.c_double(tau),
                                      C.c_long(N), C.c_long(nm), _p(L2), _p(U2), _p(V2), _p(uN),
                                      _p(vN)), "anchor_modes_ld")
        return uN, vN

    def hist_trace(self, kernels, U: np.ndarray, stride: int, threads: int):
        """Reference histories (standalone) over U[n_steps, dofs] split evenly into
        len(kernels) groups, `threads` workers; returns D at levels stride-1, 2 stride-1, ...
        as an array [n_steps // stride, dofs]."""
        assert self.kind == "reference"
        U = _arr(U)
        n_steps, dofs = U.shape
        G = len(kernels)
        keep = []

        def ptrs(name):
            arrs = [_arr(getattr(k, name)) if len(getattr(k, name)) else np.zeros(1)
                    for k in kernels]
            keep.extend(arrs)
            return (_dp * G)(*[_p(a) for a in arrs])
        gam = (C.c_double * G)(*[k.gamma for k in kernels])
        nh = (C.c_int * G)(*[k.n_head for k in kernels])
        n1 = (C.c_int * G)(*[k.np1 for k in kernels])
        n2 = (C.c_int * G)(*[k.np2 for k in kernels])
        D = np.zeros((n_steps // stride, dofs))
        _raise(self.lib.ref_hist_trace(
            C.c_int(int(kernels[0].sbd)), C.c_int(G), gam, C.c_double(kernels[0].tau), nh, n1,
            n2, ptrs("head"), ptrs("m1"), ptrs("r1"), ptrs("m2"), ptrs("r2"), C.c_long(dofs),
            C.c_long(n_steps), _p(U), C.c_long(stride), _p(D), C.c_int(threads)), "hist_trace")
        return D

    def modal_run(self, k1: Kernel, k2: Kernel, a: float, tau: float, N: int, lam, u0, v0,
                  threads: int = 1):
        """Mode-space fast FFPE stepping (test_fpfp.cpp:79-134 with fast histories; lam = the
        Laplacian eigenvalue of each mode, u0/v0 = initial DST coefficients).  Port: fo_modal_run
        (single thread); reference: the reference's BeHistory/SbdHistory lanes, `threads`
        workers over mode slices.  Returns (uN, vN, seconds)."""
        lam, u0, v0 = _arr(lam), _arr(u0), _arr(v0)
        nm = len(lam)
        uN, vN = np.zeros(nm), np.zeros(nm)
        if self.kind == "port":
            f1, f2 = _to_fo(k1), _to_fo(k2)
            import time as _t
            t0 = _t.perf_counter()
            _raise(self.lib.fo_modal_run(C.byref(f1), C.byref(f2), C.c_double(a), C.c_double(tau),
                                         C.c_long(N), C.c_long(nm), _p(lam), _p(u0), _p(v0),
                                         _p(uN), _p(vN)), "modal_run")
            return uN, vN, _t.perf_counter() - t0
        ks = [k1, k2]
        keep = []

        def ptrs(name):
            arrs = [_arr(getattr(k, name)) if len(getattr(k, name)) else np.zeros(1) for k in ks]
            keep.extend(arrs)
            return (_dp * 2)(*[_p(x) for x in arrs])
        secs = C.c_double()
        _raise(self.lib.ref_modal_run(
            C.c_int(int(k1.sbd)), (C.c_double * 2)(k1.gamma, k2.gamma), C.c_double(tau),
            (C.c_int * 2)(k1.n_head, k2.n_head), (C.c_int * 2)(k1.np1, k2.np1),
            (C.c_int * 2)(k1.np2, k2.np2), ptrs("head"), ptrs("m1"), ptrs("r1"), ptrs("m2"),
            ptrs("r2"), C.c_double(a), C.c_long(N), C.c_long(nm), _p(lam), _p(u0), _p(v0),
            _p(uN), _p(vN), C.c_int(threads), C.byref(secs)), "modal_run")
        return uN, vN, secs.value
