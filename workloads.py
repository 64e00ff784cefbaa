"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved: BASELINE.json's configs are synthetic and the paper's data are
analytic initial functions.  numpy PCG64 generators with seeds 1901051281..1901051285 (C1..C5);
draw order is documented per function.  Pure numpy (host); the bench builds the same signals on
the device with torch from the returned parameters.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEEDS = {"C1": 1901051281, "C2": 1901051282, "C3": 1901051283, "C4": 1901051284, "C5": 1901051285}


@dataclass
class SignalParams:
    """u_k(t) = a_k t^{b_k} + c_k sin(w_k t) per DOF, group (CQ exponent gamma) per DOF."""
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray
    w: np.ndarray
    gamma: np.ndarray
    tau: float
    n_steps: int

    @property
    def dofs(self) -> int:
        return len(self.a)

    def signal(self, n0: int, n1: int, dof_idx=None) -> np.ndarray:
        """U[n, k] for time indices n0 <= n < n1 (t_n = n tau), shape (n1-n0, #dofs)."""
        sel = slice(None) if dof_idx is None else dof_idx
        t = (np.arange(n0, n1, dtype=np.float64) * self.tau)[:, None]
        a, b, c, w = self.a[sel], self.b[sel], self.c[sel], self.w[sel]
        out = a[None, :] * np.power(t, b[None, :])
        nz = c != 0.0
        if np.any(nz):
            out = out + c[None, :] * np.sin(w[None, :] * t)
        return out


def c1_params(dofs: int = 1024) -> SignalParams:
    """C1: BE, gamma = 1 - alpha = 0.5, u_k(t) = t^{b_k}, b_k ~ U[0.1, 2], T = 1, N = 4096."""
    rng = np.random.Generator(np.random.PCG64(SEEDS["C1"]))
    b = rng.uniform(0.1, 2.0, dofs)
    n = 4096
    return SignalParams(a=np.ones(dofs), b=b, c=np.zeros(dofs), w=np.zeros(dofs),
                        gamma=np.full(dofs, 0.5), tau=1.0 / n, n_steps=n)


def c2_params(dofs: int = 65536) -> SignalParams:
    """C2: BDF2, alpha1 = 0.3 on the first half of the DOFs, alpha2 = 0.7 on the second half;
    the CQ exponent is gamma = 1 - alpha (0.7 then 0.3), as for C1 and the FFPE.  Draws in order:
    a ~ N(0,1), c ~ N(0,1), b ~ U[0.1,2], w ~ U[1,20] (each of length dofs).  T = 1, N = 65536."""
    rng = np.random.Generator(np.random.PCG64(SEEDS["C2"]))
    a = rng.standard_normal(dofs)
    c = rng.standard_normal(dofs)
    b = rng.uniform(0.1, 2.0, dofs)
    w = rng.uniform(1.0, 20.0, dofs)
    half = dofs // 2
    gamma = np.concatenate([np.full(half, 1.0 - 0.3), np.full(dofs - half, 1.0 - 0.7)])
    n = 65536
    return SignalParams(a=a, b=b, c=c, w=w, gamma=gamma, tau=1.0 / n, n_steps=n)


@dataclass
class FfpeInstance:
    alpha1: float
    alpha2: float
    m_transition: float
    coupling_a: float
    g1: np.ndarray
    g2: np.ndarray


def coupling(m: float) -> float:
    """a = (1-m)/(2m-1) (cq_weights.cpp:61-67)."""
    return (1.0 - m) / (2.0 * m - 1.0)


def c3_instance(grid_m: int = 4095) -> FfpeInstance:
    """C3: m = 0.45 (a = -5.5), alpha = (0.4, 0.8); G0_1 = 1 on (0, 0.5), G0_2 = 1 on (0.5, 1),
    both 0 at x = 0.5 (open intervals, as fpfp.cpp:58-59)."""
    h = 1.0 / (grid_m + 1)
    x = (np.arange(grid_m) + 1) * h
    g1 = np.where(x < 0.5, 1.0, 0.0)
    g2 = np.where(x > 0.5, 1.0, 0.0)
    return FfpeInstance(0.4, 0.8, 0.45, coupling(0.45), g1, g2)


def c4_instance(grid_m: int = 1023) -> FfpeInstance:
    """C4 (2D, unit square, grid_m^2 interior points, row-major with x fastest): m = 0.4 (a = -3),
    alpha = (0.3, 0.6); G0_1 = 1 on [0, 0.5]^2 (closed), G0_2 = 1 + U[-0.1, 0.1] at every
    interior node (one draw per node in storage order)."""
    rng = np.random.Generator(np.random.PCG64(SEEDS["C4"]))
    h = 1.0 / (grid_m + 1)
    x = (np.arange(grid_m) + 1) * h
    X, Y = np.meshgrid(x, x)
    g1 = ((X <= 0.5) & (Y <= 0.5)).astype(float).ravel()
    g2 = 1.0 + rng.uniform(-0.1, 0.1, grid_m * grid_m)
    return FfpeInstance(0.3, 0.6, 0.4, coupling(0.4), g1, g2)


def c5_instances(n_inst: int = 4096, grid_m: int = 4095) -> list[FfpeInstance]:
    """C5: per instance alpha1, alpha2 ~ U[0.1, 0.9]; m from U on [0.1,0.45] u [0.55,0.9] (draw
    U[0, 0.7) then map); per field 8 sorted U(0,1) breakpoints and 9 levels ~ U[0,1], left-closed
    pieces sampled at x_j = j h.  Draw order per instance: alpha1, alpha2, m, then field 1
    (breakpoints, levels), field 2 (breakpoints, levels)."""
    rng = np.random.Generator(np.random.PCG64(SEEDS["C5"]))
    h = 1.0 / (grid_m + 1)
    x = (np.arange(grid_m) + 1) * h
    out = []
    for _ in range(n_inst):
        a1 = rng.uniform(0.1, 0.9)
        a2 = rng.uniform(0.1, 0.9)
        u = rng.uniform(0.0, 0.7)
        m = 0.1 + u if u < 0.35 else 0.55 + (u - 0.35)
        fields = []
        for _f in range(2):
            bp = np.sort(rng.uniform(0.0, 1.0, 8))
            lv = rng.uniform(0.0, 1.0, 9)
            fields.append(lv[np.searchsorted(bp, x, side="right")])
        out.append(FfpeInstance(a1, a2, m, coupling(m), fields[0], fields[1]))
    return out
