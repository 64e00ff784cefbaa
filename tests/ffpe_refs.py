"""Test-side restatements for the FFPE checks (TEST INFRASTRUCTURE; numpy, CPU).

* ``fast_stepper_nd``: the reference's FastStepper algebra (fpfp.cpp:180-349) in physical space
  for a 1D or 2D grid with the (five-point in 2D) Dirichlet Laplacian and a dense solve of the
  coupled two-field system -- small grids only.  In 1D it is the reference scheme itself; in 2D it
  is the restatement SURVEY.md §8(c) prescribes for C4 (the reference has no 2D capability).
* ``modespace_fastbe``: the same scheme in the DST eigenbasis (the reference's mode-space oracle,
  test_fpfp.cpp:21-180, with fast histories), the fp64 accuracy anchor at large grids.
Node tables come from the CPU oracle (the reference's own auto-sizer / builders).
"""
from __future__ import annotations

import numpy as np


def laplacian(m: int, dim: int) -> np.ndarray:
    """Dense -Delta_h on m (1D) or m*m (2D, row-major, x fastest) interior points, h = 1/(m+1)."""
    h = 1.0 / (m + 1)
    T = (2 * np.eye(m) - np.eye(m, k=1) - np.eye(m, k=-1)) / h ** 2
    if dim == 1:
        return T
    I = np.eye(m)
    return np.kron(I, T) + np.kron(T, I)


class FastHist:
    """numpy restatement of BeHistory/SbdHistory in the scheme variant (fast_kernel.cpp:261-409)."""

    def __init__(self, k, n_dof):
        self.k = k
        self.r = np.concatenate([k.r1, k.r2])
        if k.sbd:
            self.f = np.concatenate([k.m1 * k.r1 ** (k.n_head - 3), k.m2 * k.r2 ** (k.n_head - 3)])
            self.L = k.n_head
        else:
            self.f = k.m1.copy()
            self.L = 2
        self.y = np.zeros((len(self.r), n_dof))

    def advance(self, n, G):
        """Level n: y <- r y + f G^{n-L} (G^0 is never fed: lo = 1)."""
        self.y *= self.r[:, None]
        src = n - self.L
        if src >= 1:
            self.y += self.f[:, None] * G[src][None, :]

    def history_sum(self):
        return self.y.sum(axis=0)


def fast_stepper_nd(orc, alpha1, alpha2, a, m, dim, t_final, N, sbd, g1, g2):
    tau = t_final / N
    A = laplacian(m, dim)
    nd = A.shape[0]
    ks = [orc.build_kernel_auto(sbd, 1 - al, tau, N) for al in (alpha1, alpha2)]
    hs = [FastHist(k, nd) for k in ks]
    G = [[np.asarray(g1, float).copy()], [np.asarray(g2, float).copy()]]
    d0 = [k.head[0] for k in ks]
    I = np.eye(nd)

    def system(scale, lead):
        return np.block([[lead / tau * I + scale * d0[0] * (a * I + A), -a * scale * d0[1] * I],
                         [-a * scale * d0[0] * I, lead / tau * I + scale * d0[1] * (a * I + A)]])
    main = system(1.0, 1.5 if sbd else 1.0)
    first = system(2.0 / 3.0, 1.0) if sbd else None
    corr_p = [[np.ones(len(k.r1)), np.ones(len(k.r2))] for k in ks]
    corr_e = [0, 0]
    for n in range(1, N + 1):
        for f in range(2):
            hs[f].advance(n, G[f])
        if sbd and n == 1:
            u0, v0 = G[0][0], G[1][0]
            r1 = u0 / tau - (d0[0] / 3.0) * (a * u0 + A @ u0) + (a * d0[1] / 3.0) * v0
            r2 = v0 / tau - (d0[1] / 3.0) * (a * v0 + A @ v0) + (a * d0[0] / 3.0) * u0
            x = np.linalg.solve(first, np.concatenate([r1, r2]))
        else:
            s = []
            for f in range(2):
                k = ks[f]
                sf = hs[f].history_sum()
                if sbd:
                    top = min(k.n_head - 1, n - 1)
                    for i in range(1, top + 1):
                        sf = sf + k.head[i] * G[f][n - i]
                    if n - 1 < k.n_head:
                        c = k.head[n - 1]
                    else:  # CorrPowers::value_at (fpfp.cpp:240-250): running powers, e = n-4
                        while corr_e[f] < n - 4:
                            corr_p[f][0] *= k.r1
                            corr_p[f][1] *= k.r2
                            corr_e[f] += 1
                        c = np.dot(k.m1, corr_p[f][0]) + np.dot(k.m2, corr_p[f][1])
                    sf = sf + 0.5 * c * G[f][0]
                elif n >= 2:
                    sf = sf + k.head[1] * G[f][n - 1]
                s.append(sf)
            if sbd:
                l1 = (2 * G[0][n - 1] - 0.5 * G[0][n - 2]) / tau
                l2 = (2 * G[1][n - 1] - 0.5 * G[1][n - 2]) / tau
            else:
                l1, l2 = G[0][n - 1] / tau, G[1][n - 1] / tau
            r1 = l1 - a * s[0] - A @ s[0] + a * s[1]
            r2 = l2 - a * s[1] - A @ s[1] + a * s[0]
            x = np.linalg.solve(main, np.concatenate([r1, r2]))
        G[0].append(x[:nd])
        G[1].append(x[nd:])
    return G[0][N], G[1][N]


def modespace_fastbe(orc, g1, g2, M, N, a, al1, al2, tau=1.0 / 16384):
    """FastBE in mode space, fp64 (per-mode 2x2 solves + per-mode fast histories)."""
    ks = [orc.build_kernel_auto(False, 1 - al1, tau, N), orc.build_kernel_auto(False, 1 - al2, tau, N)]
    h = 1.0 / (M + 1)
    k = np.arange(1, M + 1)
    V = np.sin(np.outer(k, k) * np.pi * h)
    lam = 4 / h ** 2 * np.sin(k * np.pi * h / 2) ** 2
    G = [[2 / (M + 1) * (V @ g1)], [2 / (M + 1) * (V @ g2)]]
    y = [np.zeros((len(kk.r1), M)) for kk in ks]
    d0 = [kk.head[0] for kk in ks]
    d1 = [kk.head[1] for kk in ks]
    for n in range(1, N + 1):
        s = []
        for f in range(2):
            y[f] *= ks[f].r1[:, None]
            if n - 2 >= 1:
                y[f] += ks[f].m1[:, None] * G[f][n - 2][None, :]
            sf = y[f].sum(axis=0)
            s.append(sf + d1[f] * G[f][n - 1] if n >= 2 else sf)
        r1 = G[0][n - 1] / tau - (a + lam) * s[0] + a * s[1]
        r2 = G[1][n - 1] / tau - (a + lam) * s[1] + a * s[0]
        a11, a12 = 1 / tau + d0[0] * (a + lam), -a * d0[1]
        a21, a22 = -a * d0[0], 1 / tau + d0[1] * (a + lam)
        det = a11 * a22 - a12 * a21
        G[0].append((r1 * a22 - a12 * r2) / det)
        G[1].append((a11 * r2 - a21 * r1) / det)
        if n > 3:
            G[0][n - 3] = G[1][n - 3] = None
    return V.T @ G[0][N], V.T @ G[1][N]
