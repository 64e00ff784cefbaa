"""Independent check at full C3 size: FastBE in mode space (DST-diagonalised, per-mode scalar
2x2 solves, per-mode fast histories with the same auto-sized node tables) in fp64, vs the
physical-space reference and the B200 path.  Mode space avoids the ill-conditioned stencil and
block solve, so it is the more accurate fp64 evaluation of the same discrete scheme."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from oracle.oracle import Oracle
from workloads import c3_instance

M, N = 4095, int(sys.argv[1]) if len(sys.argv) > 1 else 16384
T = N / 16384
inst = c3_instance(M)
orc = Oracle("reference")
k1 = orc.build_kernel_auto(False, 0.6, 1 / 16384, N)
k2 = orc.build_kernel_auto(False, 0.2, 1 / 16384, N)
h = 1.0 / (M + 1); tau = T / N; a = -5.5
k = np.arange(1, M + 1)
V = np.sin(np.outer(k, k) * np.pi * h)
lam = 4 / h**2 * np.sin(k * np.pi * h / 2) ** 2
c = [2 / (M + 1) * (V @ inst.g1), 2 / (M + 1) * (V @ inst.g2)]
ks = [k1, k2]
y = [np.zeros((len(kk.r1), M)) for kk in ks]
G = [[c[0]], [c[1]]]
d0 = [kk.head[0] for kk in ks]; d1 = [kk.head[1] for kk in ks]
t0 = time.time()
for n in range(1, N + 1):
    s = []
    for f in range(2):
        kk = ks[f]
        feed = G[f][n - 2] if n - 2 >= 1 else None   # scheme variant: G^0 never fed
        y[f] *= kk.r1[:, None]
        if feed is not None:
            y[f] += kk.m1[:, None] * feed[None, :]
        sf = y[f].sum(axis=0)
        if n >= 2:
            sf = sf + d1[f] * G[f][n - 1]
        s.append(sf)
    r1 = G[0][n - 1] / tau - (a + lam) * s[0] + a * s[1]
    r2 = G[1][n - 1] / tau - (a + lam) * s[1] + a * s[0]
    a11, a12 = 1 / tau + d0[0] * (a + lam), -a * d0[1]
    a21, a22 = -a * d0[0], 1 / tau + d0[1] * (a + lam)
    det = a11 * a22 - a12 * a21
    G[0].append((r1 * a22 - a12 * r2) / det); G[1].append((a11 * r2 - a21 * r1) / det)
    if n > 3:
        G[0][n - 3] = None; G[1][n - 3] = None
t1, t2 = V.T @ G[0][N], V.T @ G[1][N]
print("mode-space solve %.1f s" % (time.time() - t0))
g1, g2, _, _ = orc.run(0.4, 0.8, -5.5, M, T, N, "FastBE", "custom", inst.g1, inst.g2)
ad = lambda x, y: np.max(np.abs(np.asarray(x) - y))
print("N=%d reference vs mode-space fp64: abs g1 %.3e g2 %.3e" % (N, ad(g1, t1), ad(g2, t2)))
import paper_1901_05128_b200 as fraq
spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=M, t_final=T, n_steps=N,
                        initial="custom", custom_g1=list(inst.g1), custom_g2=list(inst.g2))
rr = fraq.run(spec, fraq.Scheme.FastBE)
print("N=%d B200 vs mode-space fp64:      abs g1 %.3e g2 %.3e" % (N, ad(rr.final_state.g1, t1), ad(rr.final_state.g2, t2)))
print("N=%d B200 vs reference:             abs g1 %.3e g2 %.3e" % (N, ad(rr.final_state.g1, g1), ad(rr.final_state.g2, g2)))
