"""Ground truth for the 1D FFPE at large M: the reference's own mode-space oracle
(test_fpfp.cpp:21-180) evaluated in float128 (np.longdouble) for the classical BE scheme."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle.oracle import Oracle
from workloads import c3_instance

def modespace_be(M, N, T, a, al1, al2, g1, g2, dt=np.longdouble):
    h = dt(1) / (M + 1); tau = dt(T) / N
    k = np.arange(1, M + 1, dtype=dt); j = np.arange(1, M + 1, dtype=dt)
    pi = dt(np.pi) if dt is np.float64 else np.arccos(dt(-1))
    V = np.sin(np.outer(k, j) * pi * h)
    lam = 4 / h**2 * np.sin(k * pi * h / 2) ** 2
    c1 = 2 / dt(M + 1) * (V @ g1.astype(dt)); c2 = 2 / dt(M + 1) * (V @ g2.astype(dt))
    def bew(g):
        w = np.empty(N + 1, dtype=dt); w[0] = 1
        for i in range(1, N + 1): w[i] = w[i-1] * ((i - 1 - dt(g)) / i)
        return w * tau ** (-dt(g))
    d1, d2 = bew(1 - al1), bew(1 - al2)
    U = np.zeros((N + 1, M), dtype=dt); W = np.zeros((N + 1, M), dtype=dt)
    U[0], W[0] = c1, c2
    a = dt(a)
    for n in range(1, N + 1):
        s1 = np.tensordot(d1[1:n], U[n-1:0:-1], axes=1) if n > 1 else np.zeros(M, dt)
        s2 = np.tensordot(d2[1:n], W[n-1:0:-1], axes=1) if n > 1 else np.zeros(M, dt)
        r1 = U[n-1] / tau - (a + lam) * s1 + a * s2
        r2 = W[n-1] / tau - (a + lam) * s2 + a * s1
        a11 = 1 / tau + d1[0] * (a + lam); a12 = -a * d2[0]; a21 = -a * d1[0]; a22 = 1 / tau + d2[0] * (a + lam)
        det = a11 * a22 - a12 * a21
        U[n] = (r1 * a22 - a12 * r2) / det; W[n] = (a11 * r2 - a21 * r1) / det
    return (V.T @ U[N]), (V.T @ W[N])

M, N, T = 4095, int(sys.argv[1]) if len(sys.argv) > 1 else 128, None
T = N / 16384
inst = c3_instance(M)
t1, t2 = modespace_be(M, N, T, -5.5, 0.4, 0.8, inst.g1, inst.g2)
t1 = t1.astype(np.float64); t2 = t2.astype(np.float64)
port = Oracle("port")
p1, p2, _, _ = port.run(0.4, 0.8, -5.5, M, T, N, "BE", "custom", inst.g1, inst.g2)
rel = lambda a, b: np.max(np.abs(a - b)) / np.max(np.abs(b))
print("port(=reference) vs float128 mode-space: g1 %.3e g2 %.3e" % (rel(p1, t1), rel(p2, t2)))
try:
    import paper_1901_05128_b200 as fraq
    spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=M, t_final=T, n_steps=N,
                            initial="custom", custom_g1=list(inst.g1), custom_g2=list(inst.g2))
    rr = fraq.run(spec, fraq.Scheme.BE)
    print("GPU vs float128 mode-space:             g1 %.3e g2 %.3e" % (rel(rr.final_state.g1, t1), rel(rr.final_state.g2, t2)))
    print("GPU vs port:                            g1 %.3e g2 %.3e" % (rel(rr.final_state.g1, p1), rel(rr.final_state.g2, p2)))
except Exception as e:
    print("no GPU:", e)
