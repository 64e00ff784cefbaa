"""The fold on the REFERENCE's own CPU histories (oracle/_ref, unmodified SbdHistory): C2 kernels
as built by the reference against the same kernels rewritten by fraq.fold_kernel (host only)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1901_05128_b200 as fraq  # noqa: E402
from oracle.oracle import Kernel, Oracle  # noqa: E402

orc = Oracle("reference")
tau = 1.0 / 65536
ks = [orc.build_kernel_auto(True, g, tau, 65536, 1e-12) for g in (0.7, 0.3)]
kf = []
for k in ks:
    pk = fraq.make_sbd_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1), list(k.m2),
                              list(k.r2))
    f, M = fraq.fold_kernel(pk, 96)
    kf.append(Kernel(True, k.gamma, k.tau, np.array(f.head), np.array(f.mult1), np.array(f.ratio1),
                     np.array(f.mult2), np.array(f.ratio2)))
    print("gamma", k.gamma, "nodes", k.np1 + k.np2, "->", kf[-1].np1 + kf[-1].np2, "head", k.n_head,
          "->", kf[-1].n_head)
threads = os.cpu_count() or 1
dofs, levels = 16384, 1024
rng = np.random.default_rng(3)
U = rng.uniform(-1, 1, (levels, dofs))
for name, kk in (("reference kernels", ks), ("folded kernels", kf)):
    secs, _ = orc.bench_history(kk, U, threads)
    print(f"{name}: {dofs * levels / secs:.3e} DOF-steps/s on {threads} threads ({secs:.2f} s)")
D0 = orc.hist_run(ks[0], U[:, :4])
D1 = orc.hist_run(kf[0], U[:, :4])
print("max rel diff (gamma 0.7, 4 DOFs x 1024 levels):",
      float(np.max(np.abs(D1 - D0)) / np.max(np.abs(D0))))
