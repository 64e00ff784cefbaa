"""Generates tests/golden/golden.npz from the REFERENCE (oracle/_ref: the unmodified reference
sources compiled by oracle/Makefile).  Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

Contents (all produced by the reference's own code path):
  c1_*   C1 workload sample: BE auto kernel at (0.5, 1/4096, 4096), 4 DOFs x 4096 steps of
         u_k = t^{b_k} (workloads.c1_params), reference derivatives;
  c4a/b  SBD auto sizing at the C4 exponents (0.7, 0.4), tau = 1/8192, horizon 8192;
  ffpe*  reference fraq::run final states for small poly_sin problems, all four schemes.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle  # noqa: E402
from workloads import c1_params  # noqa: E402  (pure numpy, no GPU)


def main():
    ref = Oracle("reference")
    out = {}
    p = c1_params()
    k = ref.build_kernel_auto(False, 0.5, p.tau, p.n_steps)
    U = p.signal(0, p.n_steps, np.arange(4))
    out.update(c1_np=k.np1, c1_m=k.m1, c1_U=U, c1_D=ref.hist_run(k, U))
    for name, g in (("c4a", 0.7), ("c4b", 0.4)):
        kk = ref.build_kernel_auto(True, g, 1 / 8192, 8192)
        out[name + "_cfg"] = np.array([g, 1 / 8192, 8192.0])
        out[name + "_sizes"] = np.array([kk.np1, kk.n_head])
        out[name + "_eps"] = kk.achieved_eps
    cases = [(0.3, 0.6, 2.0, 31, 0.25, 32, s) for s in ("BE", "FastBE", "SBD", "FastSBD")]
    cases += [(0.4, 0.8, -5.5, 63, 1.0, 128, "FastBE"), (0.45, 0.75, 0.0, 63, 0.2, 40, "FastSBD")]
    for i, c in enumerate(cases):
        g1, g2, _, _ = ref.run(*c[:6], c[6], "poly_sin")
        out[f"ffpe{i}_cfg"] = np.array(c[:6], dtype=float)
        out[f"ffpe{i}_scheme"] = np.array(c[6])
        out[f"ffpe{i}_g1"] = g1
        out[f"ffpe{i}_g2"] = g2
    out["ffpe_n"] = len(cases)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
