"""Generates tests/golden/c5_sizes.npz: the REFERENCE auto-sizer's decision for every exponent of
the C5 parameter sweep (BASELINE.json configs[4]).  oracle/_ref is the unmodified reference
(fast_kernel.cpp:182-256, build_be_kernel_auto / build_sbd_kernel_auto) compiled by
oracle/Makefile.  Run in the build container, where /root/reference exists:

    python tests/golden/make_c5_sizes.py [--procs 8]

The C5 instances are workloads.c5_instances() (seed 1901051285); each has two CQ exponents
gamma = 1 - alpha_f, sized for tau = 1/16384 and horizon 16384 with the reference's defaults
(KernelConfig{}: eps_tol 1e-12, max_points 256, max_head 256; fpfp.cpp:180-238).

Contents (index i = 2 * instance + field):
  gamma[8192]               the exponents
  be_np[8192], be_eps[8192]  BE:  N_p and achieved eps
  sbd_sizes[8192, 3]         SBD: (N_p1, N_p2, n_head)
  sbd_eps[8192]              SBD achieved eps
"""
import argparse
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

TAU = 1.0 / 16384
HORIZON = 16384
_ORC = None


def _size_one(g):
    global _ORC
    if _ORC is None:
        from oracle.oracle import Oracle
        _ORC = Oracle("reference")
    kb = _ORC.build_kernel_auto(False, g, TAU, HORIZON)
    ks = _ORC.build_kernel_auto(True, g, TAU, HORIZON)
    return kb.np1, kb.achieved_eps, (ks.np1, ks.np2, ks.n_head), ks.achieved_eps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    ap.add_argument("--instances", type=int, default=4096)
    args = ap.parse_args()
    from workloads import c5_instances
    inst = c5_instances(args.instances)
    gammas = np.array([1.0 - x for i in inst for x in (i.alpha1, i.alpha2)])
    t0 = time.time()
    with Pool(args.procs) as pool:
        res = pool.map(_size_one, list(gammas), chunksize=8)
    out = dict(gamma=gammas,
               be_np=np.array([r[0] for r in res], dtype=np.int32),
               be_eps=np.array([r[1] for r in res]),
               sbd_sizes=np.array([r[2] for r in res], dtype=np.int32),
               sbd_eps=np.array([r[3] for r in res]),
               tau=TAU, horizon=HORIZON)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "c5_sizes.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes) in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
