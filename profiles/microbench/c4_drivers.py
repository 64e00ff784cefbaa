"""C4 phase times (M = 1023, FastSBD, argv[1] levels) through both mode-sharded drivers at
world = 1: run_2d_sharded (full DST, ky slab, all-gather) and run_2d_transposed (x pass,
all-to-all, y pass, kx slab)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq  # noqa: E402
from paper_1901_05128_b200.parallel import FraqOps, run_2d_sharded, run_2d_transposed  # noqa: E402
from workloads import c4_instance  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
M = 1023
i = c4_instance(M)
ops = FraqOps(fraq, torch)
kc = fraq.KernelConfig()
kc.solver = fraq.SOLVER_MODAL
g1, g2 = ops.tensor(i.g1), ops.tensor(i.g2)
drivers = (("sharded", run_2d_sharded), ("transposed", run_2d_transposed))
if len(sys.argv) > 2:
    drivers = [d for d in drivers if d[0] == sys.argv[2]]
import gc
for rep in range(2):
    for name, fn in drivers:
        gc.collect()
        gc.disable()  # no collection pauses inside the timed phases
        T = {}
        r1, r2 = fn(ops, i.alpha1, i.alpha2, i.coupling_a, M, N / 8192, N, "FastSBD", g1, g2,
                    kconf=kc, scheme_arg=fraq.Scheme.FastSBD, timings=T)
        gc.enable()
        print(name, {k: round(v * 1e3, 3) for k, v in T.items()}, "ms",
              float(r1.abs().sum()), float(r2.abs().sum()))
