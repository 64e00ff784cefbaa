"""Small K5d stress runs (repeat under a timeout to catch intermittent hangs): two groups of 20 and 28
DOFs on 512-node SBD kernels and a BE pair, TMA and register-staged inputs, split calls."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

rng = np.random.default_rng(3)
tau = 1e-3
for sbd in (True, False):
    if sbd:
        ks = [fraq.build_sbd_kernel(0.7, tau, 256, 256, 17), fraq.build_sbd_kernel(0.3, tau, 250, 256, 15)]
    else:
        ks = [fraq.build_be_kernel(0.7, tau, 512), fraq.build_be_kernel(0.3, tau, 480)]
    U = rng.uniform(-1, 1, (140, 48))
    outs = []
    for no_tma in ("", "1"):
        os.environ["FRAQ_NO_TMA"] = no_tma
        h = fraq.MultiHistory(ks, [20, 28])
        outs.append(np.concatenate([h.run(U[:70]), h.run(U[70:107]), h.run(U[107:])]))
        assert h.last_path == 3
    assert np.array_equal(outs[0], outs[1], equal_nan=True)
print("stress run ok")
