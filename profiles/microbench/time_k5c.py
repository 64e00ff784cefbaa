"""Times the temporally blocked history kernel on the C2 workload shape (65536 DOFs, SBD
256+256 nodes, 512 levels per call) for the package found first on sys.path."""
import sys
import time

import torch

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

tau = 1.0 / 65536
ks = []
for g in (0.7, 0.3):
    b = fraq.KernelBudget(horizon=65536, eps_tol=1e-12)
    ks.append(fraq.build_sbd_kernel_auto(g, tau, b))
D0 = 65536
lv = 512
U = torch.rand((lv * 4, D0), dtype=torch.float64, device="cuda")
D = torch.empty_like(U)
h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
stream = torch.cuda.ExternalStream(fraq.context_stream())
h.run_device(U.data_ptr(), D0, lv, D.data_ptr(), D0)
fraq.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for s in range(4):
    off = s * lv * D0 * 8
    h.run_device(U.data_ptr() + off, D0, lv, D.data_ptr() + off, D0)
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1)
print(f"{sys.argv[1] if len(sys.argv) > 1 else '.':45s} {4 * lv * D0 / (ms * 1e-3):.3e} DOF-steps/s "
      f"{ms / 4:.3f} ms/call path={h.last_path}")
