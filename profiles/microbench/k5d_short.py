"""One K5d launch shape per invocation (C2 DOFs, 512 nodes per group): argv[1] levels per call."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

lv = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12))
      for g in (0.7, 0.3)]
D0 = 65536
U = torch.rand((512, D0), dtype=torch.float64, device="cuda")
D = torch.empty_like(U)
h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
for s in range(8):
    h.run_device(U.data_ptr() + (s * lv % 256) * D0 * 8, D0, lv, D.data_ptr(), D0)
fraq.synchronize()
print("ok", lv)
