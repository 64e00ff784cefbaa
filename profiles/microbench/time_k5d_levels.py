"""K5d time per call vs levels per call (C2 shape, 65536 DOFs, 512 nodes per group): separates
the per-launch state load/store cost from the per-level cost."""
import sys

import torch

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12))
      for g in (0.7, 0.3)]
D0 = 65536
U = torch.rand((1024, D0), dtype=torch.float64, device="cuda")
D = torch.empty_like(U)
stream = torch.cuda.ExternalStream(fraq.context_stream())
h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
h.run_device(U.data_ptr(), D0, 64, D.data_ptr(), D0)
for lv in (4, 8, 16, 32, 64, 128, 256, 512):
    reps = max(2, 1024 // lv)
    fraq.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(reps):
        off = (s * lv % 512) * D0 * 8
        h.run_device(U.data_ptr() + off, D0, lv, D.data_ptr() + off, D0)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{sys.argv[1] if len(sys.argv) > 1 else '.':28s} levels {lv:4d}: {ms:.4f} ms/call "
          f"{lv * D0 / (ms * 1e-3):.3e} DOF-steps/s")
