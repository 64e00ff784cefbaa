"""Times K5d (C2 shape: 65536 DOFs, SBD 256+256 nodes per group, 512 levels per call) for the
package at argv[1] and prints a checksum of the derivatives so variants can be compared."""
import sys

import torch

sys.path.insert(0, sys.argv[1] if len(sys.argv) > 1 else ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12))
      for g in (0.7, 0.3)]
D0, lv, reps = 65536, 512, 8
gen = torch.Generator(device="cuda").manual_seed(5)
U = torch.rand((lv * reps, D0), dtype=torch.float64, device="cuda", generator=gen)
D = torch.empty_like(U)
stream = torch.cuda.ExternalStream(fraq.context_stream())
best = None
for trial in range(3):
    h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
    h.run_device(U.data_ptr(), D0, lv, D.data_ptr(), D0)  # warm-up call (levels 0..511)
    fraq.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for s in range(1, reps):
        off = s * lv * D0 * 8
        h.run_device(U.data_ptr() + off, D0, lv, D.data_ptr() + off, D0)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (reps - 1)
    best = ms if best is None else min(best, ms)
chk = torch.nan_to_num(D, nan=0.0)
print(f"{sys.argv[1] if len(sys.argv) > 1 else '.':28s} {lv * D0 / (best * 1e-3):.4e} DOF-steps/s "
      f"{best:.4f} ms/call sum={chk.sum().item():.15e} abs={chk.abs().sum().item():.15e}")
