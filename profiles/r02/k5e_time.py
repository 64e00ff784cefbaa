"""Times the blocked history run at C2's kernels (K5e unless FRAQ_NO_K5E is set):
python profiles/r02/k5e_time.py [DOFs] [levels per call] [calls]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

D0 = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
lv = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12))
      for g in (0.7, 0.3)]
gen = torch.Generator(device="cuda").manual_seed(5)
U = torch.rand((lv * reps, D0), dtype=torch.float64, device="cuda", generator=gen)
D = torch.empty_like(U)
stream = torch.cuda.ExternalStream(fraq.context_stream())
h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
print("first call", flush=True)
h.run_device(U.data_ptr(), D0, lv, D.data_ptr(), D0)
fraq.synchronize()
print("first call done, path", h.last_path, flush=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for s in range(1, reps):
    off = s * lv * D0 * 8
    h.run_device(U.data_ptr() + off, D0, lv, D.data_ptr() + off, D0)
e1.record(stream)
e1.synchronize()
ms = e0.elapsed_time(e1) / (reps - 1)
chk = torch.nan_to_num(D, nan=0.0)
print(f"DOFs {D0} levels/call {lv}: {lv * D0 / (ms * 1e-3):.4e} DOF-steps/s {ms:.4f} ms/call path {h.last_path} "
      f"sum={chk.sum().item():.15e} abs={chk.abs().sum().item():.15e}", flush=True)
