"""Per-level history step at C2's kernels: K5 (every node's state per level) against K5f (K5e's
fold per level), device pointers, one launch per level:
python profiles/r02/k5f_time.py [DOFs]"""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq  # noqa: E402

D0 = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12))
      for g in (0.7, 0.3)]
gen = torch.Generator(device="cuda").manual_seed(5)
n = 512
U = torch.rand((n, D0), dtype=torch.float64, device="cuda", generator=gen)
stream = torch.cuda.ExternalStream(fraq.context_stream())
res = {}
for name in ("K5", "K5f"):
    if name == "K5":
        os.environ["FRAQ_NO_K5F"] = "1"
    else:
        os.environ.pop("FRAQ_NO_K5F", None)
    D = torch.zeros_like(U)
    h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
    h.run_device(U.data_ptr(), D0, 256, D.data_ptr(), D0)
    for i in range(256, 264):
        h.run_device(U.data_ptr() + i * D0 * 8, D0, 1, D.data_ptr() + i * D0 * 8, D0)
    fraq.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(264, n):
        h.run_device(U.data_ptr() + i * D0 * 8, D0, 1, D.data_ptr() + i * D0 * 8, D0)
    e1.record(stream)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (n - 264)
    res[name] = D
    print(f"{name}: {ms * 1e3:.2f} us per level, {D0 / (ms * 1e-3):.4e} DOF-steps/s, launches {list(h.launches)}",
          flush=True)
d = (res["K5"] - res["K5f"]).abs().max().item()
print("max |K5 - K5f| =", d, "scale", tau ** -0.7)
