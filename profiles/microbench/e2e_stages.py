"""C2 e2e (MultiHistory.run with pinned host arrays, 1024 levels per call as in bench.py) for the
staging depth / chunk height given by FRAQ_HOST_STAGES / FRAQ_HOST_CHUNK."""
import os, sys, time
sys.path.insert(0, ".")
import torch
import paper_1901_05128_b200 as fraq

tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12)) for g in (0.7, 0.3)]
D0, lv, K = 65536, 1024, 6
U = torch.rand((lv * K, D0), dtype=torch.float64).pin_memory()
D = torch.empty_like(U).pin_memory()
h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
for _ in range(2):
    h.run(U[:lv].numpy(), True, D[:lv].numpy())
best = 0
for rep in range(2):
    t = time.perf_counter()
    for s in range(K):
        rows = slice(s * lv, (s + 1) * lv)
        h.run(U[rows].numpy(), True, D[rows].numpy())
    el = time.perf_counter() - t
    best = max(best, K * lv * D0 / el)
print(f"stages={os.environ.get('FRAQ_HOST_STAGES', '2')} chunk={os.environ.get('FRAQ_HOST_CHUNK', 'auto')} "
      f"e2e {best:.3e} DOF-steps/s ({16 * best / 1e9:.1f} GB/s of PCIe)")
