"""e2e of the C2 host path (MultiHistory.run with pinned host arrays, 512 levels per call) and the
raw pinned H2D / D2H / concurrent bandwidth of this box."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_1901_05128_b200 as fraq

tau = 1.0 / 65536
ks = [fraq.build_sbd_kernel_auto(g, tau, fraq.KernelBudget(horizon=65536, eps_tol=1e-12)) for g in (0.7, 0.3)]
D0, lv, K = 65536, 512, 8
U = torch.rand((lv * K, D0), dtype=torch.float64).pin_memory()
D = torch.empty_like(U).pin_memory()
h = fraq.MultiHistory(ks, [D0 // 2, D0 // 2])
h.run(U[:lv].numpy(), True, D[:lv].numpy())
t = time.perf_counter()
for s in range(K):
    rows = slice(s * lv, (s + 1) * lv)
    h.run(U[rows].numpy(), True, D[rows].numpy())
el = time.perf_counter() - t
print(f"e2e {K * lv * D0 / el:.3e} DOF-steps/s, {1e3 * el / K:.2f} ms per 512-level call")
dev = torch.empty((lv, D0), dtype=torch.float64, device="cuda")
src = U[:lv]
torch.cuda.synchronize()
t = time.perf_counter(); dev.copy_(src, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t
t = time.perf_counter(); D[:lv].copy_(dev, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dev2 = torch.empty_like(dev)
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1): dev.copy_(src, non_blocking=True)
with torch.cuda.stream(s2): D[lv:2 * lv].copy_(dev2, non_blocking=True)
torch.cuda.synchronize(); both = time.perf_counter() - t
nb = lv * D0 * 8
print(f"H2D {nb / h2d / 1e9:.1f} GB/s  D2H {nb / d2h / 1e9:.1f} GB/s  concurrent {2 * nb / both / 1e9:.1f} GB/s total")
