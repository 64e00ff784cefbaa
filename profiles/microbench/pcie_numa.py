"""Concurrent H2D + D2H bandwidth of pinned buffers (the e2e path's bound) with the process bound
to each NUMA node's CPUs in turn (first-touch places the pinned pages on that node)."""
import os, subprocess, sys, time
import torch

def nodes():
    out = {}
    base = "/sys/devices/system/node"
    for d in sorted(os.listdir(base)):
        if d.startswith("node") and d[4:].isdigit():
            cl = open(f"{base}/{d}/cpulist").read().strip()
            cpus = set()
            for part in cl.split(","):
                if "-" in part:
                    a, b = part.split("-"); cpus |= set(range(int(a), int(b) + 1))
                elif part:
                    cpus.add(int(part))
            out[int(d[4:])] = cpus
    return out

def bw(nbytes=256 << 20, reps=8):
    h_in = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
    h_out = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
    h_in.fill_(1.0); h_out.fill_(0.0)
    d_in = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    d_out = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return 2 * nbytes * reps / dt / 1e9

print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("nvml numa node:", getattr(pynvml, "nvmlDeviceGetNumaNodeId", lambda x: None)(h))
    print("nvml cpu affinity words:", pynvml.nvmlDeviceGetCpuAffinity(h, 4))
except Exception as e:
    print("nvml:", e)
ns = nodes()
print("numa nodes:", {k: (min(v), max(v), len(v)) for k, v in ns.items() if v})
print("default affinity:", len(os.sched_getaffinity(0)), "cpus; concurrent GB/s", round(bw(), 1))
for k, cpus in ns.items():
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    print(f"node {k}: concurrent GB/s", round(bw(), 1))
