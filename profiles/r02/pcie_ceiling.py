"""Concurrent pinned H2D + D2H ceiling of this box (two streams, 537 MB each way, the sizes of one
C2 bench step), next to the C2 e2e line's implied rate."""
import torch
n = 536870912 // 8
hin = torch.empty(n, dtype=torch.float64).pin_memory()
hout = torch.empty(n, dtype=torch.float64).pin_memory()
din = torch.empty(n, dtype=torch.float64, device="cuda")
dout = torch.ones(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both(reps, chunk=None):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0); s2.wait_event(e0)
    for _ in range(reps):
        if chunk is None:
            with torch.cuda.stream(s1):
                din.copy_(hin, non_blocking=True)
            with torch.cuda.stream(s2):
                hout.copy_(dout, non_blocking=True)
        else:
            for o in range(0, n, chunk):
                with torch.cuda.stream(s1):
                    din[o:o + chunk].copy_(hin[o:o + chunk], non_blocking=True)
                with torch.cuda.stream(s2):
                    hout[o:o + chunk].copy_(dout[o:o + chunk], non_blocking=True)
    ev1 = torch.cuda.Event(); ev2 = torch.cuda.Event()
    ev1.record(s1); ev2.record(s2)
    torch.cuda.current_stream().wait_event(ev1); torch.cuda.current_stream().wait_event(ev2)
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
def one(direction, reps):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        if direction == "h2d":
            din.copy_(hin, non_blocking=True)
        else:
            hout.copy_(dout, non_blocking=True)
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps
both(2)
for d in ("h2d", "d2h"):
    ms = one(d, 5)
    print(f"{d} alone: {ms:.2f} ms per 537 MB = {0.536870912 / ms * 1e3:.1f} GB/s")
ms = both(5)
print(f"both ways, whole buffers: {ms:.2f} ms per 537 MB each way = {2 * 0.536870912 / ms * 1e3:.1f} GB/s aggregate"
      f" -> e2e ceiling {65536 * 1024 / (ms * 1e-3):.3e} DOF-steps/s")
ms = both(5, chunk=64 * 65536)
print(f"both ways, 32 MB chunks: {ms:.2f} ms = {2 * 0.536870912 / ms * 1e3:.1f} GB/s aggregate"
      f" -> e2e ceiling {65536 * 1024 / (ms * 1e-3):.3e} DOF-steps/s")
