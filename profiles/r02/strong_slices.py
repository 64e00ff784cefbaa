"""Strong-scaling slices of C2 timed on ONE GPU (no multi-GPU box in this pool): the device time
of rank r's share of the 65536-DOF job at world size G (parallel.c2_strong_slice), K5d over 1024
levels, for G = 1, 2, 4, 8.  The path has no data-path collective, so the job time at G GPUs is
the slowest rank's slice time; this prints that prediction next to the measured G = 1 rate.
(Independent per-rank work timed one rank at a time -- not ranks waiting on each other.)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1901_05128_b200 as fraq  # noqa: E402
from paper_1901_05128_b200.parallel import c2_strong_slice  # noqa: E402
from workloads import c2_params  # noqa: E402

DOFS, LV = 65536, 1024
p = c2_params(DOFS)
ks = []
for g in (0.7, 0.3):
    b = fraq.KernelBudget(horizon=65536, eps_tol=1e-12)
    ks.append(fraq.build_sbd_kernel_auto(g, p.tau, b))
dev = torch.device("cuda", 0)
stream = torch.cuda.ExternalStream(fraq.context_stream())
out = {}
for G in (1, 2, 4, 8):
    worst = 0.0
    for r in sorted({0, G // 2, G - 1}):
        lo, hi, groups = c2_strong_slice(r, G, DOFS)
        n = hi - lo
        sel = slice(lo, hi)
        a, bb, c, w = (torch.from_numpy(x[sel].copy()).to(dev) for x in (p.a, p.b, p.c, p.w))
        t = (torch.arange(0, LV, device=dev, dtype=torch.float64) * p.tau)[:, None]
        U = (a * torch.pow(t, bb) + c * torch.sin(w * t)).contiguous()
        D = torch.empty_like(U)
        torch.cuda.synchronize()
        h = fraq.MultiHistory([ks[g] for g, _ in groups], [cnt for _, cnt in groups])
        for _ in range(3):
            h.run_device(U.data_ptr(), n, LV, D.data_ptr(), n)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(stream)
        for _ in range(reps):
            h.run_device(U.data_ptr(), n, LV, D.data_ptr(), n)
        e1.record(stream)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        worst = max(worst, ms)
    rate = DOFS * LV / (worst * 1e-3)
    out[G] = {"slice_dofs": DOFS // G, "max_rank_ms_per_1024_levels": worst,
              "predicted_job_rate": rate}
base = out[1]["predicted_job_rate"]
for G, v in out.items():
    v["predicted_efficiency"] = v["predicted_job_rate"] / (G * base)
print(json.dumps(out, indent=1))
