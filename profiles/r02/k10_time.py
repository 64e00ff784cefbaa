"""K10 (direct CQ as a lower-triangular Toeplitz GEMM on DMMA): device time and DMMA rate."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1901_05128_b200 as fraq  # noqa: E402

N, D = 16384, 8192
U = torch.randn(N, D, dtype=torch.float64, device="cuda")
O = torch.empty_like(U)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(fraq.context_stream())
fraq.direct_cq_device(True, 0.4, 1.0 / N, U.data_ptr(), D, N, D, O.data_ptr(), D)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(3):
    fraq.direct_cq_device(True, 0.4, 1.0 / N, U.data_ptr(), D, N, D, O.data_ptr(), D)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1) / 3
fl = (N * (N + 1) / 2) * D * 2  # algorithmic (lower triangle)
print(f"K10 N = {N}, {D} lanes: {ms:.1f} ms, {fl / (ms * 1e-3) / 1e12:.2f} TF/s algorithmic "
      f"(DMMA peak {fraq.diag_dmma_peak()[0]:.1f})")
