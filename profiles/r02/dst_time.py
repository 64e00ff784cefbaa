"""Device time of one C4-shaped DST pass (K12: 1023 x 1023 sine matrix times 1023 x 2046) and
its DMMA rate."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1901_05128_b200 as fraq  # noqa: E402

M, C = 1023, 2046
x = torch.randn(M, C, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
torch.cuda.synchronize()
st = torch.cuda.ExternalStream(fraq.context_stream())
for _ in range(3):
    fraq.dst_cols_device(M, C, x.data_ptr(), y.data_ptr(), False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(20):
    fraq.dst_cols_device(M, C, x.data_ptr(), y.data_ptr(), False)
e1.record(st)
e1.synchronize()
ms = e0.elapsed_time(e1) / 20
print(f"C4 DST pass: {ms * 1e3:.1f} us, {2 * M * M * C / (ms * 1e-3) / 1e12:.2f} TF/s "
      f"(DMMA peak {fraq.diag_dmma_peak()[0]:.1f})")
# correctness vs float64 torch matmul with the sine matrix
k = torch.arange(1, M + 1, dtype=torch.float64, device="cuda")
S = torch.sin(torch.outer(k, k) * torch.pi / (M + 1))
ref = (2.0 / (M + 1)) * S @ x
print("max rel err", float((y - ref).abs().max() / ref.abs().max()))
