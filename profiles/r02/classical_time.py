"""Classical (direct O(N^2)) BE / SBD stepper on the device at the C3 grid: loop time for a
horizon N, next to the reference's own ClassicalStepper on the host (oracle/_ref) when present."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1901_05128_b200 as fraq  # noqa: E402
from workloads import c3_instance  # noqa: E402

i = c3_instance()
for N in (2048, 16384):
    spec = fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=4095,
                            t_final=N / 16384, n_steps=N, initial="custom", custom_g1=list(i.g1),
                            custom_g2=list(i.g2))
    for sch in ("BE", "SBD"):
        rr = fraq.run(spec, getattr(fraq.Scheme, sch))
        print(f"C3 grid classical {sch} N = {N}: loop {rr.loop_seconds:.3f} s "
              f"({2 * 4095 * N / rr.loop_seconds:.3g} DOF-steps/s)", flush=True)
