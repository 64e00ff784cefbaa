import os, sys, time
sys.path.insert(0, ".")
os.environ["FRAQ_SETUP_TRACE"] = "1"
import numpy as np
import paper_1901_05128_b200 as fraq
from workloads import c3_instance
inst = c3_instance()
spec = fraq.ProblemSpec(alpha1=inst.alpha1, alpha2=inst.alpha2, coupling_a=inst.coupling_a,
                        grid_m=4095, t_final=1.0, n_steps=16384, initial="custom",
                        custom_g1=list(inst.g1), custom_g2=list(inst.g2))
for i in range(4):
    t = time.perf_counter()
    rr = fraq.run(spec, fraq.Scheme.FastBE, fraq.KernelConfig())
    print("run wall %.2f ms loop %.2f ms" % (1e3 * (time.perf_counter() - t), 1e3 * rr.loop_seconds), file=sys.stderr)
