import sys, numpy as np
sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq
from oracle.oracle import Oracle
from workloads import c3_instance
orc = Oracle("reference")
def rel(a, b):
    a, b = np.asarray(a), np.asarray(b); return np.max(np.abs(a - b)) / np.max(np.abs(b))
for M, N, T, sch, auto in [(255, 2048, 0.125, "FastBE", True), (4095, 256, 1/64, "FastBE", True),
                           (4095, 2048, 0.125, "FastBE", True), (4095, 2048, 0.125, "FastBE", False),
                           (4095, 2048, 0.125, "BE", True), (1023, 4096, 0.25, "FastBE", True),
                           (4095, 512, 0.03125, "FastBE", False)]:
    inst = c3_instance(M)
    spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=M, t_final=T,
                            n_steps=N, initial="custom", custom_g1=list(inst.g1), custom_g2=list(inst.g2))
    kc = fraq.KernelConfig(); kc.auto_size = auto; kc.be_points = 64
    rr = fraq.run(spec, getattr(fraq.Scheme, sch), kc)
    g1, g2, e1, e2 = orc.run(0.4, 0.8, -5.5, M, T, N, sch, "custom", inst.g1, inst.g2,
                             kconf=dict(auto_size=auto, be_points=64))
    print(M, N, sch, auto, "rel g1 %.3e g2 %.3e" % (rel(rr.final_state.g1, g1), rel(rr.final_state.g2, g2)),
          "eps", rr.kernel_eps1, e1, flush=True)
