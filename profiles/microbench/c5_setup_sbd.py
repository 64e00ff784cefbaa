"""One C5 BDF2 run_batch (64 instances, full horizon) for an ncu launch list of the setup."""
import sys
sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq
from workloads import c5_instances
kc = fraq.KernelConfig()
kc.solver = fraq.SOLVER_MODAL
specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=4095,
                          t_final=1.0, n_steps=16384, initial="custom", custom_g1=list(i.g1),
                          custom_g2=list(i.g2)) for i in c5_instances(64)]
out = fraq.run_batch(specs, fraq.Scheme.FastSBD, kc)
print("setup", out[0].setup_seconds, "loop", out[0].loop_seconds)
