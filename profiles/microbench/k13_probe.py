"""One K13 launch per scheme on a C5-like batch (for ncu)."""
import sys
sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq
from workloads import c5_instances

scheme = sys.argv[1] if len(sys.argv) > 1 else "FastBE"
n_inst = int(sys.argv[2]) if len(sys.argv) > 2 else 32
N = int(sys.argv[3]) if len(sys.argv) > 3 else 512
kc = fraq.KernelConfig()
kc.solver = fraq.SOLVER_MODAL
specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=4095,
                          t_final=N / 16384, n_steps=N, initial="custom", custom_g1=list(i.g1),
                          custom_g2=list(i.g2)) for i in c5_instances(n_inst)]
out = fraq.run_batch(specs, getattr(fraq.Scheme, scheme), kc)
print(scheme, n_inst, N, out[0].loop_seconds, 2 * 4095 * N * n_inst / out[0].loop_seconds)
