import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_1901_05128_b200 as fraq
from workloads import c5_instances
insts = c5_instances(256)
t0 = time.perf_counter()
specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=4095,
                          t_final=1.0, n_steps=16384, initial="custom", custom_g1=list(i.g1),
                          custom_g2=list(i.g2)) for i in insts]
t1 = time.perf_counter()
kc = fraq.KernelConfig(); kc.solver = fraq.SOLVER_MODAL
for rep in range(2):
    t2 = time.perf_counter()
    rs = fraq.run_batch(specs, fraq.Scheme.FastBE, kc)
    t3 = time.perf_counter()
    print(f"specs {t1-t0:.3f} s  run_batch wall {t3-t2:.3f} s  loop {rs[0].loop_seconds:.3f} s  setup {rs[0].setup_seconds:.3f} s")
