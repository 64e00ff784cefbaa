"""Loop time of the 1D FFPE configurations on the GPU (C3 full; C5 subsets)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1901_05128_b200 as fraq
from paper_1901_05128_b200.workloads import c3_instance, c5_instances

inst = c3_instance()
for sch in ("FastBE", "FastSBD"):
    spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=4095, t_final=1.0,
                            n_steps=16384, initial="custom", custom_g1=list(inst.g1), custom_g2=list(inst.g2))
    rr = fraq.run(spec, getattr(fraq.Scheme, sch))
    dofs = 2 * 4095 * 16384
    print(f"C3 {sch}: loop {rr.loop_seconds:.3f} s setup {rr.setup_seconds:.3f} s -> {dofs / rr.loop_seconds:.3e} DOF-steps/s")
for n_inst in (16, 64):
    insts = c5_instances(n_inst)
    for sch in ("FastBE",):
        N = 1024
        specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=4095,
                                  t_final=N / 16384, n_steps=N, initial="custom", custom_g1=list(i.g1),
                                  custom_g2=list(i.g2)) for i in insts]
        out = fraq.run_batch(specs, getattr(fraq.Scheme, sch))
        dofs = 2 * 4095 * N * n_inst
        print(f"C5 subset {n_inst} inst x {N} levels {sch}: loop {out[0].loop_seconds:.3f} s -> {dofs / out[0].loop_seconds:.3e} DOF-steps/s")
