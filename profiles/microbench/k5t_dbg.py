import sys
sys.path.insert(0, ".")
import numpy as np
import paper_1901_05128_b200 as fraq
spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.7, coupling_a=-1.0, grid_m=15, t_final=0.1, n_steps=12)
seen = []
if len(sys.argv) > 1:
    rr = fraq.run(spec, fraq.Scheme.FastBE, fraq.KernelConfig(), lambda n, f: seen.append((n, f.g1[3])))
    print("observer run", len(seen), rr.final_state.g1[:2])
specs = [fraq.ProblemSpec(alpha1=0.2 + 0.1 * i, alpha2=0.5, coupling_a=1.0, grid_m=15, t_final=0.1, n_steps=12) for i in range(3)]
kc = fraq.KernelConfig(); kc.solver = fraq.SOLVER_PHYSICAL
outs = fraq.run_batch(specs, fraq.Scheme.FastSBD, kc)
print("batch nan", [int(np.isnan(np.array(o.final_state.g1)).sum()) for o in outs])
for s, o in zip(specs, outs):
    single = fraq.run(s, fraq.Scheme.FastSBD, kc)
    print("single nan", int(np.isnan(np.array(single.final_state.g1)).sum()), np.nanmax(np.abs(np.array(o.final_state.g1) - np.array(single.final_state.g1))))
kc2 = fraq.KernelConfig(); kc2.solver = fraq.SOLVER_AUTO
outs = fraq.run_batch(specs, fraq.Scheme.FastSBD, kc2)
print("AUTO batch nan", [int(np.isnan(np.array(o.final_state.g1)).sum()) for o in outs])
for s in specs:
    single = fraq.run(s, fraq.Scheme.FastSBD, kc2)
    print("AUTO single nan", int(np.isnan(np.array(single.final_state.g1)).sum()))
