"""Reproduce uninitialised device reads: fill freed device memory with NaN, then run the batch."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
x = torch.full((256 * 1024 * 1024,), float("nan"), dtype=torch.float64, device="cuda")
torch.cuda.synchronize(); del x; torch.cuda.empty_cache()
import paper_1901_05128_b200 as fraq
specs = [fraq.ProblemSpec(alpha1=0.2 + 0.1 * i, alpha2=0.5, coupling_a=1.0, grid_m=15, t_final=0.1, n_steps=12) for i in range(3)]
for solver in ("SOLVER_PHYSICAL", "SOLVER_MODAL"):
    kc = fraq.KernelConfig(); kc.solver = getattr(fraq, solver)
    outs = fraq.run_batch(specs, fraq.Scheme.FastSBD, kc)
    print(solver, "batch nan", [int(np.isnan(np.array(o.final_state.g1)).sum()) for o in outs], flush=True)
