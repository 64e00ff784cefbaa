"""Loop time of the FFPE configurations on the GPU: C3 (physical vs modal), C5 subsets and
extrapolation, C4 (2D, modal)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import paper_1901_05128_b200 as fraq
from workloads import c3_instance, c5_instances

def kc(modal):
    k = fraq.KernelConfig()
    k.solver = fraq.SOLVER_MODAL if modal else fraq.SOLVER_PHYSICAL
    return k

inst = c3_instance()
for sch in ("FastBE", "FastSBD"):
    for modal in (False, True):
        spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=4095, t_final=1.0,
                                n_steps=16384, initial="custom", custom_g1=list(inst.g1), custom_g2=list(inst.g2))
        rr = fraq.run(spec, getattr(fraq.Scheme, sch), kc(modal))
        dofs = 2 * 4095 * 16384
        print(f"C3 {sch} {'modal' if modal else 'physical'}: loop {rr.loop_seconds:.4f} s -> {dofs / rr.loop_seconds:.3e} DOF-steps/s", flush=True)
for n_inst, N in ((64, 2048), (256, 2048)):
    insts = c5_instances(n_inst)
    for sch in ("FastBE", "FastSBD"):
        for modal in (False, True):
            if not modal and n_inst > 64: continue
            specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=4095,
                                      t_final=N / 16384, n_steps=N, initial="custom", custom_g1=list(i.g1),
                                      custom_g2=list(i.g2)) for i in insts]
            out = fraq.run_batch(specs, getattr(fraq.Scheme, sch), kc(modal))
            dofs = 2 * 4095 * N * n_inst
            print(f"C5 subset {n_inst} inst x {N} lv {sch} {'modal' if modal else 'physical'}: loop {out[0].loop_seconds:.3f} s -> {dofs / out[0].loop_seconds:.3e} DOF-steps/s", flush=True)
M, N = 1023, 8192
rng = np.random.default_rng(1901051284)
x = (np.arange(M) + 1) / (M + 1)
X, Y = np.meshgrid(x, x)
g1 = ((X <= 0.5) & (Y <= 0.5)).astype(float).ravel()
g2 = 1.0 + rng.uniform(-0.1, 0.1, M * M)
t0 = time.time()
out = fraq.run_2d(0.3, 0.6, -3.0, M, 1.0, N, fraq.Scheme.FastSBD, g1, g2)
print(f"C4 2D FastSBD 1023^2 N=8192: loop {out.loop_seconds:.2f} s (wall {time.time()-t0:.1f} s) -> {2*M*M*N/out.loop_seconds:.3e} DOF-steps/s; finite={np.isfinite(out.final_state.g1).all()}", flush=True)
