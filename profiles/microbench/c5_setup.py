"""C5 setup vs loop split (run_batch with 256 instances, full horizon): setup_seconds is the
device auto-sizing + K13 tables + transfers, loop_seconds the DST + K13 + inverse."""
import sys, time
sys.path.insert(0, ".")
import paper_1901_05128_b200 as fraq
from workloads import c5_instances

N = 16384
kc = fraq.KernelConfig()
kc.solver = fraq.SOLVER_MODAL
for scheme in ("FastBE", "FastSBD"):
    for rep in range(2):
        specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                                  grid_m=4095, t_final=1.0, n_steps=N, initial="custom",
                                  custom_g1=list(i.g1), custom_g2=list(i.g2))
                 for i in c5_instances(256)]
        t = time.perf_counter()
        out = fraq.run_batch(specs, getattr(fraq.Scheme, scheme), kc)
        wall = time.perf_counter() - t
        print(scheme, f"wall {wall:.3f} s  setup {out[0].setup_seconds:.3f} s  loop {out[0].loop_seconds:.3f} s")
