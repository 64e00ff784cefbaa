"""Small drivers for ncu captures of round 2 (run under ncu on the GPU box; never timed).

    python profiles/r02/ncu_drivers.py c3phys [levels]   # physical C3: K5 (FFPE mode) + K6 per level
    python profiles/r02/ncu_drivers.py c4dst             # one C4-shaped DST pass (K12, DMMA GEMM)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1901_05128_b200 as fraq  # noqa: E402
from workloads import c3_instance  # noqa: E402


def c3phys(levels=64):
    i = c3_instance()
    spec = fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                            grid_m=4095, t_final=levels / 16384, n_steps=levels,
                            initial="custom", custom_g1=list(i.g1), custom_g2=list(i.g2))
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_PHYSICAL
    r = fraq.run(spec, fraq.Scheme.FastBE, kc)
    print("c3phys", levels, r.loop_seconds)


def c4dst():
    import torch
    M = 1023
    x = torch.randn(M, 2 * M, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    torch.cuda.synchronize()
    for _ in range(3):
        fraq.dst_cols_device(M, 2 * M, x.data_ptr(), y.data_ptr(), False)
    fraq.synchronize()
    print("c4dst ok", float(y.abs().max()))


if __name__ == "__main__":
    what = sys.argv[1]
    if what == "c3phys":
        c3phys(int(sys.argv[2]) if len(sys.argv) > 2 else 64)
    elif what == "c4dst":
        c4dst()


def c3modal():
    from workloads import c3_instance as _c3
    i = _c3()
    spec = fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                            grid_m=4095, t_final=1.0, n_steps=16384, initial="custom",
                            custom_g1=list(i.g1), custom_g2=list(i.g2))
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_MODAL
    for _ in range(2):
        r = fraq.run(spec, fraq.Scheme.FastBE, kc)
    print("c3modal", r.loop_seconds)


if __name__ == "__main__" and sys.argv[1] == "c3modal":
    c3modal()


def k6split(levels=1024):
    """Per-level K5 / K6 device time of the physical C3 stepper (events around every launch)."""
    from workloads import c3_instance as _c3
    i = _c3()
    spec = fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                            grid_m=4095, t_final=1.0, n_steps=16384, initial="custom",
                            custom_g1=list(i.g1), custom_g2=list(i.g2))
    st = fraq.FastStepper(spec, False, fraq.KernelConfig())
    st.step_n(1024)
    a, b = st.time_split(levels)
    import time
    fraq.synchronize()
    t0 = time.perf_counter()
    st.step_n(levels)
    fraq.synchronize()
    dt = time.perf_counter() - t0
    print(f"k5 {1e3 * a / levels:.2f} us  k6 {1e3 * b / levels:.2f} us  loop {1e6 * dt / levels:.2f} us"
          " per level")


if __name__ == "__main__" and sys.argv[1] == "k6split":
    k6split()


def c5batch(scheme="FastSBD", n_inst=37, N=4096):
    """A C5-shaped K13 launch (instances of workloads.c5_instances, M = 4095)."""
    from workloads import c5_instances as _c5
    insts = _c5(n_inst)
    specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                              grid_m=4095, t_final=N / 16384, n_steps=N, initial="custom",
                              custom_g1=list(i.g1), custom_g2=list(i.g2)) for i in insts]
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_MODAL
    rs = fraq.run_batch(specs, getattr(fraq.Scheme, scheme), kc)
    print("c5batch", scheme, rs[0].loop_seconds)


if __name__ == "__main__" and sys.argv[1] == "c5batch":
    c5batch(sys.argv[2] if len(sys.argv) > 2 else "FastSBD")
