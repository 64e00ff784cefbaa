"""FFPE workloads of bench.py (--workload C3 | C4 | C5 | C5-SBD): the fast FFPE steppers of
BASELINE.json configs[2..4] through the reference-facing API (fraq.run / run_batch / run_2d,
mode-space solver: DST on DMMA + K13 DMMA block stepping).

One bench step = one complete solve of the workload unit over its full horizon:
  C3      one 1D instance, M = 4095, N = 16384, FastBE                       (2 x 4095 DOFs)
  C4      one 2D instance, 1023^2, N = 8192, FastSBD                          (2 x 1023^2 DOFs)
  C5      CHUNK (256) 1D instances per GPU, M = 4095, N = 16384, FastBE        (weak scaling)
  C5-SBD  the same with FastSBD
`value` = DOF-steps / (sum of device-timed loop seconds over the K steps; CUDA events around DST +
stepping + inverse DST, inputs resident), max over ranks.  `e2e` = the same DOF-steps over the
wall time of the API calls themselves (host arrays in, host arrays out, kernel setup included).
The reference CPU path (oracle/_ref: unmodified fraq::run, or -- C4, which the reference cannot
run -- the mode-space restatement over the reference's SbdHistory lanes) is timed on a bounded
sample on the host cores."""
from __future__ import annotations

import concurrent.futures as cf
import json
import os
import time

import numpy as np

UNIT = "DOF-steps/s"
CHUNK = 256


def _modal_kc(fraq, solver="modal"):
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_PHYSICAL if solver == "physical" else fraq.SOLVER_MODAL
    return kc


class Workload:
    def __init__(self, name, rank, world, solver="modal"):
        from workloads import c3_instance, c4_instance, c5_instances
        self.name = name
        self.rank = rank
        if name == "C3":
            self.M, self.N, self.scheme, self.units = 4095, 16384, "FastBE", 1
            self.insts = [c3_instance()]
        elif name == "C4":
            self.M, self.N, self.scheme, self.units = 1023, 8192, "FastSBD", 1
            self.insts = [c4_instance()]
        else:
            self.M, self.N = 4095, 16384
            self.scheme = "FastSBD" if name == "C5-SBD" else "FastBE"
            self.units = CHUNK
            self.all = c5_instances(4096)
        self.world = world
        self.solver = solver
        if solver == "physical" and name == "C4":
            raise ValueError("C4 (2D) has no physical-space solver; the reference is 1D only")

    def dofs(self):
        """DOFs advanced per step by THIS rank's call (C4: the whole job, strong scaling)."""
        return 2 * (self.M * self.M if self.name == "C4" else self.M) * self.units

    def specs(self, fraq, step):
        if self.name == "C4":
            return None
        if self.name == "C3":
            insts = self.insts
        else:  # rank-sharded chunks of the 4096 C5 instances (wrapping)
            base = ((step * self.world + self.rank) * CHUNK) % 4096
            insts = [self.all[(base + i) % 4096] for i in range(CHUNK)]
        return [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                                 grid_m=self.M, t_final=1.0, n_steps=self.N, initial="custom",
                                 custom_g1=list(i.g1), custom_g2=list(i.g2)) for i in insts]

    def solve(self, fraq, specs, torch=None, device_inputs=True):
        """One step through the public API; returns (device loop seconds, results).  C4 runs the
        mode-sharded driver (parallel.run_2d_transposed) at every world size: x pass of the DST on
        the rank's rows, NCCL all-to-all transpose, y pass, K13 on the rank's kx slab of modes,
        and the mirror image for the inverse (device phase times, setup excluded)."""
        sch = getattr(fraq.Scheme, self.scheme)
        if self.name == "C4":
            from paper_1901_05128_b200.parallel import FraqOps, run_2d_transposed
            i = self.insts[0]
            ops = getattr(self, "_ops", None) or FraqOps(fraq, torch)
            self._ops = ops
            if device_inputs:
                if getattr(self, "_g_dev", None) is None:
                    self._g_dev = (ops.tensor(i.g1), ops.tensor(i.g2))
                g1, g2 = self._g_dev
            else:
                g1, g2 = i.g1, i.g2
            T = {}
            r1, r2 = run_2d_transposed(ops, i.alpha1, i.alpha2, i.coupling_a, self.M, 1.0,
                                       self.N, self.scheme, g1, g2, kconf=_modal_kc(fraq),
                                       scheme_arg=sch, timings=T)

            class R:  # RunResult-like
                pass
            r = R()
            fs = R()
            fs.g1 = r1.cpu().numpy()
            fs.g2 = r2.cpu().numpy()
            r.final_state = fs
            return sum(T.values()), [r]
        if self.name == "C3":
            r = fraq.run(specs[0], sch, _modal_kc(fraq, self.solver))
            return r.loop_seconds, [r]
        rs = fraq.run_batch(specs, sch, _modal_kc(fraq, self.solver))
        return rs[0].loop_seconds, rs

    def config(self):
        """The workload description both arms print (identical dicts)."""
        desc = {"C3": "C3: 1D two-state FFPE, M = 4095, N = 16384, FastBE (m = 0.45, alpha = 0.4/0.8)",
                "C4": "C4: 2D two-state FFPE, 1023^2, N = 8192, FastSBD (m = 0.4, alpha = 0.3/0.6)",
                "C5": "C5 (BE): 1D FFPE sweep, 256 instances per GPU per step, M = 4095, N = 16384",
                "C5-SBD": "C5 (BDF2): 1D FFPE sweep, 256 instances per GPU per step, M = 4095, "
                          "N = 16384"}[self.name]
        w = self.world
        if self.solver == "physical":
            desc += "; physical-space solver (K5 history + K6 RHS / block solve per level)"
        return {"workload": desc, "dofs_per_gpu_per_step": self.dofs(), "levels": self.N,
                "l2": "L2 flushed (256 MB write) before every step",
                "parallelism": (f"instance-sharded x{w}" if self.units > 1 else
                                f"row / kx-mode slabs x{w} + two NCCL all-to-all transposes" if
                                self.name == "C4" else f"replicas x{w}")}

    def scaling(self):
        return "strong" if self.name == "C4" else "weak"

    def launches(self):
        """Our kernels inside the device-timed region of one step.  1D modal: DST (DMMA),
        transpose, K13, transpose, inverse DST.  1D physical: K5 + K6 per level (the first BDF2
        level has no K5).  C4: two DST passes (sine table + DMMA GEMM each), K13, and two inverse
        passes (K13's tables are built at setup, outside the loop timer; the slab permutes around
        the all-to-alls are torch copies)."""
        if self.solver == "physical":
            return 2 * self.N - (1 if self.scheme == "FastSBD" else 0)
        return 9 if self.name == "C4" else 5

    def io_bytes(self):
        return 8 * self.dofs()


# ----------------------------------------------------------------------------- CPU sample
def cpu_sample(wl: Workload, orc, threads, target_s):
    """The reference's CPU path on a bounded sample of the workload; returns (rate, sample)."""
    sbd = wl.scheme == "FastSBD"
    tau = 1.0 / wl.N
    if wl.name == "C4":
        i = wl.insts[0]
        k1 = orc.build_kernel_auto(True, 1 - i.alpha1, tau, wl.N)
        k2 = orc.build_kernel_auto(True, 1 - i.alpha2, tau, wl.N)
        M = wl.M
        h = 1.0 / (M + 1)
        lam1 = 4.0 / h ** 2 * np.sin(np.arange(1, M + 1) * np.pi * h / 2) ** 2
        rng = np.random.default_rng(0)
        ky, kx = rng.integers(0, M, 2), rng.integers(0, M, 2)

        def go(nm, levels):
            sel = rng.integers(0, M, (nm, 2))
            lam = lam1[sel[:, 0]] + lam1[sel[:, 1]]
            c = rng.standard_normal((2, nm))
            _, _, secs = orc.modal_run(k1, k2, i.coupling_a, tau, levels, lam, c[0], c[1],
                                       threads=threads)
            return 2 * nm * levels / secs
        nm = 64 * threads
        rate = go(nm, 256)
        levels = int(min(wl.N, max(256, target_s * rate / (2 * nm))))
        rate = go(nm, levels)
        return rate, (f"{nm} sampled (ky,kx) modes x {levels} levels, mode-space restatement over "
                      f"the reference SbdHistory lanes ({threads} threads; the reference has no "
                      f"2D stepper, SURVEY.md §8(c))")
    # 1D: unmodified fraq::run per instance (FastBE/FastSBD), kernels sized as at the full
    # horizon; a bounded number of levels; instances in parallel over the host threads
    insts = wl.insts if wl.name == "C3" else wl.all[:max(threads, 1)]
    kcs = []
    for i in insts:
        ks = [orc.build_kernel_auto(sbd, 1 - al, tau, wl.N) for al in (i.alpha1, i.alpha2)]
        if sbd:
            kcs.append(dict(auto_size=False, sbd_points_1=max(k.np1 for k in ks),
                            sbd_points_2=max(k.np2 for k in ks), sbd_head=max(k.n_head for k in ks)))
        else:
            kcs.append(dict(auto_size=False, be_points=max(k.np1 for k in ks)))

    def one(ii, levels):
        from oracle.oracle import Oracle
        o = Oracle("reference")
        i = insts[ii]
        o.run(i.alpha1, i.alpha2, i.coupling_a, wl.M, levels * tau, levels, wl.scheme, "custom",
              custom_g1=i.g1, custom_g2=i.g2, kconf=kcs[ii])
        return o.last_loop_seconds

    def batch(levels):
        n = len(insts)
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(max_workers=min(threads, n)) as ex:
            loops = list(ex.map(lambda ii: one(ii, levels), range(n)))
        wall = time.perf_counter() - t0
        return 2 * wl.M * levels * n / max(loops) if n == 1 else 2 * wl.M * levels * n / wall
    rate = batch(64)
    per_inst = rate / len(insts)
    levels = int(min(wl.N, max(128, target_s * per_inst / (2 * wl.M))))
    rate = batch(levels)
    cores = min(threads, len(insts))
    return rate, (f"{len(insts)} instance(s) x {levels} levels, unmodified fraq::run {wl.scheme} "
                  f"(kernels sized for the full horizon N = {wl.N}), {cores} thread(s)"), cores


def run_reference(args, rank, world, METRIC):
    if rank != 0:
        return
    from oracle.oracle import Oracle, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    wl = Workload(args.workload, 0, world, args.solver)
    orc = Oracle("reference")
    threads = os.cpu_count() or 1
    vals = []
    res = None
    for s in range(args.warmup + args.steps):
        res = cpu_sample(wl, orc, threads, 1.0 if s < args.warmup else 4.0)
        if s >= args.warmup:
            vals.append(res[0])
    value = float(np.median(vals))
    cores = res[2] if len(res) > 2 else threads
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None,
        "higher_is_better": True, "scaling": wl.scaling(), "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": wl.config(),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": res[1]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
        flush=True)


def run_gpu(args, rank, world, local, pg, METRIC, Clocks, fraq, torch):
    wl = Workload(args.workload, rank, world, args.solver)
    dev = torch.device("cuda", local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > L2
    K, W = args.steps, args.warmup
    for s in range(W):
        wl.solve(fraq, wl.specs(fraq, s), torch)
    specs = [wl.specs(fraq, s) for s in range(K)]
    loops, walls = [], []
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    import gc
    with Clocks(local) as clk:
        for s in range(K):
            # no Python garbage collection inside a step: a full collection stalls the host
            # thread that issues the next phase's launches, and C4's device phase times
            # (events around host-issued phases) then include 20-150 ms of idle GPU
            gc.collect()
            gc.disable()
            flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            loop, rs = wl.solve(fraq, specs[s], torch, device_inputs=False)
            walls.append(time.perf_counter() - t0)
            if wl.name == "C4":  # device-resident inputs for the device-timed value
                flush.zero_()
                torch.cuda.synchronize()
                loop, rs = wl.solve(fraq, specs[s], torch, device_inputs=True)
            gc.enable()
            loops.append(loop)
        torch.cuda.synchronize()
    r0 = rs[0]
    assert all(np.isfinite(np.asarray(r.final_state.g1)).all() for r in rs)
    tl = torch.tensor([sum(loops), sum(walls)], dtype=torch.float64, device=dev)
    if pg:
        pg.all_reduce(tl, op=pg.ReduceOp.MAX)
    loop_s, wall_s = float(tl[0]), float(tl[1])
    dof_steps = wl.dofs() * wl.N * K
    scale = 1 if wl.name == "C4" else world  # C4: strong scaling (one job split over ranks)
    value = scale * dof_steps / loop_s
    e2e = scale * dof_steps / wall_s
    # roofline: K13 is bound by the fp64 tensor pipe; algorithmic flops per DOF-step
    # F = 4 N_nodes + 2 N_head, N_nodes / N_head of each field's kernel
    info = r0
    sbd = wl.scheme == "FastSBD"
    tau = 1.0 / wl.N
    if wl.name == "C5" or wl.name == "C5-SBD":
        gams = [(1 - i.alpha1, 1 - i.alpha2) for i in wl.all[:CHUNK]]
    else:
        gams = [(1 - wl.insts[0].alpha1, 1 - wl.insts[0].alpha2)]
    F, Fx = [], []

    def folded(ratios, L):
        # the head fold of modal_plan (modal.cu): M = 8 floor((cap - L) / 8) levels, nodes with
        # |r|^M <= 2^-70 move into the head window; executed flops 4 N_left + 2 (L + M)
        M = max(0, 80 - L) // 8 * 8
        if os.environ.get("FRAQ_K13_FOLD") is not None:
            M = max(0, min(M, int(os.environ["FRAQ_K13_FOLD"]) // 8 * 8))
        left = int(np.sum(np.abs(np.asarray(ratios)) ** M > 2.0 ** -70)) if M else len(ratios)
        return 4 * left + 2 * (L + M)

    for g1_, g2_ in gams[:32]:  # node counts of a sample of the kernels (device auto-sizer)
        for g in (g1_, g2_):
            b = fraq.KernelBudget(horizon=wl.N, eps_tol=1e-12)
            if sbd:
                k = fraq.build_sbd_kernel_auto(g, tau, b)
                F.append(4 * (len(k.ratio1) + len(k.ratio2)) + 2 * k.n_head)
                Fx.append(folded(list(k.ratio1) + list(k.ratio2), k.n_head))
            else:
                k = fraq.build_be_kernel_auto(g, tau, b)
                F.append(4 * len(k.ratios) + 2 * 2)
                Fx.append(folded(list(k.ratios), 2))
    Fm = float(np.mean(F))
    Fxm = float(np.mean(Fx))
    achieved = Fm * dof_steps / loop_s / 1e12
    executed = Fxm * dof_steps / loop_s / 1e12
    peak = fraq.diag_dmma_peak()[0]
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "peak_source": "measured DMMA stream (fraq_diag_dmma_peak)",
                "flops_per_dof_step": Fm, "kernel": "k13_kernel (modal, DMMA)",
                "executed": {"flops_per_dof_step": Fxm, "achieved": executed,
                             "frac": executed / peak,
                             "note": "frac counts SURVEY.md 8(d)'s flops of the reference's "
                                     "recurrences; K13 runs on kernels whose fast-decaying nodes "
                                     "(r^M <= 2^-70) are folded into the exact head window, so "
                                     "it executes fewer (padding to the warp tile not counted)"}}
    split = None
    if wl.solver == "physical" and wl.name != "C3":
        # C5 physical: the history pass of every instance is one HBM-bound K5 launch per level
        # (state 256 inst x 2 fields x 4095 x N_nodes x 8 B read + written); the K6 solves of a
        # level run beside the next level's K5 (CUDA graph), so the whole loop time is charged
        # to K5 here -- a lower bound on its bandwidth
        nodes = Fm / 4 - 1 if not sbd else (Fm - 2 * 17) / 4
        B = 8 * (2 * nodes + 2)
        gbs = B * dof_steps / loop_s / 1e9
        try:
            hbm = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                              "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            hbm = 6543.7
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                    "frac": gbs / hbm, "kernel": "step_kernel (K5, FFPE mode) + K6 overlapped",
                    "bytes_per_dof_step": B, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "note": "whole loop time charged to K5 (lower bound)"}
    if wl.solver == "physical" and wl.name == "C3":
        # per-kernel split of the physical stepper (events around every launch, 1024 levels in
        # the middle of a run): K5 = one fused HBM pass over the history state per level,
        # K6 = RHS + block cyclic reduction + refinement (one CTA per instance, latency-bound)
        i = wl.insts[0]
        spec = fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                                grid_m=wl.M, t_final=1.0, n_steps=wl.N, initial="custom",
                                custom_g1=list(i.g1), custom_g2=list(i.g2))
        st = fraq.FastStepper(spec, sbd, fraq.KernelConfig())
        st.step_n(2048)
        L = 1024
        ms5, ms6 = st.time_split(L)
        nodes = Fm / 4 - 1  # N_nodes (F = 4 N_nodes + 2 N_head, N_head = 2 for BE)
        if sbd:
            nodes = (Fm - 2 * 17) / 4
        B = 8 * (2 * nodes + 2)               # SURVEY.md §8(d) bytes per DOF-step
        dofs = 2 * wl.M
        gbs = B * dofs * L / (ms5 * 1e-3) / 1e9
        try:
            hbm = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                              "MEASURED_PEAKS.json")))["hbm_gbs"]
        except Exception:
            hbm = 6543.7  # the pool's measured copy bandwidth in round 1
        split = {"levels": L, "k5_us_per_level": 1e3 * ms5 / L, "k6_us_per_level": 1e3 * ms6 / L,
                 "k6_share": ms6 / (ms5 + ms6), "loop_us_per_level": 1e6 * loop_s / K / wl.N,
                 "k5_state_mb": 2 * wl.M * nodes * 8 / 1e6}
        roofline = {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s",
                    "frac": gbs / hbm, "kernel": "step_kernel (K5, FFPE mode)",
                    "bytes_per_dof_step": B,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                    "note": "the 16.8 MB C3 state is L2-resident (126 MB L2), so K5 can exceed "
                            "the HBM figure; K6 (one CTA, latency-bound) dominates the level"}
    traffic = None
    try:
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                         "r01_k13_traffic.json")))
        traffic = tr.get(wl.name)
    except Exception:
        pass
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Oracle, ref_available
            if not ref_available():
                raise RuntimeError("oracle/_ref not built")
            orc = Oracle("reference")
            threads = os.cpu_count() or 1
            res = cpu_sample(wl, orc, threads, 12.0)
            cpu = {"value": res[0], "unit": UNIT, "cores": res[2] if len(res) > 2 else threads,
                   "kind": "reference", "sample": res[1]}
        except Exception as e:
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": 1e3 * loop_s / K, "higher_is_better": True,
            "scaling": wl.scaling(), "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": wl.config(),
            "path": ("physical-space solver: K5 (history, FFPE mode) + K6 (RHS, block cyclic "
                     "reduction, refinement) per level" if wl.solver == "physical" else
                     "mode-space solver: DST (DMMA) + K13 (DMMA block stepping, solver warp) + "
                     "inverse DST"),
            "roofline": dict(roofline, traffic=traffic if wl.solver != "physical" else None,
                             traffic_unit="DRAM bytes per K13 launch (ncu, profiles/)"),
            "physical_split": split,
            "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": wl.io_bytes(),
                    "d2h_bytes_per_step": wl.io_bytes(),
                    "path": "fraq.run / run_batch / run_2d with host arrays (setup included)"},
            "gpu_launches": wl.launches() * K,
            "clocks": clk.summary(),
            "cpu_baseline": cpu}), flush=True)
