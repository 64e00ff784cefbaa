#!/usr/bin/env python
"""Benchmark of the B200 fast-CQ path on BASELINE.json's headline configuration (configs[1], C2).

Workload C2: batched Riemann-Liouville derivative with the BDF2 (SBD) fast CQ, 65536 DOFs per GPU
(CQ exponent 0.7 on the first half, 0.3 on the second), tau = 1/65536, reference auto-sized
kernels (256 + 256 nodes, N_s = 17 / 15).  Signals u_k(t) = a_k t^b_k + c_k sin(w_k t), seeded
(workloads.py), generated on the device before timing.

One bench step = one pass of the hot path over the batch for LEVELS_PER_STEP (1024) time levels:
push + derivative for every DOF at every level, through MultiHistory.run_device on device buffers
(temporally blocked kernels on the fp64 tensor cores: K5d for the first 96 levels of a history,
K5e -- the fast-decaying nodes folded into an exact FIR window -- from there on).  K timed steps
advance a fresh history from level 0; the default K = 64 covers the whole C2 horizon N = 65536.
Warm-up steps run on a separate history.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload C2 | C3 | C4 | C5 | C5-SBD]     (FFPE configs: bench_ffpe.py)

Prints one JSON line (rank 0).  --impl reference times the reference's own CPU implementation
(oracle/_ref: the unmodified reference sources) on the host cores with the same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fast-CQ DOF-steps/s (fp64) and % of HBM roofline at 1/2/4/8 B200 vs CPU"
UNIT = "DOF-steps/s"
LEVELS_PER_STEP = 1024
DOFS = 65536
N_LEVELS = 65536


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ----------------------------------------------------------------------------- clocks sampling
class Clocks:
    """nvidia-smi samples (SM clock, throttle reasons) during a timed region.  The sampler is
    started and its first line awaited before the region begins, and it polls every 50 ms, so
    even a ~100 ms region (C2: 20 steps x 5 ms) gets samples; the pre-region line is dropped."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            import select
            ready, _, _ = select.select([self.proc.stdout], [], [], 5.0)
            if ready:
                self.proc.stdout.readline()  # sampler is up; this line predates the region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) >= 7 and f[0].isdigit():
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(int(r[0]) for r in rows),
                "sm_max_mhz": int(rows[0][1]), "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- reference arm
def reference_kernels(orc, tau):
    """The reference's own auto-sized C2 kernels (fast_kernel.cpp:207-256), horizon N."""
    return [orc.build_kernel_auto(True, 1.0 - 0.3, tau, N_LEVELS),
            orc.build_kernel_auto(True, 1.0 - 0.7, tau, N_LEVELS)]


def c2_config(world, nodes, n_head, scaling="weak"):
    """The workload description both arms print (identical dicts: same_config)."""
    per = DOFS if scaling == "weak" else -(-DOFS // world)
    return {
        "workload": "C2: BDF2 fast CQ, 65536 DOFs (gamma 0.7 | 0.3), tau = 1/65536, N = 65536 "
                    "levels; one step = 1024 levels x all DOFs (push+derivative)",
        "dofs_per_gpu": per, "levels_per_step": LEVELS_PER_STEP,
        "nodes": list(nodes), "n_head": list(n_head),
        "l2": "inputs larger than L2 (537 MB of signal per step)",
        "parallelism": (f"dof-sharded x{world}, no data-path collective" if scaling == "weak" else
                        f"65536 / {world} DOFs per GPU (strong), no data-path collective")}


def cpu_sample(orc, kernels, params, threads, levels, dofs=DOFS, U=None):
    """Times the reference SbdHistory (push + derivative per level) on the FULL C2 DOF set (both
    exponent halves; each of `threads` host threads owns a contiguous DOF slice, the run_convergence
    worker-pool pattern of bench.cpp:194-223) for `levels` levels from level 0.  Per-level cost does
    not depend on the level index once the lag window is full, so DOF-steps/s over the sample equals
    the full-run rate.  Returns (DOF-steps/s, sample description, seconds)."""
    if U is None:
        U = params.signal(0, levels, np.arange(dofs))
    secs, _ = orc.bench_history(kernels, U[:levels], threads)
    return (dofs * levels / secs, f"all {dofs} DOFs x {levels} levels (per-thread DOF slices "
            f"as in a full run)", secs)


def run_reference_arm(args):
    """The reference's own CPU implementation (oracle/_ref = the unmodified reference sources) on
    the host cores, on the GPU arm's workload: one step = all 65536 DOFs x 1024 levels.  Maps no
    library of the B200 package (checked)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle.oracle import Oracle, ref_available
    from workloads import c2_params
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    orc = Oracle("reference")
    params = c2_params()
    kernels = reference_kernels(orc, params.tau)
    threads = os.cpu_count() or 1
    U = params.signal(0, LEVELS_PER_STEP, np.arange(DOFS))
    for _ in range(args.warmup):
        cpu_sample(orc, kernels, params, threads, LEVELS_PER_STEP // 8, U=U)
    vals, times = [], []
    for _ in range(args.steps):
        v, sample, secs = cpu_sample(orc, kernels, params, threads, LEVELS_PER_STEP, U=U)
        vals.append(v)
        times.append(secs)
    value = DOFS * LEVELS_PER_STEP * args.steps / sum(times)
    loaded = sorted(m for m in sys.modules if m.startswith("paper_1901_05128_b200"))
    assert not loaded, f"reference arm imported the B200 package: {loaded}"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": c2_config(world, [len(k.r1) + len(k.r2) for k in kernels],
                            [k.n_head for k in kernels], args.scaling),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample + " per step; reference SbdHistory push+derivative, "
                                            "per-thread DOF slices (bench.cpp:194-223 pattern)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=N_LEVELS // LEVELS_PER_STEP)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--solver", default="modal", choices=["modal", "physical"],
                    help="FFPE workloads: mode-space (default) or the physical-space stepper")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="C2: 65536 DOFs per GPU (weak, default) or 65536 / N per GPU (strong, "
                         "SURVEY.md §8(e))")
    ap.add_argument("--workload", default="C2", choices=["C2", "C3", "C4", "C5", "C5-SBD"],
                    help="C2 (default, BASELINE configs[1]) or an FFPE config (bench_ffpe.py)")
    args = ap.parse_args()
    if args.workload != "C2":
        import bench_ffpe
        if args.steps == N_LEVELS // LEVELS_PER_STEP:
            args.steps = {"C3": 20, "C4": 3, "C5": 4, "C5-SBD": 4}[args.workload]
        if args.impl == "reference":
            rank, world, _ = dist_env()
            bench_ffpe.run_reference(args, rank, world, METRIC)
            return
    if args.impl == "reference":
        run_reference_arm(args)
        return

    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    os.environ.setdefault("FRAQ_DEVICE", str(local))
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    import paper_1901_05128_b200 as fraq
    from workloads import c2_params
    if args.workload != "C2":
        import bench_ffpe
        bench_ffpe.run_gpu(args, rank, world, local, pg, METRIC, Clocks, fraq, torch)
        if pg:
            pg.barrier()
            pg.destroy_process_group()
        return

    params = c2_params(DOFS)
    tau = params.tau
    # device setup (K1-K4): auto-sized kernels for both exponents, as the reference picks them
    t0 = time.time()
    kernels = []
    for g in (1.0 - 0.3, 1.0 - 0.7):
        b = fraq.KernelBudget(horizon=N_LEVELS, eps_tol=1e-12)
        kernels.append((fraq.build_sbd_kernel_auto(g, tau, b), b.achieved_eps))
    setup_s = time.time() - t0
    ks = [k for k, _ in kernels]
    n_nodes = [len(k.ratio1) + len(k.ratio2) for k in ks]
    n_head = [k.n_head for k in ks]

    dev = torch.device("cuda", local)
    stream = torch.cuda.ExternalStream(fraq.context_stream())
    K, W = args.steps, args.warmup
    # input / output buffers for at most one horizon of steps (reused cyclically beyond that;
    # every step's signal is larger than L2 either way)
    nbuf = max(1, min(K, N_LEVELS // LEVELS_PER_STEP))
    levels = nbuf * LEVELS_PER_STEP
    if args.scaling == "strong":
        # contiguous DOF blocks of the ONE 65536-DOF job, 65536/N per GPU
        from paper_1901_05128_b200.parallel import c2_strong_slice
        lo, hi, groups = c2_strong_slice(rank, world, DOFS)
        sel = slice(lo, hi)
        a, bb, c, w = (torch.from_numpy(x[sel].copy()) for x in (params.a, params.b, params.c,
                                                                  params.w))
        dims = [0, 0]
        for g, cnt in groups:
            dims[g] = cnt
    else:
        # weak: each rank owns 65536 DOFs (rank 0 the seeded C2 set, others rank-seeded draws)
        gen = torch.Generator(device="cpu").manual_seed(1901051282 + rank)
        if rank == 0:
            a = torch.from_numpy(params.a); bb = torch.from_numpy(params.b)
            c = torch.from_numpy(params.c); w = torch.from_numpy(params.w)
        else:
            a = torch.randn(DOFS, generator=gen, dtype=torch.float64)
            c = torch.randn(DOFS, generator=gen, dtype=torch.float64)
            bb = 0.1 + 1.9 * torch.rand(DOFS, generator=gen, dtype=torch.float64)
            w = 1.0 + 19.0 * torch.rand(DOFS, generator=gen, dtype=torch.float64)
        dims = [DOFS // 2, DOFS - DOFS // 2]
    gk = [k for k, d in zip(ks, dims) if d > 0]
    dims = [d for d in dims if d > 0]
    NL = sum(dims)  # DOFs on this rank
    a, bb, c, w = (x.to(dev) for x in (a, bb, c, w))
    U = torch.empty((levels, NL), dtype=torch.float64, device=dev)
    for n0 in range(0, levels, 1024):
        n1 = min(levels, n0 + 1024)
        t = (torch.arange(n0, n1, device=dev, dtype=torch.float64) * tau)[:, None]
        U[n0:n1] = a * torch.pow(t, bb) + c * torch.sin(w * t)
    D = torch.empty_like(U)
    Uw = U[:LEVELS_PER_STEP].clone()
    Dw = torch.empty_like(Uw)
    torch.cuda.synchronize()

    # warm-up on a scratch history
    hw = fraq.MultiHistory(gk, dims)
    for _ in range(W):
        hw.run_device(Uw.data_ptr(), NL, LEVELS_PER_STEP, Dw.data_ptr(), NL)
    fraq.synchronize()
    del hw

    h = fraq.MultiHistory(gk, dims)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    if pg:
        pg.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        ev[0].record(stream)
        for s in range(K):
            off = (s % nbuf) * LEVELS_PER_STEP * NL * 8
            h.run_device(U.data_ptr() + off, NL, LEVELS_PER_STEP, D.data_ptr() + off, NL)
            ev[s + 1].record(stream)
        ev[K].synchronize()
        torch.cuda.synchronize()
    assert h.last_path >= 1, "temporally blocked kernel did not run"
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(K)]
    total_ms = ev[0].elapsed_time(ev[K])
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if pg:
        pg.all_reduce(t_local, op=pg.ReduceOp.MAX)
    total_ms = float(t_local.item())
    dof_steps_local = NL * LEVELS_PER_STEP * K
    job_dofs = DOFS if args.scaling == "strong" else world * DOFS
    value = job_dofs * LEVELS_PER_STEP * K / (total_ms * 1e-3)

    # sanity: outputs finite after the first level
    assert torch.isfinite(D[1:]).all().item()

    # roofline of the dominant kernel (K5e): fp64 tensor-pipe bound; algorithmic flops per DOF-step
    # F = 4 N_nodes + 2 N_head, averaged over the two exponent halves.  K5e
    # EXECUTES fewer: per 16 DOFs x 8 levels 8 DMMAs per tile of 8 slow nodes + 2 per 4 rows of the
    # combined input window (head taps + the FIR of the fast-decaying nodes); both are reported.
    F = 0.5 * sum(4 * nn + 2 * hh for nn, hh in zip(n_nodes, n_head))
    achieved_tf = F * dof_steps_local / (total_ms * 1e-3) / 1e12
    launches = list(h.launches)
    fir = list(h.fir_info)
    fir_groups = [{"fir_levels": fir[3 * i], "recurrence_nodes": fir[3 * i + 1],
                   "window_rows": fir[3 * i + 2]} for i in range(len(dims))]
    k5e = h.last_path == 4 and all(fg["window_rows"] > 0 for fg in fir_groups)
    if k5e:
        dmma_blk = [8 * ((fg["recurrence_nodes"] + 7) // 8) + 2 * (fg["window_rows"] // 4)
                    for fg in fir_groups]
        F_exec = sum(d * 512.0 / 128.0 * dm for d, dm in zip(dmma_blk, dims)) / NL
    else:
        F_exec = F
    executed_tf = F_exec * dof_steps_local / (total_ms * 1e-3) / 1e12
    dmma_peak = fraq.diag_dmma_peak()[0]   # fp64 tensor core (DMMA) stream, measured live
    fp64_peak = fraq.diag_fp64_peak()      # DFMA stream, for reference
    # HBM figures: algorithmic bytes of one state pass per level, B = 8 (2 N_nodes + 2)
    B = 0.5 * sum(8 * (2 * nn + 2) for nn in n_nodes)
    pk = peaks()
    try:  # DRAM traffic per K5d launch from the committed ncu --set full capture (profiles/)
        tr = json.load(open(os.path.join(ROOT, "profiles", "r02",
                                         "k5e_traffic.json" if k5e else "k5d_traffic.json")))
        assert tr["levels_per_launch"] == LEVELS_PER_STEP
        traffic = tr["dram_bytes_per_launch"] / 1e9  # GB per launch (one step)
    except Exception:
        traffic = None

    # per-level fused kernel K5 (one HBM pass over the state per level) on the same workload
    hs = fraq.MultiHistory(gk, dims)
    nstep = 24
    hs.run_device(U.data_ptr(), NL, 3, D.data_ptr(), NL)  # levels 0..2 (n_steps < 4: per-level K5)
    torch.cuda.synchronize()
    # force the per-level path: push/derivative on device pointers level by level
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for n in range(3, 3 + nstep):
        hs.run_device(U.data_ptr() + n * NL * 8, NL, 1, D.data_ptr() + n * NL * 8, NL)
    e1.record(stream)
    e1.synchronize()
    assert hs.last_path == 0
    step_level_ms = e0.elapsed_time(e1) / nstep
    hbm_step = B * NL / (step_level_ms * 1e-3) / 1e9
    # the same per-level calls in the steady state: K5f (K5e's fold, per level: only the slow
    # nodes keep a state in HBM, the fast-decaying ones are an exact FIR over the input ring)
    fold = None
    n0f = 3 + nstep
    hs.run_device(U.data_ptr() + n0f * NL * 8, NL, 160, D.data_ptr() + n0f * NL * 8, NL)
    n0f += 160
    lf0 = list(hs.launches)
    for n in range(n0f, n0f + 4):
        hs.run_device(U.data_ptr() + n * NL * 8, NL, 1, D.data_ptr() + n * NL * 8, NL)
    n0f += 4
    e0.record(stream)
    for n in range(n0f, n0f + nstep):
        hs.run_device(U.data_ptr() + n * NL * 8, NL, 1, D.data_ptr() + n * NL * 8, NL)
    e1.record(stream)
    e1.synchronize()
    lf1 = list(hs.launches)
    if len(lf1) > 5 and lf1[5] - lf0[5] == nstep + 4:
        fold_ms = e0.elapsed_time(e1) / nstep
        fi = list(hs.fir_info)
        # bytes K5f moves per DOF-step: the kept nodes' states read + written, the window rows
        # (head + FIR taps, from the L2-resident input ring), input and output
        Bf = 0.5 * sum(8 * (2 * fi[3 * g + 1] + (n_head[g] + fi[3 * g]) + 2) for g in range(2))
        fold = {"kernel": "step_fir_kernel (K5f)", "ms_per_level": fold_ms,
                "speedup_vs_K5": step_level_ms / fold_ms,
                "bytes_per_dof_step_moved": Bf,
                "moved_gbs": Bf * NL / (fold_ms * 1e-3) / 1e9,
                "algorithmic_gbs": B * NL / (fold_ms * 1e-3) / 1e9,
                "note": "algorithmic_gbs counts SURVEY.md 8(d)'s B (every node's state read and "
                        "written per level) and can exceed the HBM peak: K5f keeps only the "
                        "slow nodes' states"}
    del hs

    # e2e: the same metric through the C-ABI call with HOST buffers (pinned), copies inside
    ke = max(1, min(args.e2e_steps, K, nbuf))
    Uh = U[:ke * LEVELS_PER_STEP].cpu().pin_memory()
    Dh = torch.empty_like(Uh).pin_memory()
    he = fraq.MultiHistory(gk, dims)
    # untimed warm-up calls (first-call device state, staging buffers, streams, fragment tables)
    for s in range(min(args.warmup, ke)):
        rows = slice(s * LEVELS_PER_STEP, (s + 1) * LEVELS_PER_STEP)
        he.run(Uh[rows].numpy(), True, Dh[rows].numpy())
    torch.cuda.synchronize()
    t_e = time.perf_counter()
    for s in range(ke):
        rows = slice(s * LEVELS_PER_STEP, (s + 1) * LEVELS_PER_STEP)
        # host in, host out: H2D + K5d + D2H inside fraq_hist_run (pinned buffers)
        he.run(Uh[rows].numpy(), True, Dh[rows].numpy())
    e2e_s = time.perf_counter() - t_e
    del he
    t_e = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if pg:
        pg.all_reduce(t_e, op=pg.ReduceOp.MAX)
    e2e_val = job_dofs * LEVELS_PER_STEP * ke / float(t_e.item())
    step_bytes = LEVELS_PER_STEP * NL * 8

    # CPU baseline: the reference (oracle/_ref) on the host cores, rank 0 only, bounded sample
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            from oracle.oracle import Oracle, ref_available
            kind = "reference" if ref_available() else "port"
            orc = Oracle(kind)
            rk = reference_kernels(orc, tau)
            threads = os.cpu_count() or 1
            # ~10-15 s of CPU work: all DOFs x 256 levels
            v, sample, secs = cpu_sample(orc, rk, params, threads, LEVELS_PER_STEP // 4)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": kind,
                   "sample": sample + f" ({secs:.1f} s), reference SbdHistory push+derivative"}
        except Exception as e:  # report, never fake
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": total_ms / K, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": c2_config(world, n_nodes, n_head, args.scaling),
            "setup": {"kernel_eps": [e for _, e in kernels], "setup_s": setup_s,
                      "path": "MultiHistory.run_device -> " +
                              ("K5e (temporally blocked, fp64 tensor cores; fast-decaying nodes "
                               "as an exact FIR window; K5d on a history's first 96 levels)"
                               if k5e else "K5d (temporally blocked, fp64 tensor cores)"),
                      "k5e_groups": fir_groups,
                      "launches_by_path": dict(zip(["K5", "short_state", "K5c", "K5d", "K5e",
                                                    "K5f"], launches))},
            "roofline": {"bound": "tensor", "achieved": achieved_tf, "peak": dmma_peak,
                         "unit": "TFLOP/s", "frac": achieved_tf / dmma_peak,
                         "traffic": traffic, "traffic_unit": "GB per launch (ncu, profiles/)",
                         "peak_source": "measured fp64 tensor-core (DMMA) stream on this GPU "
                                        "(fraq_diag_dmma_peak); DFMA stream %.1f TF/s" % fp64_peak,
                         "dtype": "f64",
                         "flops_per_dof_step": F,
                         "kernel": "run4_kernel (K5e, DMMA)" if k5e else "run3_kernel (K5d, DMMA)",
                         "executed": {"flops_per_dof_step": F_exec, "achieved": executed_tf,
                                      "frac": executed_tf / dmma_peak,
                                      "note": "achieved / frac above count SURVEY.md 8(d)'s "
                                              "algorithmic flops of the reference's recurrences "
                                              "(one state update + one readout term per node and "
                                              "level); K5e replaces the nodes with r^M <= 2^-70 "
                                              "by an exact M-tap FIR, so it executes fewer flops "
                                              "and frac can exceed 1; executed.frac is the share "
                                              "of the DMMA peak the kernel's own DMMAs reach"},
                         "hbm_equiv_gbs": B * dof_steps_local / (total_ms * 1e-3) / 1e9},
            "roofline_step_kernel": {"bound": "hbm", "achieved": hbm_step,
                                     "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                                     "frac": hbm_step / pk.get("hbm_gbs"),
                                     "bytes_per_dof_step": B, "kernel": "step_kernel (K5)",
                                     "ms_per_level": step_level_ms,
                                     "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                                     "folded": fold},
            "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": step_bytes,
                    "d2h_bytes_per_step": step_bytes, "steps": ke,
                    "path": "MultiHistory.run(host numpy) -> fraq_hist_run(FRAQ_HOST)"},
            "gpu_launches": int(sum(launches)),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "step_ms_min_max": [min(step_ms), max(step_ms)],
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
