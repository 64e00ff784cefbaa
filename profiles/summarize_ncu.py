"""Summarise ncu captures (run here, no GPU): launch list shares and key metrics of full captures.

    python profiles/summarize_ncu.py gpurun_out/launches.csv gpurun_out/prof_k5b.ncu-rep ...
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def launches(path):
    txt = open(path).read()
    lines = [l for l in txt.splitlines() if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, data = rows[0], rows[1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ik].split("(")[0][:80]
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    print(f"== launch list {path}: {sum(v[0] for v in agg.values())} launches, {tot/1e6:.3f} ms "
          "(cold-cache, serialised: compare shares)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:20]:
        print(f"{v[0]:6d} x {v[1]/1e6/v[0]:9.4f} ms = {v[1]/1e6:9.3f} ms {100*v[1]/tot:5.1f}%  "
              f"[{role(k)}] {k}")
    # the bench's timed step is the history kernel alone; everything else is setup, the live
    # peak diagnostics behind roofline.peak, or the side measurements (K5 roofline, e2e)
    roles = collections.defaultdict(float)
    for k, v in agg.items():
        roles[role(k)] += v[1]
    print("   by role: " + ", ".join(f"{r} {100 * t / tot:.1f}%" for r, t in
                                      sorted(roles.items(), key=lambda x: -x[1])))


def role(name):
    if any(x in name for x in ("run3_kernel", "run4_kernel", "note_rows_kernel", "k13_kernel")):
        return "timed step (and its e2e / warm-up repeats)"
    if "dmma_kernel" in name or "dfma_kernel" in name:
        return "peak diagnostic"
    if any(x in name for x in ("scan_kernel", "chain_kernel", "cauchy_kernel", "rule_kernel",
                               "frag_tables", "reconstruct", "k13_tables")):
        return "setup"
    if "step_kernel" in name:
        return "K5 roofline side run"
    return "other (torch input generation / checks)"


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    print(f"== full capture {path}")
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name"))
        for k in KEYS:
            if k in d:
                print(f"   {k:70s} {d[k]} {u.get(k, '')}")
        stalls = [(k, d[k]) for k in d if k.startswith("smsp__pcsamp_warps_issue_stalled")
                  and not k.endswith("not_issued")]
        stalls = sorted(((k, float(v.replace(",", ""))) for k, v in stalls
                         if v.replace(",", "").replace(".", "", 1).isdigit()), key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        print("   top stall reasons (pc sampling):",
              ", ".join(f"{k.split('stalled_')[1]} {100*v/tot:.0f}%" for k, v in stalls[:6]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        (launches if p.endswith(".csv") else full)(p)
