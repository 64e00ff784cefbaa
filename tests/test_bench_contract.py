"""bench.py's JSON contract: the reference arm on CPU (runs here), the GPU arm on a B200."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(*args, timeout=900):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("workload", ["C2", "C3"])
def test_reference_arm_contract(workload):
    from oracle.oracle import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0", "--workload", workload)
    assert d["impl"] == "reference" and KEYS <= set(d)
    assert d["value"] > 0 and d["unit"] == "DOF-steps/s" and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    # same_config: the reference arm prints exactly the dict the GPU arm prints
    if workload == "C2":
        import bench
        assert d["config"] == bench.c2_config(1, [512, 512], [17, 15])
    else:
        import bench_ffpe
        assert d["config"] == bench_ffpe.Workload(workload, 0, 1).config()


def test_reference_arm_maps_no_product_library():
    """The CPU arm must not load the B200 package (its __init__ maps _fraq / libfraqcu.so):
    everything it imports -- workloads, oracle -- lives outside the package."""
    code = ("import sys; sys.argv = ['bench.py']; import bench, bench_ffpe, workloads, oracle.oracle; "
            "workloads.c2_params(64); bench_ffpe.Workload('C3', 0, 1).config(); "
            "bad = [m for m in sys.modules if m.startswith('paper_1901_05128_b200')]; "
            "assert not bad, bad")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.gpu
def test_gpu_arm_contract():
    d = _run("--steps", "4", "--warmup", "3", "--e2e-steps", "1")
    assert KEYS <= set(d) and "impl" not in d
    assert d["value"] > 1e9 and d["n_gpus"] == 1 and d["scaling"] == "weak"
    rf = d["roofline"]
    # frac counts SURVEY.md 8(d)'s algorithmic flops (the reference's recurrences), which K5e
    # undercuts by folding the fast-decaying nodes into a FIR: only the executed share is <= 1
    assert rf["bound"] in ("hbm", "tensor") and 0 < rf["frac"] <= 3.0
    assert rf["achieved"] == pytest.approx(rf["frac"] * rf["peak"], rel=1e-9)
    ex = rf["executed"]
    assert 0 < ex["frac"] <= 1.05 and ex["flops_per_dof_step"] <= rf["flops_per_dof_step"]
    assert ex["achieved"] == pytest.approx(ex["frac"] * rf["peak"], rel=1e-9)
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= d["steps"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["value"] > 0
    # the per-level lines: K5 against the HBM roofline, K5f (the same calls in the steady state)
    rs = d["roofline_step_kernel"]
    assert rs["bound"] == "hbm" and 0 < rs["frac"] <= 1.0
    fo = rs["folded"]
    assert fo is not None and 0 < fo["ms_per_level"] < rs["ms_per_level"]
    assert fo["bytes_per_dof_step_moved"] < rs["bytes_per_dof_step"]
    assert d["setup"]["launches_by_path"]["K5e"] >= d["steps"] - 1
