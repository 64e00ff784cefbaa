"""GPU: the `fraq` CLI and the harness drivers end to end -- the reference's cli_smoke.cmake checks
restated, plus output parity: the weights CSV is byte-identical to the reference's own table
written at 17 digits, the `solve` snapshot equals the reference's run, and the convergence /
timing drivers behave as test_bench.cpp:136-175 requires."""
import math
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1901_05128_b200", "fraq")


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def run(*args, cwd):
    r = subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=300)
    assert r.returncode == 0, r.stderr
    return r


def test_cli_smoke(tmp_path, orc):
    w = tmp_path
    run("weights", "--scheme", "be", "--alpha", "0.5", "--tau", "1", "--n", "3", "--out",
        str(w / "w.csv"), cwd=w)
    txt = (w / "w.csv").read_text()
    assert "-0.0625" in txt
    run("kernel-error", "--scheme", "sbd", "--alpha", "0.3", "--tau", "1/1000", "--np1", "15",
        "--np2", "15", "--ns", "15", "--n-max", "50", "--out", str(w / "ke.csv"), cwd=w)
    ke = (w / "ke.csv").read_text().splitlines()
    assert ke[0] == "i,eps_abs" and ke[3] == "2,0"
    run("solve", "--scheme", "fastsbd", "--alpha1", "0.3", "--alpha2", "0.6", "--a", "2",
        "--grid-m", "31", "--n-steps", "20", "--t-final", "0.5", "--init", "indicator", "--out",
        str(w / "snap.csv"), cwd=w)
    assert len((w / "snap.csv").read_text().splitlines()) == 32
    (w / "exp.cfg").write_text("# tiny study\nscheme = be\nalpha1 = 0.3\nalpha2 = 0.6\na = 2\n"
                               "grid-m = 15\ntaus = 1/8,1/16\nref-tau = 1/128\nt-final = 1\n")
    run("--config", str(w / "exp.cfg"), "convergence", "--scheme", "fastbe", "--out-dir",
        str(w / "conv"), cwd=w)
    assert (w / "conv" / "convergence_fastbe.csv").exists()
    assert not (w / "conv" / "convergence_be.csv").exists()
    assert (w / "conv" / "meta.txt").exists()
    run("bench", "--scheme", "fastbe", "--alpha1", "0.4", "--alpha2", "0.6", "--grid-m", "15",
        "--n-list", "1,2", "--out", str(w / "bench.csv"), cwd=w)
    b = (w / "bench.csv").read_text().splitlines()
    assert b[0] == "scheme,N,seconds_loop,seconds_setup" and len(b) == 3


@pytest.mark.parametrize("scheme,alpha,tau,n", [("be", "0.3777", "0.0123", "200"),
                                                 ("sbd", "0.65", "1/4096", "300")])
def test_weights_csv_identical_to_reference(tmp_path, orc, scheme, alpha, tau, n):
    import paper_1901_05128_b200 as fraq
    run("weights", "--scheme", scheme, "--alpha", alpha, "--tau", tau, "--n", n, "--out",
        str(tmp_path / "w.csv"), cwd=tmp_path)
    a, t = fraq.parse_fraction(alpha), fraq.parse_fraction(tau)
    ref = (orc.sbd_weights if scheme == "sbd" else orc.be_weights)(a, t, int(n))
    expect = "i,d_i\n" + "".join(f"{i},{fraq.format_double(v)}\n" for i, v in enumerate(ref))
    got = (tmp_path / "w.csv").read_text()
    if scheme == "be":  # K1 reproduces the reference's serial chain bit for bit
        assert got == expect
    else:               # Cauchy product: same order; compare values
        vals = np.array([float(r.split(",")[1]) for r in got.splitlines()[1:]])
        assert np.abs(vals - ref).max() <= 1e-13 * np.abs(ref).max()


def test_cli_solve_matches_reference(tmp_path, orc):
    run("solve", "--scheme", "fastbe", "--alpha1", "0.35", "--alpha2", "0.7", "--m", "0.3",
        "--grid-m", "63", "--tau", "1/400", "--t-final", "0.5", "--init", "poly_sin", "--out",
        str(tmp_path / "s.csv"), cwd=tmp_path)
    rows = [r.split(",") for r in (tmp_path / "s.csv").read_text().splitlines()[1:]]
    g1 = np.array([float(r[1]) for r in rows])
    g2 = np.array([float(r[2]) for r in rows])
    a = (1 - 0.3) / (2 * 0.3 - 1)
    r1, r2, _, _ = orc.run(0.35, 0.7, a, 63, 0.5, 200, "FastBE", "poly_sin")
    assert np.abs(g1 - r1).max() <= 1e-10 * np.abs(r1).max()
    assert np.abs(g2 - r2).max() <= 1e-10 * np.abs(r2).max()


def test_convergence_driver_tiny():  # test_bench.cpp:136-161
    import paper_1901_05128_b200 as fraq
    cfg = fraq.ExperimentConfig()
    cfg.schemes = [fraq.Scheme.BE, fraq.Scheme.FastBE]
    cfg.alpha1, cfg.alpha2, cfg.coupling_a, cfg.grid_m, cfg.t_final = 0.3, 0.6, 2.0, 31, 0.25
    cfg.taus = [cfg.t_final / 8, cfg.t_final / 16, cfg.t_final / 32]
    cfg.ref_tau = cfg.t_final / 256
    reps = fraq.run_convergence(cfg)
    assert len(reps) == 2
    for rep in reps:
        assert len(rep.rows) == 3 and math.isnan(rep.rows[0].rate1)
        for i in range(1, 3):
            assert rep.rows[i].e1 < rep.rows[i - 1].e1
            assert 0.5 < rep.rows[i].rate1 < 2.0
    for i in range(3):
        assert reps[0].rows[i].e1 == pytest.approx(reps[1].rows[i].e1, rel=1e-6)


def test_timing_sweep():  # test_bench.cpp:163-175
    import paper_1901_05128_b200 as fraq
    cfg = fraq.ExperimentConfig()
    cfg.schemes = [fraq.Scheme.FastBE]
    cfg.alpha1, cfg.alpha2, cfg.grid_m, cfg.t_final = 0.4, 0.6, 15, 0.1
    rows = fraq.timing_sweep(cfg, [1, 4])
    assert len(rows) == 2 and rows[0].scheme == "fastbe" and rows[0].n_steps == 1
    assert rows[0].seconds_loop > 0 and rows[1].seconds_loop > 0
