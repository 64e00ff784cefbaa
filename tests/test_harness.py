"""CPU: the experiment harness (fraq_bench.cpp, the reference's src/bench.cpp) and the `fraq` CLI's
argument handling -- the reference's own test_bench.cpp cases restated (parse_fraction,
parse_config_text, resolve_config precedence, validation, compute_rates, 17-digit formatting) and
the usage-error exit codes of tests/cli_smoke.cmake.  No GPU needed: nothing here solves."""
import math
import os
import random
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1901_05128_b200", "fraq")


@pytest.fixture(scope="module")
def fq():
    import paper_1901_05128_b200 as fraq
    return fraq


def test_parse_fraction(fq):  # test_bench.cpp:13-25
    assert fq.parse_fraction("1/3200") == 1.0 / 3200.0
    assert fq.parse_fraction("0.5") == 0.5
    assert fq.parse_fraction(" 3/4 ") == 0.75
    assert fq.parse_fraction("-2") == -2.0
    for bad in ("1/0", "abc", "1/2x"):
        with pytest.raises(ValueError):
            fq.parse_fraction(bad)
    lst = fq.parse_fraction_list("1/100,1/200, 0.25")
    assert lst == [0.01, 1.0 / 200.0, 0.25]


def test_parse_config_text(fq):  # test_bench.cpp:27-40
    m = fq.parse_config_text("# comment line\nalpha1 = 0.3\ntaus = 1/100,1/200\n\n"
                             "scheme= be,fastbe # trailing comment\n")
    assert m == {"alpha1": "0.3", "taus": "1/100,1/200", "scheme": "be,fastbe"}
    with pytest.raises(ValueError):
        fq.parse_config_text("no equals sign here\n")


def test_resolve_config_precedence(fq):  # test_bench.cpp:42-70 (property style)
    file_vals = {"alpha1": "0.25", "alpha2": "0.65", "grid-m": "127", "t-final": "2",
                 "np": "96", "eps-tol": "1e-10"}
    cli_vals = {"alpha1": "0.35", "alpha2": "0.45", "grid-m": "63", "t-final": "4",
                "np": "128", "eps-tol": "1e-8"}
    rng = random.Random(99)
    for _ in range(50):
        f = {k: v for k, v in file_vals.items() if rng.random() < 0.5}
        c = {k: v for k, v in cli_vals.items() if rng.random() < 0.5}
        cfg = fq.resolve_config(f, c)

        def expect(k, d):
            return fq.parse_fraction(c[k]) if k in c else (fq.parse_fraction(f[k]) if k in f else d)
        assert cfg.alpha1 == expect("alpha1", 0.5)
        assert cfg.alpha2 == expect("alpha2", 0.5)
        assert cfg.grid_m == int(expect("grid-m", 255))
        assert cfg.t_final == expect("t-final", 1.0)
        assert cfg.kernel.be_points == int(expect("np", 64))
        assert cfg.kernel.eps_tol == expect("eps-tol", 1e-12)


def test_resolve_config_details(fq):  # test_bench.cpp:72-83
    cfg = fq.resolve_config({"m": "0.75"}, {"scheme": "sbd,fastsbd", "taus": "1/20,1/40",
                                            "ref-tau": "1/640"})
    assert cfg.coupling_a == pytest.approx(0.5)
    assert list(cfg.schemes) == [fq.Scheme.SBD, fq.Scheme.FastSBD]
    assert len(cfg.taus) == 2
    assert fq.resolve_config({"m": "0.75"}, {"a": "-1"}).coupling_a == -1.0
    with pytest.raises(ValueError):
        fq.resolve_config({}, {"init": "bogus"})


def test_config_validation(fq):  # test_bench.cpp:85-95
    cfg = fq.ExperimentConfig()
    cfg.taus = [1 / 100, 1 / 200]
    cfg.ref_tau = 1 / 3200
    cfg.validate()
    cfg.ref_tau = 1 / 200
    with pytest.raises(ValueError):
        cfg.validate()
    cfg.ref_tau = 1 / 3200
    cfg.taus = [1 / 200, 1 / 100]
    with pytest.raises(ValueError):
        cfg.validate()


def test_compute_rates_and_format(fq):  # test_bench.cpp:97-107
    r = fq.compute_rates([(1 / 100, 8.434e-6), (1 / 200, 4.141e-6)])
    assert r[0] == pytest.approx(1.0263, rel=2e-4)
    assert fq.compute_rates([(0.5, 4.0), (0.25, 2.0)])[0] == pytest.approx(1.0, abs=1e-12)
    assert fq.compute_rates([(0.5, 4.0), (0.25, 1.0)])[0] == pytest.approx(2.0, abs=1e-12)
    with pytest.raises(ValueError):
        fq.compute_rates([(0.5, 1.0), (0.3, 0.5)])
    blank = fq.compute_rates([(0.5, 0.0), (0.25, 1.0)])
    assert math.isnan(blank[0]) and fq.format_double(blank[0]) == ""
    rng = random.Random(1)
    for _ in range(1000):  # 17 significant digits: exact round trip
        x = rng.uniform(-1, 1) * 10 ** rng.randint(-300, 300)
        assert float(fq.format_double(x)) == x


def _cli(*args, cwd=None):
    return subprocess.run([CLI, *args], capture_output=True, text=True, cwd=cwd, timeout=120)


def test_cli_usage_errors_exit_2():  # cli_smoke.cmake:79-80 and the parse-error path
    assert _cli("weights", "--scheme", "nope", "--alpha", "0.5", "--tau", "1", "--n", "3").returncode == 2
    assert _cli("convergence", "--taus", "1/8,1/16", "--ref-tau", "1/4").returncode == 2
    assert _cli("bogus").returncode == 2
    assert _cli().returncode == 2
    assert _cli("weights", "--unknown", "1").returncode == 2
    assert _cli("weights", "--alpha").returncode == 2
    h = _cli("--help")
    assert h.returncode == 0 and "kernel-error" in h.stdout
