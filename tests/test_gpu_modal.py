"""GPU: mode-space (DST) FFPE stepping, 1D (solver=MODAL) and 2D (BASELINE C4).

1D: equals the reference's physical-space FastStepper (oracle/_ref) on well-conditioned grids,
and the fp64 mode-space evaluation at the C3 grid.  2D: equals the numpy restatement of the
FastStepper algebra with the five-point Laplacian (tests/ffpe_refs.py) on small grids."""
import numpy as np
import pytest

from ffpe_refs import fast_stepper_nd, modespace_fastbe

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.max(np.abs(a - b)) / np.max(np.abs(b))


def modal_kc(fraq, **kw):
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_MODAL
    for k, v in kw.items():
        setattr(kc, k, v)
    return kc


@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
@pytest.mark.parametrize("m,a,init", [(31, -1.0, "indicator"), (63, 2.0, "poly_sin"),
                                      (50, 0.5, "poly_sin"), (127, -2.0, "indicator")])
def test_modal_1d_matches_reference(fraq, orc, scheme, m, a, init):
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.65, coupling_a=a, grid_m=m, t_final=0.5,
                            n_steps=96, initial=init)
    rr = fraq.run(spec, getattr(fraq.Scheme, scheme), modal_kc(fraq))
    g1, g2, e1, e2 = orc.run(0.3, 0.65, a, m, 0.5, 96, scheme, init)
    assert rel(rr.final_state.g1, g1) <= 1e-10
    assert rel(rr.final_state.g2, g2) <= 1e-10
    assert rr.kernel_eps1 == pytest.approx(e1, rel=1e-3)


def test_modal_1d_fixed_kernels_and_batch(fraq, orc):
    kc = modal_kc(fraq, auto_size=False, be_points=24, sbd_points_1=24, sbd_points_2=24, sbd_head=9)
    kconf = dict(auto_size=False, be_points=24, sbd_points_1=24, sbd_points_2=24, sbd_head=9)
    specs = [fraq.ProblemSpec(alpha1=0.2 + 0.15 * i, alpha2=0.7 - 0.1 * i, coupling_a=1.0 - i,
                              grid_m=31, t_final=0.5, n_steps=64, initial="indicator")
             for i in range(3)]
    for scheme in ("FastBE", "FastSBD"):
        outs = fraq.run_batch(specs, getattr(fraq.Scheme, scheme), kc)
        for s, o in zip(specs, outs):
            g1, g2, _, _ = orc.run(s.alpha1, s.alpha2, s.coupling_a, 31, 0.5, 64, scheme,
                                   "indicator", kconf=kconf)
            assert rel(o.final_state.g1, g1) <= 1e-10
            assert rel(o.final_state.g2, g2) <= 1e-10


def test_modal_rejects_classical_and_observer(fraq):
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.6, grid_m=15, n_steps=8)
    with pytest.raises(ValueError):
        fraq.run(spec, fraq.Scheme.BE, modal_kc(fraq))


@pytest.mark.slow
def test_modal_c3_full_against_fp64_modespace(fraq, orc):
    """C3 (M = 4095, N = 16384, FastBE): the modal GPU solver equals the fp64 mode-space
    evaluation to ~1e-13 (the physical-space paths carry ~5e-8 rounding drift here)."""
    from workloads import c3_instance
    inst = c3_instance()
    spec = fraq.ProblemSpec(alpha1=0.4, alpha2=0.8, coupling_a=-5.5, grid_m=4095, t_final=1.0,
                            n_steps=16384, initial="custom", custom_g1=list(inst.g1),
                            custom_g2=list(inst.g2))
    rr = fraq.run(spec, fraq.Scheme.FastBE, modal_kc(fraq))
    t1, t2 = modespace_fastbe(orc, inst.g1, inst.g2, 4095, 16384, -5.5, 0.4, 0.8)
    ad = max(np.max(np.abs(np.array(rr.final_state.g1) - t1)),
             np.max(np.abs(np.array(rr.final_state.g2) - t2)))
    assert ad <= 1e-11


@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
@pytest.mark.parametrize("m,a", [(7, -3.0), (15, 2.0)])
def test_2d_matches_physical_restatement(fraq, orc, scheme, m, a):
    rng = np.random.default_rng(1901051284)
    h = 1.0 / (m + 1)
    x = (np.arange(m) + 1) * h
    X, Y = np.meshgrid(x, x)                            # row-major, x fastest
    g1 = ((X <= 0.5) & (Y <= 0.5)).astype(float).ravel()  # indicator of [0, 1/2]^2 (closed)
    g2 = (1.0 + rng.uniform(-0.1, 0.1, m * m))
    N, T = 48, 0.25
    sbd = scheme == "FastSBD"
    r1, r2 = fast_stepper_nd(orc, 0.3, 0.6, a, m, 2, T, N, sbd, g1, g2)
    out = fraq.run_2d(0.3, 0.6, a, m, T, N, getattr(fraq.Scheme, scheme), g1, g2)
    assert rel(out.final_state.g1, r1) <= 1e-10
    assert rel(out.final_state.g2, r2) <= 1e-10


@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
@pytest.mark.parametrize("m,N", [(37, 61), (255, 200), (1000, 123)])
def test_k13_tensor_core_path_matches_k11(fraq, scheme, m, N, monkeypatch):
    """K13 (DMMA block GEMMs + solver warp) against K11 (per-level warp sweep): same scheme,
    different association; ragged mode counts (not multiples of 8/16) and level counts."""
    spec = fraq.ProblemSpec(alpha1=0.35, alpha2=0.75, coupling_a=-2.5, grid_m=m, t_final=0.7,
                            n_steps=N, initial="poly_sin")
    k13 = fraq.run(spec, getattr(fraq.Scheme, scheme), modal_kc(fraq))
    monkeypatch.setenv("FRAQ_MODAL_K11", "1")
    k11 = fraq.run(spec, getattr(fraq.Scheme, scheme), modal_kc(fraq))
    assert rel(k13.final_state.g1, k11.final_state.g1) <= 1e-12
    assert rel(k13.final_state.g2, k11.final_state.g2) <= 1e-12


@pytest.mark.parametrize("scheme,pts", [("FastBE", 200), ("FastBE", 256), ("FastBE", 300),
                                        ("FastBE", 509), ("FastSBD", 100), ("FastSBD", 150),
                                        ("FastSBD", 256)])
def test_k13_warp_shapes_agree(fraq, scheme, pts, monkeypatch):
    """Every K13 CTA shape on a ragged mode count (1000) and level count (77): the default shape
    for the node count (128-node GEMM warps for J in (192, 256], 104 / 128-node warps in the
    wide CTA for J in (256, 416] / (416, 512]) against 64-node warps (FRAQ_K13_NT=8), the
    8-mode path (FRAQ_K13_NARROW, J > 256) and K11.  J = 200, 256, 300, 509 (BE) and 2 x 100,
    2 x 150, 2 x 256 (SBD families)."""
    spec = fraq.ProblemSpec(alpha1=0.35, alpha2=0.75, coupling_a=-2.5, grid_m=1000, t_final=0.7,
                            n_steps=77, initial="poly_sin")
    kc = modal_kc(fraq, auto_size=False, be_points=pts, sbd_points_1=pts, sbd_points_2=pts)
    sch = getattr(fraq.Scheme, scheme)
    runs = [fraq.run(spec, sch, kc)]
    monkeypatch.setenv("FRAQ_K13_NT", "8")
    runs.append(fraq.run(spec, sch, kc))
    monkeypatch.delenv("FRAQ_K13_NT")
    monkeypatch.setenv("FRAQ_K13_NARROW", "1")
    runs.append(fraq.run(spec, sch, kc))
    monkeypatch.setenv("FRAQ_MODAL_K11", "1")
    runs.append(fraq.run(spec, sch, kc))
    for g in ("g1", "g2"):
        ref = np.array(getattr(runs[-1].final_state, g))
        for r in runs[:-1]:
            assert rel(np.array(getattr(r.final_state, g)), ref) <= 1e-12


@pytest.mark.parametrize("scheme,pts", [("FastBE", 140), ("FastBE", 150), ("FastBE", 170),
                                        ("FastBE", 190), ("FastSBD", 70), ("FastSBD", 150),
                                        ("FastSBD", 190), ("FastBE", 256), ("FastSBD", 256)])
def test_k13_head_fold_and_mid_shapes(fraq, scheme, pts, monkeypatch):
    """The K13 head fold (modal_plan: fast-decaying nodes moved into a longer exact head) and the
    9..12-tile GEMM-warp shapes it needs, on a ragged mode count (1000) and level count (200,
    past every folded head): the default (fold up to 64 / 72 head levels), no fold (the node
    counts 140 / 150 / 170 / 190 and 2 x 150 / 2 x 190 then hit the 72 / 80 / 88 / 96-node warps
    directly), shorter and longer head caps, all against K11 on the original tables."""
    spec = fraq.ProblemSpec(alpha1=0.35, alpha2=0.75, coupling_a=-2.5, grid_m=1000,
                            t_final=200.0 / 16384, n_steps=200, initial="poly_sin")
    kc = modal_kc(fraq, auto_size=False, be_points=pts, sbd_points_1=pts, sbd_points_2=pts)
    sch = getattr(fraq.Scheme, scheme)
    runs = [fraq.run(spec, sch, kc)]
    for var, val in (("FRAQ_K13_FOLD", "0"), ("FRAQ_K13_FOLD", "16"), ("FRAQ_K13_LCAP", "40"),
                     ("FRAQ_K13_LCAP", "104")):
        monkeypatch.setenv(var, val)
        runs.append(fraq.run(spec, sch, kc))
        monkeypatch.delenv(var)
    monkeypatch.setenv("FRAQ_MODAL_K11", "1")
    ref = fraq.run(spec, sch, kc)
    for g in ("g1", "g2"):
        want = np.array(getattr(ref.final_state, g))
        for r in runs:
            assert rel(np.array(getattr(r.final_state, g)), want) <= 1e-12


def test_k13_batch_mixed_instances(fraq, orc):
    """C5-like batch through K13 with per-instance kernels (different J and L per field)."""
    from workloads import c5_instances
    insts = c5_instances(6)
    N = 80
    for scheme in ("FastBE", "FastSBD"):
        specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a,
                                  grid_m=63, t_final=N / 16384, n_steps=N, initial="custom",
                                  custom_g1=list(i.g1[::64][:63]), custom_g2=list(i.g2[::64][:63]))
                 for i in insts]
        outs = fraq.run_batch(specs, getattr(fraq.Scheme, scheme), modal_kc(fraq))
        for s, o in zip(specs, outs):
            g1, g2, _, _ = orc.run(s.alpha1, s.alpha2, s.coupling_a, 63, s.t_final, N, scheme,
                                   "custom", custom_g1=s.custom_g1, custom_g2=s.custom_g2)
            assert rel(o.final_state.g1, g1) <= 1e-10
            assert rel(o.final_state.g2, g2) <= 1e-10


# ------------------------------------------------------------------ full-size sampled-mode checks
def _sines(idx, M):
    """Rows sin((k+1)(j+1) pi/(M+1)) for k in idx, j = 0..M-1."""
    return np.sin(np.outer(np.asarray(idx) + 1, np.arange(1, M + 1)) * np.pi / (M + 1))


def _eig(M):
    h = 1.0 / (M + 1)
    return 4.0 / h ** 2 * np.sin(np.arange(1, M + 1) * np.pi * h / 2) ** 2


def _sample_modes(M, n, seed):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([[0, 1, M // 2, M - 2, M - 1], rng.integers(0, M, n)]))


@pytest.mark.slow
def test_c4_full_size_sampled_modes(fraq, orc):
    """C4 at full size (1023^2, N = 8192, FastSBD): DST coefficients of the GPU result on sampled
    (ky, kx) modes -- extremes of lambda included -- equal the mode-space restatement over the
    reference's SbdHistory lanes run on the same modes."""
    from workloads import c4_instance
    M, N = 1023, 8192
    inst = c4_instance(M)
    out = fraq.run_2d(inst.alpha1, inst.alpha2, inst.coupling_a, M, 1.0, N, fraq.Scheme.FastSBD,
                      inst.g1, inst.g2)
    ky = _sample_modes(M, 12, 7)
    kx = _sample_modes(M, 12, 8)
    Sy, Sx = _sines(ky, M), _sines(kx, M)
    sc = (2.0 / (M + 1)) ** 2

    def coef(g):
        return (sc * Sy @ np.asarray(g).reshape(M, M) @ Sx.T).ravel()  # [ky][kx]
    lam1 = _eig(M)
    lam = (lam1[ky][:, None] + lam1[kx][None, :]).ravel()
    tau = 1.0 / N
    k1 = orc.build_kernel_auto(True, 1 - inst.alpha1, tau, N)
    k2 = orc.build_kernel_auto(True, 1 - inst.alpha2, tau, N)
    c1, c2 = coef(inst.g1), coef(inst.g2)
    uN, vN, _ = orc.modal_run(k1, k2, inst.coupling_a, tau, N, lam, c1, c2, threads=8)
    s = max(np.abs(c1).max(), np.abs(c2).max())
    assert np.abs(coef(out.final_state.g1) - uN).max() <= 1e-10 * s
    assert np.abs(coef(out.final_state.g2) - vN).max() <= 1e-10 * s


@pytest.mark.slow
@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
def test_c3_full_size_sampled_modes(fraq, orc, scheme):
    """C3 (M = 4095, N = 16384) through the modal solver vs the mode-space restatement on sampled
    modes (both schemes)."""
    from workloads import c3_instance
    M, N = 4095, 16384
    inst = c3_instance(M)
    spec = fraq.ProblemSpec(alpha1=inst.alpha1, alpha2=inst.alpha2, coupling_a=inst.coupling_a,
                            grid_m=M, t_final=1.0, n_steps=N, initial="custom",
                            custom_g1=list(inst.g1), custom_g2=list(inst.g2))
    rr = fraq.run(spec, getattr(fraq.Scheme, scheme), modal_kc(fraq))
    k = _sample_modes(M, 40, 3)
    S = _sines(k, M) * (2.0 / (M + 1))
    sbd = scheme == "FastSBD"
    tau = 1.0 / N
    k1 = orc.build_kernel_auto(sbd, 1 - inst.alpha1, tau, N)
    k2 = orc.build_kernel_auto(sbd, 1 - inst.alpha2, tau, N)
    c1, c2 = S @ inst.g1, S @ inst.g2
    uN, vN, _ = orc.modal_run(k1, k2, inst.coupling_a, tau, N, _eig(M)[k], c1, c2, threads=8)
    s = max(np.abs(c1).max(), np.abs(c2).max())
    assert np.abs(S @ np.array(rr.final_state.g1) - uN).max() <= 1e-10 * s
    assert np.abs(S @ np.array(rr.final_state.g2) - vN).max() <= 1e-10 * s


@pytest.mark.slow
@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
def test_c5_batch_full_horizon_sampled(fraq, orc, scheme):
    """C5: a batch of 16 instances (full M = 4095, N = 16384) in one modal launch; two instances
    checked on sampled modes against the mode-space restatement."""
    from workloads import c5_instances
    M, N = 4095, 16384
    insts = c5_instances(16)
    specs = [fraq.ProblemSpec(alpha1=i.alpha1, alpha2=i.alpha2, coupling_a=i.coupling_a, grid_m=M,
                              t_final=1.0, n_steps=N, initial="custom", custom_g1=list(i.g1),
                              custom_g2=list(i.g2)) for i in insts]
    outs = fraq.run_batch(specs, getattr(fraq.Scheme, scheme), modal_kc(fraq))
    sbd = scheme == "FastSBD"
    tau = 1.0 / N
    k = _sample_modes(M, 24, 11)
    S = _sines(k, M) * (2.0 / (M + 1))
    for ii in (0, 13):
        inst, o = insts[ii], outs[ii]
        k1 = orc.build_kernel_auto(sbd, 1 - inst.alpha1, tau, N)
        k2 = orc.build_kernel_auto(sbd, 1 - inst.alpha2, tau, N)
        c1, c2 = S @ inst.g1, S @ inst.g2
        uN, vN, _ = orc.modal_run(k1, k2, inst.coupling_a, tau, N, _eig(M)[k], c1, c2, threads=8)
        s = max(np.abs(c1).max(), np.abs(c2).max())
        assert np.abs(S @ np.array(o.final_state.g1) - uN).max() <= 1e-10 * s
        assert np.abs(S @ np.array(o.final_state.g2) - vN).max() <= 1e-10 * s


def test_dst2d_roundtrip_and_modal_run_blocks(fraq):
    """fraq_dst2d forward/inverse against the dense sine transform, and fraq_modal_run on the
    full mode set equals run_2d (the building blocks of the mode-sharded C4 driver)."""
    M = 37
    rng = np.random.default_rng(2)
    g = rng.standard_normal(2 * M * M)
    S = np.sin(np.outer(np.arange(1, M + 1), np.arange(1, M + 1)) * np.pi / (M + 1))
    c = fraq.dst2d(M, g)
    ref = np.concatenate([((2 / (M + 1)) ** 2 * S @ gi.reshape(M, M) @ S).ravel()
                          for gi in g.reshape(2, -1)])
    assert np.abs(c - ref).max() <= 1e-13 * np.abs(ref).max()
    back = fraq.dst2d(M, c, inverse=True)
    assert np.abs(back - g).max() <= 1e-12 * np.abs(g).max()
    from paper_1901_05128_b200.parallel import eig_2d
    for scheme in ("FastBE", "FastSBD"):
        sch = getattr(fraq.Scheme, scheme)
        full = fraq.run_2d(0.3, 0.6, -3.0, M, 0.5, 64, sch, g[:M * M], g[M * M:])
        cN, rr = fraq.modal_run(0.3, 0.6, -3.0, 0.5, 64, sch, eig_2d(M), c)
        out = fraq.dst2d(M, cN, inverse=True)
        assert np.abs(out[:M * M] - np.array(full.final_state.g1)).max() <= 1e-12 * np.abs(g).max()
        assert np.abs(out[M * M:] - np.array(full.final_state.g2)).max() <= 1e-12 * np.abs(g).max()
        assert rr.loop_seconds > 0


def test_sharded_driver_single_rank_equals_run_2d(fraq):
    """parallel.run_2d_sharded with the device ops (world = 1: one slab, no gather) equals
    run_2d; the multi-rank slab/gather logic is covered on CPU (tests/test_dist.py)."""
    import torch
    from paper_1901_05128_b200.parallel import FraqOps, run_2d_sharded
    M = 63
    rng = np.random.default_rng(3)
    g1, g2 = rng.uniform(0, 1, M * M), rng.uniform(0, 1, M * M)
    ops = FraqOps(fraq, torch)
    T = {}
    r1, r2 = run_2d_sharded(ops, 0.3, 0.6, -3.0, M, 1.0, 200, "FastSBD", g1, g2,
                            scheme_arg=fraq.Scheme.FastSBD, timings=T)
    full = fraq.run_2d(0.3, 0.6, -3.0, M, 1.0, 200, fraq.Scheme.FastSBD, g1, g2)
    assert np.abs(r1.cpu().numpy() - np.array(full.final_state.g1)).max() <= 1e-12
    assert np.abs(r2.cpu().numpy() - np.array(full.final_state.g2)).max() <= 1e-12
    assert set(T) == {"forward", "step", "gather", "inverse"} and T["step"] > 0


@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
def test_transposed_driver_single_rank_equals_run_2d(fraq, scheme):
    """parallel.run_2d_transposed with the device ops (world = 1: x pass, identity exchange,
    y pass via fraq_dst_cols; K13 over all modes) equals run_2d; the multi-rank all-to-all logic
    is covered on CPU (tests/test_dist.py)."""
    import torch
    from paper_1901_05128_b200.parallel import FraqOps, run_2d_transposed
    M = 63
    rng = np.random.default_rng(4)
    g1, g2 = rng.uniform(0, 1, M * M), rng.uniform(0, 1, M * M)
    ops = FraqOps(fraq, torch)
    T = {}
    r1, r2 = run_2d_transposed(ops, 0.3, 0.6, -3.0, M, 1.0, 200, scheme, g1, g2,
                               scheme_arg=getattr(fraq.Scheme, scheme), timings=T)
    full = fraq.run_2d(0.3, 0.6, -3.0, M, 1.0, 200, getattr(fraq.Scheme, scheme), g1, g2)
    assert np.abs(r1.cpu().numpy() - np.array(full.final_state.g1)).max() <= 1e-12
    assert np.abs(r2.cpu().numpy() - np.array(full.final_state.g2)).max() <= 1e-12
    assert set(T) == {"forward", "step", "exchange", "inverse"} and T["step"] > 0


@pytest.mark.parametrize("M,C", [(1, 3), (7, 5), (63, 130), (1023, 17)])
def test_dst_cols_matches_projection(fraq, M, C):
    """fraq_dst_cols (K12 DMMA GEMM along the leading axis) against the direct sine sums, both
    directions, device pointers; forward then inverse returns the input."""
    import torch
    rng = np.random.default_rng(M + C)
    X = rng.uniform(-1, 1, (M, C))
    S = np.sin(np.outer(np.arange(1, M + 1), np.arange(1, M + 1)) * np.pi / (M + 1))
    xd = torch.tensor(X, dtype=torch.float64, device="cuda")
    fd, bd = torch.empty_like(xd), torch.empty_like(xd)
    fraq.dst_cols_device(M, C, xd.data_ptr(), fd.data_ptr(), False)
    fraq.dst_cols_device(M, C, fd.data_ptr(), bd.data_ptr(), True)
    F = fd.cpu().numpy()
    assert np.abs(F - (2.0 / (M + 1)) * S @ X).max() <= 1e-13 * max(1.0, np.abs(F).max())
    assert np.abs(bd.cpu().numpy() - X).max() <= 1e-12
