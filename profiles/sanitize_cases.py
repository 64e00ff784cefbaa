"""Tiny invocations of every kernel family, each cross-checked against a second path (another
kernel, the per-level API, or a direct sum).  SURVEY.md §5 asks for compute-sanitizer runs on
small configs.  compute-sanitizer is closed on this GPU pool (runs under it have left GPUs
needing a reset), so these cases run plainly.  They exercise odd sizes and the edges of each
kernel's shape range, and the same script runs under the sanitizer where it is allowed:

    python profiles/sanitize_cases.py [case ...]
    compute-sanitizer --tool memcheck python profiles/sanitize_cases.py   # where permitted

Cases: setup (K1-K4, K7 auto sizing), k5 (per-level history, both variants), k5d (blocked,
TMA-staged), k5c (head window > 32 levels), k10 (direct CQ), host (chunked host-buffer run),
k13 (modal BE/SBD, two-CTA shape), k13w (wide CTA, J > 256), k11 (modal fallback), k6 (physical
stepper), dst2d (2D DST + K13); round 2: graph (the physical stepper's 64-level CUDA graph, K5 and
K6 on two streams), blocks (BlockSystem CR + Thomas + refinement, BandedLU, Laplacian), dsts
(the skinny DST K12s against the tile DST K12); session 5: k5e (FIR-folded blocked run against
K5d), k5f (the per-level fold against plain K5, odd sizes), fold (fold_kernel's rewritten kernel
through K5, and the physical stepper with and without folded kernels).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1901_05128_b200 as fraq  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def case_setup():
    b = fraq.KernelBudget(horizon=600, eps_tol=1e-12)
    k = fraq.build_sbd_kernel_auto(0.6, 1.0 / 600, b)
    e = fraq.KernelBudget(horizon=600, eps_tol=1e-12)
    kb = fraq.build_be_kernel_auto(0.35, 1.0 / 600, e)
    assert len(k.ratio1) > 0 and len(kb.ratios) > 0 and b.achieved_eps > 0


def case_k5():
    k = fraq.build_sbd_kernel(0.4, 0.05, 20, 20, 8)
    rng = np.random.default_rng(1)
    U = rng.uniform(-1, 1, (24, 5))
    for var in (fraq.HistoryVariant.standalone, fraq.HistoryVariant.scheme):
        h = fraq.SbdHistory(k, var, 5)
        h2 = fraq.SbdHistory(k, var, 5)
        out = []
        for n in range(24):
            h.push(list(U[n]))
            if n >= 1:
                out.append(np.array(h.derivative()))
        D = h2.run(U)
        assert rel(np.array(out), D[1:]) <= 1e-10


def _blocked(points, dim, levels):
    k = fraq.build_be_kernel(0.5, 1.0 / 4096, points)
    rng = np.random.default_rng(2)
    U = rng.uniform(-1, 1, (levels, dim))
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, dim)
    D = h.run(U)
    hs = fraq.BeHistory(k, fraq.HistoryVariant.standalone, dim)
    ref = []
    for n in range(levels):
        hs.push(list(U[n]))
        ref.append(np.array(hs.derivative()) if n >= 1 else np.full(dim, np.nan))
    assert rel(D[1:], np.array(ref[1:])) <= 1e-10
    return h.last_path


def case_k5d():
    # (K5d on the first chunks; since K5e exists the last 32-level chunk of this call is K5e's)
    assert _blocked(64, 16, 96) in (3, 4)
    os.environ["FRAQ_NO_K5E"] = "1"
    try:
        assert _blocked(64, 16, 96) == 3
    finally:
        del os.environ["FRAQ_NO_K5E"]


def case_k5c():
    k = fraq.build_sbd_kernel(0.7, 1.0 / 1024, 16, 16, 40)  # head window 40 > 32
    rng = np.random.default_rng(3)
    U = rng.uniform(-1, 1, (80, 8))
    h = fraq.SbdHistory(k, fraq.HistoryVariant.standalone, 8)
    D = h.run(U)
    hs = fraq.SbdHistory(k, fraq.HistoryVariant.standalone, 8)
    for n in range(80):
        hs.push(list(U[n]))
        if n >= 1:
            assert rel(D[n], np.array(hs.derivative())) <= 1e-10


def case_k10():
    rng = np.random.default_rng(4)
    U = rng.uniform(-1, 1, (130, 3))
    Dd = fraq.direct_cq(True, 0.4, 1.0 / 512, U)
    w = list(fraq.sbd_weights(0.4, 1.0 / 512, 129).weights)
    ref = np.array([[sum(w[i] * U[n - i, j] for i in range(n + 1)) for j in range(3)]
                    for n in range(130)])
    assert rel(Dd, ref) <= 1e-10


def case_host():
    k = fraq.build_be_kernel(0.5, 1.0 / 4096, 64)
    rng = np.random.default_rng(5)
    U = rng.uniform(-1, 1, (200, 48))
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 48)
    os.environ["FRAQ_HOST_CHUNK"] = "32"
    D = h.run(U)
    os.environ["FRAQ_HOST_CHUNK"] = ""
    h2 = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 48)
    assert rel(D[1:], h2.run(U)[1:]) <= 1e-12


def _modal(scheme, m, N, **kw):
    spec = fraq.ProblemSpec(alpha1=0.35, alpha2=0.75, coupling_a=-2.5, grid_m=m, t_final=0.7,
                            n_steps=N, initial="poly_sin")
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_MODAL
    for a, v in kw.items():
        setattr(kc, a, v)
    return fraq.run(spec, getattr(fraq.Scheme, scheme), kc), spec, kc


def case_k13():
    for sc in ("FastBE", "FastSBD"):
        r, spec, kc = _modal(sc, 37, 29)
        os.environ["FRAQ_MODAL_K11"] = "1"
        r11 = fraq.run(spec, getattr(fraq.Scheme, sc), kc)
        os.environ["FRAQ_MODAL_K11"] = ""
        assert rel(r.final_state.g1, r11.final_state.g1) <= 1e-12


def case_k13w():
    r, spec, kc = _modal("FastSBD", 40, 21, auto_size=False, be_points=64, sbd_points_1=150,
                         sbd_points_2=150)
    os.environ["FRAQ_MODAL_K11"] = "1"
    r11 = fraq.run(spec, fraq.Scheme.FastSBD, kc)
    os.environ["FRAQ_MODAL_K11"] = ""
    assert rel(r.final_state.g2, r11.final_state.g2) <= 1e-12


def case_k11():
    os.environ["FRAQ_MODAL_K11"] = "1"
    r, _, _ = _modal("FastBE", 21, 17)
    os.environ["FRAQ_MODAL_K11"] = ""
    assert np.all(np.isfinite(r.final_state.g1))


def case_k6():
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.6, coupling_a=2.0, grid_m=31, t_final=0.25,
                            n_steps=20)
    out = {}
    for solver in (fraq.SOLVER_PHYSICAL, fraq.SOLVER_MODAL):
        kc = fraq.KernelConfig()
        kc.solver = solver
        out[solver] = fraq.run(spec, fraq.Scheme.FastSBD, kc).final_state.g1
    assert rel(out[fraq.SOLVER_PHYSICAL], out[fraq.SOLVER_MODAL]) <= 1e-9


def case_dst2d():
    m = 7
    rng = np.random.default_rng(6)
    g1 = rng.uniform(0, 1, m * m)
    g2 = rng.uniform(0, 1, m * m)
    out = fraq.run_2d(0.3, 0.6, -3.0, m, 0.25, 12, fraq.Scheme.FastSBD, g1, g2)
    assert np.all(np.isfinite(out.final_state.g1))


def case_graph():
    # 2 graph replays + an eager remainder (odd grid: Thomas-free CR grid 63; and 21: Thomas)
    for m in (63, 21):
        spec = fraq.ProblemSpec(alpha1=0.35, alpha2=0.7, coupling_a=-1.5, grid_m=m,
                                t_final=0.3, n_steps=141)
        kc = fraq.KernelConfig()
        kc.solver = fraq.SOLVER_PHYSICAL
        for sch, sbd in ((fraq.Scheme.FastBE, False), (fraq.Scheme.FastSBD, True)):
            rr = fraq.run(spec, sch, kc)
            st = fraq.FastStepper(spec, sbd, fraq.KernelConfig())
            for _ in range(141):
                st.step()
            assert np.array_equal(st.state().g1, rr.final_state.g1)


def case_blocks():
    for m in (1, 3, 7, 20, 63):
        lap = fraq.DiscreteLaplacian(m, 1.0)
        rng = np.random.default_rng(m)
        x1, x2 = rng.uniform(-1, 1, m), rng.uniform(-1, 1, m)
        ax1, ax2 = np.array(lap.apply(list(x1))), np.array(lap.apply(list(x2)))
        d01, d02, a, tau, lead = 1.7, 0.4, -1.3, 0.02, 1.5
        r1 = lead / tau * x1 + d01 * (a * x1 + ax1) - a * d02 * x2
        r2 = lead / tau * x2 + d02 * (a * x2 + ax2) - a * d01 * x1
        y1, y2 = fraq.BlockSystem(d01, d02, a, tau, lap, lead).solve(list(r1), list(r2))
        assert rel(y1, x1) < 1e-12 and rel(y2, x2) < 1e-12
    lu = fraq.BandedLU(5, 1, 2)
    for i in range(5):
        lu.set(i, i, 3.0)
        if i + 1 < 5:
            lu.set(i, i + 1, 1.0)
            lu.set(i + 1, i, -1.0)
    lu.factorize()
    assert np.all(np.isfinite(lu.solve([1.0] * 5)))


def case_dsts():
    import torch
    for M, C in ((7, 1), (31, 2), (63, 8), (63, 9)):
        x = torch.randn(M, C, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        torch.cuda.synchronize()
        fraq.dst_cols_device(M, C, x.data_ptr(), y.data_ptr(), False)
        k = torch.arange(1, M + 1, dtype=torch.float64, device="cuda")
        S = torch.sin(torch.outer(k, k) * torch.pi / (M + 1))
        ref = (2.0 / (M + 1)) * S @ x
        assert float((y - ref).abs().max() / ref.abs().max()) < 1e-13


def case_k5e():
    k = fraq.build_be_kernel(0.5, 1.0 / 4096, 144)
    rng = np.random.default_rng(11)
    U = rng.uniform(-1, 1, (264, 18))
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 18)
    D = h.run(U)
    assert h.launches[4] >= 1, list(h.launches)
    os.environ["FRAQ_NO_K5E"] = "1"
    try:
        h2 = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 18)
        D2 = h2.run(U)
        assert h2.launches[4] == 0
    finally:
        del os.environ["FRAQ_NO_K5E"]
    assert rel(D[1:], D2[1:]) <= 1e-12


def case_k5f():
    k = fraq.build_sbd_kernel(0.4, 1.0 / 4096, 60, 60, 15)
    rng = np.random.default_rng(12)
    dims = [1, 3, 14, 7]
    U = rng.uniform(-1, 1, (220, sum(dims)))
    outs = []
    for no in (False, True):
        if no:
            os.environ["FRAQ_NO_K5F"] = "1"
        try:
            h = fraq.MultiHistory([k] * len(dims), dims)
            D = [np.asarray(h.run(U[i:i + 1]), dtype=float)[0] for i in range(len(U))]
            assert (h.launches[5] == 0) == no, list(h.launches)
            outs.append(np.array(D))
        finally:
            os.environ.pop("FRAQ_NO_K5F", None)
    assert rel(outs[0], outs[1]) <= 1e-12


def case_fold():
    k = fraq.build_be_kernel(0.6, 1.0 / 4096, 96)
    kf, M = fraq.fold_kernel(k, 64)
    assert M > 0
    rng = np.random.default_rng(13)
    U = rng.uniform(-1, 1, (150, 9))
    h = fraq.BeHistory(k, fraq.HistoryVariant.standalone, 9)
    hf = fraq.SbdHistory(kf, fraq.HistoryVariant.standalone, 9)
    D, Df = h.run(U), hf.run(U)
    assert rel(Df[1:], D[1:]) <= 1e-12
    spec = fraq.ProblemSpec(alpha1=0.3, alpha2=0.6, coupling_a=2.0, grid_m=31, t_final=0.125,
                            n_steps=128)
    kc = fraq.KernelConfig()
    kc.solver = fraq.SOLVER_PHYSICAL
    res = []
    for no in (False, True):
        if no:
            os.environ["FRAQ_NO_PHYS_FOLD"] = "1"
        try:
            for sch in (fraq.Scheme.FastBE, fraq.Scheme.FastSBD):
                rr = fraq.run(spec, sch, kc)
                res.append(np.concatenate([rr.final_state.g1, rr.final_state.g2]))
        finally:
            os.environ.pop("FRAQ_NO_PHYS_FOLD", None)
    assert rel(res[0], res[2]) <= 1e-11 and rel(res[1], res[3]) <= 1e-11


CASES = {n[5:]: f for n, f in globals().items() if n.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print("ok", n, flush=True)
    fraq.synchronize()
