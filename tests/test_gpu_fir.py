"""GPU parity of K5e (history_fir.cu): the blocked history evaluation with the fast-decaying
nodes folded into an exact FIR, against the CPU oracle (the reference compiled from its own
sources when present) and against K5d on the same inputs.

K5e takes over a blocked run once the history is past its first levels (path 4); K5d (path 3)
runs the first levels and ragged tails, and the per-level kernel K5 the single pushes.  The
short-node states K5e skips are rebuilt before any of those reads them, so every mix of the
three paths must equal the reference's push/derivative sequence (fast_kernel.cpp:261-409).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def kernel_from_oracle(fraq, k):
    if k.sbd:
        return fraq.make_sbd_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1),
                                    list(k.m2), list(k.r2))
    return fraq.make_be_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1))


def make(fraq, o, variant, dim):
    k = kernel_from_oracle(fraq, o)
    cls = fraq.SbdHistory if o.sbd else fraq.BeHistory
    return cls(k, getattr(fraq.HistoryVariant, variant), dim)


def check(D, D_ref, scale, tol):
    D, D_ref = np.asarray(D, dtype=float), np.asarray(D_ref, dtype=float)
    assert np.array_equal(np.isnan(D), np.isnan(D_ref))
    ok = ~np.isnan(D_ref)
    err = np.max(np.abs(D[ok] - D_ref[ok]) / np.maximum(np.abs(D_ref[ok]), scale))
    assert err <= tol, err


C2_TAU = 1.0 / 65536


@pytest.fixture(scope="module")
def c2_kernels(orc):
    # the C2 tables: the reference's auto-sized 256 + 256 nodes, heads 17 / 15
    return [orc.build_kernel_auto(True, g, C2_TAU, 65536, 1e-12) for g in (0.7, 0.3)]


@pytest.mark.parametrize("variant", ["standalone", "scheme"])
def test_k5e_c2_tables_match_reference(fraq, orc, c2_kernels, variant):
    """C2's kernels, 40 + 24 DOFs, 720 levels in one call: K5d on the first levels, K5e on the
    rest; every level equals the reference history to 1e-12 of the output scale."""
    rng = np.random.default_rng(41)
    dims = [40, 24]
    n = 720
    U = rng.uniform(-1, 1, (n, sum(dims)))
    ks = [kernel_from_oracle(fraq, o) for o in c2_kernels]
    sch = variant == "scheme"
    ref = np.concatenate([orc.hist_run(c2_kernels[0], U[:, :40], sch),
                          orc.hist_run(c2_kernels[1], U[:, 40:], sch)], axis=1)
    h = fraq.MultiHistory(ks, dims) if not sch else None
    if sch:
        # (MultiHistory is the standalone variant; the scheme variant through SbdHistory)
        for c0, c1, o in ((0, 40, c2_kernels[0]), (40, 64, c2_kernels[1])):
            hh = make(fraq, o, variant, c1 - c0)
            D = hh.run(np.ascontiguousarray(U[:, c0:c1]))
            assert hh.last_path == 4
            check(D, ref[:, c0:c1], C2_TAU ** -o.gamma, 1e-12)
        return
    D = h.run(U)
    assert h.last_path == 4
    check(D[:, :40], ref[:, :40], C2_TAU ** -0.7, 1e-12)
    check(D[:, 40:], ref[:, 40:], C2_TAU ** -0.3, 1e-12)


def test_k5e_equals_k5d(fraq, orc, c2_kernels, monkeypatch):
    """The same calls with K5e switched off (FRAQ_NO_K5E: everything on K5d): the two blocked
    forms agree to a few ulps of the output scale, and so do the states they leave behind
    (one further per-level push + derivative after the runs reads every node's state)."""
    rng = np.random.default_rng(43)
    o = c2_kernels[0]
    dim, n = 32, 512
    U = rng.uniform(-1, 1, (n + 1, dim))
    outs, paths = [], []
    for off in (False, True):
        if off:
            monkeypatch.setenv("FRAQ_NO_K5E", "1")
        else:
            monkeypatch.delenv("FRAQ_NO_K5E", raising=False)
        h = make(fraq, o, "standalone", dim)
        D = np.concatenate([h.run(U[:256]), h.run(U[256:n])])
        paths.append(h.last_path)
        h.push(list(U[n]))
        D = np.concatenate([D, np.array(h.derivative())[None, :]])
        outs.append(D)
    assert paths == [4, 3]
    scale = C2_TAU ** -o.gamma
    assert np.max(np.abs(outs[0] - outs[1])) <= 2e-14 * scale * 4


@pytest.mark.parametrize("sbd", [False, True])
def test_k5e_mixed_with_pushes_and_ragged_calls(fraq, orc, sbd):
    """Blocked runs of ragged lengths (K5e on the 8-level blocks, K5d on the remainders)
    interleaved with single pushes (K5, which needs the short states rebuilt and keeps the
    input ring current): the whole sequence equals the reference history."""
    rng = np.random.default_rng(47 + sbd)
    tau = 1.0 / 16384
    o = orc.build_kernel_auto(sbd, 0.6, tau, 16384, 1e-12)
    dim = 24
    n = 900
    U = rng.uniform(-1, 1, (n, dim))
    ref = orc.hist_run(o, U)
    h = make(fraq, o, "standalone", dim)
    out = []
    pos = 0
    seen = set()
    for ln in (200, -3, 136, 77, -2, 64, 203, -1, 214):
        if ln < 0:
            for _ in range(-ln):
                h.push(list(U[pos]))
                out.append(np.array(h.derivative())[None, :])
                pos += 1
        else:
            out.append(np.asarray(h.run(U[pos:pos + ln]), dtype=float))
            seen.add(h.last_path)
            pos += ln
    assert pos == n
    assert 4 in seen
    check(np.concatenate(out), ref, tau ** -0.6, 1e-12)


def test_k5e_small_kernels_and_ragged_groups(fraq, orc):
    """Groups of ragged sizes with small kernels (some with no short node at all, some with no
    long tile per warp): tasks straddle no group boundary and every group equals its own
    reference history.  The same with odd group starts, which TMA cannot address (boxes must
    start 16-byte aligned): those histories stay on K5d's register-staged path."""
    rng = np.random.default_rng(53)
    dims = [2, 4, 16, 18, 34, 6]  # (even group starts: K5e stages its inputs by TMA)
    taus = [1e-3, 1e-4, 1e-5, 1e-3, 1e-5, 1e-4]
    os_ = [orc.build_be_kernel(0.25 + 0.1 * i, taus[i], 24 + 37 * i) for i in range(len(dims))]
    ks = [kernel_from_oracle(fraq, o) for o in os_]
    h = fraq.MultiHistory(ks, dims)
    n = 480
    U = rng.uniform(-1, 1, (n, sum(dims)))
    D = np.concatenate([np.asarray(h.run(U[:200]), dtype=float),
                        np.asarray(h.run(U[200:]), dtype=float)])
    assert h.last_path == 4
    c = 0
    for o, dm, tau in zip(os_, dims, taus):
        D_ref = orc.hist_run(o, np.ascontiguousarray(U[:, c:c + dm]))
        check(D[:, c:c + dm], D_ref, tau ** -o.gamma, 1e-12)
        c += dm
    odd = [1, 3, 16, 17, 33, 6]  # total 76 (even leading dimension), odd group starts
    h = fraq.MultiHistory(ks, odd)
    D = np.asarray(h.run(U[:, :sum(odd)]), dtype=float)
    assert h.last_path == 3
    c = 0
    for o, dm, tau in zip(os_, odd, taus):
        D_ref = orc.hist_run(o, np.ascontiguousarray(U[:, c:c + dm]))
        check(D[:, c:c + dm], D_ref, tau ** -o.gamma, 1e-12)
        c += dm


def test_k5e_long_run_device(fraq, orc, c2_kernels):
    """run_device (device buffers, torch) in 256-level calls over 2048 levels, compared on the
    last levels with the reference history: no drift between the FIR form and the recurrences."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(59)
    o = c2_kernels[1]
    dim, n = 32, 2048
    U = rng.uniform(-1, 1, (n, dim))
    ref = orc.hist_run(o, U)
    k = kernel_from_oracle(fraq, o)
    h = fraq.MultiHistory([k], [dim])
    Ud = torch.from_numpy(U).cuda()
    Dd = torch.empty_like(Ud)
    for s in range(0, n, 256):
        h.run_device(Ud.data_ptr() + s * dim * 8, dim, 256, Dd.data_ptr() + s * dim * 8, dim)
    fraq.synchronize()
    assert h.last_path == 4
    check(Dd.cpu().numpy(), ref, C2_TAU ** -0.3, 1e-12)


def test_k5e_padded_rows_and_no_output(fraq, orc, c2_kernels):
    """run_device with leading dimensions above the DOF count (rows of a wider device array)
    and a null output pointer on part of the sequence (state only, as a solver that needs no
    derivative there would call it): the levels that are written equal the reference history."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(61)
    o = c2_kernels[0]
    dim, ld, n = 48, 80, 1024
    U = rng.uniform(-1, 1, (n, dim))
    ref = orc.hist_run(o, U)
    k = kernel_from_oracle(fraq, o)
    h = fraq.MultiHistory([k], [dim])
    Ud = torch.zeros((n, ld), dtype=torch.float64, device="cuda")
    Ud[:, :dim] = torch.from_numpy(U).cuda()
    Dd = torch.full((n, ld), -7.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    row = ld * 8
    h.run_device(Ud.data_ptr(), ld, 256, Dd.data_ptr(), ld)
    h.run_device(Ud.data_ptr() + 256 * row, ld, 384, 0, ld)           # no output
    h.run_device(Ud.data_ptr() + 640 * row, ld, 384, Dd.data_ptr() + 640 * row, ld)
    fraq.synchronize()
    assert h.last_path == 4 and h.launches[4] == 3
    D = Dd.cpu().numpy()
    assert np.all(D[:, dim:] == -7.0) and np.all(D[256:640, :dim] == -7.0)
    scale = C2_TAU ** -o.gamma
    check(D[:256, :dim], ref[:256], scale, 1e-12)
    check(D[640:, :dim], ref[640:], scale, 1e-12)


# ------------------------------------------------------------------------------------- K5f
# The per-level step in K5e's folded form (history_fir.cu step_fir_kernel): push / derivative /
# history_sum of a pure push sequence past the first levels.  launches[5] counts its launches.

@pytest.mark.parametrize("sbd,variant", [(False, "standalone"), (True, "standalone"),
                                         (True, "scheme"), (False, "scheme")])
def test_k5f_pure_push_sequence(fraq, orc, sbd, variant):
    """push + derivative level by level from a fresh history (the reference's own calling
    pattern, fast_kernel.cpp:291-300, 317-325, 366-376, 397-409): K5 on the first levels (which
    also records the inputs), K5f from the level its window is on record, equal to the reference
    history throughout."""
    rng = np.random.default_rng(71 + 2 * sbd + (variant == "scheme"))
    tau = 1.0 / 16384
    o = orc.build_kernel_auto(sbd, 0.45, tau, 16384, 1e-12)
    dim, n = 22, 260
    U = rng.uniform(-1, 1, (n, dim))
    if variant == "scheme":
        U[0] = 0.0  # (scheme histories start from the initial value G^0 = 0 convention of the tests)
    ref = orc.hist_run(o, U, scheme_variant=variant == "scheme")
    h = make(fraq, o, variant, dim)
    out = np.full((n, dim), np.nan)
    for i in range(n):
        h.push(list(U[i]))
        if sbd or i >= 1:
            out[i] = h.derivative()
    lz = list(h.launches)
    assert lz[5] > 100 and lz[0] > 20
    check(out, ref, tau ** -0.45, 1e-12)


def test_k5f_mixed_with_runs_and_read_only_outputs(fraq, orc, c2_kernels, monkeypatch):
    """Blocked runs (K5d / K5e) interleaved with single pushes on K5f, history_sum and repeated
    derivative reads without a new push (read-only K5f), lagged values, and a separate
    advance() / append() pair (K5, after the short states were rebuilt): the same sequence with
    FRAQ_NO_K5F=1 (K5 for every per-level call) gives the same numbers, and both equal the
    reference history."""
    rng = np.random.default_rng(83)
    o = c2_kernels[0]
    dim, n = 20, 700
    U = rng.uniform(-1, 1, (n, dim))
    ref = orc.hist_run(o, U)

    def sequence():
        h = make(fraq, o, "standalone", dim)
        D = np.full((n, dim), np.nan)
        sums, lag = [], []
        pos = 0
        for ln in (208, -40, 136, -3, 99, -60, 154):
            if ln > 0:
                D[pos:pos + ln] = np.asarray(h.run(U[pos:pos + ln]), dtype=float)
                pos += ln
                continue
            for q in range(-ln):
                if q == 5:
                    # the reference's split calls (fast_kernel.cpp:268-289, 343-365)
                    h.advance()
                    h.append(list(U[pos]))
                else:
                    h.push(list(U[pos]))
                if q % 4 == 1:
                    sums.append(np.array(h.history_sum()))
                D[pos] = h.derivative()
                if q % 7 == 2:
                    assert np.array_equal(np.array(h.derivative()), D[pos])  # read-only repeat
                    lag.append(np.array(h.lagged(3)))
                pos += 1
        assert pos == n
        return h, D, np.array(sums), np.array(lag)

    h1, D1, s1, l1 = sequence()
    assert h1.launches[5] > 60
    monkeypatch.setenv("FRAQ_NO_K5F", "1")
    h2, D2, s2, l2 = sequence()
    assert h2.launches[5] == 0
    scale = C2_TAU ** -o.gamma
    check(D1, ref, scale, 1e-12)
    check(D2, ref, scale, 1e-12)
    assert np.max(np.abs(s1 - s2)) <= 1e-12 * scale
    assert np.array_equal(l1, l2)


def test_k5f_ragged_groups_odd_starts(fraq, orc):
    """Groups of ragged sizes with odd first DOFs (rows K5e cannot stage by TMA): the per-level
    fold has no alignment precondition; every group equals its own reference history."""
    rng = np.random.default_rng(89)
    dims = [1, 3, 16, 17, 33, 6]
    taus = [1e-3, 1e-4, 1e-5, 1e-3, 1e-5, 1e-4]
    os_ = [orc.build_be_kernel(0.25 + 0.1 * i, taus[i], 24 + 37 * i) for i in range(len(dims))]
    ks = [kernel_from_oracle(fraq, o) for o in os_]
    h = fraq.MultiHistory(ks, dims)
    n = 300
    U = rng.uniform(-1, 1, (n, sum(dims)))
    D = np.full((n, sum(dims)), np.nan)
    D[:160] = np.asarray(h.run(U[:160]), dtype=float)
    for i in range(160, n):
        D[i] = np.asarray(h.run(U[i:i + 1]), dtype=float)[0]  # one-level calls
    assert h.launches[5] == n - 160
    c = 0
    for o, dm, tau in zip(os_, dims, taus):
        D_ref = orc.hist_run(o, np.ascontiguousarray(U[:, c:c + dm]))
        check(D[:, c:c + dm], D_ref, tau ** -o.gamma, 1e-12)
        c += dm


@pytest.mark.parametrize("sbd,max_head", [(False, 96), (True, 96), (True, 64), (False, 40)])
def test_folded_kernel_history_equals_reference(fraq, orc, sbd, max_head, monkeypatch):
    """fraq_fold_kernel's rewrite (longer exact head, only the slow nodes; the kernels the
    physical FFPE stepper hands to its K5 pass) driven through the plain history kernels: an
    SbdHistory over the folded kernel reproduces the reference history of the ORIGINAL kernel,
    level by level (K5) and in one blocked run."""
    monkeypatch.setenv("FRAQ_NO_K5F", "1")  # plain K5: every node of the folded kernel streamed
    rng = np.random.default_rng(97 + sbd)
    tau = 1.0 / 16384
    o = orc.build_kernel_auto(sbd, 0.6, tau, 16384, 1e-12)
    folded, M = fraq.fold_kernel(kernel_from_oracle(fraq, o), max_head)
    assert M > 0
    dim, n = 10, 320
    U = rng.uniform(-1, 1, (n, dim))
    ref = orc.hist_run(o, U)
    h = fraq.SbdHistory(folded, fraq.HistoryVariant.standalone, dim)
    out = np.full((n, dim), np.nan)
    for i in range(n):
        h.push(list(U[i]))
        out[i] = h.derivative()
    first = 0 if sbd else 1  # (the reference's BE derivative needs two pushed values)
    check(out[first:], ref[first:], tau ** -0.6, 1e-12)
    h2 = fraq.SbdHistory(folded, fraq.HistoryVariant.standalone, dim)
    D = np.asarray(h2.run(U), dtype=float)
    check(D[first:], ref[first:], tau ** -0.6, 1e-12)


def test_k5f_padded_rows_and_guard_bands(fraq, orc, c2_kernels):
    """One-level run_device calls (K5f) on rows of wider device arrays, odd DOF count: the
    padding columns and the rows around the call stay untouched, the written levels equal the
    reference history."""
    torch = pytest.importorskip("torch")
    rng = np.random.default_rng(103)
    o = c2_kernels[1]
    dim, ld, n = 37, 64, 200
    U = rng.uniform(-1, 1, (n, dim))
    ref = orc.hist_run(o, U)
    k = kernel_from_oracle(fraq, o)
    h = fraq.MultiHistory([k], [dim])
    Ud = torch.full((n, ld), 3.0, dtype=torch.float64, device="cuda")
    Ud[:, :dim] = torch.from_numpy(U).cuda()
    Dd = torch.full((n + 2, ld), -7.0, dtype=torch.float64, device="cuda")  # guard rows 0, n + 1
    torch.cuda.synchronize()
    row = ld * 8
    h.run_device(Ud.data_ptr(), ld, 128, Dd.data_ptr() + row, ld)
    for i in range(128, n):
        h.run_device(Ud.data_ptr() + i * row, ld, 1, Dd.data_ptr() + (i + 1) * row, ld)
    fraq.synchronize()
    assert h.launches[5] == n - 128
    D = Dd.cpu().numpy()
    assert np.all(D[0] == -7.0) and np.all(D[n + 1] == -7.0) and np.all(D[:, dim:] == -7.0)
    assert np.all(Ud.cpu().numpy()[:, dim:] == 3.0)
    check(D[1:n + 1, :dim], ref, C2_TAU ** -o.gamma, 1e-12)
