"""The identity behind K5e (history_fir.cu) and the K13 head fold (modal.cu), checked on the CPU
against the reference's own kernels (oracle): folding the fast-decaying nodes into the head does
not change the convolution weights the compressed kernel stands for.

A fast kernel (fast_kernel.cpp:54-124) with head d_0..d_(L-1) and nodes (r_j, f_j) fed at lag L
represents the weights  w_i = d_i (i < L),  w_i = sum_j f_j r_j^(i-L) (i >= L)
(fast_kernel.cpp:38-52, reconstruct).  With S = {j : |r_j|^M <= 2^-70}:

  head'  c_i = d_i (i < L),  c_i = sum_{all j} f_j r_j^(i-L)  (L <= i < L + M)
  nodes' (r_j, f_j r_j^M) for j not in S, fed at lag L + M

represent  w'_i = w_i  for i < L + M  and  w'_i = w_i - sum_{j in S} f_j r_j^(i-L)  beyond, and
the dropped sum is below 2^-70 sum_S |f_j|.
"""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def orc():
    from oracle.oracle import Oracle, ref_available
    return Oracle("reference" if ref_available() else "port")


def weights(head, r, f, L, n):
    w = np.zeros(n, dtype=np.longdouble)
    w[:L] = head[:L]
    p = f.astype(np.longdouble).copy()
    rl = r.astype(np.longdouble)
    for i in range(L, n):
        w[i] = p.sum()
        p *= rl
    return w


@pytest.mark.parametrize("sbd,g,tau,M", [(True, 0.7, 1.0 / 65536, 48), (True, 0.3, 1.0 / 65536, 48),
                                          (True, 0.55, 1.0 / 16384, 24), (False, 0.5, 1.0 / 16384, 56),
                                          (False, 0.9, 1.0 / 16384, 40)])
def test_fold_preserves_weights(orc, sbd, g, tau, M):
    k = orc.build_kernel_auto(sbd, g, tau, int(round(1 / tau)), 1e-12)
    r = np.concatenate([k.r1, k.r2])
    m = np.concatenate([k.m1, k.m2])
    L = k.n_head if sbd else 2
    # feeds: BE node weights; SBD mult * ratio^(n_head - 3) (fast_kernel.cpp:337-340)
    f = m * r ** (k.n_head - 3) if sbd else m
    n = 4096
    w = weights(np.asarray(k.head), r, f, L, n)
    short = np.abs(r.astype(np.longdouble)) ** M <= np.longdouble(2.0) ** -70
    assert short.sum() >= 0.3 * len(r)  # the fold is worth something on the reference's tables
    rl, fl = r.astype(np.longdouble), f.astype(np.longdouble)
    head2 = np.zeros(L + M, dtype=np.longdouble)
    head2[:L] = np.asarray(k.head)[:L]
    p = fl.copy()
    for i in range(M):
        head2[L + i] = p.sum()
        p *= rl
    r2 = r[~short]
    f2 = (fl[~short] * rl[~short] ** M).astype(np.float64)
    w2 = weights(head2.astype(np.float64), r2, f2, L + M, n)
    scale = abs(float(k.head[0]))
    assert float(np.max(np.abs(w2 - w))) <= 1e-15 * scale
    # what is dropped: bounded by 2^-70 sum |f_j| / (1 - |r_j|) over the folded nodes
    bound = float(np.sum(np.abs(fl[short]) * np.abs(rl[short]) ** M / (1 - np.abs(rl[short]))))
    assert bound <= 2.0 ** -60 * scale


def test_fold_sbd_is_a_kernel_rewrite(orc):
    """For the SBD families the folded kernel is again a reference-format kernel: the feed
    convention mult * ratio^(n_head - 3) absorbs r^M when n_head grows by M, so the node tables
    of the kept nodes are unchanged."""
    k = orc.build_kernel_auto(True, 0.7, 1.0 / 65536, 65536, 1e-12)
    r = np.concatenate([k.r1, k.r2])
    m = np.concatenate([k.m1, k.m2])
    M = 48
    keep = np.abs(r) ** M > 2.0 ** -70
    f_fold = (m * r ** (k.n_head - 3))[keep] * r[keep] ** M
    f_rewritten = m[keep] * r[keep] ** (k.n_head + M - 3)
    assert np.max(np.abs(f_fold - f_rewritten) / np.abs(f_rewritten)) <= 1e-13


# ---------------------------------------------------------------------------- fraq_fold_kernel
# The product's own rewrite (history_fir.cu fold_kernel, C ABI fraq_fold_kernel; host only), on
# the reference's kernels: the folded kernel is a reference-format SBD kernel that stands for the
# same convolution weights.

def _pkg_kernel(fraq, k):
    if k.sbd:
        return fraq.make_sbd_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1),
                                    list(k.m2), list(k.r2))
    return fraq.make_be_kernel(k.gamma, k.tau, list(k.head), list(k.m1), list(k.r1))


@pytest.mark.parametrize("sbd,g,tau", [(True, 0.7, 1.0 / 65536), (True, 0.3, 1.0 / 65536),
                                       (False, 0.6, 1.0 / 16384), (False, 0.2, 1.0 / 16384),
                                       (True, 0.45, 1.0 / 16384), (False, 0.9, 1.0 / 16384)])
def test_fold_kernel_abi_preserves_weights(orc, sbd, g, tau):
    import paper_1901_05128_b200 as fraq
    k = orc.build_kernel_auto(sbd, g, tau, int(round(1 / tau)), 1e-12)
    folded, M = fraq.fold_kernel(_pkg_kernel(fraq, k), 96)
    L = k.n_head if sbd else 2
    assert M > 0 and M % 8 == 0 and folded.n_head == L + M <= 96
    r = np.concatenate([k.r1, k.r2])
    m = np.concatenate([k.m1, k.m2])
    f = m * r ** (k.n_head - 3) if sbd else m
    n = 4096
    w = weights(np.asarray(k.head), r, f, L, n)
    r2 = np.concatenate([folded.ratio1, folded.ratio2])
    m2 = np.concatenate([folded.mult1, folded.mult2])
    assert 0 < len(r2) < len(r)
    assert set(r2.tolist()) <= set(r.tolist())  # kept nodes keep their ratios
    if sbd:
        assert set(m2.tolist()) <= set(m.tolist())  # ... and, for SBD families, their multipliers
    f2 = m2 * r2 ** (folded.n_head - 3)  # the reference's feed convention, fast_kernel.cpp:337-340
    w2 = weights(np.asarray(folded.head), r2, f2, folded.n_head, n)
    scale = abs(float(k.head[0]))
    assert float(np.max(np.abs(w2 - w))) <= 2e-15 * scale
    # the bytes a per-level pass moves (16 per node state, 8 per head tap) went down
    assert 16 * len(r2) + 8 * folded.n_head < 16 * len(r) + 8 * L
    # a head cap below L + 8 leaves the kernel alone (returned in the generic-head format)
    same, M0 = fraq.fold_kernel(_pkg_kernel(fraq, k), L + 7)
    assert M0 == 0 and same.n_head == L and len(same.ratio1) + len(same.ratio2) == len(r)
    f0 = np.concatenate([same.mult1, same.mult2]) * \
        np.concatenate([same.ratio1, same.ratio2]) ** (same.n_head - 3)
    assert np.max(np.abs(f0 - f) / np.abs(f)) <= 4e-16


@pytest.mark.parametrize("sbd,g", [(False, 0.6), (True, 0.7)])
def test_reference_history_on_the_folded_kernel(orc, sbd, g):
    """The rewrite is an algorithmic identity, not a property of the CUDA kernels: the
    REFERENCE's own SbdHistory (fast_kernel.cpp:327-409), built from the folded kernel, reproduces
    the reference history of the original kernel while carrying a fraction of the node states."""
    import paper_1901_05128_b200 as fraq
    from oracle.oracle import Kernel
    tau = 1.0 / 16384
    k = orc.build_kernel_auto(sbd, g, tau, 16384, 1e-12)
    folded, M = fraq.fold_kernel(_pkg_kernel(fraq, k), 96)
    assert M > 0
    kf = Kernel(True, k.gamma, k.tau, np.array(folded.head), np.array(folded.mult1),
                np.array(folded.ratio1), np.array(folded.mult2), np.array(folded.ratio2))
    assert kf.np1 + kf.np2 <= 0.75 * (k.np1 + k.np2)
    rng = np.random.default_rng(101 + sbd)
    U = rng.uniform(-1, 1, (600, 6))
    ref = orc.hist_run(k, U)
    got = orc.hist_run(kf, U)
    first = 0 if sbd else 1  # (BeHistory::derivative needs two pushed values)
    scale = tau ** -g
    err = np.max(np.abs(got[first:] - ref[first:]) / np.maximum(np.abs(ref[first:]), scale))
    assert err <= 1e-13, err
