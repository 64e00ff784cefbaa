"""Multi-GPU plumbing for the sharded configurations.

The fast-CQ path has no exchange step: DOFs (C2) and instances (C5) are independent, so each rank
owns a contiguous shard and runs the single-GPU path on it.  torch.distributed (NCCL on the GPU
box, gloo in the CPU tests) is used only for a barrier, the max-over-ranks device time, and an
optional gather of per-shard checksums -- never on the data path.
"""
from __future__ import annotations

import os


def dist_env() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment (defaults: single process)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous range [lo, hi) of n units for `rank` of `world` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def c2_groups(lo: int, hi: int, n_dofs: int = 65536) -> list[tuple[int, int]]:
    """C2 has two CQ exponents: DOFs [0, n/2) use gamma 0.7, [n/2, n) gamma 0.3.  For a
    contiguous DOF block [lo, hi) returns the (group index, DOF count) pairs it spans, empty
    groups dropped -- the MultiHistory groups a rank builds."""
    half = n_dofs // 2
    counts = [max(0, min(hi, half) - lo), max(0, hi - max(lo, half))]
    return [(g, c) for g, c in enumerate(counts) if c > 0]


def c2_strong_slice(rank: int, world: int, n_dofs: int = 65536):
    """SURVEY.md §8(e) strong scaling of C2: rank r owns the contiguous DOF block
    shard(n_dofs, r, world) of the ONE 65536-DOF job (the exponent halves map to rank halves when
    world is even).  Returns (lo, hi, groups)."""
    lo, hi = shard(n_dofs, rank, world)
    return lo, hi, c2_groups(lo, hi, n_dofs)


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (the job time is the slowest rank's device time)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(value: float, device=None) -> list[float]:
    """All ranks' scalars on every rank (e.g. per-shard checksums of the results)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return [float(value)]
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]


# ----------------------------------------------------------------------------- C4: mode shards
def eig_2d(M: int):
    """lambda_k + lambda_l of the five-point Dirichlet Laplacian on the unit square, [ky][kx]
    flattened (block_solver.cpp:21-24 per axis)."""
    import numpy as np
    h = 1.0 / (M + 1)
    lam1 = 4.0 / h ** 2 * np.sin(np.arange(1, M + 1) * np.pi * h / 2) ** 2
    return (lam1[:, None] + lam1[None, :]).ravel()


def slab_rows(M: int, rank: int, world: int) -> tuple[int, int, int]:
    """ky rows [lo, hi) owned by `rank` and the padded slab height (equal on every rank, so the
    coefficient gather is a plain all-gather of equal buffers)."""
    per = -(-M // world)
    lo = min(M, rank * per)
    return lo, min(M, lo + per), per


class FraqOps:
    """Device building blocks (fraq_dst2d, fraq_modal_run) on the library's CUDA stream; tensors
    on the current GPU.  The all-gather runs on the same stream (NCCL over NVLink)."""

    def __init__(self, fraq, torch):
        self.fraq, self.torch = fraq, torch
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self.stream = torch.cuda.ExternalStream(fraq.context_stream())

    def tensor(self, x):
        return self.torch.as_tensor(x, dtype=self.torch.float64).to(self.dev).contiguous()

    def empty(self, *shape):
        return self.torch.empty(*shape, dtype=self.torch.float64, device=self.dev)

    def mark(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    @staticmethod
    def seconds(a, b):
        b.synchronize()
        return a.elapsed_time(b) * 1e-3

    def dst2d(self, M, x, inverse):
        out = self.empty(*x.shape)
        self.fraq.dst2d_device(M, x.numel() // (M * M), x.data_ptr(), out.data_ptr(), inverse)
        return out

    def dst_cols(self, M, x, inverse):
        """1D DST pass along the leading axis of x (M x C): K12 via fraq_dst_cols."""
        out = self.empty(*x.shape)
        self.fraq.dst_cols_device(M, x.numel() // M, x.data_ptr(), out.data_ptr(), inverse)
        return out

    def step(self, alpha1, alpha2, a, t_final, N, scheme, lam, c0, kconf):
        cN = self.empty(*c0.shape)
        rr = self.fraq.modal_run_device(alpha1, alpha2, a, t_final, N, scheme, lam.numel(),
                                        lam.data_ptr(), c0.data_ptr(), cN.data_ptr(),
                                        kconf if kconf is not None else self.fraq.KernelConfig())
        return cN, rr.loop_seconds


def run_2d_sharded(ops, alpha1, alpha2, a, M, t_final, N, scheme, g1_0, g2_0, kconf=None,
                   scheme_arg=None, timings=None):
    """C4 across the ranks of the default process group.  Every rank projects
    the initial data (the forward 2D DST is ~1e-3 of the stepping), steps its slab of ky rows of
    modes -- independent 2x2 recursions, no exchange -- and one all-gather of the coefficient
    slabs (2 x M^2 doubles in total) precedes the inverse DST.  g1_0 / g2_0: numpy arrays or
    tensors already on the ops' device.  Returns (g1, g2) as tensors on the ops' device.
    `scheme_arg` is what ops.step receives (the fraq.Scheme value on the GPU, the scheme name for
    the oracle ops).  If `timings` is a dict it receives the device seconds of the phases
    (forward, step -- the library's own loop timer, setup excluded --, gather, inverse)."""
    import contextlib
    import numpy as np
    import torch
    import torch.distributed as dist
    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    lo, hi, per = slab_rows(M, rank, world)
    ctx = torch.cuda.stream(ops.stream) if ops.stream is not None else contextlib.nullcontext()
    T = timings if timings is not None else {}
    with ctx:
        if isinstance(g1_0, torch.Tensor):
            g = torch.cat([g1_0.reshape(-1), g2_0.reshape(-1)]).to(torch.float64).contiguous()
        else:
            g = ops.tensor(np.concatenate([np.asarray(g1_0), np.asarray(g2_0)]))
        lam = ops.tensor(eig_2d(M)[lo * M:hi * M])
        send = ops.empty(2, per * M)
        send.zero_()
        m0 = ops.mark()
        c = ops.dst2d(M, g, inverse=False).view(2, M * M)
        m1 = ops.mark()
        T["forward"] = ops.seconds(m0, m1)
        T["step"] = 0.0
        if hi > lo:
            cN, T["step"] = ops.step(alpha1, alpha2, a, t_final, N,
                                     scheme if scheme_arg is None else scheme_arg, lam,
                                     c[:, lo * M:hi * M].contiguous(), kconf)
            send[:, :(hi - lo) * M] = cN
        m2 = ops.mark()
        if world > 1:
            recv = ops.empty(world * 2, per * M)  # concatenated along dim 0 (NCCL and gloo)
            dist.all_gather_into_tensor(recv, send)
            recv = recv.view(world, 2, per * M)
        else:
            recv = send.view(1, 2, per * M)
        full = ops.empty(2, M * M)
        for r in range(world):
            rlo, rhi, _ = slab_rows(M, r, world)
            if rhi > rlo:
                full[:, rlo * M:rhi * M] = recv[r, :, :(rhi - rlo) * M]
        m3 = ops.mark()
        out = ops.dst2d(M, full.contiguous().view(-1), inverse=True).view(2, M * M)
        m4 = ops.mark()
        T["gather"] = ops.seconds(m2, m3)
        T["inverse"] = ops.seconds(m3, m4)
    return out[0], out[1]


def _alltoall(ops, send):
    """Equal-chunk all-to-all along dim 0 (NCCL over NVLink on the GPU box; gloo in the tests)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return send
    recv = ops.empty(*send.shape)
    dist.all_to_all_single(recv, send.contiguous())
    return recv


def run_2d_transposed(ops, alpha1, alpha2, a, M, t_final, N, scheme, g1_0, g2_0, kconf=None,
                      scheme_arg=None, timings=None, gather=True):
    """C4 across the ranks of the default process group with the 2D DST split at the transpose
    (north_star "(4)"): rank r owns the physical rows y in slab r and the modes
    kx in slab r (all ky).

      forward:  x pass on its rows (fraq_dst_cols)  ->  all-to-all transpose  ->  y pass
      stepping: its kx slab of modes (fraq_modal_run, K13), no exchange
      inverse:  ky pass  ->  all-to-all transpose  ->  kx pass on its rows

    Slabs are padded to ceil(M / world) so both exchanges are equal-chunk all-to-alls
    (2 x M x per doubles per rank each).  Each rank reads only its rows of g1_0 / g2_0 and ends
    with its rows of the result; `gather=True` all-gathers them (outside the timed phases) and
    returns the full (g1, g2), else the rank's (2, rows, M) slab.  `timings` (dict) receives the
    device seconds of forward, step (the library's loop timer), exchange and inverse."""
    import contextlib
    import numpy as np
    import torch
    import torch.distributed as dist
    rank = dist.get_rank() if dist.is_initialized() else 0
    world = dist.get_world_size() if dist.is_initialized() else 1
    lo, hi, per = slab_rows(M, rank, world)
    n = hi - lo
    ctx = torch.cuda.stream(ops.stream) if ops.stream is not None else contextlib.nullcontext()
    T = timings if timings is not None else {}

    def to_cols(recv):
        # recv block q = [i (per)][f][j (per)] from rank q -> rows q*per + j, columns (f, i)
        return recv.view(world, per, 2, per).permute(0, 3, 2, 1).reshape(world * per, 2 * per)[:M]

    with ctx:
        if isinstance(g1_0, torch.Tensor):
            g = torch.stack([g1_0.reshape(M, M)[lo:hi], g2_0.reshape(M, M)[lo:hi]]).to(torch.float64)
        else:
            g = ops.tensor(np.stack([np.asarray(g1_0).reshape(M, M)[lo:hi],
                                     np.asarray(g2_0).reshape(M, M)[lo:hi]]))
        xs = ops.empty(M, 2, per)
        xs.zero_()
        xs[:, :, :n] = g.permute(2, 0, 1)                      # [x][f][y_local]
        m0 = ops.mark()
        w = ops.dst_cols(M, xs.reshape(M, 2 * per), inverse=False)  # [kx][f][y_local]
        send = ops.empty(world * per, 2, per)
        send.zero_()
        send[:M] = w.view(M, 2, per)
        m1 = ops.mark()
        recv = _alltoall(ops, send)                            # block q: [kx_local][f][y of q]
        m2 = ops.mark()
        c = ops.dst_cols(M, to_cols(recv).contiguous(), inverse=False).view(M, 2, per)  # [ky][f][kxl]
        m3 = ops.mark()
        T["forward"] = ops.seconds(m0, m1) + ops.seconds(m2, m3)
        T["exchange"] = ops.seconds(m1, m2)
        T["step"] = 0.0
        z_in = ops.empty(M, 2, per)
        z_in.zero_()
        if n > 0:
            c0 = c[:, :, :n].permute(1, 0, 2).reshape(2, M * n).contiguous()  # [f][ky * n + kxl]
            lam1 = 4.0 * (M + 1) ** 2 * np.sin(np.arange(1, M + 1) * np.pi / (2 * (M + 1))) ** 2
            lam = ops.tensor((lam1[:, None] + lam1[None, lo:hi]).ravel())
            cN, T["step"] = ops.step(alpha1, alpha2, a, t_final, N,
                                     scheme if scheme_arg is None else scheme_arg, lam, c0, kconf)
            z_in[:, :, :n] = cN.view(2, M, n).permute(1, 0, 2)
        m4 = ops.mark()
        z = ops.dst_cols(M, z_in.reshape(M, 2 * per), inverse=True)  # [y][f][kx_local]
        send2 = ops.empty(world * per, 2, per)
        send2.zero_()
        send2[:M] = z.view(M, 2, per)
        m5 = ops.mark()
        recv2 = _alltoall(ops, send2)                          # block q: [y_local][f][kx of q]
        m6 = ops.mark()
        gx = ops.dst_cols(M, to_cols(recv2).contiguous(), inverse=True).view(M, 2, per)  # [x][f][yl]
        slab = gx[:, :, :n].permute(1, 2, 0).contiguous()      # [f][y_local][x]
        m7 = ops.mark()
        T["inverse"] = ops.seconds(m4, m5) + ops.seconds(m6, m7)
        T["exchange"] += ops.seconds(m5, m6)
        if not gather:
            return slab
        if world > 1:
            pad = ops.empty(2, per, M)
            pad.zero_()
            pad[:, :n] = slab
            allp = ops.empty(world * 2, per, M)  # concatenated along dim 0 (NCCL and gloo)
            dist.all_gather_into_tensor(allp, pad)
            full = allp.view(world, 2, per, M).permute(1, 0, 2, 3).reshape(2, world * per, M)[:, :M]
        else:
            full = slab
    return full[0].reshape(-1), full[1].reshape(-1)
