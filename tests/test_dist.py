"""Multi-rank host logic on CPU (gloo, world_size 2): DOF / instance sharding, max-over-ranks
timing, checksum gathers.  Each rank evaluates its shard with the CPU oracle (the GPU kernels run
the identical per-shard computation on the box); the concatenated shards must equal the
single-process result, which is what makes the weak/strong scaling runs exact."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1901_05128_b200.parallel import shard


def test_shard_partitions():
    for n in (0, 1, 7, 65536, 4096):
        for world in (1, 2, 3, 8):
            ranges = [shard(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_1901_05128_b200.parallel import gather_scalars, max_over_ranks
    orc = Oracle("port")
    k = orc.build_sbd_kernel(0.6, 1e-3, 24, 24, 12)
    rng = np.random.default_rng(1234)
    U = rng.uniform(-1, 1, (120, 10))
    lo, hi = shard(U.shape[1], rank, world)
    D = orc.hist_run(k, U[:, lo:hi])
    t = max_over_ranks(float(rank + 1))
    sums = gather_scalars(float(np.nansum(D)))
    dist.barrier()
    q.put((rank, lo, hi, D, t, sums))
    dist.destroy_process_group()


def test_two_rank_shards_match_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from oracle.oracle import Oracle
    orc = Oracle("port")
    k = orc.build_sbd_kernel(0.6, 1e-3, 24, 24, 12)
    rng = np.random.default_rng(1234)
    U = rng.uniform(-1, 1, (120, 10))
    full = orc.hist_run(k, U)
    stitched = np.concatenate([r[3] for r in res], axis=1)
    assert np.array_equal(stitched, full)  # lanes are independent: bitwise
    assert all(r[4] == 2.0 for r in res)   # max over ranks
    assert res[0][5] == res[1][5] and len(res[0][5]) == 2


def _worker_2d(rank, world, port, q, scheme):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from oracle_ops import OracleOps
    from paper_1901_05128_b200.parallel import run_2d_sharded
    g1, g2 = _c4_like(9)
    ops = OracleOps(Oracle("port"), torch)
    try:
        r1, r2 = run_2d_sharded(ops, 0.3, 0.6, -3.0, 9, 0.25, 40, scheme, g1, g2)
        q.put((rank, r1.numpy(), r2.numpy()))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None))
    dist.destroy_process_group()


def _c4_like(M):
    h = 1.0 / (M + 1)
    x = (np.arange(M) + 1) * h
    X, Y = np.meshgrid(x, x)
    g1 = ((X <= 0.5) & (Y <= 0.5)).astype(float).ravel()
    g2 = 1.0 + np.random.default_rng(1901051284).uniform(-0.1, 0.1, M * M)
    return g1, g2


@pytest.mark.parametrize("scheme", ["FastBE", "FastSBD"])
def test_c4_mode_shards_two_ranks(scheme):
    """C4's mode-sharded driver (parallel.run_2d_sharded) on 2 gloo ranks: odd row split (9 rows ->
    5 + 4, padded slabs), one all-gather of the coefficient slabs; every rank's result equals the
    single-process run of the same driver and the physical-space 2D restatement to 1e-10."""
    import torch
    from oracle.oracle import Oracle
    from oracle_ops import OracleOps
    from paper_1901_05128_b200.parallel import run_2d_sharded
    from ffpe_refs import fast_stepper_nd
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d, args=(r, 2, port, q, scheme)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[2] is not None for r in res), res
    g1, g2 = _c4_like(9)
    orc = Oracle("port")
    s1, s2 = run_2d_sharded(OracleOps(orc, torch), 0.3, 0.6, -3.0, 9, 0.25, 40, scheme, g1, g2)
    p1, p2 = fast_stepper_nd(orc, 0.3, 0.6, -3.0, 9, 2, 0.25, 40, scheme == "FastSBD", g1, g2)
    for _, r1, r2 in res:
        assert np.abs(r1 - s1.numpy()).max() <= 1e-14 * np.abs(s1.numpy()).max()
        assert np.abs(r2 - s2.numpy()).max() <= 1e-14 * np.abs(s2.numpy()).max()
        assert np.abs(r1 - p1).max() <= 1e-10 * np.abs(p1).max()
        assert np.abs(r2 - p2).max() <= 1e-10 * np.abs(p2).max()


def _worker_2d_t(rank, world, port, q, scheme):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from oracle_ops import OracleOps
    from paper_1901_05128_b200.parallel import run_2d_transposed
    g1, g2 = _c4_like(9)
    ops = OracleOps(Oracle("port"), torch)
    try:
        T = {}
        r1, r2 = run_2d_transposed(ops, 0.3, 0.6, -3.0, 9, 0.25, 40, scheme, g1, g2, timings=T)
        slab = run_2d_transposed(ops, 0.3, 0.6, -3.0, 9, 0.25, 40, scheme, g1, g2, gather=False)
        q.put((rank, r1.numpy(), r2.numpy(), slab.numpy(), sorted(T)))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e), None, None, None))
    dist.destroy_process_group()


@pytest.mark.parametrize("scheme,world", [("FastBE", 2), ("FastSBD", 3)])
def test_c4_transposed_dst_ranks(scheme, world):
    """C4 with the 2D DST split at the transpose (parallel.run_2d_transposed) on gloo ranks: x pass
    on each rank's rows, equal-chunk all-to-all, y pass, K13 over the rank's kx slab, and the
    mirror image for the inverse.  9 rows over 2 ranks (5 + 4, padded) and 3 ranks (3 + 3 + 3):
    every rank's gathered result equals the single-process run of the all-gather driver and the
    physical-space 2D restatement, and each rank's slab is its rows of the result."""
    import torch
    from oracle.oracle import Oracle
    from oracle_ops import OracleOps
    from paper_1901_05128_b200.parallel import run_2d_sharded, slab_rows
    from ffpe_refs import fast_stepper_nd
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_2d_t, args=(r, world, port, q, scheme))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[2] is not None for r in res), res
    g1, g2 = _c4_like(9)
    orc = Oracle("port")
    s1, s2 = run_2d_sharded(OracleOps(orc, torch), 0.3, 0.6, -3.0, 9, 0.25, 40, scheme, g1, g2)
    p1, p2 = fast_stepper_nd(orc, 0.3, 0.6, -3.0, 9, 2, 0.25, 40, scheme == "FastSBD", g1, g2)
    for rank, r1, r2, slab, keys in res:
        assert keys == ["exchange", "forward", "inverse", "step"]
        assert np.abs(r1 - s1.numpy()).max() <= 1e-13 * np.abs(s1.numpy()).max()
        assert np.abs(r2 - s2.numpy()).max() <= 1e-13 * np.abs(s2.numpy()).max()
        assert np.abs(r1 - p1).max() <= 1e-10 * np.abs(p1).max()
        assert np.abs(r2 - p2).max() <= 1e-10 * np.abs(p2).max()
        lo, hi, _ = slab_rows(9, rank, world)
        assert np.array_equal(slab[0], r1.reshape(9, 9)[lo:hi])
        assert np.array_equal(slab[1], r2.reshape(9, 9)[lo:hi])


def _strong_worker(rank, world, port, q):
    """One rank of the C2 strong split: its DOF block and exponent groups, evaluated with the
    oracle on a shortened horizon, and the all-gathered coverage of the job."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import Oracle
    from paper_1901_05128_b200.parallel import c2_strong_slice
    from workloads import c2_params
    n = 96  # a scaled-down C2 job: 96 DOFs, exponent halves 0.7 | 0.3
    lo, hi, groups = c2_strong_slice(rank, world, n)
    p = c2_params(n)
    orc = Oracle("port")
    ks = [orc.build_sbd_kernel(g, 1e-3, 24, 24, 12) for g in (0.7, 0.3)]
    U = p.signal(0, 64, np.arange(lo, hi))
    cols, off = [], 0
    for g, cnt in groups:
        cols.append(orc.hist_run(ks[g], U[:, off:off + cnt]))
        off += cnt
    D = np.concatenate(cols, axis=1) if cols else np.zeros((64, 0))
    cover = torch.tensor([lo, hi], dtype=torch.int64)
    allc = [torch.zeros(2, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allc, cover)
    q.put((rank, lo, hi, D, [tuple(x.tolist()) for x in allc]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c2_strong_split(world):
    """bench.py --scaling strong: the ranks' DOF blocks tile the one 65536-DOF job (here a
    96-DOF stand-in), each block picks the right exponent per DOF, and the stitched result equals
    the single-process evaluation bitwise."""
    from paper_1901_05128_b200.parallel import c2_groups, c2_strong_slice
    assert c2_strong_slice(0, 8)[2] == [(0, 8192)] and c2_strong_slice(7, 8)[2] == [(1, 8192)]
    assert c2_groups(30000, 40000) == [(0, 2768), (1, 7232)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    cover = res[0][4]
    assert cover[0][0] == 0 and cover[-1][1] == 96
    assert all(a[1] == b[0] for a, b in zip(cover, cover[1:]))
    from oracle.oracle import Oracle
    from workloads import c2_params
    orc = Oracle("port")
    p = c2_params(96)
    U = p.signal(0, 64, np.arange(96))
    ks = [orc.build_sbd_kernel(g, 1e-3, 24, 24, 12) for g in (0.7, 0.3)]
    full = np.concatenate([orc.hist_run(ks[0], U[:, :48]), orc.hist_run(ks[1], U[:, 48:])], axis=1)
    stitched = np.concatenate([r[3] for r in res], axis=1)
    assert np.array_equal(stitched, full)
