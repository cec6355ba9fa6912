"""Host-side multi-rank plumbing of bench.py on CPU with gloo, world size 2:
NCCL unique-id broadcast through the torch store, max-over-ranks timing,
z-slab decomposition (MPIPlusX layout) and the oracle's view of
a slab-partitioned problem (concatenation equivalence)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    import torch
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = bench.broadcast_uid(bytes(range(128)) if rank == 0 else None, rank, dist)
        ms = bench.max_over_ranks(1.0 + rank, dist, world, "cpu")
        z0, nzl, Lz = bench.slab(rank, world, 8)
        # each rank's slab of the global state, gathered on every rank
        got = [None] * world
        dist.all_gather_object(got, (z0, nzl))
        q.put((rank, uid, ms, z0, nzl, Lz, got))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_plumbing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, uid, ms, z0, nzl, Lz, got in res:
        assert uid == bytes(range(128))                   # same NCCL id on every rank
        assert ms == 2.0                                  # slowest rank's time
        assert Lz == 2.0 and nzl == 8
        planes = sorted(got)
        assert planes == [(0, 8), (8, 8)]                 # disjoint, covering slabs


def test_slab_concatenation_matches_global_oracle():
    """The global problem on [0,1]^2 x [0,P] split into P z-slabs: the
    oracle's advection of the global state restricted to each slab equals
    the stencil applied to the slab plus its halo plane (what each rank
    computes), so rank-local results concatenate to the global ones."""
    import oracle
    nx = ny = 6
    P, nzl = 3, 4
    nz = P * nzl
    y = np.random.default_rng(3).random(3 * nx * ny * nz)
    k = (0.5, 0.25, 0.125)
    f = oracle.advection(y, nx, ny, nz, *k).reshape(nz, ny, nx, 3)
    Y = y.reshape(nz, ny, nx, 3)
    for r in range(P):
        sl = Y[r * nzl:(r + 1) * nzl]
        halo = Y[(r * nzl - 1) % nz]
        # local stencil with the halo as plane -1 (what BW_AdvectionRHS does)
        ext = np.concatenate([halo[None], sl], 0)
        loc = np.empty_like(sl)
        for kk in range(nzl):
            q = ext[kk + 1]
            acc = k[0] * (np.roll(q, 1, axis=1) - q)
            acc = acc + k[1] * (np.roll(q, 1, axis=0) - q)
            acc = acc + k[2] * (ext[kk] - q)
            loc[kk] = acc
        assert np.array_equal(loc, f[r * nzl:(r + 1) * nzl])


def test_reference_arm_rank1_exits_cleanly(monkeypatch, capsys):
    import sys
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--gpus", "2",
                                      "--steps", "1", "--warmup", "0"])
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    monkeypatch.setenv("LOCAL_RANK", "1")
    bench.main()
    assert capsys.readouterr().out == ""                  # only rank 0 prints
