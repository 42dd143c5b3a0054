"""Multi-process (world_size 2, gloo, CPU) tests of the row/head-sharded launcher.

The device kernels are exercised by the GPU tests; here each rank computes its
shard with the float64 oracle, standing in for the kernel, to check the host
logic a multi-GPU run relies on: shard boundaries, the per-row independence
that makes sharding exchange-free, the max-over-ranks reduction, and the
optional all-gather.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_07829_b200.launcher import gather_rows, max_over_ranks, shard


def test_shard_covers_range_without_overlap():
    for total, world, align in [(8192, 8, 128), (1000, 3, 128), (7, 4, 1), (300, 2, 128), (64, 8, 128)]:
        shards = [shard(total, r, world, align) for r in range(world)]
        assert shards[0].start == 0 and shards[-1].stop == total
        for a, b in zip(shards, shards[1:]):
            assert a.stop == b.start
        for s in shards[:-1]:
            assert s.start % align == 0
        sizes = [s.size for s in shards]
        assert max(sizes) - min(sizes) <= align


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cpu

        rng = np.random.default_rng(0)  # identical inputs on every rank (seeded, no broadcast)
        M, D, F, N = 300, 32, 48, 16
        X = rng.standard_normal((M, D))
        Wt, Vt = rng.standard_normal((F, D)) / 6, rng.standard_normal((F, D)) / 6
        Ut = rng.standard_normal((N, F)) / 7
        shards = [shard(M, r, world, align=128) for r in range(world)]
        me = shards[rank]
        local = torch.from_numpy(cpu.rms_ffn_swiglu(X[me.start:me.stop], Wt, Vt, Ut, threads=1))
        full = gather_rows(local, shards)
        ref = cpu.rms_ffn_swiglu(X, Wt, Vt, Ut, threads=1)
        t = max_over_ranks(1.0 + rank)
        result_q.put((rank, float(np.abs(full.numpy() - ref).max()), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_row_sharding_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(world)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    for rank, err, t in res:
        assert err == 0.0  # row sharding is exact: rows are independent
        assert t == float(world)  # max over ranks of (1 + rank)


def test_c_abi_shard_range_matches_python_shards():
    """bf_shard_range (the C-ABI's sharding, no GPU needed) equals launcher.shard with 128-row
    alignment for rows and whole heads for attention; shards tile [0, units) in order."""
    from paper_2505_07829_b200 import launcher

    for units, world in [(8192, 8), (32768, 8), (1000, 3), (130, 4), (65536, 2), (5, 8)]:
        prev = 0
        for r in range(world):
            a, b = launcher.shard_range("rms_ffn_swiglu", units, world, r)
            s = launcher.shard(units, r, world, 128)
            assert (a, b) == (s.start, s.stop)
            assert a == prev
            prev = b
        assert prev == units
    for heads, world in [(256, 8), (7, 3)]:
        got = [launcher.shard_range("attention", heads, world, r) for r in range(world)]
        assert got == [(launcher.shard(heads, r, world).start, launcher.shard(heads, r, world).stop)
                       for r in range(world)]
