"""Host logic of the filter-sharded multi-GPU path, on CPU:
partition math, and a world-size-2 gloo run of broadcast + per-rank slice +
all-gather reassembling exactly the full oracle output.  (`-m "not gpu"`;
per-rank compute here is the oracle, injected by the test — the product's
sharded_multi calls the CUDA kernels and is covered by the GPU tests.)"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2212_00404_b200.shard import allgather_output, broadcast_input, shard_range, shard_sizes


@pytest.mark.parametrize("M,world", [(4096, 8), (10, 3), (5, 8), (1, 1), (256, 2), (7, 7)])
def test_shard_ranges_partition_m(M, world):
    ranges = [shard_range(M, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == M
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    sizes = shard_sizes(M, world)
    assert max(sizes) - min(sizes) <= 1 and sum(sizes) == M


def test_shard_range_errors():
    with pytest.raises(ValueError):
        shard_range(8, 0, 0)
    with pytest.raises(ValueError):
        shard_range(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, M, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        C, W, K = 3, 9, 3
        I = torch.from_numpy(synth.uniform01(5, (C, W, W))) if rank == 0 else torch.zeros(C, W, W)
        broadcast_input(I, src=0)
        F = synth.uniform_pm1(6, (M, C, K, K))
        m0, m1 = shard_range(M, world, rank)
        Oloc, _ = oracle.conv_multi(I.numpy(), F[m0:m1]) if m1 > m0 else (np.zeros((0, W - K + 1, W - K + 1)), None)
        Ofull = allgather_output(torch.from_numpy(Oloc), M)
        Oref, _ = oracle.conv_multi(I.numpy(), F)
        q.put((rank, bool(np.array_equal(Ofull.numpy(), Oref))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("M", [8, 5])
def test_gloo_world2_broadcast_shard_allgather(M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, M, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]
