"""N>1 path on CPU: the batch sharder with world_size 2 over gloo.

The per-rank compute is injected by the test (the CPU oracle stands in for the GPU
kernels, which the product never does); what is tested is the product's partitioning and
gather logic: every polynomial is processed exactly once, in order, with uneven shards."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2402_00675_b200.shard import Sharder, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 16, 4097):
        for world in (1, 2, 3, 8):
            ranges = [shard_range(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c and b - a >= d - c >= b - a - 1
    with pytest.raises(ValueError):
        shard_range(5, 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle.oracle import IMPROVED, Oracle

        o = Oracle()
        P = o.params(3329, 256, 16, (IMPROVED,), exact=True)
        full = o.rng(12345, 3329, total * 256).reshape(total, 256)
        sh = Sharder.from_env()
        local = sh.run(lambda part: P.forward(IMPROVED, part), full)
        got = sh.gather(torch.from_numpy(local.astype(np.int64)), total)
        if rank == 0:
            want = P.forward(IMPROVED, full).astype(np.int64)
            q.put(bool((got.numpy() == want).all()) and got.shape[0] == total)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [9, 16])
def test_gloo_world2_shard_and_gather(total):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) is True
