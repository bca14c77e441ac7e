"""World-size-2 gloo test of the multi-GPU host logic on CPU: sharding,
parameter broadcast from rank 0, checksum all-gather and output gather. The per-shard compute is
the CPU oracle (the product kernels need a GPU); what is under test is that
the sharded job reproduces the single-process result exactly."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2507_01040_b200 import dist as D
from paper_2507_01040_b200 import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        B, C, d, g = 5, 3, 6, (1, 1)
        nb = 4
        rng = np.random.default_rng(0)
        if rank == 0:
            f = torch.from_numpy(rng.uniform(-0.2, 0.2, (nb, C, C, 9)).astype(np.float32))
            b = torch.from_numpy((rng.standard_normal((nb, C)) * 0.1).astype(np.float32))
        else:
            f = torch.zeros((nb, C, C, 9))
            b = torch.zeros((nb, C))
        D.broadcast_params([f, b])
        lo, hi = D.shard(B, rank, world)
        xr = np.random.default_rng(1).standard_normal((B, C, d * d, nb)).astype(np.float32)
        y = O.conv_ref(xr[lo:hi], f.numpy(), b.numpy(), g, d, 3, 1)
        cs = D.sample_checksums(torch.from_numpy(y))
        allcs = D.gather_checksums(cs, B, rank, world)
        yall = D.gather_outputs(torch.from_numpy(y), B, rank, world)
        if rank == 0:
            full = O.conv_ref(xr, f.numpy(), b.numpy(), g, d, 3, 1)
            assert np.array_equal(yall.numpy(), full)  # the gathered outputs, bit for bit
            q.put((allcs.numpy(), D.sample_checksums(torch.from_numpy(full)).numpy()))
        else:
            assert yall is None
    finally:
        dist.destroy_process_group()


def test_sharded_job_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("B,world", [(256, 1), (256, 2), (256, 8), (5, 2), (3, 4), (0, 2)])
def test_shard_partition(B, world):
    parts = [W.shard(B, r, world) for r in range(world)]
    assert parts[0][0] == 0 and parts[-1][1] == B
    for (a, b), (c, d) in zip(parts, parts[1:]):
        assert b == c
    sizes = [b - a for a, b in parts]
    assert max(sizes) - min(sizes) <= 1
