"""The batch-sharded job with the REAL B200 kernels per shard: two ranks
(gloo, world size 2) share cuda:0 -- no kernel of one rank waits on the
other, each runs the block on its own contiguous slice -- with the
parameters broadcast from rank 0, the per-sample checksums all-gathered and
the outputs gathered to rank 0. The sharded result must equal the
single-process B200 result bit for bit (samples are independent,
conv.py:151-182) and stay on the oracle. In-round GPU access is one GPU; the
driver's round-end scaling run exercises the same code over NCCL on 1/2/4/8
GPUs (bench.py)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params():
    rng = np.random.default_rng(0)
    g, C, d, nb = (1, 1, 1), 4, 6, 8
    fan = C * nb * 27
    f1 = (rng.uniform(-1, 1, (nb, C, C, 27)) / np.sqrt(fan)).astype(np.float32)
    f2 = (rng.uniform(-1, 1, (nb, C, C, 27)) / np.sqrt(fan)).astype(np.float32)
    b1 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    b2 = (rng.standard_normal((nb, C)) * 0.1).astype(np.float32)
    return g, C, d, nb, f1, b1, f2, b2


def _worker(rank, world, port, B, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2507_01040_b200 as M
    from paper_2507_01040_b200 import dist as D
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        g, C, d, nb, f1, b1, f2, b2 = _params()
        params = [torch.from_numpy(a) if rank == 0 else torch.zeros(a.shape) for a in (f1, b1, f2, b2)]
        D.broadcast_params(params)  # gloo: host tensors
        lo, hi = D.shard(B, rank, world)
        x = np.random.default_rng(1).standard_normal((B, C, d ** 3, nb)).astype(np.float32)
        blk = M.make_basic_block(M.Signature(g), hi - lo, C, C, C, d, params[0], params[1], 2, params[2],
                                 params[3], padding="same", residual=True)
        y = M.block_forward(torch.from_numpy(x[lo:hi]).cuda(), blk).cpu()
        allcs = D.gather_checksums(D.sample_checksums(y), B, rank, world)
        yall = D.gather_outputs(y, B, rank, world)
        if rank == 0:
            q.put((yall.numpy(), allcs.numpy()))
    finally:
        dist.destroy_process_group()


def test_sharded_block_with_b200_kernels_matches_single_process():
    import oracle as O
    import paper_2507_01040_b200 as M
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    B = 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, B, q)) for r in range(2)]
    for p in procs:
        p.start()
    yall, allcs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the same job in one process, same kernels
    g, C, d, nb, f1, b1, f2, b2 = _params()
    x = np.random.default_rng(1).standard_normal((B, C, d ** 3, nb)).astype(np.float32)
    blk = M.make_basic_block(M.Signature(g), B, C, C, C, d, f1, b1, 2, f2, b2, padding="same", residual=True)
    y1 = M.block_forward(torch.from_numpy(x).cuda(), blk).cpu().numpy()
    assert np.array_equal(yall, y1)
    np.testing.assert_allclose(allcs, y1.reshape(B, -1).astype(np.float64).sum(axis=1), rtol=1e-12, atol=0)
    ref = O.block_ref(x, g, d, f1, b1, 2, tuple(range(nb)), None, None, f2, b2, padding="same", residual=True)
    assert O.max_rel_error(yall, ref) <= 1e-4
