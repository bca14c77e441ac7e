"""Batch-sharded data parallelism: contiguous sample slices
per rank, NCCL (or gloo on CPU) broadcast of the compact parameters from
rank 0, all-gather of per-sample checksums and a gather of the outputs to
rank 0. No collective on the data path (samples are independent)."""

from __future__ import annotations

from .workloads import shard  # noqa: F401  (re-exported)


def broadcast_params(tensors, src: int = 0):
    """In-place broadcast of parameter tensors from `src` (compact filters,
    biases, activation weights: 3.5 MB per cfg5 conv)."""
    import torch.distributed as dist
    for t in tensors:
        if t is not None:
            dist.broadcast(t, src=src)
    return tensors


def sample_checksums(y):
    """Per-sample fp64 sums of a (B, ...) output tensor (cheap gather payload)."""
    return y.reshape(y.shape[0], -1).double().sum(dim=1)


def gather_checksums(local, B_total: int, rank: int, world: int):
    """All-gather per-sample checksums of contiguous shards into one (B_total,) vector."""
    import torch
    import torch.distributed as dist
    sizes = [shard(B_total, r, world) for r in range(world)]
    n_max = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros(n_max, dtype=local.dtype, device=local.device)
    buf[: local.numel()] = local
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.cat([p[: hi - lo] for p, (lo, hi) in zip(parts, sizes)])


def gather_outputs(y_local, B_total: int, rank: int, world: int, dst: int = 0):
    """Gather the sharded (B_total, ...) output to rank `dst` (NCCL point-to-point
    over NVLink: every rank sends its contiguous slice). Returns the full tensor on
    `dst`, None elsewhere."""
    import torch
    import torch.distributed as dist
    if rank != dst:
        dist.send(y_local.contiguous(), dst=dst)
        return None
    out = torch.empty((B_total,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=y_local.device)
    for r in range(world):
        lo, hi = shard(B_total, r, world)
        if r == dst:
            out[lo:hi].copy_(y_local)
        else:
            dist.recv(out[lo:hi], src=r)
    return out
