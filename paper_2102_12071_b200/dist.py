"""Multi-process plumbing (torch.distributed): one process per GPU.

The hot path shards without a data-path collective: independent
problems (config 4's batch) are split across ranks, and throughput runs place
one replica per rank.  The only collectives are control-plane: a barrier around
timed regions, the max-over-ranks step time, and gathering per-problem
histories.  NCCL on GPUs, gloo for the CPU tests."""

from __future__ import annotations

import os

import numpy as np


def env():
    """(world, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None, device=None):
    import torch
    import torch.distributed as dist
    world, rank, local = env()
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl" and device is not None:
            kw["device_id"] = device
        dist.init_process_group(backend, **kw)
    return world, rank, local


def shard(count: int, rank: int, world: int):
    """Contiguous [lo, hi) share of `count` independent problems for `rank`
    (sizes differ by at most one; every problem is owned by exactly one rank)."""
    base, extra = divmod(count, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def gather_rows(local: np.ndarray, count: int, device=None) -> np.ndarray | None:
    """Gather per-problem rows (e.g. residual histories) sharded by `shard` onto
    rank 0 in global problem order; other ranks get None."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return np.asarray(local)
    world, rank = dist.get_world_size(), dist.get_rank()
    width = local.shape[1]
    lo, hi = shard(count, rank, world)
    maxn = count // world + 1
    buf = torch.zeros((maxn, width), dtype=torch.float64, device=device)
    if hi > lo:
        buf[: hi - lo] = torch.as_tensor(local, dtype=torch.float64, device=device)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    if rank != 0:
        return None
    rows = []
    for r in range(world):
        a, b = shard(count, r, world)
        rows.append(outs[r][: b - a].cpu().numpy())
    return np.concatenate(rows, axis=0)
