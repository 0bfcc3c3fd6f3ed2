"""Frame sharding across the GPUs of one node.

Frames are independent at inference (no cross-frame state; the reference's
temporal metric is evaluation-only, analysis.py:350-377), so a batch or a
temporal window is split into contiguous per-rank shards and every rank runs
the whole hot path on its own frames with no data-path collective. One
process per GPU (torchrun); ``torch.distributed`` (NCCL over NVLink on the
GPU box, gloo in the CPU tests) is used only to gather per-rank timings and,
optionally, the visibility images back on rank 0.
"""

from __future__ import annotations

import os

import numpy as np


def shard_bounds(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous shard; sizes differ by at most one
    and earlier ranks take the remainder."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(n_frames, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard(items, rank: int, world: int):
    a, b = shard_bounds(len(items), rank, world)
    return list(items[a:b])


def dist_env():
    """(rank, world, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str | None = None):
    """Initialise the process group for this node (127.0.0.1 rendezvous)."""
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(local)
            kw["device_id"] = torch.device("cuda", local)
        dist.init_process_group(backend, **kw)
    return rank, world, local


def max_over_ranks(value: float, device=None) -> float:
    """Max of a scalar over all ranks (the job's time is the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_frames(local, n_frames: int, device=None):
    """All-gather per-rank (n_i, ...) shards into the full (n_frames, ...)
    batch in frame order (shards may differ in size by one frame)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return local
    world, rank = dist.get_world_size(), dist.get_rank()
    sizes = [shard_bounds(n_frames, r, world) for r in range(world)]
    cap = max(b - a for a, b in sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad)
    return torch.cat([bufs[r][: b - a] for r, (a, b) in enumerate(sizes)], dim=0)


def window_seed(rank: int, base: int = 0) -> int:
    """Seed of rank's own temporal window in the weak-scaling benchmark."""
    return int(np.uint32(base * 1000003 + rank))
