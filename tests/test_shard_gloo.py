"""Multi-process (world_size 2, gloo, CPU) coverage of the frame-sharding
path: shard bounds, the all-gather that restores frame order, and the
max-over-ranks timing reduction bench.py uses."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_05262_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover_exactly_once():
    for n in (0, 1, 7, 8, 9, 64):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                a, b = shard.shard_bounds(n, r, world)
                seen += list(range(a, b))
                assert (b - a) in (n // world, n // world + 1)
            assert seen == list(range(n))
    with pytest.raises(ValueError):
        shard.shard_bounds(8, 2, 2)


def _worker(rank, world, port, n_frames, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard.shard_bounds(n_frames, rank, world)
        # each rank "renders" its frames: frame i is filled with i
        local = torch.stack([torch.full((1, 4, 6), float(i)) for i in range(a, b)])
        full = shard.gather_frames(local, n_frames)
        t = shard.max_over_ranks(1.5 + rank)
        q.put((rank, full.numpy(), t))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [8, 7])
def test_gather_restores_frame_order_world2(n_frames):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, full, t in res:
        assert full.shape == (n_frames, 1, 4, 6)
        np.testing.assert_array_equal(full[:, 0, 0, 0], np.arange(n_frames, dtype=np.float32))
        assert t == 2.5                                   # max over ranks
