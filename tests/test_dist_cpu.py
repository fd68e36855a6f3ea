"""World-size-2 gloo test of the data-parallel host logic (CPU)."""
import os

import pytest
import torch.multiprocessing as mp

from paper_2506_13695_b200.dist import max_over_ranks, shard_users, split_users


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        begin, n = shard_users(rank, world, 128)
        t = max_over_ranks(10.0 + rank)
        out[rank] = (begin, n, t)
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_max():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    got = [out[r] for r in range(world)]
    assert [g[:2] for g in got] == [(0, 128), (128, 128)]  # disjoint, contiguous, weak scaling
    assert all(g[2] == 11.0 for g in got)  # every rank sees the max step time


def test_split_users_covers_all():
    for n in (0, 1, 7, 1024):
        for w in (1, 2, 3, 8):
            parts = [split_users(n, r, w) for r in range(w)]
            assert sum(c for _, c in parts) == n
            pos = 0
            for b, c in parts:
                assert b == pos
                pos += c
    with pytest.raises(ValueError):
        shard_users(2, 2, 8)
