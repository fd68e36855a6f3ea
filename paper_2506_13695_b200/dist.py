"""Data-parallel plumbing for one process per GPU (torch.distributed).

Users are independent end to end (harness.cpp:506-522), so each
rank owns a disjoint contiguous block of users with its own weight replica and
there is no data-path collective. The only collectives are the timing barrier
and the max-over-ranks reduction of the measured step time.
"""
from __future__ import annotations


def shard_users(rank: int, world: int, users_per_rank: int):
    """Contiguous user block of `rank`: (user_begin, n_users)."""
    if not (0 <= rank < world):
        raise ValueError("rank outside world")
    return rank * users_per_rank, users_per_rank


def split_users(n_users: int, rank: int, world: int):
    """Balanced contiguous split of n_users over world ranks: (begin, count)."""
    base, rem = divmod(n_users, world)
    begin = rank * base + min(rank, rem)
    return begin, base + (1 if rank < rem else 0)


def ep_unique_id(device=None) -> bytes:
    """NCCL unique id for the engines' expert-parallel communicator: made on
    rank 0 (orx_ep_unique_id) and broadcast over the default process group."""
    import ctypes as C

    import torch
    import torch.distributed as dist

    from ._lib import check, lib
    buf = (C.c_uint8 * 128)()
    if dist.get_rank() == 0:
        check(lib().orx_ep_unique_id(buf))
    t = torch.tensor(list(bytes(buf)), dtype=torch.uint8, device=device)
    dist.broadcast(t, src=0)
    return bytes(t.cpu().tolist())


def max_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
