"""Expert-parallel MoE exchange on CPU (gloo, world size 2 and 4).

Drives the host plan (csrc/ep_plan.hpp through orx_debug_ep_plan; the
device plan ep_plan_kernel computes the same layout: per owner, local experts
in order, source-rank-major rows within each expert segment, segments padded
to the grouped-GEMM tile) with the same dispatch / regroup / return / combine
steps as EngineT::moe_ep, with gloo all_to_all standing in for the peer-memory
stores and numpy experts standing in for the grouped GEMMs, and checks the result
against the single-process MoE (every rank holding all experts): identical
per-token outputs, ascending-expert combine (nn.cpp:152-169).
"""
import ctypes as C
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

E, K, D, TILE = 8, 2, 6, 4


def _experts():
    rng = np.random.default_rng(123)
    return rng.standard_normal((E, D, D)).astype(np.float64)


def _tokens(rank):
    """Rank-local tokens with skewed routing; rank 1 of 4 has no tokens at all."""
    rng = np.random.default_rng(1000 + rank)
    n = 0 if rank == 3 else [37, 21, 50][rank % 3]
    x = rng.standard_normal((n, D))
    # skew: experts 0 and 5 are hot, expert 6 never used
    p = np.array([6, 1, 1, 1, 1, 5, 0, 1], dtype=np.float64)
    sel = np.stack([np.sort(rng.choice(E, K, replace=False, p=p / p.sum())) for _ in range(n)]) if n else \
        np.zeros((0, K), dtype=np.int64)
    w = rng.random((n, K))
    return x, sel.astype(np.int64), w


def _moe_reference(x, sel, w, W_e):
    out = np.zeros_like(x)
    for r in range(x.shape[0]):
        acc = np.zeros(D)
        for j in range(K):  # ascending expert id
            acc = acc + w[r, j] * (W_e[sel[r, j]] @ x[r])
        out[r] = acc
    return out


def _plan(world, rank, counts, max_tiles):
    from paper_2506_13695_b200._lib import check, lib
    L = lib()
    El = E // world
    I64 = C.c_int64 * world
    sc, so, rc, ro = I64(), I64(), I64(), I64()
    tab = (C.c_int32 * (world * El * 3))()
    tiles = (C.c_int32 * max_tiles)()
    nt = C.c_int32()
    cnt = (C.c_int32 * (world * E))(*[int(v) for v in counts.reshape(-1)])
    check(L.orx_debug_ep_plan(world, rank, E, cnt, TILE, max_tiles, sc, so, rc, ro, tab, tiles, C.byref(nt)))
    return (np.array(sc), np.array(so), np.array(rc), np.array(ro), np.array(tab).reshape(world, El, 3),
            np.array(tiles), nt.value)


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W_e = _experts()
        x, sel, w = _tokens(rank)
        n = x.shape[0]
        El, e0 = E // world, rank * (E // world)
        # 1. routing histogram, all-gathered
        counts = np.bincount(sel.reshape(-1), minlength=E).astype(np.int32)
        allc = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(counts))
        allc = torch.stack(allc).numpy()
        max_tiles = (world * 64 * K) // TILE + E + 1
        sc, so, rc, ro, tab, tiles, nt = _plan(world, rank, allc, max_tiles)
        # 2. compact send order by expert (ep_send_plan + moe_scatter)
        cursor = np.concatenate([[0], np.cumsum(counts)[:-1]])
        xs = np.zeros((n * K, D))
        ws = np.zeros(n * K)
        slot = np.zeros((n, K), dtype=np.int64)
        for r in range(n):
            for j in range(K):
                s = cursor[sel[r, j]]
                cursor[sel[r, j]] += 1
                xs[s], ws[s], slot[r, j] = x[r], w[r, j], s
        assert so[-1] + sc[-1] == n * K
        # 3. dispatch (NCCL send/recv in the engine)
        xr = torch.zeros((int(rc.sum()), D), dtype=torch.float64)
        wr = torch.zeros(int(rc.sum()), dtype=torch.float64)
        dist.all_to_all_single(xr, torch.from_numpy(xs), [int(v) for v in rc], [int(v) for v in sc])
        dist.all_to_all_single(wr, torch.from_numpy(ws), [int(v) for v in rc], [int(v) for v in sc])
        xr, wr = xr.numpy(), wr.numpy()
        # 4. regroup expert-major (ep_permute_kernel), run local experts per tile
        S = nt * TILE
        xg = np.zeros((S, D))
        rs = np.zeros(S)
        perm = np.full(xr.shape[0], -1)
        for p in range(world):
            for el in range(El):
                src, dst, c = tab[p, el]
                xg[dst:dst + c], rs[dst:dst + c] = xr[src:src + c], wr[src:src + c]
                perm[src:src + c] = np.arange(dst, dst + c)
        assert (perm >= 0).all() and len(set(perm.tolist())) == len(perm)
        assert (tiles[nt:] == -1).all() and np.all(np.diff(tiles[:nt]) >= 0)
        yg = np.zeros((S, D))
        for t in range(nt):
            e = e0 + tiles[t]
            rows = slice(t * TILE, (t + 1) * TILE)
            yg[rows] = rs[rows, None] * (xg[rows] @ W_e[e].T)
        ys = yg[perm]
        # 5. return and combine in ascending expert order (moe_combine)
        yr = torch.zeros((n * K, D), dtype=torch.float64)
        dist.all_to_all_single(yr, torch.from_numpy(ys), [int(v) for v in sc], [int(v) for v in rc])
        yr = yr.numpy()
        got = np.zeros((n, D))
        for r in range(n):
            acc = np.zeros(D)
            for j in range(K):
                acc = acc + yr[slot[r, j]]
            got[r] = acc
        want = _moe_reference(x, sel, w, W_e)
        out[rank] = (n, float(np.abs(got - want).max()) if n else 0.0, int(rc.sum()), nt)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_ep_exchange_gloo(world):
    port = 29700 + world + (os.getpid() % 200)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    got = [out[r] for r in range(world)]
    assert sum(g[2] for g in got) == sum(g[0] for g in got) * K  # every (token, expert) row served once
    for n, err, _, _ in got:
        assert err < 1e-12, got


def test_ep_plan_rejects_bad_world():
    from paper_2506_13695_b200._lib import lib
    tab = (C.c_int32 * 64)()
    tiles = (C.c_int32 * 8)()
    cnt = (C.c_int32 * (3 * E))()
    assert lib().orx_debug_ep_plan(3, 0, E, cnt, TILE, 8, None, None, None, None, tab, tiles, None) != 0
