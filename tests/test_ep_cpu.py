"""Expert-parallel MoE exchange on CPU (gloo, world size 2 and 4).

Drives the host restatement of the device plan (csrc/ep_plan.hpp
ep_plan_placed through orx_debug_ep_plan; ep_plan_kernel computes the same
layout: per rank, local expert slots in order -- replicated experts first,
then owned ones -- each segment holding every rank's rows source-rank major
for an owned expert and the rank's own rows for a replicated one, padded to
the grouped-GEMM tile) with the same dispatch / grouped experts / return /
combine steps as EngineT::moe_ep, gloo object all-gathers standing in for the
peer-memory stores and numpy experts for the grouped GEMMs, and checks the
result against the single-process MoE (every rank holding all experts):
identical per-token outputs, ascending-expert combine (nn.cpp:152-169). Also
the load-balanced placement (ep_place_balanced) and placed weight shards.
"""
import ctypes as C
import os

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

E, K, D, TILE = 8, 2, 6, 4
# placements of the one MoE layer: contiguous, and replicated + permuted owners
PLACEMENTS = {
    "contiguous": None,
    "replicated": {2: [-1, 1, 0, 1, 0, -1, 0, 1], 4: [-1, 3, 0, 1, 2, -1, 0, 3]},
}


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


def _owner(world, placement):
    if PLACEMENTS[placement] is None:
        return np.arange(E) // (E // world)
    return np.array(PLACEMENTS[placement][world])


def _local(owner, rank):
    """local slots of a rank: replicated experts, then owned ones (ascending ids)"""
    return [e for e in range(E) if owner[e] < 0] + [e for e in range(E) if owner[e] == rank]


def _plan(world, rank, counts, owner, slots, max_tiles):
    from paper_2506_13695_b200._lib import check, lib
    I32 = C.c_int32
    cnt = (I32 * (world * E))(*[int(v) for v in counts.reshape(-1)])
    own = (I32 * E)(*[int(v) for v in owner])
    cursor, seg, tiles = (I32 * E)(), (I32 * (2 * slots))(), (I32 * max_tiles)()
    nt, need = I32(), C.c_int64()
    check(lib().orx_debug_ep_plan(world, rank, E, cnt, own, TILE, max_tiles, slots, cursor, seg, tiles, C.byref(nt),
                                  C.byref(need)))
    return np.array(cursor), np.array(seg).reshape(slots, 2), np.array(tiles), nt.value, need.value


def _worker(rank, world, port, placement, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W_e = _experts()
        x, sel, w = _tokens(rank)
        n = x.shape[0]
        owner = _owner(world, placement)
        slots = max(len(_local(owner, p)) for p in range(world))
        # 1. routing histogram, all-gathered (ep_counts)
        counts = np.bincount(sel.reshape(-1), minlength=E).astype(np.int32)
        allc = [torch.zeros(E, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allc, torch.from_numpy(counts))
        allc = torch.stack(allc).numpy()
        max_tiles = (world * 64 * K) // TILE + E + 1
        cursor, seg, tiles, nt, need = _plan(world, rank, allc, owner, slots, max_tiles)
        # 2. dispatch: pair gw = r * K + j, in order, to its computing rank at cursor[e]++ (ep_dispatch)
        sends = []
        for r in range(n):
            for j in range(K):
                e = int(sel[r, j])
                dest = rank if owner[e] < 0 else int(owner[e])
                sends.append((dest, int(cursor[e]), x[r], w[r, j], (rank, r * K + j)))
                cursor[e] += 1
        gathered = [None] * world
        dist.all_gather_object(gathered, sends)
        xr = np.zeros((need, D))
        wr = np.zeros(need)
        src = [None] * need
        for lst in gathered:
            for dest, pos, xv, wv, code in lst:
                if dest != rank:
                    continue
                assert src[pos] is None, "two rows dispatched to one position"
                xr[pos], wr[pos], src[pos] = xv, wv, code
        # every row of every local segment has exactly one source; padding none
        local = _local(owner, rank)
        for j in range(slots):
            s0, cnt_j = seg[j]
            g = local[j] if j < len(local) else -1
            want = 0 if g < 0 else (allc[rank, g] if owner[g] < 0 else allc[:, g].sum())
            assert cnt_j == want
            assert all(src[i] is not None for i in range(s0, s0 + cnt_j))
        assert sum(c is not None for c in src) == seg[:, 1].sum()
        assert (tiles[nt:] == -1).all() and np.all(np.diff(tiles[:nt]) >= 0)
        # 3. grouped experts over the received rows (tile -> local slot -> global expert)
        yr_back = []
        covered = 0
        for t in range(nt):
            g = local[tiles[t]]
            s0 = seg[tiles[t], 0] + TILE * (t - int(np.argmax(tiles[:nt] == tiles[t])))
            for i in range(s0, min(s0 + TILE, need)):
                if src[i] is not None:
                    yr_back.append((src[i], wr[i] * (W_e[g] @ xr[i])))
                    covered += 1
        assert covered == seg[:, 1].sum()
        # 4. return (the W2 epilogue's peer stores) and combine in ascending expert order
        gathered = [None] * world
        dist.all_gather_object(gathered, yr_back)
        yr = np.full((n * K, D), np.nan)
        for lst in gathered:
            for (q, gw), y in lst:
                if q == rank:
                    yr[gw] = y
        got = np.zeros((n, D))
        for r in range(n):
            acc = np.zeros(D)
            for j in range(K):
                acc = acc + yr[r * K + j]
            got[r] = acc
        want = _moe_reference(x, sel, w, W_e)
        out[rank] = (n, float(np.abs(got - want).max()) if n else 0.0, int(seg[:, 1].sum()), nt)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("placement", sorted(PLACEMENTS))
@pytest.mark.parametrize("world", [2, 4])
def test_ep_exchange_gloo(world, placement):
    port = 29700 + world + 7 * len(placement) + (os.getpid() % 200)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, placement, out), nprocs=world, join=True)
    got = [out[r] for r in range(world)]
    assert sum(g[2] for g in got) == sum(g[0] for g in got) * K  # every (token, expert) row served once
    for n, err, _, _ in got:
        assert err < 1e-12, got


def test_ep_plan_rejects_bad_placement():
    from paper_2506_13695_b200._lib import lib
    I32 = C.c_int32
    cursor, seg, tiles, nt = (I32 * E)(), (I32 * 16)(), (I32 * 8)(), I32()
    cnt = (I32 * (2 * E))()
    bad_owner = (I32 * E)(*([5] * E))  # rank 5 of 2
    assert lib().orx_debug_ep_plan(2, 0, E, cnt, bad_owner, TILE, 8, 8, cursor, seg, tiles, C.byref(nt), None) != 0
    ok_owner = (I32 * E)(*([0] * 4 + [1] * 4))
    assert lib().orx_debug_ep_plan(2, 0, E, cnt, ok_owner, TILE, 8, 2, cursor, seg, tiles, C.byref(nt), None) != 0
    assert lib().orx_debug_ep_plan(2, 0, E, cnt, ok_owner, TILE, 8, 4, cursor, seg, tiles, C.byref(nt), None) == 0


def _rank_loads(load, owner, world):
    r = np.zeros(world)
    for e, o in enumerate(owner):
        if o < 0:
            r += load[e] / world
        else:
            r[o] += load[e]
    return r


def test_ep_place_balances_and_replicates_hot_experts():
    import paper_2506_13695_b200 as P
    rng = np.random.default_rng(5)
    layers, E24, world = 6, 24, 4
    load = rng.integers(1000, 5000, size=(layers, E24)).astype(np.int64)
    load[0, 7] = 60000  # one expert above a rank's fair share: must be replicated
    load[3, [2, 3]] = 30000
    owner, pred = P.ep_place(load, world, 4)
    owner2, pred2 = P.ep_place(load, world, 4)
    assert (owner == owner2).all() and (pred == pred2).all()  # deterministic
    assert owner[0, 7] == -1
    for li in range(layers):
        own = owner[li]
        assert ((own >= -1) & (own < world)).all()
        n_rep = int((own < 0).sum())
        assert n_rep <= 4
        cap = (E24 - n_rep + world - 1) // world + 1
        assert all((own == p).sum() <= cap for p in range(world))
        r = _rank_loads(load[li], own, world)
        assert abs(r.max() / r.mean() - pred[li]) < 1e-9
        contiguous = _rank_loads(load[li], np.arange(E24) // (E24 // world), world)
        assert r.max() <= contiguous.max() + 1e-9
        assert pred[li] <= 1.05 or n_rep == 4
    # no replicas allowed: plain packing, still no worse than contiguous blocks
    owner0, _ = P.ep_place(load, world, 0)
    assert (owner0 >= 0).all()
    # at least 3 replicated (the hottest) per layer: fewer rows cross NVLink
    owner3, pred3 = P.ep_place(load, world, 6, min_replicas=3)
    for li in range(layers):
        rep = np.flatnonzero(owner3[li] < 0)
        assert len(rep) >= 3
        hottest = np.argsort(-load[li], kind="stable")[:len(rep)]
        assert set(rep) == set(hottest.tolist())
    with pytest.raises(Exception):
        P.ep_place(load, world, 2, min_replicas=3)


def test_placed_weights_materialise_the_computed_experts():
    import paper_2506_13695_b200 as P
    cfg = P.PolicyConfig.preset("tiny", moe_enabled=True, n_experts=8, experts_active=2, moe_location="enc_and_dec")
    L = P.moe_layers(cfg)
    assert L == 4  # tiny: 2 encoder + 2 decoder layers, all MoE
    owner = np.tile(np.array(PLACEMENTS["replicated"][2], dtype=np.int32), (L, 1))
    owner[1] = np.arange(8) % 2  # a different placement in layer 1
    full = P.Weights.random(cfg)
    for rank in range(2):
        shard = P.Weights.random_ep(cfg, rank, 2, owner=owner)
        for li, name in enumerate(["enc0", "enc1", "dec0", "dec1"]):
            for e in range(8):
                t = shard.get(f"{name}.moe.expert{e}.w1.w")
                keep = owner[li, e] < 0 or owner[li, e] == rank
                if keep:
                    np.testing.assert_array_equal(t, full.get(f"{name}.moe.expert{e}.w1.w"))
                else:
                    assert t.size == 0  # not materialised on this rank
    with pytest.raises(Exception):
        P.Weights.random_ep(cfg, 0, 2, owner=owner[:2])
