"""Multi-rank partitioning on CPU: world_size 2, 4 and 8 over the gloo backend.

Each rank plans its shard, builds a planning context (device -1) for it,
computes its slab of head outputs with the fp64 oracle (standing in for the
GPU kernels, which the -m gpu tests cover), and all-gathers them with
``gather_heads``.  The gathered tensor must equal the unsharded oracle output
bit for bit, in both shard modes, for decode and prefill layouts.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

B, N, HQ, HKV, D, S = 8, 40, 16, 8, 64, 3
WINDOWS = [1, 5, 0, 40, 7, 7, 2, 30, 3, 3, 40, 39, 11, 0, 6, 9]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs():
    g = np.random.default_rng(0)
    q = g.standard_normal((B, N, HQ, D))
    k = g.standard_normal((B, N, HKV, D))
    v = g.standard_normal((B, N, HKV, D))
    return q, k, v


def _costs():
    from paper_2406_14909_b200 import dist as mdist
    return mdist.group_costs([WINDOWS], S, HQ // HKV)


def _worker(rank, world, port, mode, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2406_14909_b200 import dist as mdist
        shards = mdist.plan_shards(world, HKV, B, mode, group_cost=_costs())
        shard = shards[rank]
        # planning context of this shard: its windows are its q-heads' windows
        ctx = mdist.make_context(shard, 1, HQ, HKV, D, device=None)
        ctx.set_spans(0, WINDOWS, S, N)
        G = HQ // HKV
        heads = list(range(shard.g0 * G, shard.g1 * G))
        assert [ctx.window(0, h) for h in range(len(heads))] == [WINDOWS[h] for h in heads]
        q, k, v = _inputs()
        qt, kt, vt = (torch.from_numpy(x) for x in (q, k, v))
        ql = mdist.local_slice_q(qt, shard, G).numpy()
        kl = mdist.local_slice_kv(kt, shard).numpy()
        vl = mdist.local_slice_kv(vt, shard).numpy()
        o_local, _ = oracle.prefill(ql, kl, vl, [WINDOWS[h] for h in heads], S, 0.25)
        full_pref = mdist.gather_heads(torch.from_numpy(o_local), shard, shards, G)
        # decode layout: last row of each sequence, through the preallocated gather (kv mode)
        if mode == "kv":
            hg = mdist.HeadGather(shards, rank, B, G, D, dtype=torch.float64, device="cpu")
            hg.local_out().copy_(torch.from_numpy(o_local[:, -1].copy()))
            full_dec, _ = hg.gather()
        else:
            full_dec = mdist.gather_heads(torch.from_numpy(o_local[:, -1].copy()), shard, shards, G)
        results[rank] = (full_pref.numpy(), full_dec.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "batch"), (2, "kv"), (4, "kv"), (4, "batch"), (3, "kv"), (3, "batch"),
                                        (8, "kv"), (8, "batch")])
def test_sharded_outputs_gather_to_unsharded(world, mode):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, results)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    q, k, v = _inputs()
    ref, _ = oracle.prefill(q, k, v, WINDOWS, S, 0.25)
    for r in range(world):
        pref, dec = results[r]
        assert np.array_equal(pref, ref)
        assert np.array_equal(dec, ref[:, -1])


def test_plan_shards_cover_units_once():
    from paper_2406_14909_b200 import dist as mdist
    for world, mode in [(1, "auto"), (2, "batch"), (4, "kv"), (8, "kv"), (8, "batch")]:
        hkv, batch = 8, 32
        shards = mdist.plan_shards(world, hkv, batch, mode)
        units = [(b, g) for s in shards for b in range(s.b0, s.b1) for g in range(s.g0, s.g1)]
        assert sorted(units) == [(b, g) for b in range(batch) for g in range(hkv)]
    assert mdist.plan_shards(3, 8, 6, "auto")[0].mode == "batch"
    assert mdist.plan_shards(4, 8, 6, "auto")[0].mode == "kv"
    with pytest.raises(ValueError):
        mdist.plan_shards(9, 8, 7, "kv")       # a rank without a group
    with pytest.raises(ValueError):
        mdist.plan_shards(8, 8, 7, "batch")    # a rank without a sequence


def test_cost_balanced_kv_split_is_optimal():
    """The kv split minimises the heaviest rank over ALL contiguous partitions (brute force),
    and never loses to the equal-count split (SURVEY §8(e) "assign units by cost")."""
    import itertools
    import random

    from paper_2406_14909_b200 import dist as mdist
    rng = random.Random(3)
    for _ in range(200):
        n = rng.randint(1, 9)
        world = rng.randint(1, n)
        cost = [rng.choice([1, 2, 5, 64, 300, 4096]) for _ in range(n)]
        shards = mdist.plan_shards(world, n, 4, "kv", group_cost=cost)
        assert [s.g0 for s in shards][0] == 0 and shards[-1].g1 == n
        assert all(s.g1 > s.g0 for s in shards) and all(a.g1 == b.g0 for a, b in zip(shards, shards[1:]))
        got = max(sum(cost[s.g0:s.g1]) for s in shards)
        best = min(max(sum(cost[a:b]) for a, b in zip((0,) + cut, cut + (n,)))
                   for cut in itertools.combinations(range(1, n), world - 1))
        assert got == best
        if n % world == 0:
            per = n // world
            assert got <= max(sum(cost[r * per:(r + 1) * per]) for r in range(world))


def test_group_costs_are_in_window_rows():
    from paper_2406_14909_b200 import dist as mdist
    # two layers, G = 2: W_g = max over the pair; rows = s + W_g, capped at pos + 1
    wl = [[3, 10, 0, 0], [100, 1, 5, 6]]
    assert mdist.group_costs(wl, 4, 2) == [(4 + 10) + (4 + 100), (4 + 0) + (4 + 6)]
    assert mdist.group_costs(wl, 4, 2, pos=20) == [14 + 21, 4 + 10]
