"""Rank invariance of the sharded hot path (SURVEY §4 tier 4, §8(c) "Multi-GPU" pin:
sharded + all-gathered O == 1-GPU O bitwise).

Heads are masked independently, so a kv-group shard computes the same
numbers as the unsharded context for its heads -- provided every reduction order is a
function of the (sequence, kv-group) region alone.  The decode split cuts each region into
fixed chunks from its first row (decode_mma.cu, rank-invariant split), independent of the
batch, the other groups and the SM count; prefill items are whole (head, q-tile) units.
These tests run the shards as separate contexts on one GPU (a shard's context sees only its
groups, so its launch has a different grid and a different CTA -> row assignment) and
compare the concatenated outputs with the unsharded context's BIT FOR BIT, every step,
through ring wrap-around.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import bits, f64
from moa_workloads.inputs import normal

pytestmark = pytest.mark.gpu
CHUNK = 256   # moa_set_decode_split: rank-invariant chunks


def _run(moa, shard_groups, B_sel, q, k, v, qd, kd, vd, W, s, G, steps):
    """Prefill + `steps` fused decode steps of the sequences B_sel on kv-groups
    [g0, g1); returns (prefill O, [decode o per step]) restricted to those heads."""
    g0, g1 = shard_groups
    dev = torch.device("cuda")
    Hq, d = q.shape[2], q.shape[3]
    Hkv = k.shape[2]
    N = q.shape[1]
    Bl = len(B_sel)
    ctx = moa.MoAContext(1, Hq, Hkv, d, Bl, dtype=torch.bfloat16, kv_group_begin=g0, kv_group_end=g1)
    ctx.set_decode_split(CHUNK)
    ctx.set_spans(0, W, s, N)
    ctx.alloc_cache(Bl)
    ws = ctx.alloc_workspace(Bl)
    sel = torch.tensor(B_sel)
    ql = q[sel][:, :, g0 * G:g1 * G].contiguous().to(dev)
    kl = k[sel][:, :, g0:g1].contiguous().to(dev)
    vl = v[sel][:, :, g0:g1].contiguous().to(dev)
    o = torch.empty_like(ql)
    scale = 1 / math.sqrt(d)
    ctx.prefill(0, ql, kl, vl, o, scale)
    outs = []
    for t in range(steps):
        qt = qd[t][sel][:, g0 * G:g1 * G].contiguous().to(dev)
        kt = kd[t][sel][:, g0:g1].contiguous().to(dev)
        vt = vd[t][sel][:, g0:g1].contiguous().to(dev)
        od = torch.empty_like(qt)
        ctx.decode_step_fused(0, qt, kt, vt, od, N + t, scale, ws)
        outs.append(od)
    torch.cuda.synchronize()
    return o.cpu(), [x.cpu() for x in outs]


@pytest.mark.parametrize("world", [2, 3, 4])
def test_kv_shards_bitwise_equal_unsharded(moa, world):
    """Cost-balanced (uneven) kv-group ranges from dist.plan_shards, concatenated by heads."""
    from paper_2406_14909_b200 import dist as mdist
    B, N, Hq, Hkv, d, s, T = 3, 1100, 16, 8, 128, 16, 40
    G = Hq // Hkv
    # heterogeneous windows: several chunks per region, tiny and zero windows, one > N
    W = [1000, 7, 600, 600, 0, 33, 257, 256, 1, 1500, 300, 90, 512, 511, 64, 900]
    q = normal((B, N, Hq, d), 901, torch.bfloat16)
    k = normal((B, N, Hkv, d), 902, torch.bfloat16)
    v = normal((B, N, Hkv, d), 903, torch.bfloat16)
    qd = normal((T, B, Hq, d), 904, torch.bfloat16)
    kd = normal((T, B, Hkv, d), 905, torch.bfloat16)
    vd = normal((T, B, Hkv, d), 906, torch.bfloat16)
    full_o, full_dec = _run(moa, (0, Hkv), list(range(B)), q, k, v, qd, kd, vd, W, s, G, T)
    shards = mdist.plan_shards(world, Hkv, B, "kv", group_cost=mdist.group_costs([W], s, G))
    shard = [_run(moa, (sh.g0, sh.g1), list(range(B)), q, k, v, qd, kd, vd, W, s, G, T) for sh in shards]
    cat_o = torch.cat([x[0] for x in shard], dim=2)
    assert np.array_equal(bits(cat_o), bits(full_o))
    for t in range(T):
        cat = torch.cat([x[1][t] for x in shard], dim=1)
        assert np.array_equal(bits(cat), bits(full_dec[t])), t
    # and the unsharded result is the masked attention of the oracle (not merely self-consistent)
    Kh = torch.cat([k, kd.permute(1, 0, 2, 3)], 1)
    Vh = torch.cat([v, vd.permute(1, 0, 2, 3)], 1)
    for t in (0, T - 1):
        Od, _ = oracle.decode(f64(qd[t]), f64(Kh[:, :N + t + 1]), f64(Vh[:, :N + t + 1]), N + t, W, s,
                              1 / math.sqrt(d))
        assert np.abs(f64(full_dec[t]) - Od).max() < 2e-2


def test_batch_shards_bitwise_equal_unsharded(moa):
    """Sequences are independent too: a context serving a subset of the batch computes the
    same bits for those sequences (the split does not depend on the batch size)."""
    B, N, Hq, Hkv, d, s, T = 4, 700, 8, 2, 128, 64, 12
    G = Hq // Hkv
    W = [600, 20, 128, 0, 300, 299, 1, 700]
    q = normal((B, N, Hq, d), 911, torch.bfloat16)
    k = normal((B, N, Hkv, d), 912, torch.bfloat16)
    v = normal((B, N, Hkv, d), 913, torch.bfloat16)
    qd = normal((T, B, Hq, d), 914, torch.bfloat16)
    kd = normal((T, B, Hkv, d), 915, torch.bfloat16)
    vd = normal((T, B, Hkv, d), 916, torch.bfloat16)
    full_o, full_dec = _run(moa, (0, Hkv), list(range(B)), q, k, v, qd, kd, vd, W, s, G, T)
    for sel in ([0, 1], [2, 3], [3]):
        o, dec = _run(moa, (0, Hkv), sel, q, k, v, qd, kd, vd, W, s, G, T)
        assert np.array_equal(bits(o), bits(full_o[sel]))
        for t in range(T):
            assert np.array_equal(bits(dec[t]), bits(full_dec[t][sel])), (sel, t)
