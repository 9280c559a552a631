"""Fused head-output all-gather (moa_set_peer_outputs + moa_wait_flag)
on one GPU: two kv-group shard contexts play two ranks.  Each shard's decode epilogue writes
its finished head rows into BOTH ranks' gathered [L, B, Hq, d] buffers and bumps both
counters; after waiting on its own counter each "rank" holds the full head output.

Pins (heads are masked independently; rank-invariant split, SURVEY §4
tier 4): both gathered buffers equal the unsharded context's output BIT FOR BIT, every step,
single-layer and cross-layer launches; each counter advances by B * Hkv per layer-step; the
shard's own o equals its slice of the gathered buffer.
"""
import math

import numpy as np
import pytest
import torch

from tests.gpu_util import bits
from moa_workloads.inputs import normal

pytestmark = pytest.mark.gpu
CHUNK = 128


def _ctx(moa, L, Hq, Hkv, d, B, g0, g1, wins, s, N, K, V):
    dev = torch.device("cuda")
    G = Hq // Hkv
    c = moa.MoAContext(L, Hq, Hkv, d, B, dtype=torch.bfloat16, kv_group_begin=g0, kv_group_end=g1)
    c.set_decode_split(CHUNK)
    for l in range(L):
        c.set_spans(l, wins[l], s, N)
    c.alloc_cache(B)
    for l in range(L):
        c.cache_fill(l, K[l][:, :, g0:g1].contiguous().to(dev), V[l][:, :, g0:g1].contiguous().to(dev))
    return c


@pytest.mark.parametrize("cross", [False, True])
def test_peer_gather_two_shards_bitwise(cross):
    import paper_2406_14909_b200 as moa
    dev = torch.device("cuda")
    L, B, N, Hq, Hkv, d, s, steps = 3, 3, 333, 8, 4, 128, 8, 5
    G = Hq // Hkv
    rng = np.random.default_rng(11)
    wins = [[int(x) for x in rng.integers(0, N + 4, size=Hq)] for _ in range(L)]
    K = [normal((B, N, Hkv, d), 500 + l, torch.bfloat16) for l in range(L)]
    V = [normal((B, N, Hkv, d), 600 + l, torch.bfloat16) for l in range(L)]
    full = _ctx(moa, L, Hq, Hkv, d, B, 0, Hkv, wins, s, N, K, V)
    shards = [(0, 1), (1, Hkv)]           # unequal shards: 1 and 3 kv-groups
    sc = [_ctx(moa, L, Hq, Hkv, d, B, g0, g1, wins, s, N, K, V) for g0, g1 in shards]
    gathered = [torch.zeros(L, B, Hq, d, dtype=torch.bfloat16, device=dev) for _ in shards]
    flags = [torch.zeros(L, dtype=torch.int32, device=dev) for _ in shards]
    for (g0, g1), c in zip(shards, sc):
        c.set_peer_outputs([x.data_ptr() for x in gathered], [f.data_ptr() for f in flags],
                           batch_stride=Hq * d, layer_stride=B * Hq * d, head0=g0 * G)
    scale = 1 / math.sqrt(d)
    ws_f = full.alloc_workspace(B, L)
    ws_s = [c.alloc_workspace(B, L) for c in sc]
    qd = normal((steps, L, B, Hq, d), 701, torch.bfloat16).to(dev)
    kd = normal((steps, L, B, Hkv, d), 702, torch.bfloat16).to(dev)
    vd = normal((steps, L, B, Hkv, d), 703, torch.bfloat16).to(dev)
    o_full = torch.empty(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    o_loc = [torch.empty(L, B, (g1 - g0) * G, d, dtype=torch.bfloat16, device=dev) for g0, g1 in shards]
    for t in range(steps):
        p = N + t
        if cross:
            full.decode_step_fused_layers(0, qd[t], kd[t], vd[t], o_full, p, scale, ws_f)
        else:
            for l in range(L):
                full.decode_step_fused(l, qd[t, l], kd[t, l], vd[t, l], o_full[l], p, scale, ws_f)
        for (g0, g1), c, ol, w in zip(shards, sc, o_loc, ws_s):
            q = qd[t][:, :, g0 * G:g1 * G].contiguous()
            k = kd[t][:, :, g0:g1].contiguous()
            v = vd[t][:, :, g0:g1].contiguous()
            if cross:
                c.decode_step_fused_layers(0, q, k, v, ol, p, scale, w)
            else:
                for l in range(L):
                    c.decode_step_fused(l, q[l], k[l], v[l], ol[l], p, scale, w)
        # each "rank" waits for every region of every layer of this step, then reads
        for r in range(len(shards)):
            for l in range(L):
                moa.wait_flag(flags[r][l:l + 1], (t + 1) * B * Hkv)
        torch.cuda.synchronize()
        ref = bits(o_full)
        for r, (g0, g1) in enumerate(shards):
            assert np.array_equal(bits(gathered[r]), ref), (cross, t, r)
            assert np.array_equal(bits(o_loc[r]), ref[:, :, g0 * G:g1 * G]), (cross, t, r)
            assert flags[r].cpu().tolist() == [(t + 1) * B * Hkv] * L, (t, r)


def test_peer_outputs_errors_and_off():
    import paper_2406_14909_b200 as moa
    from paper_2406_14909_b200._lib import MoAError
    dev = torch.device("cuda")
    c = moa.MoAContext(1, 4, 2, 128, 1, dtype=torch.bfloat16, kv_group_begin=1, kv_group_end=2)
    buf = torch.zeros(1, 1, 4, 128, dtype=torch.bfloat16, device=dev)
    fl = torch.zeros(1, dtype=torch.int32, device=dev)
    with pytest.raises(MoAError, match="SHAPE"):      # head0 2 + 2 heads > 3 heads per row
        c.set_peer_outputs([buf.data_ptr()], [fl.data_ptr()], batch_stride=3 * 128, layer_stride=0, head0=2)
    with pytest.raises(MoAError, match="INVALID_ARG"):
        c.set_peer_outputs([buf.data_ptr()], [fl.data_ptr() + 1], batch_stride=4 * 128, layer_stride=0, head0=2)
    c.set_peer_outputs([buf.data_ptr()], [fl.data_ptr()], batch_stride=4 * 128, layer_stride=0, head0=2)
    c.set_peer_outputs([], [], 0, 0, 0)               # off again
    f32 = moa.MoAContext(1, 4, 2, 128, 1, dtype=torch.float32)
    with pytest.raises(MoAError, match="UNSUPPORTED"):
        f32.set_peer_outputs([buf.data_ptr()], [fl.data_ptr()], batch_stride=4 * 128, layer_stride=0, head0=0)
    # wait_flag on an already-reached counter returns at once
    fl.fill_(7)
    moa.wait_flag(fl, 7)
    moa.wait_flag(fl, 3)
    torch.cuda.synchronize()


def test_peer_gather_class_two_shards():
    """dist.PeerGather (the bench's multi-GPU path) with two shard contexts on one GPU: the
    per-layer wait + next_token bookkeeping gives every 'rank' the unsharded output."""
    import paper_2406_14909_b200 as moa
    from paper_2406_14909_b200 import dist as mdist
    dev = torch.device("cuda")
    L, B, N, Hq, Hkv, d, s, steps = 2, 2, 200, 4, 2, 128, 4, 3
    G = Hq // Hkv
    wins = [[40, 7, 200, 0], [1, 64, 9, 33]]
    K = [normal((B, N, Hkv, d), 800 + l, torch.bfloat16) for l in range(L)]
    V = [normal((B, N, Hkv, d), 900 + l, torch.bfloat16) for l in range(L)]
    full = _ctx(moa, L, Hq, Hkv, d, B, 0, Hkv, wins, s, N, K, V)
    shards = mdist.plan_shards(2, Hkv, B, "kv")
    sc = [_ctx(moa, L, Hq, Hkv, d, B, sh.g0, sh.g1, wins, s, N, K, V) for sh in shards]
    outs = [torch.zeros(L, B, Hq, d, dtype=torch.bfloat16, device=dev) for _ in shards]
    flags = [torch.zeros(L, dtype=torch.int32, device=dev) for _ in shards]
    pgs = [mdist.PeerGather(c, sh, G, Hkv, B, outs[r], flags[r], [o.data_ptr() for o in outs],
                            [f.data_ptr() for f in flags]) for r, (c, sh) in enumerate(zip(sc, shards))]
    scale = 1 / math.sqrt(d)
    ws = full.alloc_workspace(B)
    wss = [c.alloc_workspace(B) for c in sc]
    o_full = torch.empty(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    for t in range(steps):
        q = normal((B, Hq, d), 1000 + t, torch.bfloat16).to(dev)
        k = normal((B, Hkv, d), 1100 + t, torch.bfloat16).to(dev)
        v = normal((B, Hkv, d), 1200 + t, torch.bfloat16).to(dev)
        for l in range(L):
            full.decode_step_fused(l, q, k, v, o_full[l], N + t, scale, ws)
            for r, (c, sh) in enumerate(zip(sc, shards)):
                ol = torch.empty(B, (sh.g1 - sh.g0) * G, d, dtype=torch.bfloat16, device=dev)
                c.decode_step_fused(l, mdist.local_slice_q(q, sh, G).contiguous(),
                                    mdist.local_slice_kv(k, sh).contiguous(), mdist.local_slice_kv(v, sh).contiguous(),
                                    ol, N + t, scale, wss[r])
            for pg in pgs:
                pg.wait(l)
        for pg in pgs:
            pg.next_token()
        torch.cuda.synchronize()
        for r in range(len(shards)):
            assert np.array_equal(bits(outs[r]), bits(o_full)), (t, r)
