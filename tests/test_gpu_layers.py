"""Cross-layer decode (moa_decode_step_fused_layers) against the oracle
and against the single-layer launches.

One launch appends and decodes the token of every layer of a range: each layer is the decode
step of PAPER.md:704 (fixed span, oldest ring entry replaced) with the per-head masks applied
independently.  Checks, every step and through ring wrap-around:
  * o of every layer vs oracle.decode over the FULL history (2e-2 bf16, north_star);
  * the cache image of every layer vs oracle.cache_image, bitwise;
  * with the rank-invariant split (moa_set_decode_split) o and lse are BITWISE those of the
    single-layer calls (the split, the reduction order and the merge order are functions of
    the region alone);
  * graph capture of a token step after moa_prepare_layers, and the state errors.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import bits, check_cache_image, f64
from moa_workloads.inputs import normal

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _layer_windows(L, Hq, N, seed):
    rng = np.random.default_rng(seed)
    out = []
    for l in range(L):
        w = [int(x) for x in rng.integers(0, N + 8, size=Hq)]
        w[0] = 1 if l % 2 else N + 4   # a minimal and a full-span head
        out.append(w)
    return out


def _setup(moa, L, B, N, Hq, Hkv, d, s, wins, chunk, seed):
    ctx = moa.MoAContext(L, Hq, Hkv, d, B, dtype=torch.bfloat16)
    if chunk:
        ctx.set_decode_split(chunk)
    for l in range(L):
        ctx.set_spans(l, wins[l], s, N)
    ctx.alloc_cache(B)
    dev = torch.device("cuda")
    K = [normal((B, N, Hkv, d), seed + 10 * l + 2, torch.bfloat16) for l in range(L)]
    V = [normal((B, N, Hkv, d), seed + 10 * l + 3, torch.bfloat16) for l in range(L)]
    for l in range(L):
        ctx.cache_fill(l, K[l].to(dev), V[l].to(dev))
    return ctx, K, V


@pytest.mark.parametrize("L,B,N,Hq,Hkv,d,s,chunk,steps", [
    (3, 2, 300, 4, 4, 128, 4, 0, 24),       # MHA, balanced split, wraps of the small windows
    (4, 3, 200, 8, 2, 128, 8, 128, 12),     # GQA G=4, rank-invariant split
    (2, 2, 150, 8, 1, 64, 2, 0, 8),         # G=8, d=64
    (40, 1, 96, 2, 2, 64, 4, 0, 3),         # > 32 layers: two launches per token
])
def test_layers_vs_oracle(L, B, N, Hq, Hkv, d, s, chunk, steps):
    import paper_2406_14909_b200 as moa
    dev = torch.device("cuda")
    G = Hq // Hkv
    wins = _layer_windows(L, Hq, N, 7 + L)
    ctx, K, V = _setup(moa, L, B, N, Hq, Hkv, d, s, wins, chunk, 100)
    ws = ctx.alloc_workspace(B, L)
    scale = 1 / math.sqrt(d)
    qd = normal((steps, L, B, Hq, d), 11, torch.bfloat16)
    kd = normal((steps, L, B, Hkv, d), 12, torch.bfloat16)
    vd = normal((steps, L, B, Hkv, d), 13, torch.bfloat16)
    o = torch.empty(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    lse = torch.empty(L, B, Hq, dtype=torch.float32, device=dev)
    Kh = [torch.cat([K[l], kd[:, l].transpose(0, 1)], 1) for l in range(L)]
    Vh = [torch.cat([V[l], vd[:, l].transpose(0, 1)], 1) for l in range(L)]
    for t in range(steps):
        p = N + t
        ctx.decode_step_fused_layers(0, qd[t].to(dev), kd[t].to(dev), vd[t].to(dev), o, p, scale, ws, lse=lse)
        torch.cuda.synchronize()
        for l in range(L):
            Od, Ld = oracle.decode(f64(qd[t, l]), f64(Kh[l]), f64(Vh[l]), p, wins[l], s, scale)
            err = np.abs(f64(o[l]) - Od).max()
            assert err < TOL, (t, l, err)
            assert np.abs(lse[l].cpu().double().numpy() - Ld).max() < 1e-2, (t, l)
        if t in (0, steps - 1):
            for l in range(L):
                check_cache_image(ctx, l, Kh[l][:, :p + 1], Vh[l][:, :p + 1], p, wins[l], s, B, G)


def test_layers_bitwise_equal_single_layer_calls():
    """Rank-invariant split: the cross-layer launch reproduces the per-layer launches bit for bit."""
    import paper_2406_14909_b200 as moa
    dev = torch.device("cuda")
    L, B, N, Hq, Hkv, d, s, steps = 5, 4, 700, 8, 4, 128, 16, 6
    wins = _layer_windows(L, Hq, N, 3)
    scale = 1 / math.sqrt(d)
    qd = normal((steps, L, B, Hq, d), 21, torch.bfloat16).to(dev)
    kd = normal((steps, L, B, Hkv, d), 22, torch.bfloat16).to(dev)
    vd = normal((steps, L, B, Hkv, d), 23, torch.bfloat16).to(dev)
    c1, _, _ = _setup(moa, L, B, N, Hq, Hkv, d, s, wins, 128, 200)
    c2, _, _ = _setup(moa, L, B, N, Hq, Hkv, d, s, wins, 128, 200)
    ws1, ws2 = c1.alloc_workspace(B), c2.alloc_workspace(B, L)
    o1 = torch.empty(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    o2 = torch.empty_like(o1)
    l1 = torch.empty(L, B, Hq, dtype=torch.float32, device=dev)
    l2 = torch.empty_like(l1)
    for t in range(steps):
        for l in range(L):
            c1.decode_step_fused(l, qd[t, l], kd[t, l], vd[t, l], o1[l], N + t, scale, ws1, lse=l1[l])
        c2.decode_step_fused_layers(0, qd[t], kd[t], vd[t], o2, N + t, scale, ws2, lse=l2)
        torch.cuda.synchronize()
        assert np.array_equal(bits(o1), bits(o2)), t
        assert np.array_equal(bits(l1), bits(l2)), t
    for l in range(L):
        for b in range(B):
            for g in range(Hkv):
                assert torch.equal(c1.cache_rows(l, b, g, "k"), c2.cache_rows(l, b, g, "k"))
                assert torch.equal(c1.cache_rows(l, b, g, "v"), c2.cache_rows(l, b, g, "v"))


def test_layers_subrange_and_graph_capture():
    """A sub-range of layers, then a CUDA-graph captured token step (after prepare_layers)
    replayed with the positions the caller's graph would see."""
    import paper_2406_14909_b200 as moa
    dev = torch.device("cuda")
    L, B, N, Hq, Hkv, d, s = 4, 2, 260, 4, 2, 128, 4
    wins = _layer_windows(L, Hq, N, 5)
    scale = 1 / math.sqrt(d)
    ctx, K, V = _setup(moa, L, B, N, Hq, Hkv, d, s, wins, 0, 300)
    ws = ctx.alloc_workspace(B, L)
    steps = 6
    qd = normal((steps, L, B, Hq, d), 31, torch.bfloat16)
    kd = normal((steps, L, B, Hkv, d), 32, torch.bfloat16)
    vd = normal((steps, L, B, Hkv, d), 33, torch.bfloat16)
    Kh = [torch.cat([K[l], kd[:, l].transpose(0, 1)], 1) for l in range(L)]
    Vh = [torch.cat([V[l], vd[:, l].transpose(0, 1)], 1) for l in range(L)]
    o = torch.zeros(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    # token N: layers 1..3 in one launch, layer 0 alone
    q0, k0, v0 = qd[0].to(dev), kd[0].to(dev), vd[0].to(dev)
    ctx.decode_step_fused(0, q0[0], k0[0], v0[0], o[0], N, scale, ws)
    ctx.decode_step_fused_layers(1, q0[1:], k0[1:], v0[1:], o[1:], N, scale, ws)
    torch.cuda.synchronize()
    for l in range(L):
        Od, _ = oracle.decode(f64(qd[0, l]), f64(Kh[l]), f64(Vh[l]), N, wins[l], s, scale)
        assert np.abs(f64(o[l]) - Od).max() < TOL, l
    # graph of one token step: static input buffers, positions advance per capture
    ctx.prepare_layers()
    sq = torch.empty(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    sk = torch.empty(L, B, Hkv, d, dtype=torch.bfloat16, device=dev)
    sv = torch.empty_like(sk)
    st = torch.cuda.Stream()
    for t in range(1, steps):
        sq.copy_(qd[t]), sk.copy_(kd[t]), sv.copy_(vd[t])
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            ctx.decode_step_fused_layers(0, sq, sk, sv, o, N + t, scale, ws, stream=st)
        g.replay()
        torch.cuda.synchronize()
        for l in range(L):
            Od, _ = oracle.decode(f64(qd[t, l]), f64(Kh[l]), f64(Vh[l]), N + t, wins[l], s, scale)
            assert np.abs(f64(o[l]) - Od).max() < TOL, (t, l)


def test_layers_errors():
    import paper_2406_14909_b200 as moa
    from paper_2406_14909_b200._lib import MoAError
    dev = torch.device("cuda")
    L, B, N, Hq, d, s = 3, 1, 128, 2, 128, 4
    wins = [[8, 16]] * L
    ctx, _, _ = _setup(moa, L, B, N, Hq, Hq, d, s, wins, 0, 400)
    q = torch.zeros(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    kv = torch.zeros(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    o = torch.empty_like(q)
    small = ctx.alloc_workspace(B)        # one layer's worth
    with pytest.raises(MoAError, match="OOM"):
        ctx.decode_step_fused_layers(0, q, kv, kv, o, N, 0.1, small)
    ws = ctx.alloc_workspace(B, L)
    with pytest.raises(MoAError, match="expects"):
        ctx.decode_step_fused_layers(0, q, kv, kv, o, N + 1, 0.1, ws)
    ctx.decode_step_fused(0, q[0], kv[0], kv[0], o[0], N, 0.1, ws)     # layer 0 now expects N + 1
    with pytest.raises(MoAError, match="expects"):
        ctx.decode_step_fused_layers(0, q, kv, kv, o, N, 0.1, ws)
    with pytest.raises(MoAError, match="INVALID_ARG"):
        ctx.decode_step_fused_layers(2, q, kv, kv, o, N, 0.1, ws)       # [2, 5) out of range
    # stale descriptors while capturing -> state error, nothing launched
    ctx.set_spans(1, [8, 16], s, N)   # marks the descriptors stale (same footprint)
    zk = torch.zeros(B, N, Hq, d, dtype=torch.bfloat16, device=dev)
    ctx.cache_fill(1, zk, zk)         # layer 1 expects N again
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with pytest.raises(MoAError, match="prepare_layers"):
        with torch.cuda.graph(g, stream=st):
            ctx.decode_step_fused_layers(1, q[1:], kv[1:], kv[1:], o[1:], N, 0.1, ws, stream=st)
