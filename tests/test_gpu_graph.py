"""CUDA-graph capture of a decode token step.

A token step = every layer's fused append + decode with DEVICE positions
(moa_decode_step_fused_ragged on uniform layers) followed by moa_advance_pos, captured
once and replayed per token.  The replayed outputs must equal the eager host-position
path bit for bit and the oracle's masked attention over the full history within the bf16
tolerance, and the cache image must be the oracle's, bit for bit, after ring wrap-around.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from tests.gpu_util import bits, check_cache_image, f64
from moa_workloads.inputs import normal

pytestmark = pytest.mark.gpu


def test_graph_token_step_matches_eager_and_oracle(moa):
    dev = torch.device("cuda")
    L, B, N, Hq, Hkv, d, s, T = 2, 3, 300, 8, 4, 128, 8, 70
    G = Hq // Hkv
    Ws = [[40, 7, 300, 0, 33, 32, 1, 64], [17, 17, 200, 90, 5, 0, 260, 11]]
    scale = 1 / math.sqrt(d)
    q = [normal((B, N, Hq, d), 1200 + 10 * l, torch.bfloat16).to(dev) for l in range(L)]
    k = [normal((B, N, Hkv, d), 1201 + 10 * l, torch.bfloat16).to(dev) for l in range(L)]
    v = [normal((B, N, Hkv, d), 1202 + 10 * l, torch.bfloat16).to(dev) for l in range(L)]
    qd = normal((T, L, B, Hq, d), 1300, torch.bfloat16).to(dev)
    kd = normal((T, L, B, Hkv, d), 1301, torch.bfloat16).to(dev)
    vd = normal((T, L, B, Hkv, d), 1302, torch.bfloat16).to(dev)

    def context():
        ctx = moa.MoAContext(L, Hq, Hkv, d, B, dtype=torch.bfloat16)
        for l in range(L):
            ctx.set_spans(l, Ws[l], s, N)
        ctx.alloc_cache(B)
        ws = ctx.alloc_workspace(B)
        for l in range(L):
            ctx.prefill(l, q[l], k[l], v[l], torch.empty_like(q[l]), scale)
        return ctx, ws

    # eager: host positions
    ctx_e, ws_e = context()
    eager = torch.empty(T, L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    for t in range(T):
        for l in range(L):
            ctx_e.decode_step_fused(l, qd[t, l], kd[t, l], vd[t, l], eager[t, l], N + t, scale, ws_e)
    # graph: static input/output buffers, device positions advanced inside the graph
    ctx_g, ws_g = context()
    pos = torch.full((B,), N, dtype=torch.int64, device=dev)
    sq, sk, sv = qd[0].clone(), kd[0].clone(), vd[0].clone()
    so = torch.empty(L, B, Hq, d, dtype=torch.bfloat16, device=dev)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with torch.cuda.graph(graph, stream=side):
            for l in range(L):
                ctx_g.decode_step_fused_ragged(l, sq[l], sk[l], sv[l], so[l], pos, scale, ws_g)
            moa.advance_pos(pos)
    got = torch.empty_like(eager)
    for t in range(T):
        sq.copy_(qd[t]), sk.copy_(kd[t]), sv.copy_(vd[t])
        graph.replay()
        got[t].copy_(so)
    torch.cuda.synchronize()
    assert pos.tolist() == [N + T] * B
    assert np.array_equal(bits(got), bits(eager))
    for l in range(L):
        Kh = torch.cat([k[l], kd[:, l].permute(1, 0, 2, 3)], 1).cpu()
        Vh = torch.cat([v[l], vd[:, l].permute(1, 0, 2, 3)], 1).cpu()
        for t in (0, 31, T - 1):
            Od, _ = oracle.decode(f64(qd[t, l]), f64(Kh[:, :N + t + 1]), f64(Vh[:, :N + t + 1]), N + t, Ws[l], s,
                                  scale)
            assert np.abs(f64(got[t, l]) - Od).max() < 2e-2, (l, t)
        check_cache_image(ctx_g, l, Kh, Vh, N + T - 1, Ws[l], s, B, G)


def test_advance_pos_skips_inactive(moa):
    pos = torch.tensor([5, -1, 0, 7], dtype=torch.int64, device="cuda")
    moa.advance_pos(pos, 3)
    assert pos.tolist() == [8, -1, 3, 10]
    with pytest.raises(moa.MoAError):
        moa.advance_pos(torch.empty(0, dtype=torch.int64, device="cuda"))
