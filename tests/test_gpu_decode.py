"""GPU parity of the cache kernels and decode path against the fp64 oracle.

Bars (BASELINE.json north_star): max-abs 1e-5 for fp32 I/O, 2e-2 for bf16
I/O; KV-cache images bit-exact.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from moa_workloads import CONFIGS, decode_tokens, normal, prefill_qkv, rule_table
from tests.gpu_util import bits, check_cache_image, f64, rule_windows

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}
LSE_TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-3}


@pytest.fixture(scope="module")
def moa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_14909_b200 as m
    return m


def _decode_run(moa, dtype, B, Hq, Hkv, d, s, windows, T, seed, fused=False, check_every=1,
                prompt=0):
    """Fill the cache by appends from position `prompt` (cache_fill of a
    prompt first if prompt > 0), decode T steps, compare every step."""
    dev = torch.device("cuda")
    G = Hq // Hkv
    ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
    N = max(prompt, 1)
    ctx.set_spans(0, windows, s, N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    total = prompt + T
    K = normal((B, total, Hkv, d), seed + 1, dtype)
    V = normal((B, total, Hkv, d), seed + 2, dtype)
    Qd = normal((T, B, Hq, d), seed + 3, dtype)
    Kg, Vg, Qg = K.to(dev), V.to(dev), Qd.to(dev)
    if prompt:
        ctx.cache_fill(0, Kg[:, :prompt].contiguous(), Vg[:, :prompt].contiguous())
    scale = 1 / math.sqrt(d)
    Kf, Vf = f64(K), f64(V)
    o = torch.empty(B, Hq, d, dtype=dtype, device=dev)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=dev)
    outs = []
    for t in range(T):
        p = prompt + t
        kn, vn = Kg[:, p].contiguous(), Vg[:, p].contiguous()
        if fused:
            ctx.decode_step_fused(0, Qg[t], kn, vn, o, p, scale, ws, lse)
        else:
            ctx.kv_append(0, kn, vn, p)
            ctx.decode_step(0, Qg[t], o, p, scale, ws, lse)
        torch.cuda.synchronize()
        ref, lref = oracle.decode(f64(Qd[t]), Kf[:, : p + 1], Vf[:, : p + 1], p, windows, s, scale)
        err = np.abs(f64(o) - ref).max()
        assert err < TOL[dtype], (t, p, err)
        assert np.abs(f64(lse) - lref).max() < LSE_TOL[dtype], (t, p)
        if t % check_every == 0 or t == T - 1:
            check_cache_image(ctx, 0, K, V, p, windows, s, B, G)
        outs.append(o.clone())
    return torch.stack(outs)


def test_c1_decode_fp32_from_empty_cache(moa):
    """C1 shape (fp32, d=64, s=4, W={16,32,64,256}); 300 positions from 0, so
    the ring of W=16 wraps ~18 times and the W=256 head fills completely."""
    _decode_run(moa, torch.float32, 1, 4, 4, 64, 4, [16, 32, 64, 256], 300, 11, check_every=7)


@pytest.mark.parametrize("d", [64, 128])
def test_gqa_bf16_decode_heterogeneous_group(moa, d):
    """G=4 with different windows inside each group (incl. W=0 sink-only and
    W=1 self-only heads): the group cache holds W_g = max, every head masks
    to its own W_h (reading c10)."""
    W = [0, 1, 5, 40, 17, 3, 64, 2]
    _decode_run(moa, torch.bfloat16, 2, 8, 2, d, 4, W, 160, 21, check_every=9)


@pytest.mark.parametrize("G", [1, 2, 8])
def test_group_sizes_bf16(moa, G):
    Hkv = 2
    W = [(7 * h + 3) % 50 + 1 for h in range(G * Hkv)]
    _decode_run(moa, torch.bfloat16, 3, G * Hkv, Hkv, 128, 3, W, 90, 31 + G, check_every=11)


def test_fused_append_decode_matches_two_calls(moa):
    """moa_decode_step_fused == moa_kv_append + moa_decode_step: both are
    checked against the oracle every step (and the cache image bitwise); the
    fused kernel folds the new token in fp32 outside the tensor-core tile path,
    so the two agree to rounding, not bit for bit (bf16)."""
    W = [9, 33, 2, 70]
    a = _decode_run(moa, torch.bfloat16, 2, 4, 2, 128, 5, W, 120, 41, fused=False, check_every=13)
    b = _decode_run(moa, torch.bfloat16, 2, 4, 2, 128, 5, W, 120, 41, fused=True, check_every=13)
    assert (a.float() - b.float()).abs().max().item() < 2e-2


def test_fused_append_fp32_is_bitwise_equal_to_two_calls(moa):
    W = [9, 33, 2, 70]
    a = _decode_run(moa, torch.float32, 1, 4, 2, 64, 5, W, 90, 43, fused=False, check_every=13)
    b = _decode_run(moa, torch.float32, 1, 4, 2, 64, 5, W, 90, 43, fused=True, check_every=13)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))


def test_cache_fill_then_decode_with_wraps(moa):
    """Prompt of 200 tokens by moa_cache_fill, then 100 decode steps."""
    W = [0, 7, 150, 300, 64, 1]
    _decode_run(moa, torch.float32, 2, 6, 3, 64, 8, W, 100, 51, prompt=200, check_every=10)


def test_structured_window_edge_and_sinks_fp32(moa):
    """Adversarial keys (SURVEY §7 hard part 8): a score spike every 16
    positions, so every window (W in {16,32,64,256}) holds W/16 spikes and an
    off-by-one at the window edge adds or drops a spike (an O(1) change of the
    output); sink keys either dominate (+20) or vanish (-20)."""
    dev = torch.device("cuda")
    B, Hq, Hkv, d, s = 1, 4, 4, 64, 4
    W = [16, 32, 64, 256]
    T = 300
    for sink_score in (20.0, -20.0):
        ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=torch.float32)
        ctx.set_spans(0, W, s, 1)
        ctx.alloc_cache(B)
        ws = ctx.alloc_workspace(B)
        u = torch.zeros(d)
        u[0] = 1.0
        spike = (torch.arange(T) % 16 == 0).float() * 10.0
        K = spike[None, :, None, None] * u
        K = K.expand(B, T, Hkv, d).clone()
        K[:, :s] = sink_score * u
        K = K + 0.01 * normal((B, T, Hkv, d), 7)
        V = normal((B, T, Hkv, d), 8)
        Q = u.expand(T, B, Hq, d).clone()
        Kg, Vg, Qg = K.to(dev), V.to(dev), Q.to(dev)
        o = torch.empty(B, Hq, d, device=dev)
        for p in range(T):
            ctx.kv_append(0, Kg[:, p].contiguous(), Vg[:, p].contiguous(), p)
            ctx.decode_step(0, Qg[p], o, p, 1.0, ws)
            if p % 5 == 0 or p > T - 20:
                torch.cuda.synchronize()
                ref, _ = oracle.decode(f64(Q[p]), f64(K)[:, : p + 1], f64(V)[:, : p + 1], p, W, s, 1.0)
                assert np.abs(f64(o) - ref).max() < 1e-5, (sink_score, p)


# ----------------------------------------------------------------------------------------
# full-size layer shapes (C2, C3, C5), sampled outputs
# ----------------------------------------------------------------------------------------

def _full_layer_decode(moa, name, layer, steps, sample_b, batch=None, fused=True):
    cfg = CONFIGS[name]
    dev = torch.device("cuda")
    B = cfg.batch if batch is None else batch
    t = rule_table(name)
    W = rule_windows(t, layer, cfg.N, cfg.n_sink)
    ctx = moa.MoAContext(1, cfg.hq, cfg.hkv, cfg.head_dim, B, dtype=torch.bfloat16)
    ctx.set_spans(0, W, cfg.n_sink, cfg.N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    seed = cfg.seed_base + 10 * layer
    Kp = normal((B, cfg.N, cfg.hkv, cfg.head_dim), seed + 2, torch.bfloat16, dev)
    Vp = normal((B, cfg.N, cfg.hkv, cfg.head_dim), seed + 3, torch.bfloat16, dev)
    ctx.cache_fill(0, Kp, Vp)
    qd, kd, vd = (x.to(dev) for x in decode_tokens(cfg, layer, steps, batch=B))
    scale = 1 / math.sqrt(cfg.head_dim)
    o = torch.empty(B, cfg.hq, cfg.head_dim, dtype=torch.bfloat16, device=dev)
    Ks = torch.cat([Kp[sample_b], kd[:, sample_b].transpose(0, 1)], dim=1)
    Vs = torch.cat([Vp[sample_b], vd[:, sample_b].transpose(0, 1)], dim=1)
    Kf, Vf = f64(Ks), f64(Vs)
    for st in range(steps):
        p = cfg.N + st
        if fused:
            ctx.decode_step_fused(0, qd[st], kd[st], vd[st], o, p, scale, ws)
        else:
            ctx.kv_append(0, kd[st], vd[st], p)
            ctx.decode_step(0, qd[st], o, p, scale, ws)
        torch.cuda.synchronize()
        ref, _ = oracle.decode(f64(qd[st][sample_b]), Kf[:, : p + 1], Vf[:, : p + 1], p, W, cfg.n_sink, scale)
        err = np.abs(f64(o[sample_b]) - ref).max()
        assert err < 2e-2, (name, st, err)
    # ring + sinks bit-exact for the sampled sequences after the last step
    wg = oracle.group_windows(W, cfg.group)
    img = oracle.cache_image(bits(Ks), bits(Vs), cfg.N + steps - 1, wg, cfg.n_sink)
    for i, b in enumerate(sample_b):
        for g in range(cfg.hkv):
            Ki, Vi, valid = img[(i, g)]
            assert np.array_equal(bits(ctx.cache_rows(0, b, g, "k"))[valid], Ki[valid])
            assert np.array_equal(bits(ctx.cache_rows(0, b, g, "v"))[valid], Vi[valid])


def test_c2_full_layer_decode(moa):
    _full_layer_decode(moa, "C2", 31, 3, [0, 7])


def test_c3_full_layer_decode(moa):
    _full_layer_decode(moa, "C3", 5, 3, [0, 15], fused=False)


def test_c5_full_layer_decode(moa):
    _full_layer_decode(moa, "C5", 70, 2, [31])


def test_decode_state_errors(moa):
    from paper_2406_14909_b200 import MoAError
    ctx = moa.MoAContext(1, 2, 2, 64, 1, dtype=torch.bfloat16)
    ctx.set_spans(0, [4, 4], 1, 8)
    dev = torch.device("cuda")
    q = torch.zeros(1, 2, 64, dtype=torch.bfloat16, device=dev)
    kn = torch.zeros(1, 2, 64, dtype=torch.bfloat16, device=dev)
    with pytest.raises(MoAError, match="STATE"):
        ctx.kv_append(0, kn, kn, 0)                  # no cache bound
    ctx.alloc_cache(1)
    ws = ctx.alloc_workspace(1)
    with pytest.raises(MoAError, match="STATE"):
        ctx.kv_append(0, kn, kn, 3)                  # not the next position
    ctx.kv_append(0, kn, kn, 0)
    with pytest.raises(MoAError, match="STATE"):
        ctx.decode_step(0, q, q.clone(), 1, 0.1, ws)  # not yet appended
    with pytest.raises(MoAError, match="OOM"):
        ctx.decode_step(0, q, q.clone(), 0, 0.1, ws[:8])
    ctx.decode_step(0, q, q.clone(), 0, 0.1, ws)
    torch.cuda.synchronize()


def test_multilayer_stream_overlap_no_sync(moa):
    """Decode launches of several layers back to back with no host sync, as a
    model would issue them: q/k_new/v_new are written into REUSED buffers by a
    torch kernel right before every launch and o is copied out right after,
    so a decode that read its inputs (or wrote o) before its predecessor
    finished, or streamed a cache the predecessor was still writing, fails.
    Covers the early cache streaming between layers (include/moa.h) and the
    full-wait path (kv_append + decode_step of the same layer)."""
    dev = torch.device("cuda")
    dtype = torch.bfloat16
    L, B, Hq, Hkv, d, s, N, T = 3, 2, 8, 4, 128, 4, 300, 40
    G = Hq // Hkv
    wins = [[1, 37, 128, 0, 299, 64, 5, 200], [300, 300, 10, 10, 90, 91, 2, 3], [0, 0, 64, 65, 17, 250, 130, 1]]
    ctx = moa.MoAContext(L, Hq, Hkv, d, B, dtype=dtype)
    for l in range(L):
        ctx.set_spans(l, wins[l], s, N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    scale = 1 / math.sqrt(d)
    K = [normal((B, N + T, Hkv, d), 700 + 10 * l, dtype) for l in range(L)]
    V = [normal((B, N + T, Hkv, d), 701 + 10 * l, dtype) for l in range(L)]
    Q = [normal((T, B, Hq, d), 702 + 10 * l, dtype) for l in range(L)]
    Kg, Vg, Qg = [x.to(dev) for x in K], [x.to(dev) for x in V], [x.to(dev) for x in Q]
    for l in range(L):
        ctx.cache_fill(l, Kg[l][:, :N].contiguous(), Vg[l][:, :N].contiguous())
    qbuf = torch.empty(B, Hq, d, dtype=dtype, device=dev)
    kbuf = torch.empty(B, Hkv, d, dtype=dtype, device=dev)
    vbuf = torch.empty(B, Hkv, d, dtype=dtype, device=dev)
    obuf = torch.empty(B, Hq, d, dtype=dtype, device=dev)
    out = torch.empty(T, L, B, Hq, d, dtype=dtype, device=dev)
    for t in range(T):
        p = N + t
        for l in range(L):
            qbuf.copy_(Qg[l][t])
            kbuf.copy_(Kg[l][:, p])
            vbuf.copy_(Vg[l][:, p])
            if l == 1 and t % 2:   # the two-call path of the same layer: the decode must fully wait
                ctx.kv_append(l, kbuf, vbuf, p)
                ctx.decode_step(l, qbuf, obuf, p, scale, ws)
            else:
                ctx.decode_step_fused(l, qbuf, kbuf, vbuf, obuf, p, scale, ws)
            out[t, l].copy_(obuf)
    torch.cuda.synchronize()
    for l in range(L):
        Kf, Vf = f64(K[l]), f64(V[l])
        for t in range(T):
            p = N + t
            ref, _ = oracle.decode(f64(Q[l][t]), Kf[:, : p + 1], Vf[:, : p + 1], p, wins[l], s, scale)
            err = np.abs(f64(out[t, l]) - ref).max()
            assert err < TOL[dtype], (l, t, err)
        check_cache_image(ctx, l, K[l], V[l], N + T - 1, wins[l], s, B, G)


@pytest.mark.parametrize("G", [1, 4])
def test_structured_window_edge_and_sinks_bf16_tensor_core(moa, G):
    """The adversarial test above on the bf16 tensor-core decode (fused append): a score spike
    every 16 positions (an off-by-one at any head's window edge adds or drops a spike: an O(1)
    change) and dominant / vanishing sinks, windows spanning several 64-row tiles, GQA with
    per-head windows inside the group, 300 positions so every ring wraps."""
    dev = torch.device("cuda")
    B, Hkv, d, s, T = 2, 2, 128, 64, 300
    Hq = Hkv * G
    W = ([16, 48, 112, 200] * 2)[:Hq] if G > 1 else [16, 112]
    dtype = torch.bfloat16
    for sink_score in (12.0, -12.0):
        ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
        ctx.set_spans(0, W, s, 1)
        ctx.alloc_cache(B)
        ws = ctx.alloc_workspace(B)
        u = torch.zeros(d)
        u[0] = 1.0
        spike = (torch.arange(T) % 16 == 0).float() * 8.0
        K = (spike[None, :, None, None] * u).expand(B, T, Hkv, d).clone()
        K[:, :s] = sink_score * u
        K = (K + 0.01 * normal((B, T, Hkv, d), 9)).to(dtype)
        V = normal((B, T, Hkv, d), 10, dtype)
        Q = u.expand(T, B, Hq, d).clone().to(dtype)
        Kg, Vg, Qg = K.to(dev), V.to(dev), Q.to(dev)
        o = torch.empty(B, Hq, d, dtype=dtype, device=dev)
        Kf, Vf = f64(K), f64(V)
        for p in range(T):
            ctx.decode_step_fused(0, Qg[p], Kg[:, p].contiguous(), Vg[:, p].contiguous(), o, p, 1.0, ws)
            if p % 7 == 0 or p > T - 20:
                torch.cuda.synchronize()
                ref, _ = oracle.decode(f64(Q[p]), Kf[:, : p + 1], Vf[:, : p + 1], p, W, s, 1.0)
                assert np.abs(f64(o) - ref).max() < 2e-2, (sink_score, p)
        check_cache_image(ctx, 0, K, V, T - 1, W, s, B, G)
