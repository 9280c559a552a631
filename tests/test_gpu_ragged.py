"""GPU parity of ragged batches against the fp64 oracle.

A ragged batch is padded to the layer's N; sequence b is the prompt of its first N_b
rows with its own spans (Eq. 2 at N_b).  Prefill (tcgen05 bf16 and FFMA
fp32 kernels, token and block masks), the ragged cache fill, and fused append+decode
at per-sequence positions (device pos array, incl. an inactive sequence) are compared
element by element with oracle.prefill_ragged / oracle.decode_ragged, and the cache
images bitwise with the oracle's image of every sequence.  Bars as the other parity
tests (BASELINE.json north_star): 1e-5 fp32 I/O, 2e-2 bf16 I/O.
"""
import math

import numpy as np
import pytest
import torch

import oracle
from moa_workloads import normal
from tests.gpu_util import bits, f64, rule_windows

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}
LSE_TOL = {torch.float32: 1e-5, torch.bfloat16: 1e-3}


@pytest.fixture(scope="module")
def moa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_14909_b200 as m
    return m


def _ragged_windows(alpha, beta, lens, s, cap):
    """Eq. 2 at every sequence's own length, clipped to the capacity (the spans at the
    padded length) -- equal for beta >= 0 (test_spans_shrink_with_length...)."""
    out = []
    for n in lens:
        w = [oracle.window_of(oracle.span_of(a, b, n), s) for a, b in zip(alpha, beta)]
        out.append([min(x, c) for x, c in zip(w, cap)])
    return out


def _prefill_case(moa, dtype, B, N, lens, Hq, Hkv, d, s, alpha, beta, seed, block=0, wins=None):
    dev = torch.device("cuda")
    cap = [oracle.window_of(oracle.span_of(a, b, N), s) for a, b in zip(alpha, beta)]
    if wins is None:
        wins = _ragged_windows(alpha, beta, lens, s, cap)
    ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
    ctx.set_spans(0, cap, s, N, block=block)
    ctx.set_ragged(0, lens, wins)
    Q = normal((B, N, Hq, d), seed, dtype)
    K = normal((B, N, Hkv, d), seed + 1, dtype)
    V = normal((B, N, Hkv, d), seed + 2, dtype)
    for b, n in enumerate(lens):  # padding: any finite values (header contract), here large ones
        Q[b, n:] = 3.0e4
        K[b, n:] = -3.0e4
        V[b, n:] = 3.0e4
    o = torch.full((B, N, Hq, d), 7.0, dtype=dtype, device=dev)  # sentinel: rows >= N_b untouched
    lse = torch.full((B, Hq, N), 7.0, dtype=torch.float32, device=dev)
    tau = 1 / math.sqrt(d)
    ctx.prefill_attn(0, Q.to(dev), K.to(dev), V.to(dev), o, tau, lse)
    torch.cuda.synchronize()
    ref, lref = oracle.prefill_ragged(f64(Q), f64(K), f64(V), lens, wins, s, tau, block)
    og, lg = f64(o), f64(lse)
    for b, n in enumerate(lens):
        err = np.abs(og[b, :n] - ref[b, :n]).max()
        assert err < TOL[dtype], (b, n, err)
        assert np.abs(lg[b, :, :n] - lref[b, :, :n]).max() < LSE_TOL[dtype], b
        assert np.all(og[b, n:] == 7.0) and np.all(lg[b, :, n:] == 7.0), f"rows past N_{b} written"
    return ctx, wins


@pytest.mark.parametrize("d", [64, 128])
def test_ragged_prefill_bf16_token_mask(moa, d):
    """tcgen05 kernel; lengths span several 128-row tiles, a ragged tail, a sequence
    shorter than one tile and one of a single token; GQA group 4 with heterogeneous
    elastic rules (one W = 0 head, one full-span head)."""
    alpha = [16.0, 40.0, 0.0, 500.0, 8.0, 100.0, 4.0, 64.0]
    beta = [0.05, 0.1, 0.0, 1.0, 0.25, 0.0, 0.5, 0.2]
    _prefill_case(moa, torch.bfloat16, 4, 700, [700, 333, 129, 1], 8, 2, d, 4, alpha, beta, 100 + d)


def test_ragged_prefill_fp32(moa):
    alpha = [16.0, 40.0, 0.0, 300.0]
    beta = [0.05, 0.1, 0.0, 1.0]
    _prefill_case(moa, torch.float32, 3, 300, [300, 201, 64], 4, 2, 64, 4, alpha, beta, 200)


def test_ragged_prefill_bf16_block_mask(moa):
    """The paper's block-64 mask with per-sequence block-multiple windows."""
    B, N, s = 3, 640, 64
    alpha, beta = [128.0, 512.0, 64.0, 640.0], [0.0, 0.0, 0.0, 0.0]  # caps 64, 448, 0, 576
    lens = [640, 300, 65]
    wins = [[64, 448, 0, 576], [0, 192, 0, 64], [64, 64, 0, 0]]
    _prefill_case(moa, torch.bfloat16, B, N, lens, 4, 1, 128, s, alpha, beta, 300, block=64, wins=wins)


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_ragged_fill_then_decode(moa, dtype):
    """moa_prefill (attention + ragged cache fill), then fused append+decode at
    per-sequence positions held in a device tensor the test advances; sequence 3 is
    inactive (pos = -1) for the first steps and must leave its cache untouched."""
    dev = torch.device("cuda")
    B, N, Hq, Hkv, d, s, T = 4, 260, 8, 2, 128 if dtype == torch.bfloat16 else 64, 4, 40
    lens = [260, 150, 9, 77]
    alpha = [16.0, 40.0, 0.0, 500.0, 8.0, 100.0, 4.0, 64.0]
    beta = [0.05, 0.1, 0.0, 1.0, 0.25, 0.0, 0.5, 0.2]
    cap = [oracle.window_of(oracle.span_of(a, b, N), s) for a, b in zip(alpha, beta)]
    wins = _ragged_windows(alpha, beta, lens, s, cap)
    ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
    ctx.set_spans(0, cap, s, N)
    ctx.set_ragged(0, lens, wins)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    total = N + T
    Q = normal((B, N, Hq, d), 400, dtype)
    Kh = normal((B, total, Hkv, d), 401, dtype)  # history: row p = position p of each sequence
    Vh = normal((B, total, Hkv, d), 402, dtype)
    Qd = normal((T, B, Hq, d), 403, dtype)
    tau = 1 / math.sqrt(d)
    o = torch.empty(B, N, Hq, d, dtype=dtype, device=dev)
    ctx.prefill(0, Q.to(dev), Kh[:, :N].contiguous().to(dev), Vh[:, :N].contiguous().to(dev), o, tau)
    # decode inputs: the token at position pos_b of sequence b
    Kf, Vf = f64(Kh), f64(Vh)
    pos = torch.tensor(lens, dtype=torch.int64, device=dev)
    inactive_until = 5
    pos[3] = -1
    od = torch.empty(B, Hq, d, dtype=dtype, device=dev)
    lse = torch.empty(B, Hq, dtype=torch.float32, device=dev)
    G = Hq // Hkv
    for t in range(T):
        if t == inactive_until:
            pos[3] = lens[3]
        ph = pos.cpu().tolist()
        kn = torch.stack([Kh[b, max(p, 0)] for b, p in enumerate(ph)]).to(dev)
        vn = torch.stack([Vh[b, max(p, 0)] for b, p in enumerate(ph)]).to(dev)
        ctx.decode_step_fused_ragged(0, Qd[t].to(dev), kn, vn, od, pos, tau, ws, lse)
        torch.cuda.synchronize()
        ref, lref = oracle.decode_ragged(f64(Qd[t]), Kf, Vf, ph, wins, s, tau)
        err = np.abs(f64(od) - ref).max()
        assert err < TOL[dtype], (t, ph, err)
        lg = f64(lse)
        fin = np.isfinite(lref)
        assert np.array_equal(np.isfinite(lg), fin)
        assert np.abs(lg[fin] - lref[fin]).max() < LSE_TOL[dtype], t
        if t in (0, inactive_until - 1, inactive_until, T - 1):
            # cache image of every sequence at its own position (inactive: still its prompt)
            wg = oracle.group_windows(cap, G)
            for b, p in enumerate(ph):
                last = p if p >= 0 else lens[b] - 1
                img = oracle.cache_image(bits(Kh[b:b + 1]), bits(Vh[b:b + 1]), last, wg, s)
                for g in range(Hkv):
                    Ki, Vi, valid = img[(0, g)]
                    assert np.array_equal(bits(ctx.cache_rows(0, b, g, "k"))[valid], Ki[valid]), (t, b, g)
                    assert np.array_equal(bits(ctx.cache_rows(0, b, g, "v"))[valid], Vi[valid]), (t, b, g)
        pos += (pos >= 0).to(torch.int64)


def test_ragged_layer_refuses_uniform_decode(moa):
    from paper_2406_14909_b200 import MoAError
    dev = torch.device("cuda")
    ctx = moa.MoAContext(1, 2, 1, 64, 2, dtype=torch.bfloat16)
    ctx.set_spans(0, [8, 8], 4, 32)
    ctx.set_ragged(0, [32, 10])
    ctx.alloc_cache(2)
    ws = ctx.alloc_workspace(2)
    q = torch.zeros(2, 2, 64, dtype=torch.bfloat16, device=dev)
    kn = torch.zeros(2, 1, 64, dtype=torch.bfloat16, device=dev)
    with pytest.raises(MoAError, match="STATE"):
        ctx.decode_step_fused(0, q, kn, kn, q.clone(), 0, 0.1, ws)
    with pytest.raises(MoAError, match="STATE"):
        ctx.kv_append(0, kn, kn, 0)


def test_c2_full_layer_ragged_prefill_and_decode(moa):
    """A full C2 layer (B=8, N=4096, 32 heads, d=128, 64 sinks) as a ragged batch with
    N_b uniform in [N/4, N] and Eq. 2 windows at N_b (the launch configuration of
    tools/time_ragged.py): sampled rows of every sequence vs oracle.prefill_rows on the
    truncated sequence, the ragged cache images bitwise, then 3 fused ragged decode steps
    vs oracle.decode on sampled sequences."""
    from moa_workloads import CONFIGS, prefill_qkv, rule_table
    cfg = CONFIGS["C2"]
    dev = torch.device("cuda")
    B, N, s, d, layer = cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim, 20
    t = rule_table("C2")
    rng = np.random.default_rng(7)
    lens = rng.integers(N // 4, N + 1, size=B).tolist()
    lens[1] = N
    cap = rule_windows(t, layer, N, s)
    wins = [[min(w, c) for w, c in zip(rule_windows(t, layer, n, s), cap)]
            for n in lens]
    ctx = moa.MoAContext(1, cfg.hq, cfg.hkv, d, B)
    ctx.set_spans(0, cap, s, N)
    ctx.set_ragged(0, lens, wins)
    ctx.alloc_cache(B)
    q, k, v = prefill_qkv(cfg, layer, device=dev)
    o = torch.empty_like(q)
    lse = torch.empty(B, cfg.hq, N, dtype=torch.float32, device=dev)
    tau = 1 / math.sqrt(d)
    ctx.prefill(0, q, k, v, o, tau, lse)
    torch.cuda.synchronize()
    for b in (0, 1, B - 1):
        n = lens[b]
        rows = []
        for h in range(0, cfg.hq, 3):
            W = wins[b][h]
            base = {0, s - 1, s, W - 1, W, W + 1, 127, 128, n - 2, n - 1}
            base |= set(int(x) for x in rng.integers(0, n, 4))
            rows += [(0, h, i) for i in sorted(base) if 0 <= i < n]
        O, L = oracle.prefill_rows(f64(q[b:b + 1, :n]), f64(k[b:b + 1, :n]), f64(v[b:b + 1, :n]), wins[b], s, tau,
                                   rows)
        got = np.stack([f64(o[b, i, h]) for _, h, i in rows])
        gl = np.array([float(lse[b, h, i]) for _, h, i in rows])
        assert np.abs(got - O).max() < 2e-2, b
        assert np.abs(gl - L).max() < 2e-3, b
        wg = oracle.group_windows(cap, cfg.group)
        img = oracle.cache_image(bits(k[b:b + 1, :n]), bits(v[b:b + 1, :n]), n - 1, wg, s)
        for g in range(0, cfg.hkv, 5):
            Ki, Vi, valid = img[(0, g)]
            assert np.array_equal(bits(ctx.cache_rows(0, b, g, "k"))[valid], Ki[valid]), (b, g)
            assert np.array_equal(bits(ctx.cache_rows(0, b, g, "v"))[valid], Vi[valid]), (b, g)
    # decode: new tokens at positions N_b (history = prompt rows + the new rows)
    ws = ctx.alloc_workspace(B)
    pos = torch.tensor(lens, dtype=torch.int64, device=dev)
    od = torch.empty(B, cfg.hq, d, dtype=torch.bfloat16, device=dev)
    T = 3
    kq = normal((T, B, cfg.hq, d), 77, torch.bfloat16)
    kn = normal((T, B, cfg.hkv, d), 78, torch.bfloat16)
    vn = normal((T, B, cfg.hkv, d), 79, torch.bfloat16)
    for t_ in range(T):
        ctx.decode_step_fused_ragged(0, kq[t_].to(dev), kn[t_].to(dev), vn[t_].to(dev), od, pos, tau, ws)
        torch.cuda.synchronize()
        for b in (0, 1, B - 1):
            n = lens[b]
            Kh = np.concatenate([f64(k[b:b + 1, :n]), f64(kn[:t_ + 1, b]).reshape(1, t_ + 1, cfg.hkv, d)], 1)
            Vh = np.concatenate([f64(v[b:b + 1, :n]), f64(vn[:t_ + 1, b]).reshape(1, t_ + 1, cfg.hkv, d)], 1)
            ref, _ = oracle.decode(f64(kq[t_, b:b + 1]), Kh, Vh, n + t_, wins[b], s, tau)
            assert np.abs(f64(od[b:b + 1]) - ref).max() < 2e-2, (t_, b)
        pos += 1


def test_ragged_kv_sharded_contexts_on_one_gpu(moa):
    """Two contexts serving kv-groups [0,2) and [2,4) of a ragged batch (each keeps its
    heads' columns of the full [B][Hq] window table), on head-sliced views: prefill and a
    fused ragged decode step, concatenated by heads, equal the oracle for all heads."""
    from paper_2406_14909_b200 import dist as mdist
    dev = torch.device("cuda")
    B, N, Hq, Hkv, d, s = 3, 300, 8, 4, 128, 4
    cap = [3, 200, 0, 77, 128, 129, 1, 300]
    lens = [300, 140, 33]
    wins = [cap, [3, 100, 0, 60, 128, 20, 1, 140], [0, 33, 0, 5, 10, 29, 1, 33]]
    G = Hq // Hkv
    q = normal((B, N, Hq, d), 311, torch.bfloat16)
    k = normal((B, N + 1, Hkv, d), 312, torch.bfloat16)
    v = normal((B, N + 1, Hkv, d), 313, torch.bfloat16)
    qd = normal((B, Hq, d), 314, torch.bfloat16)
    qg, qdg = q.to(dev), qd.to(dev)
    kg, vg = k[:, :N].contiguous().to(dev), v[:, :N].contiguous().to(dev)
    # decode token of sequence b sits at position N_b
    kd = torch.stack([k[b, n] for b, n in enumerate(lens)]).to(dev)
    vd = torch.stack([v[b, n] for b, n in enumerate(lens)]).to(dev)
    o = torch.empty_like(qg)
    od = torch.empty_like(qdg)
    pos = torch.tensor(lens, dtype=torch.int64, device=dev)
    tau = 1 / math.sqrt(d)
    for sh in mdist.plan_shards(2, Hkv, B, "kv"):
        ctx = mdist.make_context(sh, 1, Hq, Hkv, d, device=0)
        ctx.set_spans(0, cap, s, N)
        ctx.set_ragged(0, lens, wins)
        ctx.alloc_cache(B)
        ws = ctx.alloc_workspace(B)
        ctx.prefill(0, mdist.local_slice_q(qg, sh, G), mdist.local_slice_kv(kg, sh), mdist.local_slice_kv(vg, sh),
                    mdist.local_slice_q(o, sh, G), tau)
        ctx.decode_step_fused_ragged(0, mdist.local_slice_q(qdg, sh, G), mdist.local_slice_kv(kd, sh),
                                     mdist.local_slice_kv(vd, sh), mdist.local_slice_q(od, sh, G), pos, tau, ws)
    torch.cuda.synchronize()
    O, _ = oracle.prefill_ragged(f64(q), f64(k[:, :N]), f64(v[:, :N]), lens, wins, s, tau)
    for b, n in enumerate(lens):
        assert np.abs(f64(o)[b, :n] - O[b, :n]).max() < 2e-2, b
    Od, _ = oracle.decode_ragged(f64(qd), f64(k), f64(v), lens, wins, s, tau)
    assert np.abs(f64(od) - Od).max() < 2e-2
