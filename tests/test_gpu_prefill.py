"""GPU parity of moa_prefill (+ the cache fill it performs) against the oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
from moa_workloads import CONFIGS, normal, prefill_qkv, rule_table
from tests.gpu_util import bits, check_cache_image, f64, rule_windows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def moa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_14909_b200 as m
    return m


def _prefill(moa, q, k, v, W, s, dtype, scale=None, ctx_batch=None, block=0):
    dev = torch.device("cuda")
    B, N, Hq, d = q.shape
    Hkv = k.shape[2]
    ctx = moa.MoAContext(1, Hq, Hkv, d, ctx_batch or B, dtype=dtype)
    ctx.set_spans(0, W, s, N, block=block)
    ctx.alloc_cache(B)
    qg, kg, vg = q.to(dev), k.to(dev), v.to(dev)
    o = torch.full_like(qg, float("nan"))
    lse = torch.empty(B, Hq, N, dtype=torch.float32, device=dev)
    scale = 1 / math.sqrt(d) if scale is None else scale
    ctx.prefill(0, qg, kg, vg, o, scale, lse)
    torch.cuda.synchronize()
    return ctx, o, lse, scale


def test_c1_prefill_fp32_full(moa):
    """C1 in full: 1 layer, 4 heads, d=64, N=256, W={16,32,64,256}, s=4, fp32."""
    cfg = CONFIGS["C1"]
    q, k, v = prefill_qkv(cfg, 0)
    W = list(cfg.windows)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, cfg.n_sink, torch.float32)
    O, L = oracle.prefill(f64(q), f64(k), f64(v), W, cfg.n_sink, scale)
    assert np.abs(f64(o) - O).max() < 1e-5
    assert np.abs(f64(lse) - L).max() < 1e-5
    check_cache_image(ctx, 0, k, v, cfg.N - 1, W, cfg.n_sink, 1, 1)


@pytest.mark.parametrize("N", [1, 5, 127, 129, 300])
def test_prefill_fp32_ragged_gqa(moa, N):
    """Ragged tails (N not a multiple of the 128-row tile), tiny N, GQA with
    intra-group heterogeneity, W = 0 sink-only heads and W > N."""
    B, Hq, Hkv, d, s = 2, 6, 3, 64, 3
    W = [0, 1, 70, 129, 2, N + 7]
    q = normal((B, N, Hq, d), 101)
    k = normal((B, N, Hkv, d), 102)
    v = normal((B, N, Hkv, d), 103)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, s, torch.float32)
    O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale)
    assert np.abs(f64(o) - O).max() < 1e-5
    assert np.abs(f64(lse) - L).max() < 1e-5
    check_cache_image(ctx, 0, k, v, N - 1, W, s, B, 2)


def test_prefill_fp32_structured(moa):
    """Spike keys every 16 positions + dominant / vanishing sinks (cf. the
    decode structured test): window-edge and sink errors become O(1)."""
    B, N, H, d, s = 1, 256, 4, 64, 4
    W = [16, 32, 64, 256]
    u = torch.zeros(d)
    u[0] = 1.0
    for sink_score in (20.0, -20.0):
        spike = (torch.arange(N) % 16 == 0).float() * 10.0
        k = (spike[None, :, None, None] * u).expand(B, N, H, d).clone()
        k[:, :s] = sink_score * u
        k = k + 0.01 * normal((B, N, H, d), 5)
        v = normal((B, N, H, d), 6)
        q = u.expand(B, N, H, d).clone()
        ctx, o, lse, _ = _prefill(moa, q, k, v, W, s, torch.float32, scale=1.0)
        O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, 1.0)
        assert np.abs(f64(o) - O).max() < 1e-5


# ----------------------------------------------------------------------------------------
# bf16: the tcgen05 tensor-core kernel
# ----------------------------------------------------------------------------------------

@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("N", [100, 300, 513])
def test_prefill_bf16_small_full_compare(moa, d, N):
    B, Hq, Hkv, s = 2, 6, 3, 4
    W = [0, 1, 130, 257, 17, N + 3]
    q = normal((B, N, Hq, d), 201, torch.bfloat16)
    k = normal((B, N, Hkv, d), 202, torch.bfloat16)
    v = normal((B, N, Hkv, d), 203, torch.bfloat16)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, s, torch.bfloat16)
    O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale)
    err = np.abs(f64(o) - O)
    assert np.isfinite(f64(o)).all()
    assert err.max() < 2e-2, (err.max(), np.unravel_index(err.argmax(), err.shape))
    assert np.abs(f64(lse) - L).max() < 2e-3
    check_cache_image(ctx, 0, k, v, N - 1, W, s, B, 2)


def test_prefill_bf16_structured(moa):
    B, N, H, d, s = 1, 640, 4, 128, 64
    W = [16, 200, 300, 640]
    u = torch.zeros(d)
    u[0] = 1.0
    for sink_score in (12.0, -12.0):
        spike = (torch.arange(N) % 16 == 0).float() * 8.0
        k = (spike[None, :, None, None] * u).expand(B, N, H, d).clone()
        k[:, :s] = sink_score * u
        k = (k + 0.01 * normal((B, N, H, d), 5)).to(torch.bfloat16)
        v = normal((B, N, H, d), 6, torch.bfloat16)
        q = u.expand(B, N, H, d).clone().to(torch.bfloat16)
        ctx, o, lse, _ = _prefill(moa, q, k, v, W, s, torch.bfloat16, scale=1.0)
        O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, 1.0)
        assert np.abs(f64(o) - O).max() < 2e-2, sink_score


def _sample_rows(B, Hq, N, s, W, rng, n_rand=24):
    rows = []
    for b in sorted(set([0, B - 1])):
        for h in range(Hq):
            base = {0, s - 1, s, W[h] - 1, W[h], W[h] + 1, N - 1, N - 2, 127, 128}
            base |= set(int(x) for x in rng.integers(0, N, n_rand // 4))
            rows += [(b, h, i) for i in sorted(base) if 0 <= i < N]
    return rows


def _full_layer_prefill(moa, name, layer, batch=None, block=0):
    cfg = CONFIGS[name]
    dev = torch.device("cuda")
    B = cfg.batch if batch is None else batch
    t = rule_table(name)
    W = rule_windows(t, layer, cfg.N, cfg.n_sink)
    q, k, v = prefill_qkv(cfg, layer, batch=B, device=dev)
    ctx = moa.MoAContext(1, cfg.hq, cfg.hkv, cfg.head_dim, B, dtype=torch.bfloat16)
    ctx.set_spans(0, W, cfg.n_sink, cfg.N, block=block)
    ctx.alloc_cache(B)
    o = torch.empty_like(q)
    lse = torch.empty(B, cfg.hq, cfg.N, dtype=torch.float32, device=dev)
    scale = 1 / math.sqrt(cfg.head_dim)
    ctx.prefill(0, q, k, v, o, scale, lse)
    torch.cuda.synchronize()
    rng = np.random.default_rng(layer)
    rows = _sample_rows(B, cfg.hq, cfg.N, cfg.n_sink, W, rng)
    bs = sorted(set(r[0] for r in rows))
    qs, ks, vs = f64(q[bs]), f64(k[bs]), f64(v[bs])
    remap = {b: i for i, b in enumerate(bs)}
    O, L = oracle.prefill_rows(qs, ks, vs, W, cfg.n_sink, scale, [(remap[b], h, i) for b, h, i in rows],
                               block=block)
    got = np.stack([f64(o[b, i, h]) for b, h, i in rows])
    gl = np.array([float(lse[b, h, i]) for b, h, i in rows])
    assert np.abs(got - O).max() < 2e-2
    assert np.abs(gl - L).max() < 2e-3
    # the cache fill of the same call, bitwise, for the sampled sequences
    wg = oracle.group_windows(W, cfg.group)
    img = oracle.cache_image(bits(k[bs]), bits(v[bs]), cfg.N - 1, wg, cfg.n_sink)
    for bi, b in enumerate(bs):
        for g in range(cfg.hkv):
            Ki, Vi, valid = img[(bi, g)]
            assert np.array_equal(bits(ctx.cache_rows(0, b, g, "k"))[valid], Ki[valid])
            assert np.array_equal(bits(ctx.cache_rows(0, b, g, "v"))[valid], Vi[valid])


def test_c2_full_layer_prefill(moa):
    _full_layer_prefill(moa, "C2", 20)


def test_c3_gqa_prefill_slice(moa):
    _full_layer_prefill(moa, "C3", 9, batch=2)


def test_c4_full_layer_prefill(moa):
    _full_layer_prefill(moa, "C4", 33)


def test_kv_sharded_contexts_on_one_gpu(moa):
    """Two contexts serving kv-groups [0,2) and [2,4) on head-sliced views of
    full tensors (row strides of the full layout): prefill and decode outputs
    of the shards, concatenated by heads, equal the oracle for all heads."""
    from paper_2406_14909_b200 import dist as mdist
    dev = torch.device("cuda")
    B, N, Hq, Hkv, d, s = 2, 300, 8, 4, 128, 4
    W = [3, 200, 0, 77, 128, 129, 1, 300]
    G = Hq // Hkv
    q = normal((B, N, Hq, d), 301, torch.bfloat16)
    k = normal((B, N, Hkv, d), 302, torch.bfloat16)
    v = normal((B, N, Hkv, d), 303, torch.bfloat16)
    qd = normal((B, Hq, d), 304, torch.bfloat16)
    kd = normal((B, Hkv, d), 305, torch.bfloat16)
    vd = normal((B, Hkv, d), 306, torch.bfloat16)
    qg, kg, vg, qdg, kdg, vdg = (x.to(dev) for x in (q, k, v, qd, kd, vd))
    o = torch.empty_like(qg)
    od = torch.empty_like(qdg)
    scale = 1 / math.sqrt(d)
    for sh in mdist.plan_shards(2, Hkv, B, "kv"):
        ctx = mdist.make_context(sh, 1, Hq, Hkv, d, device=0)
        ctx.set_spans(0, W, s, N)
        ctx.alloc_cache(B)
        ws = ctx.alloc_workspace(B)
        ctx.prefill(0, mdist.local_slice_q(qg, sh, G), mdist.local_slice_kv(kg, sh), mdist.local_slice_kv(vg, sh),
                    mdist.local_slice_q(o, sh, G), scale)
        ctx.decode_step_fused(0, mdist.local_slice_q(qdg, sh, G), mdist.local_slice_kv(kdg, sh),
                              mdist.local_slice_kv(vdg, sh), mdist.local_slice_q(od, sh, G), N, scale, ws)
    torch.cuda.synchronize()
    O, _ = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale)
    assert np.abs(f64(o) - O).max() < 2e-2
    Kh, Vh = torch.cat([k, kd[:, None]], 1), torch.cat([v, vd[:, None]], 1)
    Od, _ = oracle.decode(f64(qd), f64(Kh), f64(Vh), N, W, s, scale)
    assert np.abs(f64(od) - Od).max() < 2e-2


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
def test_prefill_attn_plus_cache_fill_equals_prefill(moa, dtype):
    """moa_prefill_attn + moa_cache_fill is moa_prefill (include/moa.h): the same
    kernel, so outputs are bitwise equal; prefill_attn needs no bound cache and
    leaves the decode position alone."""
    B, N, Hq, Hkv, d, s = 2, 300, 4, 2, 128, 4
    W = [3, 140, 0, 290]
    q, k, v = (normal((B, N, h, d), 300 + i, dtype).cuda() for i, h in enumerate((Hq, Hkv, Hkv)))
    _, ref, _, scale = _prefill(moa, q.cpu(), k.cpu(), v.cpu(), W, s, dtype)
    ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
    ctx.set_spans(0, W, s, N)
    o = torch.full_like(q, float("nan"))
    ctx.prefill_attn(0, q, k, v, o, scale)         # no cache bound: allowed
    torch.cuda.synchronize()
    assert np.array_equal(bits(o), bits(ref))
    ctx.alloc_cache(B)
    assert ctx.next_pos(0) == 0
    ctx.prefill_attn(0, q, k, v, o, scale)
    assert ctx.next_pos(0) == 0
    ctx.cache_fill(0, k, v)
    torch.cuda.synchronize()
    assert ctx.next_pos(0) == N
    check_cache_image(ctx, 0, k.cpu(), v.cpu(), N - 1, W, s, B, 2)


# ----------------------------------------------------------------------------------------
# block mode: the paper's block sliding-window prefill mask
# ----------------------------------------------------------------------------------------

@pytest.mark.parametrize("b", [64, 16])
@pytest.mark.parametrize("d", [128, 64])
@pytest.mark.parametrize("N", [100, 300, 513, 1000])
def test_prefill_block_bf16(moa, b, d, N):
    B, Hq, Hkv, s = 2, 6, 3, b
    W = [0, b, 2 * b, 3 * b, 256, (N // b + 2) * b]
    q = normal((B, N, Hq, d), 401, torch.bfloat16)
    k = normal((B, N, Hkv, d), 402, torch.bfloat16)
    v = normal((B, N, Hkv, d), 403, torch.bfloat16)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, s, torch.bfloat16, block=b)
    O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale, block=b)
    err = np.abs(f64(o) - O)
    assert np.isfinite(f64(o)).all()
    assert err.max() < 2e-2, (err.max(), np.unravel_index(err.argmax(), err.shape))
    assert np.abs(f64(lse) - L).max() < 2e-3
    check_cache_image(ctx, 0, k, v, N - 1, W, s, B, 2)   # the cache fill is mode-independent


@pytest.mark.parametrize("N", [129, 300])
def test_prefill_block_fp32(moa, N):
    B, Hq, Hkv, d, s, b = 2, 4, 2, 64, 16, 16
    W = [16, 48, 0, 160]
    q = normal((B, N, Hq, d), 411)
    k = normal((B, N, Hkv, d), 412)
    v = normal((B, N, Hkv, d), 413)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, s, torch.float32, block=b)
    O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale, block=b)
    assert np.abs(f64(o) - O).max() < 1e-5
    assert np.abs(f64(lse) - L).max() < 1e-5


@pytest.mark.parametrize("dtype,tol", [(torch.bfloat16, 2e-2), (torch.float32, 1e-5)])
def test_prefill_block_structured(moa, dtype, tol):
    """Spike keys at the last key of every block: the token window of a row ending inside a
    block reaches the spike just before the block-aligned window start, the block window
    does not, so the two masks differ by O(1) (and so would a kernel off by one block)."""
    B, N, H, d, s, b = 1, 640, 4, 64 if dtype == torch.float32 else 128, 16, 16
    W = [16, 32, 208, 640]
    u = torch.zeros(d)
    u[0] = 1.0
    spike = (torch.arange(N) % b == b - 1).float() * 8.0
    k = (spike[None, :, None, None] * u).expand(B, N, H, d).clone()
    k = (k + 0.01 * normal((B, N, H, d), 7)).to(dtype)
    v = normal((B, N, H, d), 8, dtype)
    q = u.expand(B, N, H, d).clone().to(dtype)
    ctx, o, lse, _ = _prefill(moa, q, k, v, W, s, dtype, scale=1.0, block=b)
    O, _ = oracle.prefill(f64(q), f64(k), f64(v), W, s, 1.0, block=b)
    assert np.abs(f64(o) - O).max() < tol
    Ot, _ = oracle.prefill(f64(q), f64(k), f64(v), W, s, 1.0)   # the token mask differs here
    assert np.abs(Ot - O).max() > 0.1


def test_c4_full_layer_prefill_block64(moa):
    """C4's rule windows are multiples of 64 (alpha in multiples of 2048, beta in k/8, N=16k),
    so the layer runs with the paper's block-64 mask; sampled rows vs the oracle."""
    _full_layer_prefill(moa, "C4", 33, block=64)


def test_block_prefill_then_token_decode(moa):
    """Block mode changes prefill only: the cache and the token-granular decode that follows
    are those of the token mode."""
    dev = torch.device("cuda")
    B, N, Hq, Hkv, d, s, b = 2, 300, 4, 2, 128, 64, 64
    W = [64, 128, 0, 192]
    q = normal((B, N, Hq, d), 421, torch.bfloat16)
    k = normal((B, N, Hkv, d), 422, torch.bfloat16)
    v = normal((B, N, Hkv, d), 423, torch.bfloat16)
    qd = normal((B, Hq, d), 424, torch.bfloat16)
    kd = normal((B, Hkv, d), 425, torch.bfloat16)
    vd = normal((B, Hkv, d), 426, torch.bfloat16)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, s, torch.bfloat16, block=b)
    ws = ctx.alloc_workspace(B)
    od = torch.empty(B, Hq, d, dtype=torch.bfloat16, device=dev)
    ctx.decode_step_fused(0, qd.to(dev), kd.to(dev), vd.to(dev), od, N, scale, ws)
    torch.cuda.synchronize()
    Kh, Vh = torch.cat([k, kd[:, None]], 1), torch.cat([v, vd[:, None]], 1)
    Od, _ = oracle.decode(f64(qd), f64(Kh), f64(Vh), N, W, s, scale)
    assert np.abs(f64(od) - Od).max() < 2e-2


def test_output_rows_not_32_byte_aligned(moa):
    """The epilogue uses 256-bit stores only for 32-byte aligned output rows; an output view
    offset by 16 bytes takes the 128-bit path and must give bitwise the same result."""
    dev = torch.device("cuda")
    B, N, Hq, Hkv, d, s = 2, 300, 4, 2, 128, 4
    W = [3, 200, 0, 77]
    q = normal((B, N, Hq, d), 321, torch.bfloat16).to(dev)
    k = normal((B, N, Hkv, d), 322, torch.bfloat16).to(dev)
    v = normal((B, N, Hkv, d), 323, torch.bfloat16).to(dev)
    ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=torch.bfloat16)
    ctx.set_spans(0, W, s, N)
    o1 = torch.empty_like(q)
    flat = torch.zeros(q.numel() + 8, dtype=torch.bfloat16, device=dev)
    o2 = flat[8:].view(B, N, Hq, d)  # 16 bytes past a 256-byte aligned allocation
    assert o2.data_ptr() % 32 == 16
    tau = 1 / math.sqrt(d)
    ctx.prefill_attn(0, q, k, v, o1, tau)
    ctx.prefill_attn(0, q, k, v, o2, tau)
    torch.cuda.synchronize()
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
    O, _ = oracle.prefill(f64(q), f64(k), f64(v), W, s, tau)
    assert np.abs(f64(o2) - O).max() < 2e-2


@pytest.mark.parametrize("d", [128, 64])
def test_prefill_bf16_gqa_group_of_eight(moa, d):
    """G = 8 (the C5 / Llama3-70B grouping) through the tcgen05 kernel: 16 q-heads over 2
    kv-groups with heterogeneous windows inside each group (W = 0 sink-only, W = 1, W > N)."""
    B, N, Hkv, G, s = 2, 333, 2, 8, 5
    Hq = Hkv * G
    W = [0, 1, 64, 127, 128, 129, 300, N + 9, 2, 17, 200, 333, 31, 0, 1, 250]
    q = normal((B, N, Hq, d), 431, torch.bfloat16)
    k = normal((B, N, Hkv, d), 432, torch.bfloat16)
    v = normal((B, N, Hkv, d), 433, torch.bfloat16)
    ctx, o, lse, scale = _prefill(moa, q, k, v, W, s, torch.bfloat16)
    O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale)
    assert np.isfinite(f64(o)).all()
    assert np.abs(f64(o) - O).max() < 2e-2
    assert np.abs(f64(lse) - L).max() < 2e-3
    check_cache_image(ctx, 0, k, v, N - 1, W, s, B, G)


def test_set_spans_twice_keeps_cache_maps_for_decode(moa):
    """moa_set_spans again with the same footprint keeps the bound cache, and a
    bf16 decode must still find its TMA tensor maps (no re-bind needed, include/moa.h)."""
    dev = torch.device("cuda")
    B, N, Hq, Hkv, d, s = 2, 200, 4, 2, 128, 4
    W = [7, 150, 0, 33]
    q = normal((B, N, Hq, d), 441, torch.bfloat16).to(dev)
    k = normal((B, N, Hkv, d), 442, torch.bfloat16).to(dev)
    v = normal((B, N, Hkv, d), 443, torch.bfloat16).to(dev)
    qd = normal((B, Hq, d), 444, torch.bfloat16).to(dev)
    kd = normal((B, Hkv, d), 445, torch.bfloat16).to(dev)
    vd = normal((B, Hkv, d), 446, torch.bfloat16).to(dev)
    ctx = moa.MoAContext(1, Hq, Hkv, d, B, dtype=torch.bfloat16)
    ctx.set_spans(0, W, s, N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    ctx.set_spans(0, [9, 150, 33, 0], s, N)     # same group capacities (150, 33): same footprint
    o = torch.empty_like(q)
    tau = 1 / math.sqrt(d)
    ctx.prefill(0, q, k, v, o, tau)
    od = torch.empty_like(qd)
    ctx.decode_step_fused(0, qd, kd, vd, od, N, tau, ws)
    torch.cuda.synchronize()
    W2 = [9, 150, 33, 0]
    Kh, Vh = torch.cat([k, kd[:, None]], 1), torch.cat([v, vd[:, None]], 1)
    Od, _ = oracle.decode(f64(qd), f64(Kh), f64(Vh), N, W2, s, tau)
    assert np.abs(f64(od) - Od).max() < 2e-2


@pytest.mark.parametrize("N,s,W,Hkv", [
    (300, 4, [3, 140, 0, 290, 17, 17, 1, 0], 2),      # G=4: filler heads 3 (W=290) and 4 (first of the 17s)
    (1000, 64, [0, 0, 512, 2000], 4),                 # sink-only groups, W > N
    (40, 64, [5, 100], 2),                            # N < s: every position is a sink
    (129, 8, [128, 1, 64, 129], 4),                   # ragged last tile, W = N
    (777, 16, [600, 77, 300, 5, 700, 760, 2, 40], 4), # G=2, filler head second in its group
])
def test_fused_cache_fill_equals_separate_fill(moa, N, s, W, Hkv):
    """moa_prefill's fused cache fill (warp 10 copies the kept rows of the filler item's K/V
    tiles from shared memory) writes the same cache bytes as moa_prefill_attn + the separate
    moa_cache_fill kernel, and both match the oracle image (reading c13)."""
    B, d = 3, 128
    Hq = len(W)
    dtype = torch.bfloat16
    q, k, v = (normal((B, N, h, d), 900 + i, dtype).cuda() for i, h in enumerate((Hq, Hkv, Hkv)))
    scale = 1 / math.sqrt(d)
    c1 = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
    c2 = moa.MoAContext(1, Hq, Hkv, d, B, dtype=dtype)
    for c in (c1, c2):
        c.set_spans(0, W, s, N)
        c.alloc_cache(B)
    o1, o2 = torch.empty_like(q), torch.empty_like(q)
    c1.prefill(0, q, k, v, o1, scale)
    c2.prefill_attn(0, q, k, v, o2, scale)
    c2.cache_fill(0, k, v)
    torch.cuda.synchronize()
    assert np.array_equal(bits(o1), bits(o2))
    for which in (0, 1):
        assert torch.equal(c1._cache[which], c2._cache[which]), which
    assert c1.next_pos(0) == N
    check_cache_image(c1, 0, k.cpu(), v.cpu(), N - 1, W, s, B, Hq // Hkv)


@pytest.mark.gpu
def test_prefill_bf16_clustered_kernel():
    """The opt-in clustered prefill (MOA_PP_CLUSTER=1: two SMs per 256-row item, K/V multicast,
    double-buffered S and P, two alternating softmax groups) against the oracle -- uniform and
    structured inputs, fused cache fill bit-exact.  Runs in a subprocess with a time limit: one
    C2-scale run of a modified build was seen to hang, so a hang fails this test
    instead of stalling the suite."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, MOA_PP_CLUSTER="1")
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cl_parity_worker.py")
    r = subprocess.run([sys.executable, worker], env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "clustered parity ok" in r.stdout
