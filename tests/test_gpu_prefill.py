"""GPU parity of moa_prefill (+ the cache fill it performs) against the oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
from moa_workloads import CONFIGS, normal, prefill_qkv, rule_table
from tests.gpu_util import bits, check_cache_image, f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def moa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_14909_b200 as m
    return m


def _prefill(moa, q, k, v, W, s, dtype, scale=None, ctx_batch=None):
    dev = torch.device("cuda")
    B, N, Hq, d = q.shape
    Hkv = k.shape[2]
    ctx = moa.MoAContext(1, Hq, Hkv, d, ctx_batch or B, dtype=dtype)
    ctx.set_spans(0, W, s, N)
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
