"""GPU parity of moa_attention_influence against the fp64 oracle."""
import math

import numpy as np
import pytest
import torch

import oracle
from moa_workloads import normal
from tests.gpu_util import f64

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def moa():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2406_14909_b200 as m
    return m


def _run(moa, B, N, Hq, Hkv, d, seed, scale=None, accumulate_onto=None):
    q = normal((B, N, Hq, d), seed, torch.bfloat16)
    k = normal((B, N, Hkv, d), seed + 1, torch.bfloat16)
    v = normal((B, N, Hkv, d), seed + 2, torch.bfloat16)
    do = normal((B, N, Hq, d), seed + 3, torch.bfloat16)
    scale = 1 / math.sqrt(d) if scale is None else scale
    dev = torch.device("cuda")
    out = None if accumulate_onto is None else accumulate_onto.clone().to(dev)
    e = moa.attention_influence(q.to(dev), k.to(dev), v.to(dev), do.to(dev), scale, out=out,
                                accumulate=accumulate_onto is not None)
    torch.cuda.synchronize()
    ref = oracle.influence_blocks(f64(q), f64(k), f64(v), f64(do), scale, 64)
    return f64(e), ref


@pytest.mark.parametrize("N,d,G", [(64, 64, 1), (100, 128, 1), (200, 64, 2), (257, 128, 4)])
def test_influence_blocks_match_oracle(moa, N, d, G):
    """bf16 inputs are exact in both; the kernel's fp32 tensor-core sums and exp2 give
    relative errors ~1e-5 on E, so the block means must agree to 1e-3 of their scale."""
    Hkv = 2
    got, ref = _run(moa, 1 if N > 200 else 2, N, Hkv * G, Hkv, d, 500 + N)
    scale_ref = np.abs(ref).max()
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-3 * scale_ref + 1e-6, (np.abs(got - ref).max(), scale_ref)
    nb = got.shape[-1]
    assert np.all(got[..., np.triu_indices(nb, 1)[0], np.triu_indices(nb, 1)[1]] == 0.0)


def test_influence_accumulates(moa):
    """accumulate = 1 adds the item's block means onto the buffer (causal entries only)."""
    B, N, H, d = 1, 130, 2, 64
    nb = 3
    base = torch.arange(B * H * nb * nb, dtype=torch.float32).reshape(B, H, nb, nb)
    got, ref = _run(moa, B, N, H, H, d, 700, accumulate_onto=base)
    causal = np.tril(np.ones((nb, nb), dtype=bool))
    want = base.numpy().astype(np.float64) + ref
    assert np.abs(got[..., causal] - want[..., causal]).max() < 1e-3 * np.abs(ref).max() + 1e-5
    assert np.array_equal(got[..., ~causal], base.numpy()[..., ~causal].astype(np.float64))


@pytest.mark.parametrize("scale", [0.6, 1.0])
def test_influence_peaked_rows(moa, scale):
    """Peaked rows (score spread ~5-8 units: 1 - A of the top key down to ~1e-4..1e-6): the
    kernel splits the row max off its sums, so A/(1-A) and R - G keep fp32 accuracy where
    1 - A in fp32 would lose it; the fp64 oracle is still exact at these margins."""
    got, ref = _run(moa, 1, 160, 2, 2, 64, 800, scale=scale)
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-3 * np.abs(ref).max() + 1e-6, (np.abs(got - ref).max(), np.abs(ref).max())


def test_rule_losses_match_oracle(moa):
    """Eq. 4 on the GPU from the kernel's own influence blocks vs the oracle's Eq. 4 on the same
    blocks (fp64), over the paper's 6 x 9 rule grid at N = 1000 (ragged)."""
    from moa_workloads import ALPHA_GRID, BETA_GRID
    dev = torch.device("cuda")
    B, N, H, d, s = 1, 1000, 3, 64, 64
    q, k, v, do = (normal((B, N, H, d), 900 + i, torch.bfloat16).to(dev) for i in range(4))
    e = moa.attention_influence(q, k, v, do, 1 / math.sqrt(d))
    alphas = [a for a in ALPHA_GRID for _ in BETA_GRID]
    betas = [b for _ in ALPHA_GRID for b in BETA_GRID]
    alphas = [a / 8 for a in alphas]                       # spans at N = 1000 cover short and long windows
    got = f64(moa.rule_losses(e[0].contiguous(), N, s, alphas, betas))
    ref = oracle.rule_losses(f64(e[0]), alphas, betas, N, s, 64)
    assert np.abs(got - ref).max() <= 1e-5 * np.abs(ref).max() + 1e-7
    assert np.all(got[:, [i for i, (a, b) in enumerate(zip(alphas, betas)) if a + b * N >= N]] == 0.0)


@pytest.mark.parametrize("N,d,G,q_blocks", [(2048, 128, 1, [0, 1, 15, 16, 31]),
                                            (2113, 64, 2, [0, 7, 32, 33]),
                                            (8192, 128, 1, [0, 64, 127])])
def test_influence_long_sequences_sampled_blocks(moa, N, d, G, q_blocks):
    """Lengths the kernel is timed at: sampled query blocks (incl. the ragged last one) of
    every head against every key block vs oracle.influence_blocks_sampled, with a PER-BLOCK
    tolerance relative to the block's own mean |E| (far-from-diagonal blocks, the ones sparse
    rules mask and Eq. 4 sums, are checked at their own scale, not the diagonal's)."""
    B, Hkv = 1, 2
    Hq = Hkv * G
    seed = 1500 + N
    q = normal((B, N, Hq, d), seed, torch.bfloat16)
    k = normal((B, N, Hkv, d), seed + 1, torch.bfloat16)
    v = normal((B, N, Hkv, d), seed + 2, torch.bfloat16)
    do = normal((B, N, Hq, d), seed + 3, torch.bfloat16)
    scale = 1 / math.sqrt(d)
    dev = torch.device("cuda")
    e = f64(moa.attention_influence(q.to(dev), k.to(dev), v.to(dev), do.to(dev), scale))
    torch.cuda.synchronize()
    Q, K, V, dO = f64(q), f64(k), f64(v), f64(do)
    nb = e.shape[-1]
    for h in range(Hq):
        ref = oracle.influence_blocks_sampled(Q, K, V, dO, scale, 64, 0, h, q_blocks)
        mag = oracle.influence_blocks_sampled(Q, K, V, dO, scale, 64, 0, h, q_blocks, magnitude=True)
        got = e[0, h, q_blocks]
        tol = 2e-3 * mag + 1e-6 * mag.max()
        bad = np.abs(got - ref) > tol
        assert not bad.any(), (h, np.argwhere(bad)[:5], (np.abs(got - ref) / np.maximum(mag, 1e-30)).max())
        for r, ib in enumerate(q_blocks):
            assert np.all(got[r, ib + 1:] == 0.0)      # non-causal blocks carry nothing
        assert nb == (N + 63) // 64
