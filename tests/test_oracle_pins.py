"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a printed example, a closed
form, a library routine for a special case, an invariant or brute force.
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
from moa_workloads import ALPHA_GRID, BETA_GRID, CONFIGS, rule_table

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


# --- printed examples --------------------------------------------------------

def test_softmax_printed_example():
    """softmax([1,2,3]) = [0.09003, 0.24473, 0.66524] +- 1e-5.
    Realised through the oracle's attention row: q.k_j = j+1 (tau = 1) and
    V = identity, so O is exactly the softmax weight vector."""
    with open(os.path.join(GOLDEN, "softmax_example.txt")) as f:
        line = [l for l in f if l.strip() and not l.startswith("#")][0].split()
    scores = np.array([float(x) for x in line[:3]])
    expected = np.array([float(x) for x in line[3:6]])
    tol = float(line[6])
    q = np.array([1.0, 0.0, 0.0])
    K = np.stack([[s, 0.0, 0.0] for s in scores])
    V = np.eye(3)
    o, lse = oracle.attend(q, K, V, tau=1.0)
    assert np.max(np.abs(o - expected)) < tol
    assert abs(lse - math.log(np.exp(scores).sum())) < 1e-12


def test_span_window_density_examples():
    with open(os.path.join(GOLDEN, "span_examples.txt")) as f:
        rows = [l.split("#")[0].split() for l in f if l.strip() and not l.startswith("#")]
    n = 0
    for kind, a, b, N, s, exp in rows:
        a, b, N, s = float(a), float(b), int(N), int(s)
        span = oracle.span_of(a, b, N)
        if kind == "span":
            assert span == int(exp), (a, b, N)
        elif kind == "window":
            assert oracle.window_of(span, s) == int(exp), (a, b, N)
        elif kind == "density":
            w = oracle.window_of(span, s)
            assert abs(oracle.density([w], s, N) - float(exp)) < 1e-12
        n += 1
    assert n >= 10


def test_mask_predicate_hand_written_picture():
    """The predicate against a hand-typed N=8, W=3, s=2 mask picture."""
    with open(os.path.join(GOLDEN, "mask_N8_W3_s2.txt")) as f:
        pic = [l.strip() for l in f if l.strip() and not l.startswith("#")]
    assert len(pic) == 8
    for i in range(8):
        got = "".join("1" if oracle.visible(i, j, 3, 2) else "." for j in range(8))
        assert got == pic[i], (i, got, pic[i])
        assert list(oracle.visible_keys(i, 3, 2)) == [j for j in range(8) if pic[i][j] == "1"]


# --- special cases that reduce to a library routine / closed form ------------

@pytest.mark.parametrize("G", [1, 2])
@pytest.mark.parametrize("s", [0, 4])
@pytest.mark.parametrize("extra", [0, 7])
def test_full_span_is_causal_attention(G, s, extra):
    """Any W >= N reproduces textbook causal attention (north_star), checked
    against torch.nn.functional.scaled_dot_product_attention(is_causal=True)
    in fp64 on the CPU."""
    B, N, Hkv, d = 2, 40, 2, 16
    Hq = Hkv * G
    Q, K, V = _rand((B, N, Hq, d), 1), _rand((B, N, Hkv, d), 2), _rand((B, N, Hkv, d), 3)
    tau = 1 / math.sqrt(d)
    O, LSE = oracle.prefill(Q, K, V, [N + extra] * Hq, s, tau)
    q = torch.from_numpy(Q).permute(0, 2, 1, 3)
    k = torch.from_numpy(K).permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
    v = torch.from_numpy(V).permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=tau)
    ref = ref.permute(0, 2, 1, 3).numpy()
    assert np.max(np.abs(O - ref)) < 1e-12
    # LSE of the causal row via a plain log-sum-exp over j <= i
    S = tau * torch.einsum("bhid,bhjd->bhij", q, k)
    S = S.masked_fill(torch.triu(torch.ones(N, N, dtype=torch.bool), 1), float("-inf"))
    assert np.max(np.abs(LSE - torch.logsumexp(S, -1).numpy())) < 1e-12


def test_window_one_no_sink_is_own_value_row():
    """W = 1, s = 0: the softmax has one element, so O_i = V_i exactly."""
    B, N, H, d = 2, 33, 3, 8
    Q, K, V = _rand((B, N, H, d), 4), _rand((B, N, H, d), 5), _rand((B, N, H, d), 6)
    O, _ = oracle.prefill(Q, K, V, [1] * H, 0, 0.3)
    assert np.array_equal(O, V)


def _closed_form_visible(i, W, s):
    """Count and position-sum of V(h,i) by arithmetic series (no predicate)."""
    n1 = min(s, i + 1)
    sum1 = n1 * (n1 - 1) / 2
    if W > 0:
        lo = max(i - W + 1, n1)
        n2 = max(0, i - lo + 1)
        sum2 = (lo + i) * n2 / 2 if n2 else 0.0
    else:
        n2, sum2 = 0, 0.0
    return n1 + n2, sum1 + sum2


@pytest.mark.parametrize("W,s", [(1, 0), (5, 0), (5, 3), (0, 3), (17, 4), (64, 1), (100, 0), (3, 20)])
def test_constant_keys_average_visible_positions(W, s):
    """Constant K makes every visible score equal, so O_i is the plain mean
    of the visible V rows; with V[j] = (1, j) the second output is the mean
    visible position, known in closed form.  LSE = tau q.k + log |V(h,i)|."""
    N, d = 70, 2
    Q = _rand((1, N, 1, d), 7)
    K = np.ones((1, N, 1, d)) * 0.5
    V = np.stack([np.ones(N), np.arange(N, dtype=np.float64)], axis=1)[None, :, None, :]
    O, LSE = oracle.prefill(Q, K, V, [W], s, 0.7)
    for i in range(N):
        cnt, tot = _closed_form_visible(i, W, s)
        assert abs(O[0, i, 0, 0] - 1.0) < 1e-12
        assert abs(O[0, i, 0, 1] - tot / cnt) < 1e-9
        assert abs(LSE[0, 0, i] - (0.7 * Q[0, i, 0] @ K[0, 0, 0] + math.log(cnt))) < 1e-12


def test_rows_sum_to_one():
    """Softmax rows sum to 1: with V = 1 every output is 1."""
    B, N, Hq, Hkv, d = 1, 50, 4, 2, 8
    Q, K = _rand((B, N, Hq, d), 8), _rand((B, N, Hkv, d), 9)
    V = np.ones((B, N, Hkv, d))
    O, _ = oracle.prefill(Q, K, V, [0, 3, 17, 60], 2, 1.3)
    assert np.max(np.abs(O - 1.0)) < 1e-12


# --- brute force on tiny inputs ----------------------------------------------

def test_gather_equals_dense_mask_bruteforce():
    """Gather-set formulation == dense additive-mask formulation, exhaustive
    over W in [0, N+1] and s in {0..4} for N = 12 (and a GQA group)."""
    B, N, Hkv, G, d = 1, 12, 1, 2, 4
    Q, K, V = _rand((B, N, Hkv * G, d), 10), _rand((B, N, Hkv, d), 11), _rand((B, N, Hkv, d), 12)
    for s in range(5):
        for W in range(N + 2):
            if W == 0 and s == 0:
                continue
            w = [W, max(W - 1, 0) if s else W]
            O1, L1 = oracle.prefill(Q, K, V, w, s, 0.5)
            O2, L2 = oracle.prefill_dense_mask(Q, K, V, w, s, 0.5)
            assert np.max(np.abs(O1 - O2)) < 1e-13
            assert np.max(np.abs(L1 - L2)) < 1e-12


def test_empty_row_rejected():
    with pytest.raises(ValueError):
        oracle.prefill(_rand((1, 4, 1, 2), 1), _rand((1, 4, 1, 2), 2), _rand((1, 4, 1, 2), 3), [0], 0, 1.0)


# --- decode and the cache image ----------------------------------------------

def test_decode_is_prefill_row():
    """A decode step at position p attends exactly like prefill row p of the
    full prompt (windows frozen, reading c9)."""
    B, N, Hq, Hkv, d, s = 2, 60, 4, 2, 8, 3
    W = [5, 9, 1, 70]
    Q, K, V = _rand((B, N, Hq, d), 13), _rand((B, N, Hkv, d), 14), _rand((B, N, Hkv, d), 15)
    O, L = oracle.prefill(Q, K, V, W, s, 0.4)
    for p in (0, 2, 3, 17, 59):
        o, l = oracle.decode(Q[:, p], K[:, : p + 1], V[:, : p + 1], p, W, s, 0.4)
        assert np.max(np.abs(o - O[:, p])) < 1e-13
        assert np.max(np.abs(l - L[:, :, p])) < 1e-13


def test_cache_image_ring_invariants():
    """SPEC.md:463/470/486: resident = min(p+1, s+W); after w+k steps the ring
    holds exactly the last w positions; sinks never move; each slot's row is
    the history row of the position it holds."""
    B, T, Hkv, d, s = 1, 80, 3, 4, 4
    Wg = [0, 7, 16]
    K = _rand((B, T, Hkv, d), 16)
    V = _rand((B, T, Hkv, d), 17)
    for p in range(T):
        img = oracle.cache_image(K, V, p, Wg, s)
        for g, w in enumerate(Wg):
            Ki, Vi, valid = img[(0, g)]
            assert valid.sum() == min(p + 1, s + w)
            held = oracle.resident_positions(p, s, w)
            for pos in held:
                r = oracle.slot_of(pos, s, w)
                assert np.array_equal(Ki[r], K[0, pos, g]) and np.array_equal(Vi[r], V[0, pos, g])
            if p >= s + w:
                assert sorted(held) == list(range(min(s, p + 1))) + list(range(p - w + 1, p + 1))
            for pos in range(min(s, p + 1)):
                assert oracle.slot_of(pos, s, w) == pos
    # every ring slot is reused once per W_g positions (eviction of the oldest)
    assert [oracle.slot_of(p, 4, 7) for p in range(4, 20)] == [4 + (p - 4) % 7 for p in range(4, 20)]


def test_visible_pairs_closed_form():
    """Sum_i |V(h,i)| = W(W+1)/2 + (N-W)W + sum_{i>=W} min(s, i-W+1) for
    W <= N, and brute force for small N."""
    for N, W, s in [(30, 0, 3), (30, 7, 0), (30, 7, 5), (30, 30, 2), (31, 40, 2), (64, 17, 20)]:
        brute = sum(len(oracle.visible_keys(i, W, s)) for i in range(N))
        assert oracle.visible_pairs(N, W, s) == brute
    N, W, s = 4096, 1984, 64
    closed = W * (W + 1) // 2 + (N - W) * W + sum(min(s, i - W + 1) for i in range(W, N))
    assert oracle.visible_pairs(N, W, s) == closed
    assert abs(closed / (N * (N + 1) / 2) - 0.750) < 0.001   # 0.750 of causal


# --- the committed rule tables ---------------------------------------------

@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_rule_tables_shape_density(name):
    cfg = CONFIGS[name]
    t = rule_table(name)
    a, b = np.array(t["alpha"]), np.array(t["beta"])
    assert a.shape == (cfg.layers, cfg.hq)
    assert set(a.ravel()) <= set(ALPHA_GRID) and set(b.ravel()) <= set(BETA_GRID)
    for l in range(cfg.layers):
        assert len(set(zip(a[l], b[l]))) <= 2
        for g in range(cfg.hkv):                               # one rule per kv-group
            sl = slice(g * cfg.group, (g + 1) * cfg.group)
            assert len(set(zip(a[l, sl], b[l, sl]))) == 1
    w = [[oracle.window_of(oracle.span_of(x, y, cfg.N), cfg.n_sink) for x, y in zip(a[l], b[l])]
         for l in range(cfg.layers)]
    dens = np.mean([oracle.density(wl, cfg.n_sink, cfg.N) for wl in w])
    assert abs(dens - cfg.target_density) < 0.01


# --- block mode ("block sliding-window attention pattern with a block size of
# 64"; SPEC.md:216-224 build_mask) -------------------------------------------------------

def test_block_mask_hand_written_picture():
    """SPEC.md:216-224's worked example n=16, block=4, one sink block, window_blocks=2,
    against a hand-typed picture."""
    with open(os.path.join(GOLDEN, "block_mask_N16_b4_s4_W8.txt")) as f:
        pic = [l.strip() for l in f if l.strip() and not l.startswith("#")]
    assert len(pic) == 16
    for i in range(16):
        got = "".join("1" if oracle.visible_block(i, j, 8, 4, 4) else "." for j in range(16))
        assert got == pic[i], (i, got, pic[i])
        assert list(oracle.visible_keys(i, 8, 4, block=4)) == [j for j in range(16) if pic[i][j] == "1"]


def test_block_one_window_block_sees_sink_and_own_block():
    """window_blocks = 1, sink_blocks = 1 -> each query block sees block 0 and
    itself only (causal inside it)."""
    b = 8
    for i in range(64):
        keys = set(oracle.visible_keys(i, b, b, block=b).tolist())
        own = set(range((i // b) * b, i + 1))
        assert keys == set(range(min(b, i + 1))) | own


@pytest.mark.parametrize("N", [1, 7, 33])
def test_block_size_one_is_token_mask(N):
    """b = 1 reduces the block predicate to the token predicate (already pinned above)."""
    for W in range(0, N + 2):
        for s in range(0, 4):
            for i in range(N):
                for j in range(N):
                    assert oracle.visible_block(i, j, W, s, 1) == oracle.visible(i, j, W, s)


@pytest.mark.parametrize("b", [2, 4, 8])
def test_block_window_between_token_windows(b):
    """Containment fixed by the definitions: the block window starts at
    b*floor(i/b) - W + b, between i-W+1 and i-W+b, so token mask(W-b+1) <= block mask(W)
    <= token mask(W) (same sinks, s a multiple of b)."""
    N = 6 * b + 3
    for s in (0, b):
        for W in range(b, N + b, b):
            for i in range(N):
                blk = set(oracle.visible_keys(i, W, s, block=b).tolist())
                assert set(oracle.visible_keys(i, W - b + 1, s).tolist()) <= blk
                assert blk <= set(oracle.visible_keys(i, W, s).tolist())


@pytest.mark.parametrize("s", [0, 4])
def test_block_full_window_is_causal_attention(s):
    """window_blocks >= n_blocks -> pure causal mask, against
    torch scaled_dot_product_attention(is_causal=True) in fp64."""
    B, N, H, d, b = 1, 24, 2, 8, 4
    Q, K, V = _rand((B, N, H, d), 91), _rand((B, N, H, d), 92), _rand((B, N, H, d), 93)
    O, _ = oracle.prefill(Q, K, V, [N, N + b], s, 0.3, block=b)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.from_numpy(Q).permute(0, 2, 1, 3), torch.from_numpy(K).permute(0, 2, 1, 3),
        torch.from_numpy(V).permute(0, 2, 1, 3), is_causal=True, scale=0.3).permute(0, 2, 1, 3).numpy()
    assert np.max(np.abs(O - ref)) < 1e-12


@pytest.mark.parametrize("b", [2, 4])
def test_block_gather_matches_dense_mask(b):
    """Gather-set formulation == dense additive-mask formulation (brute force) in block mode,
    all windows multiple of b up to N, GQA."""
    B, N, Hq, Hkv, d = 1, 20, 4, 2, 8
    Q, K, V = _rand((B, N, Hq, d), 94), _rand((B, N, Hkv, d), 95), _rand((B, N, Hkv, d), 96)
    for s in (0, b):
        for W in range(0 if s else b, N + b, b):
            wq = [W, max(b, W - b), W, b]
            O1, L1 = oracle.prefill(Q, K, V, wq, s, 0.25, block=b)
            O2, L2 = oracle.prefill_dense_mask(Q, K, V, wq, s, 0.25, block=b)
            assert np.max(np.abs(O1 - O2)) < 1e-12 and np.max(np.abs(L1 - L2)) < 1e-12


def test_block_visible_pairs_brute_force():
    """visible_pairs_block against the picture's count and the b=1 token closed form."""
    with open(os.path.join(GOLDEN, "block_mask_N16_b4_s4_W8.txt")) as f:
        pic = [l.strip() for l in f if l.strip() and not l.startswith("#")]
    assert oracle.visible_pairs_block(16, 8, 4, 4) == sum(r.count("1") for r in pic)
    for N, W, s in ((50, 7, 3), (64, 64, 0), (33, 1, 0)):
        assert oracle.visible_pairs_block(N, W, s, 1) == oracle.visible_pairs(N, W, s)


# --- attention influence (Eq. 3; derivation PAPER.md:1361-1405) ----------

def _renormalised_delta(A_row, j):
    """eq:delta_A by its definition: A as exp(S)/sum exp(S); mask key j (drop its term)
    and recompute the row; the change of every entry (brute force, not the closed form)."""
    S = np.log(np.where(A_row > 0, A_row, 1.0))
    vis = A_row > 0
    w = np.where(vis, np.exp(S), 0.0)
    w_masked = w.copy()
    w_masked[j] = 0.0
    return w_masked / w_masked.sum() - w / w.sum()


def test_influence_spec_worked_example():
    """row A=[0.75, 0.25], g=[1, 2], masking key 2 -> E = -0.25; masking key 1
    gives dA = [-0.75, +0.75], sum g dA = 0.75 (the same renormalisation rule)."""
    E = oracle.attention_influence(np.array([[0.75, 0.25]]), np.array([[1.0, 2.0]]))
    assert abs(E[0, 1] - (-0.25)) < 1e-12
    assert abs(E[0, 0] - 0.75) < 1e-12


def test_influence_equals_sum_of_g_times_renormalised_change():
    """Eq. 3 == sum_n g_in dA_in|j with dA from re-normalising the softmax row without key j
    (eq:each_effect + eq:delta_A evaluated by brute force), random causal rows."""
    rng = np.random.default_rng(7)
    N = 9
    S = rng.standard_normal((N, N)) * 2
    A = np.zeros((N, N))
    for i in range(N):
        w = np.exp(S[i, :i + 1] - S[i, :i + 1].max())
        A[i, :i + 1] = w / w.sum()
    G = rng.standard_normal((N, N))
    E = oracle.attention_influence(A, G)
    for i in range(1, N):
        for j in range(i + 1):
            dA = _renormalised_delta(A[i], j)
            assert abs(dA.sum()) < 1e-12                     # SPEC.md:299 stochasticity kept
            assert abs(E[i, j] - float(G[i] @ dA)) < 1e-12
    assert E[0, 0] == 0.0                                   # single visible key: defined 0


def test_influence_zero_gradient_and_block_size_one():
    rng = np.random.default_rng(8)
    B, N, H, d = 1, 12, 2, 4
    Q, K, V = rng.standard_normal((B, N, H, d)), rng.standard_normal((B, N, H, d)), rng.standard_normal((B, N, H, d))
    assert np.all(oracle.influence_blocks(Q, K, V, np.zeros((B, N, H, d)), 0.5, 4) == 0.0)   # g = 0 -> E = 0
    dO = rng.standard_normal((B, N, H, d))
    e1 = oracle.influence_blocks(Q, K, V, dO, 0.5, 1)
    e3 = oracle.influence_blocks(Q, K, V, dO, 0.5, 3)
    # block mean of 3x3 == mean of the block-1 entries (averaging is linear)
    for ib in range(4):
        for jb in range(4):
            assert abs(e3[0, 1, ib, jb] - e1[0, 1, ib * 3:ib * 3 + 3, jb * 3:jb * 3 + 3].mean()) < 1e-12
    assert np.all(e1[0, 0][np.triu_indices(N, 1)] == 0.0)   # non-causal pairs carry no influence


def test_influence_gradient_is_chain_rule_of_o_equals_av():
    """G = dO V^T is dL/dA for O = A V: torch autograd on L = sum(dO * (A V)) in fp64."""
    rng = np.random.default_rng(9)
    N, d = 7, 5
    A = torch.tensor(rng.random((N, N)), requires_grad=True)
    V = torch.tensor(rng.standard_normal((N, d)))
    dO = torch.tensor(rng.standard_normal((N, d)))
    (dO * (A @ V)).sum().backward()
    assert torch.allclose(A.grad, dO @ V.T, atol=1e-12)


# --- rule losses (Eq. 4) ---------------------------------------------------

def _token_level_rule_loss(E_tok, W, s, b):
    """Eq. 4 at token level: sum of E over the pairs the rule's block mask hides (direct
    summation with the block predicate, independent of the block averaging)."""
    N = E_tok.shape[0]
    return sum(E_tok[i, j] for i in range(N) for j in range(i + 1) if not oracle.visible_block(i, j, W, s, b))


def test_rule_losses_equal_token_level_sums():
    """Block-averaged influence + Eq. 4 == token-level sum of E over the masked pairs
    (SPEC.md:345 'sums over masks then multiply by block token counts'), ragged N."""
    rng = np.random.default_rng(11)
    B, N, H, d, b, s = 1, 22, 2, 4, 4, 4
    Q, K, V, dO = (rng.standard_normal((B, N, H, d)) for _ in range(4))
    E_blocks = oracle.influence_blocks(Q, K, V, dO, 0.7, b)[0]
    alphas = [0.0, 4.0, 8.0, -8.0, 0.0]
    betas = [0.25, 0.0, 0.5, 0.0, 1.0]
    L = oracle.rule_losses(E_blocks, alphas, betas, N, s, b)
    for h in range(H):
        S = 0.7 * Q[0, :, h] @ K[0, :, h].T
        A = np.zeros((N, N))
        for i in range(N):
            w = np.exp(S[i, :i + 1] - S[i, :i + 1].max())
            A[i, :i + 1] = w / w.sum()
        E_tok = oracle.attention_influence(A, dO[0, :, h] @ V[0, :, h].T)
        for r, (a, be) in enumerate(zip(alphas, betas)):
            W = oracle.rule_window_blocked(a, be, N, s, b)
            assert abs(L[h, r] - _token_level_rule_loss(E_tok, W, s, b)) < 1e-12


def test_rule_losses_full_rule_zero_and_nesting():
    """the full-attention rule masks nothing (loss 0); a wider rule masks a
    subset, so with Ebar >= 0 its loss is not larger."""
    rng = np.random.default_rng(12)
    H, N, b, s = 3, 200, 8, 8
    nb = -(-N // b)
    E = rng.random((H, nb, nb))
    L = oracle.rule_losses(E, [0.0, 16.0, 64.0, 0.0], [1.0, 0.0, 0.0, 0.5], N, s, b)
    assert np.all(L[:, 0] == 0.0)
    assert np.all(L[:, 2] <= L[:, 1]) and np.all(L[:, 3] <= L[:, 1])
    # sink-only rule (span <= s): every causal block outside the sink column is masked
    Ls = oracle.rule_losses(E, [0.0], [0.0], N, s, b)
    cnt = lambda i: min(b, N - i * b)
    want = sum(E[:, ib, jb] * cnt(ib) * cnt(jb) for ib in range(nb) for jb in range(1, ib + 1))
    assert np.allclose(Ls[:, 0], want, rtol=0, atol=1e-10)


# --- ragged batches -------------------------------------

def test_ragged_full_span_sequences_are_textbook_causal():
    """Ragged batch whose every window covers its sequence: sequence b is plain causal
    attention over its own first N_b rows (torch SDPA, fp64), whatever the padding holds."""
    B, N, Hkv, G, d, s = 3, 37, 2, 2, 8, 2
    Hq = Hkv * G
    Q, K, V = _rand((B, N, Hq, d), 40), _rand((B, N, Hkv, d), 41), _rand((B, N, Hkv, d), 42)
    lens = [37, 20, 1]
    for b, n in enumerate(lens):  # garbage in the padding must not matter
        Q[b, n:] = 1e6
        K[b, n:] = -1e6
        V[b, n:] = np.nan
    wins = [[n] * Hq for n in lens]
    O, L = oracle.prefill_ragged(Q, K, V, lens, wins, s, 0.3)
    for b, n in enumerate(lens):
        q = torch.from_numpy(Q[b:b + 1, :n]).permute(0, 2, 1, 3)
        k = torch.from_numpy(K[b:b + 1, :n]).permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
        v = torch.from_numpy(V[b:b + 1, :n]).permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
        ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=0.3)
        assert np.max(np.abs(O[b, :n] - ref.permute(0, 2, 1, 3).numpy()[0])) < 1e-12
        assert np.all(np.isnan(O[b, n:])) and np.all(np.isnan(L[b, :, n:]))


def test_ragged_windows_match_dense_mask_of_truncated_sequence():
    """Per-sequence windows (Eq. 2 at each N_b): each sequence equals the dense-mask
    formulation run on that sequence alone."""
    B, N, Hkv, G, d, s = 3, 30, 1, 3, 4, 3
    Q, K, V = _rand((B, N, Hkv * G, d), 43), _rand((B, N, Hkv, d), 44), _rand((B, N, Hkv, d), 45)
    lens = [30, 17, 9]
    alpha, beta = [4.0, 8.0, 2.0], [0.2, 0.0, 0.5]
    wins = [[oracle.window_of(oracle.span_of(a, bt, n), s) for a, bt in zip(alpha, beta)] for n in lens]
    assert wins[1] != wins[0]  # the spans do depend on the sequence length
    O, L = oracle.prefill_ragged(Q, K, V, lens, wins, s, 0.7)
    for b, n in enumerate(lens):
        O2, L2 = oracle.prefill_dense_mask(Q[b:b + 1, :n], K[b:b + 1, :n], V[b:b + 1, :n], wins[b], s, 0.7)
        assert np.max(np.abs(O[b, :n] - O2[0])) < 1e-13
        assert np.max(np.abs(L[b, :, :n] - L2[0])) < 1e-12


def test_ragged_decode_rows_and_inactive_sequences():
    """decode_ragged at per-sequence positions == row p_b of the dense-mask prefill of
    sequence b; an inactive sequence (p < 0) gives O = 0, LSE = -inf."""
    B, N, Hkv, G, d, s = 3, 25, 2, 2, 4, 2
    Hq = Hkv * G
    Q, K, V = _rand((B, N, Hq, d), 46), _rand((B, N, Hkv, d), 47), _rand((B, N, Hkv, d), 48)
    wins = [[3, 0, 7, 30], [1, 2, 3, 4], [5, 5, 5, 5]]
    pos = [24, 11, -1]
    o, l = oracle.decode_ragged(Q[np.arange(B), np.maximum(pos, 0)], K, V, pos, wins, s, 0.5)
    for b in range(2):
        p = pos[b]
        O2, L2 = oracle.prefill_dense_mask(Q[b:b + 1, :p + 1], K[b:b + 1, :p + 1], V[b:b + 1, :p + 1], wins[b],
                                           s, 0.5)
        assert np.max(np.abs(o[b] - O2[0, p])) < 1e-13
        assert np.max(np.abs(l[b] - L2[0, :, p])) < 1e-12
    assert np.all(o[2] == 0) and np.all(np.isneginf(l[2]))


def test_spans_shrink_with_length_for_nonnegative_beta():
    """Eq. 2 with beta >= 0: the span at N_b <= N never exceeds the span at N, so the
    cache capacity resolved at the padded length holds every sequence's window
    (the moa_set_ragged precondition)."""
    for a in (0.0, 64.0, 1000.0, 5000.0):
        for bt in (0.0, 0.1, 0.5, 1.0):
            prev = -1
            for n in range(1, 3000, 37):
                w = oracle.window_of(oracle.span_of(a, bt, n), 64)
                assert w >= prev
                prev = w


# --- round 2 pins: block-rounded rule windows, group windows, attention matrix ---------------

def _golden_rows(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return [l.split("#")[0].strip() for l in f if l.strip() and not l.startswith("#")]


def test_rule_window_blocked_hand_computed():
    """tests/golden/rule_window_blocked.txt: span of Eq. 2 clipped to [0, N], rounded UP to a
    whole block, minus the sinks -- values typed by hand, so
    ceil -> floor (or rounding before the clip) fails here."""
    rows = _golden_rows("rule_window_blocked.txt")
    assert len(rows) >= 10
    for r in rows:
        a, be, N, s, b, want = r.split()
        got = oracle.rule_window_blocked(float(a), float(be), int(N), int(s), int(b))
        assert got == int(want), r


def test_group_windows_hand_computed():
    """tests/golden/group_windows.txt: W_g = max over the q-heads h with h // G == g (c10)."""
    rows = _golden_rows("group_windows.txt")
    for r in rows:
        G, wq, wg = (x.strip() for x in r.split("|"))
        got = oracle.group_windows([int(x) for x in wq.split()], int(G))
        assert list(got) == [int(x) for x in wg.split()], r


@pytest.mark.parametrize("G", [1, 2])
def test_attention_matrix_is_sdpa_causal(G):
    """attention_matrix (the A of influence_blocks) times V == torch SDPA(is_causal) in fp64,
    its rows sum to 1, and it is zero above the diagonal."""
    B, N, Hkv, d, tau = 1, 33, 2, 8, 0.37
    Q, K, V = _rand((B, N, Hkv * G, d), 60), _rand((B, N, Hkv, d), 61), _rand((B, N, Hkv, d), 62)
    q = torch.from_numpy(Q).permute(0, 2, 1, 3)
    k = torch.from_numpy(K).permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
    v = torch.from_numpy(V).permute(0, 2, 1, 3).repeat_interleave(G, dim=1)
    ref = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, scale=tau).numpy()
    for h in range(Hkv * G):
        A = oracle.attention_matrix(Q[0, :, h], K[0, :, h // G], tau)
        assert np.max(np.abs(A @ V[0, :, h // G] - ref[0, h])) < 1e-12
        assert np.max(np.abs(A.sum(axis=1) - 1.0)) < 1e-12
        assert np.all(A[np.triu_indices(N, 1)] == 0.0)
        sub = oracle.attention_matrix(Q[0, :, h], K[0, :, h // G], tau, rows=[0, 5, N - 1])
        assert np.array_equal(sub, A[[0, 5, N - 1]])


def test_influence_rows_equal_term_by_term():
    """attention_influence_rows (R_i - G_ij A_ij form) == the term-by-term Eq. 3, incl. a
    single-key row (A = 1 -> 0) and masked entries (A = 0 -> 0)."""
    rng = np.random.default_rng(13)
    N = 11
    S = rng.standard_normal((N, N)) * 3
    A = np.zeros((N, N))
    for i in range(N):
        w = np.exp(S[i, :i + 1] - S[i, :i + 1].max())
        A[i, :i + 1] = w / w.sum()
    G = rng.standard_normal((N, N))
    assert np.max(np.abs(oracle.attention_influence_rows(A, G) - oracle.attention_influence(A, G))) < 1e-12


def test_influence_sampled_equals_full():
    """influence_blocks_sampled == the listed rows of influence_blocks (ragged last block, GQA)."""
    rng = np.random.default_rng(14)
    B, N, Hkv, G, d, b = 2, 23, 2, 2, 4, 4
    Q, K, V, dO = (rng.standard_normal(s) for s in ((B, N, Hkv * G, d), (B, N, Hkv, d), (B, N, Hkv, d),
                                                   (B, N, Hkv * G, d)))
    full = oracle.influence_blocks(Q, K, V, dO, 0.6, b)
    for bb, h in ((0, 0), (1, 3)):
        qb = [0, 2, 5]
        got = oracle.influence_blocks_sampled(Q, K, V, dO, 0.6, b, bb, h, qb)
        assert np.max(np.abs(got - full[bb, h, qb])) < 1e-12


# --- rule selection (eq:mip) ---------------------------------------------

def test_plan_rules_spec_examples_oracle():
    """SPEC.md solve_single examples (exhaustive 1- and 4-case enumeration, typed by hand)."""
    assert oracle.plan_rules([[0, 5]], [1.0, 0.5], 1, 1, 0.5) == ((1,), 5.0, 0.5)
    assert oracle.plan_rules([[0, 3], [0, 1]], [1.0, 0.5], 1, 2, 0.75) == ((0, 1), 1.0, 0.75)
    # ADVICE r1 repro: rule 1 (density 0.5, loss 8) fits the budget and beats rule 0 (loss 10)
    assert oracle.plan_rules([[10, 8, 0]], [0.2, 0.5, 0.9], 1, 1, 0.5) == ((1,), 8.0, 0.5)
    assert oracle.plan_rules([[1, 2]], [0.6, 0.7], 1, 1, 0.5) is None           # infeasible


def test_plan_rules_layer_limit_and_budget_by_hand():
    """2 heads in one layer, 3 rules: with the limit 2 the best plan mixes two rules; with
    limit 1 both heads share one rule (values typed by hand)."""
    loss = [[0.0, 4.0, 9.0],     # head 0 is sensitive
            [5.0, 1.0, 0.0]]     # head 1 prefers the sparse rule 2
    dens = [1.0, 0.5, 0.1]
    assert oracle.plan_rules(loss, dens, 1, 2, 0.55, 2) == ((0, 2), 0.0, 0.55)
    assert oracle.plan_rules(loss, dens, 1, 2, 0.55, 1) == ((1, 1), 5.0, 0.5)
