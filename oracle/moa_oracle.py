"""Plain fp64 CPU oracle of MoA heterogeneous sliding-window attention.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  It shares no code with the CUDA path (``paper_2406_14909_b200``) and
imports nothing from it.

Every function below is the plain definition from the paper, written out in
float64 with Python/numpy, no blocking, no fusion, no reordering:

* Eq. 1 (``eq:attention_compute``):
  ``S = Q K^T,  A = softmax(S + M),  O = A V``.
* The mask ``M`` of one head is the MoA sliding-window mask with attention
  sinks ("the initial few tokens (64 tokens for MoA) are not
  masked"; "Prefix ... remain visible to all attention
  heads"; PAPER.md:625-637 visual-element table).
* The span of a head comes from the elastic rule, Eq. 2 (PAPER.md:181,
  ``eq:search_space``) ``S_h = alpha_h + beta_h * N``, clipped to [0, N]
  (PAPER.md:692).  The span includes the sinks ("The attention
  span equals the sliding-window span plus the number of initially unmasked
  tokens").
* Decode keeps a static per-head cache of sinks + the most recent window and
  "replace[s] the old KV-Cache that exceeds the span with the latest"
  (``sec:appendix/effiency_experiment_setup``).

Readings of silent / ambiguous passages are the ones listed in DESIGN.md
section "Readings".  The ones this file relies on:

* c2: windows are passed separately from the sink count; the window of a
  rule is ``W = max(0, clip(S, 0, N) - s)``.
* c3: the window counts the query itself: key j is in the window of query i
  iff ``i - j < W``.
* c6: ``alpha + beta*N`` is rounded up (ceil) before clipping.
* c7: ``W = 0`` is allowed only with ``s >= 1``.
* c8: the softmax scale tau is an explicit argument (Eq. 1 has none).
* c9: decode windows are frozen at their prefill value.
* c10: GQA: q-head h reads kv-group ``h // G``; the cache of a group holds
  ``W_g = max_{h in g} W_h`` recent rows; every q-head masks to its own W_h.
* c13: ring slot of position p: ``p`` if ``p < s`` else
  ``s + (p - s) mod W_g``.
* c5 / NEXT-1 (block mode): the paper's prefill kernel uses "the block
  sliding-window attention pattern with a block size of 64 ... The first
  block of tokens is not masked and serves as the attention sink"
  (PAPER.md:690).  With block size b (s and W multiples of b),
  query block ``i // b`` sees key block ``j // b`` iff ``j <= i`` and
  (``j // b < s // b`` or ``i // b - j // b < W // b``), causal inside the
  diagonal block (``build_mask``).  ``block = 0`` is the
  token-granular mask above.  Decode stays token-granular in both modes: the
  cache "replace[s] the old KV-Cache that exceeds the span with the latest"
  token by token.

Parity pins for every function are in ``tests/test_oracle_pins.py``; none of
them is "parity unpinned".
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "span_of",
    "window_of",
    "group_windows",
    "visible",
    "visible_block",
    "visible_keys",
    "attend",
    "prefill",
    "prefill_rows",
    "prefill_dense_mask",
    "prefill_ragged",
    "decode_ragged",
    "decode",
    "slot_of",
    "resident_positions",
    "cache_image",
    "density",
    "visible_pairs",
    "visible_pairs_block",
    "attention_matrix",
    "attention_influence",
    "attention_influence_rows",
    "influence_blocks",
    "influence_blocks_sampled",
    "rule_window_blocked",
    "rule_losses",
    "plan_rules",
]


# ---------------------------------------------------------------------------
# Elastic rule -> span -> window (Eq. 2; clip PAPER.md:692)
# ---------------------------------------------------------------------------

def span_of(alpha: float, beta: float, N: int) -> int:
    """Attention span of one head at input length N (Eq. 2).

    ``S = alpha + beta * N`` (alpha = base span in tokens, beta = expansion
    rate; reading c1 -- App. A's ``alpha x N + beta`` at PAPER.md:609 has the
    roles swapped, and the search ranges at PAPER.md:692, alpha in
    [-2048, 8192] and beta in [0, 1], only make sense this way round).
    Rounded up (reading c6) and "clipped to the range between 0 and the
    current input length".
    """
    s = math.ceil(alpha + beta * N)
    return int(min(max(s, 0), N))


def window_of(span: int, n_sink: int) -> int:
    """Sliding-window length of a head whose span is ``span`` (reading c2).

    "The attention span equals the sliding-window span plus the number of
    initially unmasked tokens", so window = span - sinks,
    floored at 0 (a sink-only head).
    """
    return int(max(0, span - n_sink))


def group_windows(windows_q, group_size: int) -> np.ndarray:
    """Cache capacity of each kv-group, ``W_g = max_{h in g} W_h`` (c10)."""
    w = np.asarray(windows_q, dtype=np.int64)
    assert w.size % group_size == 0
    return w.reshape(-1, group_size).max(axis=1)


# ---------------------------------------------------------------------------
# The mask predicate and Eq. 1
# ---------------------------------------------------------------------------

def visible(i: int, j: int, W: int, s: int) -> bool:
    """True iff key j is visible to query i: causal, and a sink or in the
    window.  ``V(h,i) = { j : 0 <= j <= i and (j < s or i - j < W) }``."""
    return 0 <= j <= i and (j < s or i - j < W)


def visible_block(i: int, j: int, W: int, s: int, b: int) -> bool:
    """Block-granular mask of block size b:
    key j is visible to query i iff causal and its block is a sink block or
    within ``W // b`` blocks of the query's block (the query's own block
    included).  Requires ``s % b == 0`` and ``W % b == 0``."""
    assert b >= 1 and s % b == 0 and W % b == 0
    return 0 <= j <= i and (j // b < s // b or i // b - j // b < W // b)


def _visible(i: int, j: int, W: int, s: int, block: int) -> bool:
    return visible(i, j, W, s) if block == 0 else visible_block(i, j, W, s, block)


def visible_keys(i: int, W: int, s: int, block: int = 0) -> np.ndarray:
    """Sorted list of visible key positions of query i (brute-force
    enumeration of the predicate, O(i)); ``block`` > 0 selects the block mask."""
    return np.array([j for j in range(i + 1) if _visible(i, j, W, s, block)],
                    dtype=np.int64)


def attend(q: np.ndarray, Kj: np.ndarray, Vj: np.ndarray, tau: float):
    """One row of Eq. 1 restricted to the visible keys.

    ``z_j = tau * q . k_j`` ; ``a = softmax(z)`` ; ``o = sum_j a_j v_j``.
    Also returns ``lse = log sum_j exp(z_j)``.  fp64 throughout.
    """
    if Kj.shape[0] == 0:
        raise ValueError("empty softmax row (W = 0 and s = 0 is invalid, c7)")
    z = tau * (Kj.astype(np.float64) @ q.astype(np.float64))
    m = z.max()
    w = np.exp(z - m)
    l = w.sum()
    o = (w @ Vj.astype(np.float64)) / l
    return o, m + math.log(l)


def _check_shapes(Q, K, V, windows_q):
    B, N, Hq, d = Q.shape
    assert K.shape[0] == B and K.shape[1] == N and K.shape[3] == d
    assert V.shape == K.shape
    Hkv = K.shape[2]
    assert Hq % Hkv == 0
    assert len(windows_q) == Hq
    return B, N, Hq, Hkv, d, Hq // Hkv


def prefill_rows(Q, K, V, windows_q, n_sink: int, tau: float, rows, block: int = 0):
    """Eq. 1 for a list of sampled outputs ``rows = [(b, h, i), ...]``.

    Returns (O [len(rows), d], LSE [len(rows)]) in fp64.  Each row gathers
    its visible set V(h,i) by enumerating the predicate and attends over it
    (``block`` > 0: the block mask of block size ``block``).
    """
    B, N, Hq, Hkv, d, G = _check_shapes(Q, K, V, windows_q)
    O = np.zeros((len(rows), d), dtype=np.float64)
    L = np.zeros(len(rows), dtype=np.float64)
    for r, (b, h, i) in enumerate(rows):
        g = h // G
        J = visible_keys(int(i), int(windows_q[h]), n_sink, block)
        O[r], L[r] = attend(Q[b, i, h], K[b, J, g], V[b, J, g], tau)
    return O, L


def prefill(Q, K, V, windows_q, n_sink: int, tau: float, block: int = 0):
    """Causal prefill with the per-head MoA mask (Eq. 1 + PAPER.md:178;
    ``block`` > 0: block mask).

    Q: [B, N, Hq, d]; K, V: [B, N, Hkv, d] (any float dtype, upcast to fp64).
    windows_q: window W_h of every q-head.  Returns O [B, N, Hq, d] and
    LSE [B, Hq, N], both fp64.
    """
    B, N, Hq, Hkv, d, G = _check_shapes(Q, K, V, windows_q)
    rows = [(b, h, i) for b in range(B) for h in range(Hq) for i in range(N)]
    o, l = prefill_rows(Q, K, V, windows_q, n_sink, tau, rows, block)
    O = o.reshape(B, Hq, N, d).transpose(0, 2, 1, 3).copy()
    LSE = l.reshape(B, Hq, N)
    return O, LSE


def prefill_dense_mask(Q, K, V, windows_q, n_sink: int, tau: float, block: int = 0):
    """Second, brute-force formulation of the same prefill: a dense N x N
    additive mask M with a finite -1e30 sentinel for masked cells
    (SPEC.md:69 design decision), A = softmax(S + M) by rows, masked
    probabilities snapped to exact 0, O = A V (Eq. 1 verbatim).
    Meant for N <= 64."""
    B, N, Hq, Hkv, d, G = _check_shapes(Q, K, V, windows_q)
    O = np.zeros((B, N, Hq, d), dtype=np.float64)
    LSE = np.zeros((B, Hq, N), dtype=np.float64)
    for b in range(B):
        for h in range(Hq):
            g = h // G
            M = np.full((N, N), -1e30)
            for i in range(N):
                for j in range(N):
                    if _visible(i, j, int(windows_q[h]), n_sink, block):
                        M[i, j] = 0.0
            S = tau * (Q[b, :, h].astype(np.float64) @ K[b, :, g].astype(np.float64).T)
            X = S + M
            mx = X.max(axis=1, keepdims=True)
            E = np.exp(X - mx)
            E[M != 0.0] = 0.0
            A = E / E.sum(axis=1, keepdims=True)
            O[b, :, h] = A @ V[b, :, g].astype(np.float64)
            LSE[b, h] = mx[:, 0] + np.log(E.sum(axis=1))
    return O, LSE


# ---------------------------------------------------------------------------
# Ragged batches: per-sequence length, per-sequence spans
# ---------------------------------------------------------------------------

def prefill_ragged(Q, K, V, seq_len, windows_bq, n_sink: int, tau: float, block: int = 0):
    """Prefill of a padded ragged batch: sequence b is the prompt of its first
    ``seq_len[b]`` rows and its heads use ``windows_bq[b]`` -- the spans of Eq. 2
    resolved at that sequence's own length (spans "scale with the
    input length").  Each sequence is its own problem (Eq. 1 per sequence), so this
    is ``prefill`` of every truncated sequence.  Rows i >= N_b are NaN (no output).
    Returns O [B, N, Hq, d], LSE [B, Hq, N] (fp64)."""
    B, N, Hq, Hkv, d, G = _check_shapes(Q, K, V, windows_bq[0])
    O = np.full((B, N, Hq, d), np.nan)
    LSE = np.full((B, Hq, N), np.nan)
    for b in range(B):
        n = int(seq_len[b])
        assert 1 <= n <= N
        o, l = prefill(Q[b:b + 1, :n], K[b:b + 1, :n], V[b:b + 1, :n], list(windows_bq[b]), n_sink, tau, block)
        O[b, :n] = o[0]
        LSE[b, :, :n] = l[0]
    return O, LSE


def decode_ragged(q, K_hist, V_hist, pos, windows_bq, n_sink: int, tau: float):
    """Decode step of a ragged batch: sequence b is at its own position pos[b]
    with its own windows (``decode`` per sequence).  pos[b] < 0 marks
    an inactive sequence: O row 0, LSE -inf (the C-ABI's convention).
    Returns O [B, Hq, d], LSE [B, Hq]."""
    B, Hq, d = q.shape
    O = np.zeros((B, Hq, d), dtype=np.float64)
    L = np.full((B, Hq), -np.inf)
    for b in range(B):
        p = int(pos[b])
        if p < 0:
            continue
        o, l = decode(q[b:b + 1], K_hist[b:b + 1, :p + 1], V_hist[b:b + 1, :p + 1], p, list(windows_bq[b]),
                      n_sink, tau)
        O[b], L[b] = o[0], l[0]
    return O, L


# ---------------------------------------------------------------------------
# Decode: one new query at absolute position p
# ---------------------------------------------------------------------------

def decode(q, K_hist, V_hist, p: int, windows_q, n_sink: int, tau: float):
    """Decode step at position p, computed from the FULL history.

    q: [B, Hq, d]; K_hist, V_hist: [B, >= p+1, Hkv, d] hold every token's K/V
    since position 0 (never the ring).  Windows are frozen at their prefill
    value (reading c9), so this is row i = p of Eq. 1 with the same mask.
    Returns O [B, Hq, d], LSE [B, Hq].
    """
    B, Hq, d = q.shape
    Hkv = K_hist.shape[2]
    G = Hq // Hkv
    O = np.zeros((B, Hq, d), dtype=np.float64)
    L = np.zeros((B, Hq), dtype=np.float64)
    for b in range(B):
        for h in range(Hq):
            g = h // G
            J = visible_keys(p, int(windows_q[h]), n_sink)
            O[b, h], L[b, h] = attend(q[b, h], K_hist[b, J, g], V_hist[b, J, g], tau)
    return O, L


# ---------------------------------------------------------------------------
# The compact cache image (readings c10, c13)
# ---------------------------------------------------------------------------

def slot_of(pos: int, n_sink: int, W_g: int):
    """Cache row of absolute position ``pos`` in a group's region of
    ``n_sink + W_g`` rows (reading c13); None if the group stores no ring."""
    if pos < n_sink:
        return pos
    if W_g == 0:
        return None
    return n_sink + (pos - n_sink) % W_g


def resident_positions(p: int, n_sink: int, W_g: int):
    """Positions a group's cache holds after position p was written: the
    sinks {0..min(s, p+1)-1} and the most recent W_g non-sink positions
    {max(s, p-W_g+1)..p} ("replace the old KV-Cache that exceeds the span
    with the latest")."""
    sinks = list(range(min(n_sink, p + 1)))
    recent = list(range(max(n_sink, p - W_g + 1), p + 1))
    return sinks + recent


def cache_image(K_hist, V_hist, p: int, windows_g, n_sink: int):
    """Expected cache contents after position p was written.

    Returns, per (b, g), a tuple (K_img, V_img, valid) with K_img, V_img
    [n_sink + W_g, d] copies of the history rows (same dtype as the inputs,
    so a bitwise comparison is possible) and ``valid`` a bool mask of the
    rows that hold a position; invalid rows are excluded from comparison.
    """
    B = K_hist.shape[0]
    Hkv = K_hist.shape[2]
    d = K_hist.shape[3]
    out = {}
    for b in range(B):
        for g in range(Hkv):
            Wg = int(windows_g[g])
            Kimg = np.zeros((n_sink + Wg, d), dtype=K_hist.dtype)
            Vimg = np.zeros((n_sink + Wg, d), dtype=V_hist.dtype)
            valid = np.zeros(n_sink + Wg, dtype=bool)
            for pos in resident_positions(p, n_sink, Wg):
                r = slot_of(pos, n_sink, Wg)
                Kimg[r] = K_hist[b, pos, g]
                Vimg[r] = V_hist[b, pos, g]
                valid[r] = True
            out[(b, g)] = (Kimg, Vimg, valid)
    return out


# ---------------------------------------------------------------------------
# Accounting (PAPER.md:375 density; Eq. 1 work)
# ---------------------------------------------------------------------------

def density(windows, n_sink: int, N: int) -> float:
    """"the ratio of the average in-memory KV-Cache length to sequence
    length during decoding": mean over heads of
    min(N, s + W_h) / N (reading c11)."""
    w = np.asarray(windows, dtype=np.int64)
    return float(np.mean(np.minimum(N, n_sink + w)) / N)


def visible_pairs_block(N: int, W: int, s: int, b: int) -> int:
    """Number of (query, key) pairs of one head under the block mask, by
    enumerating the predicate."""
    return sum(1 for i in range(N) for j in range(i + 1) if visible_block(i, j, W, s, b))


def visible_pairs(N: int, W: int, s: int) -> int:
    """Number of (query, key) pairs one head attends to in prefill, by
    enumerating the predicate row by row (sum over i of |V(h,i)|)."""
    total = 0
    for i in range(N):
        n_sink = min(s, i + 1)
        lo = max(0, i - W + 1)
        n_win = i + 1 - lo if W > 0 else 0
        # keys counted twice: sinks that are also in the window
        overlap = max(0, min(s, i + 1) - lo) if W > 0 else 0
        total += n_sink + n_win - overlap
    return total


# ---------------------------------------------------------------------------
# Attention influence (Eq. 3; derivation PAPER.md:1361-1405)
# ---------------------------------------------------------------------------

def attention_influence(A: np.ndarray, G: np.ndarray) -> np.ndarray:
    """E of one head (Eq. 3, ``eq:effect``):

        E_ij = G_ij * (-A_ij) + sum_{n != j} G_in * A_in * A_ij / (1 - A_ij)

    with A the attention matrix (rows stochastic over their visible keys) and
    G = dL/dA.  Written term by term as in Eq. 3.  Entries with A_ij = 1 (the
    row's only visible key: masking it is never a candidate) are 0 (SPEC.md:287
    degenerate-row decision); masked entries (A_ij = 0) give 0.
    """
    A = np.asarray(A, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    E = np.zeros_like(A)
    n_rows, n_cols = A.shape
    for i in range(n_rows):
        for j in range(n_cols):
            a = A[i, j]
            if a == 0.0 or a >= 1.0:
                continue
            direct = G[i, j] * (-a)
            indirect = sum(G[i, n] * A[i, n] for n in range(n_cols) if n != j) * a / (1.0 - a)
            E[i, j] = direct + indirect
    return E


def attention_matrix(Qh, Kh, tau: float, rows=None) -> np.ndarray:
    """Dense causal attention matrix of one head, ``A = softmax(tau Q K^T + causal)``
    (Eq. 1 with the unmasked causal model that profiling uses).
    Qh, Kh: [N, d].  ``rows`` (optional) selects the query rows to return; row i holds
    A_ij for j <= i and 0 above the diagonal.  Returns [len(rows), N] fp64."""
    Qh = np.asarray(Qh, dtype=np.float64)
    Kh = np.asarray(Kh, dtype=np.float64)
    N = Kh.shape[0]
    rows = range(N) if rows is None else rows
    rows = list(rows)
    A = np.zeros((len(rows), N))
    for r, i in enumerate(rows):
        z = tau * (Kh[: i + 1] @ Qh[i])
        w = np.exp(z - z.max())
        A[r, : i + 1] = w / w.sum()
    return A


def attention_influence_rows(A: np.ndarray, G: np.ndarray) -> np.ndarray:
    """Eq. 3 for whole rows at once:

        E_ij = G_ij * (-A_ij) + (R_i - G_ij A_ij) * A_ij / (1 - A_ij),   R_i = sum_n G_in A_in

    i.e. the same formula as ``attention_influence`` with the sum over n != j written as the
    row total minus the j term.  Same conventions: E = 0 where A = 0 or A = 1.  Pinned
    against the term-by-term ``attention_influence`` (tests/test_oracle_pins.py)."""
    A = np.asarray(A, dtype=np.float64)
    G = np.asarray(G, dtype=np.float64)
    R = (G * A).sum(axis=1, keepdims=True)
    live = (A > 0.0) & (A < 1.0)
    Asafe = np.where(live, A, 0.0)
    E = -G * Asafe + (R - G * Asafe) * Asafe / np.where(live, 1.0 - Asafe, 1.0)
    return np.where(live, E, 0.0)


def influence_blocks(Q, K, V, dO, tau: float, block: int):
    """Block-averaged attention influence of every head for one calibration item.

    The profiling pass of the paper: dense causal attention (PAPER.md:691
    profiles the unmasked model), ``A = softmax(tau Q K^T + causal)``
    (Eq. 1, ``attention_matrix``), ``G = dL/dA = dO V^T`` for ``O = A V`` (chain
    rule), E by Eq. 3, then "the average attention influence within
    each block" over ``block x block`` token pairs (masked pairs count
    as 0, the last block may be partial: mean over its real pairs).
    Q, dO: [B, N, Hq, d]; K, V: [B, N, Hkv, d].  Returns [B, Hq, nb, nb] fp64.
    """
    B, N, Hq, d = Q.shape
    Hkv = K.shape[2]
    G_ = Hq // Hkv
    nb = (N + block - 1) // block
    out = np.zeros((B, Hq, nb, nb), dtype=np.float64)
    for b in range(B):
        for h in range(Hq):
            g = h // G_
            A = attention_matrix(Q[b, :, h], K[b, :, g], tau)
            Gm = dO[b, :, h].astype(np.float64) @ V[b, :, g].astype(np.float64).T
            E = attention_influence(A, Gm)
            for ib in range(nb):
                for jb in range(nb):
                    blk = E[ib * block:(ib + 1) * block, jb * block:(jb + 1) * block]
                    out[b, h, ib, jb] = blk.sum() / blk.size
    return out


def influence_blocks_sampled(Q, K, V, dO, tau: float, block: int, b: int, h: int, q_blocks,
                             magnitude: bool = False):
    """Rows ``q_blocks`` of ``influence_blocks(...)[b, h]`` (the block means of the listed
    query blocks against every key block), for lengths where the full N x N computation is
    out of reach: the same steps (``attention_matrix`` of the block's rows, G = dO V^T, Eq. 3
    by ``attention_influence_rows``, block means over ``block x block`` pairs).
    ``magnitude``: block means of |E| instead (the scale a per-block test tolerance uses).
    Returns [len(q_blocks), nb] fp64."""
    B, N, Hq, d = Q.shape
    Hkv = K.shape[2]
    g = h // (Hq // Hkv)
    nb = (N + block - 1) // block
    out = np.zeros((len(q_blocks), nb), dtype=np.float64)
    for r, ib in enumerate(q_blocks):
        rows = list(range(ib * block, min(N, (ib + 1) * block)))
        A = attention_matrix(Q[b, :, h], K[b, :, g], tau, rows)
        Gm = dO[b, rows, h].astype(np.float64) @ V[b, :, g].astype(np.float64).T
        E = attention_influence_rows(A, Gm)
        if magnitude:
            E = np.abs(E)
        for jb in range(nb):
            blk = E[:, jb * block:(jb + 1) * block]
            out[r, jb] = blk.sum() / blk.size
    return out


# ---------------------------------------------------------------------------
# Rule losses (Eq. 4) from the block-averaged influence
# ---------------------------------------------------------------------------

def rule_window_blocked(alpha: float, beta: float, N: int, n_sink: int, block: int) -> int:
    """Window of a rule for the block mask: the span of Eq. 2 (clipped to
    [0, N]) rounded up to a whole block (SPEC.md:200 ``span_of``), minus the
    sinks; a multiple of ``block`` when ``n_sink`` is."""
    span = span_of(alpha, beta, N)
    span = -(-span // block) * block
    return int(max(0, span - n_sink))


def rule_losses(E_blocks: np.ndarray, alphas, betas, N: int, n_sink: int, block: int) -> np.ndarray:
    """Delta L_{h,r} = sum_{i,j} M_{r,i,j} * Ebar_{h,i,j} (Eq. 4) with M the
    masked (causal but invisible) positions of rule r's block mask at length N, evaluated on
    the block-averaged influence ``E_blocks`` [H, nb, nb] (means over block x block pairs,
    the ragged last block over its real pairs): a fully masked block contributes its mean
    times its pair count, i.e. the token-level sum.  Returns [H, R] fp64."""
    H, nb, _ = E_blocks.shape
    out = np.zeros((H, len(alphas)))
    for r, (a, b_) in enumerate(zip(alphas, betas)):
        W = rule_window_blocked(a, b_, N, n_sink, block)
        for ib in range(nb):
            rows = min(block, N - ib * block)
            for jb in range(ib + 1):
                i_any, j_any = ib * block, jb * block   # block-mask visibility is per block
                if visible_block(i_any + block - 1 if ib * block + block <= N else N - 1,
                                 j_any, W, n_sink, block):
                    continue
                cols = min(block, N - jb * block)
                out[:, r] += E_blocks[:, ib, jb] * rows * cols
    return out


# ---------------------------------------------------------------------------
# Rule selection at one length (Eq. 5 / eq:mip)
# ---------------------------------------------------------------------------

def plan_rules(loss, density, layers: int, heads_per_layer: int, density_budget: float,
               max_rules_per_layer: int = 2):
    """Exhaustive solution of eq:mip: every assignment of one rule per head
    (eq:mip:plan) with at most ``max_rules_per_layer`` distinct rules in a layer
    ("at most two per model layer") and mean density
    ``(1/H) sum_h d_{r_h} <= d_constr`` (eq:mip:latency; feasibility slack: the sum
    may exceed ``budget * H`` by at most 1e-9), minimising ``sum_h Delta L_{h,r_h}``
    (eq:mip:obj up to the constant 1/H).  Brute force, for small instances only.
    loss: [H, R], density: [R].  Returns (plan tuple, loss, mean density) of an optimum
    (lowest loss, then lowest density, then the lexicographically first plan), or None
    if no assignment is feasible."""
    import itertools
    loss = np.asarray(loss, dtype=np.float64)
    dens = np.asarray(density, dtype=np.float64)
    H, R = loss.shape
    assert H == layers * heads_per_layer and dens.shape == (R,)
    best = None
    for plan in itertools.product(range(R), repeat=H):
        if any(len(set(plan[l * heads_per_layer:(l + 1) * heads_per_layer])) > max_rules_per_layer
               for l in range(layers)):
            continue
        dsum = sum(dens[r] for r in plan)
        if dsum > density_budget * H + 1e-9:
            continue
        lsum = sum(loss[h, r] for h, r in enumerate(plan))
        key = (lsum, dsum)
        if best is None or key < best[0]:
            best = (key, plan)
    if best is None:
        return None
    (lsum, dsum), plan = best
    return plan, lsum, dsum / H
