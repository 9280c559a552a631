"""Helpers for the GPU parity tests (test-side only)."""
import math

import numpy as np
import torch

import oracle


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def bits(t: torch.Tensor) -> np.ndarray:
    """Raw bit pattern (int16 for bf16, int32 for fp32) as numpy, for bitwise checks."""
    t = t.detach().cpu().contiguous()
    return (t.view(torch.int16) if t.element_size() == 2 else t.view(torch.int32)).numpy()


def check_cache_image(ctx, layer, K_hist, V_hist, p, windows_q, n_sink, B, G):
    """Bitwise comparison of the GPU cache regions with the oracle image at p."""
    wg = oracle.group_windows(windows_q, G)
    img = oracle.cache_image(bits(K_hist), bits(V_hist), p, wg, n_sink)
    for b in range(B):
        for g in range(len(wg)):
            Ki, Vi, valid = img[(b, g)]
            kg = bits(ctx.cache_rows(layer, b, g, "k"))
            vg = bits(ctx.cache_rows(layer, b, g, "v"))
            assert kg.shape == Ki.shape
            assert np.array_equal(kg[valid], Ki[valid]), (b, g, p)
            assert np.array_equal(vg[valid], Vi[valid]), (b, g, p)


def sdpa_scale(d):
    return 1.0 / math.sqrt(d)


def rule_windows(table, layer, N, n_sink):
    """Windows of one layer of a committed rule table through the ORACLE's Eq. 2 + clip
    (span_of) and window = span - sinks (window_of) -- never through libmoa."""
    return [oracle.window_of(oracle.span_of(a, b, N), n_sink)
            for a, b in zip(table["alpha"][layer], table["beta"][layer])]
