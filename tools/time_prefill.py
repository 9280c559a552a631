"""Time moa_prefill over several layers of a config (CUDA events), print in-window TFLOP/s.

    python tools/time_prefill.py [C2|C4] [layers] [block]

block = 0: token mask; block = 64: the paper's block mask (moa_set_spans_blocked).
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from moa_workloads import CONFIGS, prefill_qkv, rule_table  # noqa: E402


def pairs(N, W, s, block=0):
    """sum_i |V(h,i)| of one head (token or block mask), vectorised host arithmetic."""
    i = np.arange(N, dtype=np.int64)
    if W > 0:
        lo = i - W + 1 if block == 0 else ((i // block) - W // block + 1) * block
        lo = np.maximum(lo, 0)
        win = i - lo + 1
        overlap = np.maximum(0, np.minimum(s, i + 1) - lo)
    else:
        win = overlap = 0
    return int((np.minimum(s, i + 1) + win - overlap).sum())


def main(name="C2", layers=4, block=0):
    cfg = CONFIGS[name]
    t = rule_table(name)
    dev = torch.device("cuda")
    L = list(range(cfg.layers - layers, cfg.layers)) if name != "C2" else list(range(8, 8 + layers))
    ctx = moa.MoAContext(len(L), cfg.hq, cfg.hkv, cfg.head_dim, cfg.batch)
    flops = 0
    for i, l in enumerate(L):
        W = moa.resolve_spans(t["alpha"][l], t["beta"][l], cfg.N, cfg.n_sink)
        ctx.set_spans(i, W, cfg.n_sink, cfg.N, block=block)
        flops += 4 * cfg.head_dim * cfg.batch * sum(pairs(cfg.N, w, cfg.n_sink, block) for w in W)
    ctx.alloc_cache(cfg.batch)
    qkv = [prefill_qkv(cfg, l, device=dev) for l in L]
    o = torch.empty_like(qkv[0][0])
    sc = 1 / math.sqrt(cfg.head_dim)
    for _ in range(2):
        for i in range(len(L)):
            ctx.prefill(i, *qkv[i], o, sc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        for i in range(len(L)):
            ctx.prefill(i, *qkv[i], o, sc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} layers={len(L)} block={block} {ms:.3f} ms  {flops / (ms / 1e3) / 1e12:.1f} TFLOP/s")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0] if a else "C2", int(a[1]) if len(a) > 1 else 4, int(a[2]) if len(a) > 2 else 0)
