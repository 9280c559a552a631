"""Decode timing study on the full C2 cache (all 32 layers resident, 8.6 GB).

    python tools/time_decode.py [--tokens 64] [--config C2]

Times the fused decode phase (tokens x layers launches) with CUDA events
around the whole phase, with and without an event pair around every launch,
and prints µs per launch and the in-window GB/s.  Diagnostic only.
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from moa_workloads import CONFIGS, decode_tokens, rule_table  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--layers", type=int, default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    L = a.layers or cfg.layers
    B, N, s, d, G = cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim, cfg.hq // cfg.hkv
    dev = torch.device("cuda")
    t = rule_table(cfg.name)
    ctx = moa.MoAContext(L, cfg.hq, cfg.hkv, d, B, dtype=torch.bfloat16)
    wins = []
    for l in range(L):
        w = moa.resolve_spans(t["alpha"][l], t["beta"][l], N, s)
        wins.append(w)
        ctx.set_spans(l, w, s, N)
    kc, vc = ctx.alloc_cache(B)
    kp = torch.randn(B, N, cfg.hkv, d, device=dev, dtype=torch.bfloat16)   # one prompt K/V for every layer
    vp = torch.randn(B, N, cfg.hkv, d, device=dev, dtype=torch.bfloat16)
    ws = ctx.alloc_workspace(B)
    T = a.tokens
    qd, kd, vd = decode_tokens(cfg, 0, T, batch=B, device=dev)
    od = torch.empty(B, cfg.hq, d, dtype=torch.bfloat16, device=dev)
    scale = 1 / math.sqrt(d)
    # in-window bytes per launch (mean over layers), p = N + t
    by = 0.0
    for t_ in range(T):
        p = N + t_
        for l in range(L):
            wg = [max(wins[l][g * G:(g + 1) * G]) for g in range(cfg.hkv)]
            by += sum(min(p + 1, s + w) for w in wg) * d * 2 * 2 * B + B * cfg.hq * d * 2 * 2 + B * cfg.hkv * d * 2 * 2 * 2
    by /= T * L
    stream = torch.cuda.current_stream()

    def phase(per_launch):
        evs = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t_ in range(T):
            for l in range(L):
                if per_launch:
                    x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    x.record(stream)
                ctx.decode_step_fused(l, qd[t_], kd[t_], vd[t_], od, N + t_, scale, ws)
                if per_launch:
                    y.record(stream)
                    evs.append((x, y))
        e1.record(stream)
        torch.cuda.synchronize()
        tot = e0.elapsed_time(e1) * 1e3 / (T * L)
        k = sum(x.elapsed_time(y) for x, y in evs) * 1e3 / (T * L) if evs else float("nan")
        return tot, k

    # positions are replayed from N: cache_fill resets every layer to next_pos = N
    def reset():
        for l in range(L):
            ctx.cache_fill(l, kp, vp)
        torch.cuda.synchronize()

    for mode in (False, True, False, True):
        reset()
        phase(mode)          # warm
        reset()
        tot, k = phase(mode)
        print(f"per-launch events={mode!s:5}  phase {tot:7.2f} us/launch ({by / tot / 1e3:7.1f} GB/s)   "
              f"kernel events {k:7.2f} us ({by / k / 1e3 if k == k else float('nan'):7.1f} GB/s)", flush=True)
    print(f"bytes/launch {by / 1e6:.1f} MB, variant {os.environ.get('MOA_DEC_VARIANT', '0')}")


if __name__ == "__main__":
    main()
