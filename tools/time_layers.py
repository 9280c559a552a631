"""Cross-layer decode vs one launch per layer on the full C2 cache (diagnostic).

    python tools/time_layers.py [--config C2] [--tokens 32] [--chunk 0]

Times T tokens x L layers of fused decode as (a) L single-layer launches per token and
(b) one moa_decode_step_fused_layers launch per token, CUDA events around the phase;
prints us per layer-token and the in-window GB/s of both.
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
    ap.add_argument("--tokens", type=int, default=32)
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=0)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    dev = torch.device("cuda")
    L = a.layers or cfg.layers
    B, N, s, d, G, T = cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim, cfg.group, a.tokens
    t = rule_table(cfg.name)
    wins = [moa.resolve_spans(t["alpha"][l], t["beta"][l], N, s) for l in range(L)]
    ctx = moa.MoAContext(L, cfg.hq, cfg.hkv, d, B, dtype=torch.bfloat16)
    if a.chunk:
        ctx.set_decode_split(a.chunk)
    for l in range(L):
        ctx.set_spans(l, wins[l], s, N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B, L)
    g = torch.Generator(device=dev).manual_seed(7)
    kp = torch.randn(B, N, cfg.hkv, d, device=dev, generator=g).to(torch.bfloat16)
    vp = torch.randn(B, N, cfg.hkv, d, device=dev, generator=g).to(torch.bfloat16)
    qd, kd, vd = decode_tokens(cfg, 0, T, device=dev)
    ql = qd[:, None].expand(T, L, *qd.shape[1:]).contiguous()
    kl = kd[:, None].expand(T, L, *kd.shape[1:]).contiguous()
    vl = vd[:, None].expand(T, L, *vd.shape[1:]).contiguous()
    o = torch.empty(L, B, cfg.hq, d, dtype=torch.bfloat16, device=dev)
    scale = 1 / math.sqrt(d)
    by = 0
    for t_ in range(T):
        for l in range(L):
            wg = [max(wins[l][x * G:(x + 1) * G]) for x in range(cfg.hkv)]
            by += B * (sum(min(N + t_ + 1, s + w) for w in wg) * d * 4 + cfg.hq * d * 4 + cfg.hkv * d * 8)

    def run(ml):
        for l in range(L):
            ctx.cache_fill(l, kp, vp)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t_ in range(T):
            if ml:
                ctx.decode_step_fused_layers(0, ql[t_], kl[t_], vl[t_], o, N + t_, scale, ws)
            else:
                for l in range(L):
                    ctx.decode_step_fused(l, ql[t_, l], kl[t_, l], vl[t_, l], o[l], N + t_, scale, ws)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    for ml in (False, True, False, True):
        run(ml)
        sec = min(run(ml) for _ in range(3))
        print(f"{'cross-layer ' if ml else 'per-layer   '}: {sec / (T * L) * 1e6:7.2f} us/layer-token, "
              f"{by / sec / 1e9:8.1f} GB/s in-window, {B * T / sec:9.1f} tokens/s ({L} layers)", flush=True)


if __name__ == "__main__":
    main()
