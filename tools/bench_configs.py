"""Throughput of every BASELINE.json config on one B200 (the bench.py line covers C2 only).

    python tools/bench_configs.py [--configs C1,C3,C4,C5] [--out profiles/r01_configs.json]

Per config, with the same synthetic recipe as the parity tests (moa_workloads):
  decode  (C1, C3, C5): fused append + split-KV decode over all layers, CUDA events around
          T tokens x L launches; tokens/s = B * T / time and in-window GB/s against the
          measured HBM peak.  C5's 80-layer cache (171.8 GB) is timed on `--c5-layers`
          resident layers and the per-launch time is scaled to 80 layers (stated in the output).
  prefill (C1, C4): moa_prefill_attn over all layers (tcgen05 kernel for bf16), tokens/s =
          B * N / time and in-window TFLOP/s against the measured sustained bf16 peak.
Diagnostic reporting only; bench.py is the measured contract.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from moa_workloads import CONFIGS, decode_tokens, prefill_qkv, rule_table  # noqa: E402


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d["hbm_gbs"], d.get("bf16_tflops_sustained", d["bf16_tflops"])
    return 6650.0, 1400.0


def windows_of(cfg, l):
    if cfg.windows is not None:
        return list(cfg.windows)
    t = rule_table(cfg.name)
    return moa.resolve_spans(t["alpha"][l], t["beta"][l], cfg.N, cfg.n_sink)


def pairs(N, W, s):
    W = min(W, N)
    if W == 0:
        m = min(s, N)
        return m * N - m * (m - 1) // 2
    return W * (W + 1) // 2 + (N - W) * W + sum(min(s, i - W + 1) for i in range(W, N))


def time_decode(cfg, layers, tokens, dtype):
    dev = torch.device("cuda")
    L, B, N, s, d, G = layers, cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim, cfg.group
    ctx = moa.MoAContext(L, cfg.hq, cfg.hkv, d, B, dtype=dtype)
    wins = [windows_of(cfg, l) for l in range(L)]
    for l in range(L):
        ctx.set_spans(l, wins[l], s, N)
    ctx.alloc_cache(B)
    g = torch.Generator(device=dev).manual_seed(cfg.seed_base + 7)
    kp = torch.randn(B, N, cfg.hkv, d, device=dev, generator=g).to(dtype)
    vp = torch.randn(B, N, cfg.hkv, d, device=dev, generator=g).to(dtype)
    ws = ctx.alloc_workspace(B)
    qd, kd, vd = decode_tokens(cfg, 0, tokens, batch=B, device=dev)
    od = torch.empty(B, cfg.hq, d, dtype=dtype, device=dev)
    scale = 1 / math.sqrt(d)
    es = torch.finfo(dtype).bits // 8
    by = 0.0
    for t_ in range(tokens):
        p = N + t_
        for l in range(L):
            wg = [max(wins[l][x * G:(x + 1) * G]) for x in range(cfg.hkv)]
            by += (sum(min(p + 1, s + w) for w in wg) * d * 2 * es * B + B * cfg.hq * d * 2 * es
                   + B * cfg.hkv * d * 2 * es * 2)

    def run():
        for l in range(L):
            ctx.cache_fill(l, kp, vp)  # positions restart at N
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t_ in range(tokens):
            for l in range(L):
                ctx.decode_step_fused(l, qd[t_], kd[t_], vd[t_], od, N + t_, scale, ws)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    run()
    sec = min(run() for _ in range(2))
    return sec, by


def time_prefill(cfg, layers, dtype):
    dev = torch.device("cuda")
    L, B, N, s, d = layers, cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim
    ctx = moa.MoAContext(L, cfg.hq, cfg.hkv, d, B, dtype=dtype)
    flops = 0
    for l in range(L):
        w = windows_of(cfg, l)
        ctx.set_spans(l, w, s, N)
        flops += 4 * d * B * sum(pairs(N, x, s) for x in w)
    qkv = [prefill_qkv(cfg, l, device=dev) for l in range(L)]
    o = torch.empty_like(qkv[0][0])
    scale = 1 / math.sqrt(d)

    def run():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for l in range(L):
            ctx.prefill_attn(l, *qkv[l], o, scale)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    run()
    sec = min(run() for _ in range(3))
    return sec, flops


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C3,C4,C5")
    ap.add_argument("--tokens", type=int, default=32)
    ap.add_argument("--c5-layers", type=int, default=16)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    hbm, tf = peaks()
    res = {}
    for name in a.configs.split(","):
        cfg = CONFIGS[name]
        dtype = torch.float32 if cfg.dtype == "f32" else torch.bfloat16
        r = {}
        if "decode" in cfg.modes:
            L = min(cfg.layers, a.c5_layers) if name == "C5" else cfg.layers
            T = min(a.tokens, cfg.decode_steps)
            sec, by = time_decode(cfg, L, T, dtype)
            per_launch = sec / (T * L)
            tps = cfg.batch / (per_launch * cfg.layers)
            r["decode"] = {"tokens_per_s": tps, "us_per_layer_token": per_launch * 1e6,
                           "in_window_GBps": by / (T * L) / per_launch / 1e9,
                           "frac_hbm": by / (T * L) / per_launch / 1e9 / hbm, "layers_timed": L,
                           "layers_model": cfg.layers, "tokens": T, "batch": cfg.batch}
        if "prefill" in cfg.modes:
            sec, flops = time_prefill(cfg, cfg.layers, dtype)
            r["prefill"] = {"tokens_per_s": cfg.batch * cfg.N / sec, "ms_all_layers": sec * 1e3,
                            "in_window_TFLOPs": flops / sec / 1e12, "frac_sustained_bf16": flops / sec / 1e12 / tf,
                            "layers": cfg.layers, "batch": cfg.batch, "N": cfg.N}
        res[name] = r
        print(name, json.dumps(r), flush=True)
        torch.cuda.empty_cache()
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"gpu": torch.cuda.get_device_name(), "peaks": {"hbm_gbs": hbm, "bf16_tflops_sustained": tf},
                       "configs": res}, f, indent=1)


if __name__ == "__main__":
    main()
