"""Time a ragged C2 batch (per-sequence lengths and Eq. 2 spans) against the uniform batch.

    python tools/time_ragged.py [layers] [seed]     (seed < 0: all N_b = N, the RAG kernel on uniform work)

Lengths N_b are drawn uniformly from [N/4, N] (seeded); windows are Eq. 2 at N_b
(moa.resolve_spans), clipped to the capacity resolved at N.  Prefill: in-window TFLOP/s
(4 d |V(h,i)| per visible pair, every sequence with its own windows) and tokens/s over
sum N_b.  Decode: fused ragged append+decode at positions N_b (device pos tensor), per
layer-token time vs the uniform decode of the same capacity (the ring capacity is what
the kernel streams).  Diagnostic reporting only.
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from moa_workloads import CONFIGS, decode_tokens, prefill_qkv, rule_table  # noqa: E402
sys.path.insert(0, os.path.join(ROOT, "tools"))
from time_prefill import pairs  # noqa: E402


def main(layers=4, seed=0):
    cfg = CONFIGS["C2"]
    t = rule_table("C2")
    dev = torch.device("cuda")
    B, N, s, d = cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim
    rng = np.random.default_rng(abs(seed))
    lens = sorted(rng.integers(N // 4, N + 1, size=B).tolist(), reverse=True)
    if seed < 0:  # control: a ragged batch with every sequence at full length (= uniform work)
        lens = [N] * B
    L = list(range(8, 8 + layers))
    ctx = moa.MoAContext(len(L), cfg.hq, cfg.hkv, d, B)
    uni = moa.MoAContext(len(L), cfg.hq, cfg.hkv, d, B)
    flops_r = flops_u = 0
    for i, l in enumerate(L):
        cap = moa.resolve_spans(t["alpha"][l], t["beta"][l], N, s)
        wins = [[min(w, c) for w, c in zip(moa.resolve_spans(t["alpha"][l], t["beta"][l], n, s), cap)]
                for n in lens]
        ctx.set_spans(i, cap, s, N)
        ctx.set_ragged(i, lens, wins)
        uni.set_spans(i, cap, s, N)
        flops_r += 4 * d * sum(pairs(n, w, s) for b, n in enumerate(lens) for w in wins[b])
        flops_u += 4 * d * B * sum(pairs(N, w, s) for w in cap)
    ctx.alloc_cache(B)
    uni.alloc_cache(B)
    qkv = [prefill_qkv(cfg, l, device=dev) for l in L]
    o = torch.empty_like(qkv[0][0])
    sc = 1 / math.sqrt(d)

    def time_prefill(c):
        for _ in range(2):
            for i in range(len(L)):
                c.prefill(i, *qkv[i], o, sc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            for i in range(len(L)):
                c.prefill(i, *qkv[i], o, sc)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 3

    ms_r, ms_u = time_prefill(ctx), time_prefill(uni)
    print(f"lens {lens}")
    print(f"prefill ragged  {ms_r:.3f} ms  {flops_r / ms_r / 1e9:.1f} TFLOP/s  "
          f"{sum(lens) * len(L) / ms_r / 1e3:.3e} layer-tokens/s")
    print(f"prefill uniform {ms_u:.3f} ms  {flops_u / ms_u / 1e9:.1f} TFLOP/s  "
          f"{B * N * len(L) / ms_u / 1e3:.3e} layer-tokens/s")

    T = 16
    qd, kd, vd = decode_tokens(cfg, 0, T, batch=B, device=dev)
    od = torch.empty(B, cfg.hq, d, dtype=torch.bfloat16, device=dev)
    ws = ctx.alloc_workspace(B)
    wsu = uni.alloc_workspace(B)
    pos = torch.tensor(lens, dtype=torch.int64, device=dev)

    def time_decode(ragged):
        c = ctx if ragged else uni
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for rep in range(3):
            for i in range(len(L)):
                c.prefill(i, *qkv[i], o, sc)  # refills the cache; positions restart
            pos.copy_(torch.tensor(lens, dtype=torch.int64))
            torch.cuda.synchronize()
            e0.record()
            for t_ in range(T):
                for i in range(len(L)):
                    if ragged:
                        c.decode_step_fused_ragged(i, qd[t_], kd[t_], vd[t_], od, pos, sc, ws)
                    else:
                        c.decode_step_fused(i, qd[t_], kd[t_], vd[t_], od, N + t_, sc, wsu)
                if ragged:
                    pos.add_(1)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                best = min(best, e0.elapsed_time(e1))
        return best * 1e3 / (T * len(L))

    us_r, us_u = time_decode(True), time_decode(False)
    print(f"decode ragged  {us_r:.2f} us/layer-token (incl. the pos += 1 kernel per token)")
    print(f"decode uniform {us_u:.2f} us/layer-token")


if __name__ == "__main__":
    a = sys.argv[1:]
    main(int(a[0]) if a else 4, int(a[1]) if len(a) > 1 else 0)
