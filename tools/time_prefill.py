"""Time moa_prefill over several layers of a config (CUDA events), print TFLOP/s."""
import math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2406_14909_b200 as moa
from moa_workloads import CONFIGS, prefill_qkv, rule_table


def pairs(N, W, s):
    W = min(W, N)
    if W == 0:
        m = min(s, N)
        return m * N - m * (m - 1) // 2
    return W * (W + 1) // 2 + (N - W) * W + sum(min(s, i - W + 1) for i in range(W, N))


def main(name="C2", layers=4, reps=3):
    cfg = CONFIGS[name]
    t = rule_table(name)
    dev = torch.device("cuda")
    L = list(range(cfg.layers - layers, cfg.layers)) if name != "C2" else list(range(8, 8 + layers))
    ctx = moa.MoAContext(len(L), cfg.hq, cfg.hkv, cfg.head_dim, cfg.batch)
    flops = 0
    for i, l in enumerate(L):
        W = moa.resolve_spans(t["alpha"][l], t["beta"][l], cfg.N, cfg.n_sink)
        ctx.set_spans(i, W, cfg.n_sink, cfg.N)
        flops += 4 * cfg.head_dim * cfg.batch * sum(pairs(cfg.N, w, cfg.n_sink) for w in W)
    ctx.alloc_cache(cfg.batch)
    qkv = [prefill_qkv(cfg, l, device=dev) for l in L]
    o = torch.empty_like(qkv[0][0])
    sc = 1 / math.sqrt(cfg.head_dim)
    for _ in range(2):
        for i in range(len(L)):
            ctx.prefill(i, *qkv[i], o, sc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for i in range(len(L)):
            ctx.prefill(i, *qkv[i], o, sc)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} layers={len(L)} {ms:.3f} ms  {flops / (ms / 1e3) / 1e12:.1f} TFLOP/s")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 4)
