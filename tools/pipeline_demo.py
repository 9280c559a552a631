"""The MoA pipeline end to end on one B200, on synthetic data (no trained weights exist here):
profile -> rule losses -> rule selection -> spans -> prefill + decode.

    python tools/pipeline_demo.py [--layers 4] [--N 4096] [--items 2] [--budget 0.5]

1. profile   moa_attention_influence on synthetic calibration items (Q, K, V and dO of a
             Vicuna-7B-shaped layer, N(0,1)), averaged over items      (Eq. 3)
2. losses    moa_rule_losses over the paper's 6 x 9 rule grid          (Eq. 4)
3. select    moa_plan_rules at the density budget, <= 2 rules / layer  (Eq. 5)
4. serve     windows of the chosen rules -> moa_set_spans_blocked (block 64) -> moa_prefill +
             a few fused decode steps
Synthetic influence has no semantic structure, so the chosen spans only exercise the
mechanics; timings are per stage (CUDA events).
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from moa_workloads import ALPHA_GRID, BETA_GRID  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = fn()
    e1.record()
    torch.cuda.synchronize()
    return r, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--items", type=int, default=2)
    ap.add_argument("--budget", type=float, default=0.5)
    a = ap.parse_args()
    dev = torch.device("cuda")
    L, N, H, d, s, B = a.layers, a.N, 32, 128, 64, 1
    sc = 1 / math.sqrt(d)
    g = torch.Generator(device=dev).manual_seed(0)
    nb = (N + 63) // 64
    alphas = [x for x in ALPHA_GRID for _ in BETA_GRID]
    betas = [y for _ in ALPHA_GRID for y in BETA_GRID]
    # 1 + 2: profile and rule losses per layer
    losses = np.zeros((L * H, len(alphas)), dtype=np.float32)
    t_prof = t_loss = 0.0
    for l in range(L):
        eb = torch.zeros(1, H, nb, nb, device=dev)
        for it in range(a.items):
            q, k, v, do = (torch.randn(1, N, H, d, device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
            _, ms = timed(lambda: moa.attention_influence(q, k, v, do, sc, out=eb, accumulate=it > 0))
            t_prof += ms
        eb /= a.items
        lo, ms = timed(lambda: moa.rule_losses(eb[0].contiguous(), N, s, alphas, betas))
        t_loss += ms
        losses[l * H:(l + 1) * H] = lo.cpu().numpy()
    # 3: select
    wins = [moa.resolve_spans([al], [be], N, s)[0] for al, be in zip(alphas, betas)]
    wins = [((w + s + 63) // 64) * 64 - s if w > 0 else 0 for w in wins]   # block-rounded spans
    dens = np.array([min(N, s + w) / N for w in wins], dtype=np.float32)
    plan, tot, D = moa.plan_rules(losses, dens, L, H, a.budget, 2)
    # 4: serve with the chosen spans
    ctx = moa.MoAContext(L, H, H, d, B)
    for l in range(L):
        ctx.set_spans(l, [wins[r] for r in plan[l * H:(l + 1) * H]], s, N, block=64)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    q, k, v = (torch.randn(B, N, H, d, device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    o = torch.empty_like(q)
    _, t_pre = timed(lambda: [ctx.prefill(l, q, k, v, o, sc) for l in range(L)])
    qd, kd, vd = (torch.randn(B, H, d, device=dev, generator=g).to(torch.bfloat16) for _ in range(3))
    od = torch.empty_like(qd)
    _, t_dec = timed(lambda: [ctx.decode_step_fused(l, qd, kd, vd, od, N, sc, ws) for l in range(L)])
    used = sorted(set(plan))
    print(f"profile {t_prof:.1f} ms ({a.items} items x {L} layers, N={N}), rule losses {t_loss:.2f} ms")
    print(f"plan: {len(used)} distinct rules, mean density {D:.3f} (budget {a.budget}), total loss {tot:.4g}")
    for l in range(L):
        rs = sorted(set(plan[l * H:(l + 1) * H]))
        print(f"  layer {l}: rules {[(alphas[r], betas[r]) for r in rs]} windows {[wins[r] for r in rs]}")
    print(f"prefill {t_pre:.2f} ms for {L} layers, decode step {t_dec:.3f} ms; finite output: "
          f"{bool(torch.isfinite(o).all())}, {bool(torch.isfinite(od).all())}")


if __name__ == "__main__":
    main()
