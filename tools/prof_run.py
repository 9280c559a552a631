"""Short driver for ncu captures of one kernel family on C2-shaped inputs.

    python tools/prof_run.py decode [--layers 4] [--tokens 8]
    python tools/prof_run.py layers [--layers 32 --first-layer 0] [--tokens 3]   (cross-layer launches)
    python tools/prof_run.py prefill [--layers 2]

Sets up C2 layers (real rule spans), runs prefill once per layer, then
`tokens` fused decode steps over the layers.  Used under
`ncu --set full -k regex:... -s <skip> -c <count>`.
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from moa_workloads import CONFIGS, decode_tokens, prefill_qkv, rule_table  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["decode", "prefill", "layers"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--layers", type=int, default=4)
    ap.add_argument("--first-layer", type=int, default=12)
    ap.add_argument("--tokens", type=int, default=8)
    ap.add_argument("--batch", type=int, default=None)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    B = a.batch or cfg.batch
    dev = torch.device("cuda")
    t = rule_table(cfg.name)
    layers = list(range(a.first_layer, a.first_layer + a.layers))
    ctx = moa.MoAContext(len(layers), cfg.hq, cfg.hkv, cfg.head_dim, B, dtype=torch.bfloat16)
    for i, l in enumerate(layers):
        ctx.set_spans(i, moa.resolve_spans(t["alpha"][l], t["beta"][l], cfg.N, cfg.n_sink), cfg.n_sink, cfg.N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B, len(layers))
    scale = 1 / math.sqrt(cfg.head_dim)
    O = None
    for i, l in enumerate(layers):
        q, k, v = prefill_qkv(cfg, l, batch=B, device=dev)
        if O is None:
            O = torch.empty_like(q)
        ctx.prefill(i, q, k, v, O, scale)
        del q, k, v
    if a.what == "decode":
        qd, kd, vd = decode_tokens(cfg, 0, a.tokens, batch=B, device=dev)
        od = torch.empty(B, cfg.hq, cfg.head_dim, dtype=torch.bfloat16, device=dev)
        for tt in range(a.tokens):
            for i in range(len(layers)):
                ctx.decode_step_fused(i, qd[tt], kd[tt], vd[tt], od, cfg.N + tt, scale, ws)
    if a.what == "layers":
        qd, kd, vd = decode_tokens(cfg, 0, a.tokens, batch=B, device=dev)
        L = len(layers)
        od = torch.empty(L, B, cfg.hq, cfg.head_dim, dtype=torch.bfloat16, device=dev)
        for tt in range(a.tokens):
            ctx.decode_step_fused_layers(0, qd[tt].expand(L, *qd[tt].shape), kd[tt].expand(L, *kd[tt].shape),
                                         vd[tt].expand(L, *vd[tt].shape), od, cfg.N + tt, scale, ws)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
