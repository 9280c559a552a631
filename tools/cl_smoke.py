"""Tiny bf16 prefill vs the fp64 oracle (hang check of a kernel change; MOA_PP_CLUSTER=1 for the clustered kernel)."""
import math, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle, paper_2406_14909_b200 as m
from moa_workloads import normal
for (N, d, W) in [(100, 128, [0, 17, 64, 300]), (300, 128, [0, 17, 64, 300]), (300, 64, [5, 130, 1, 1000])]:
    B, Hq, Hkv, s = 2, 4, 2, 4
    ctx = m.MoAContext(1, Hq, Hkv, d, B, dtype=torch.bfloat16, device=0)
    ctx.set_spans(0, W, s, N)
    ctx.alloc_cache(B)
    q, k, v = normal((B, N, Hq, d), 1, torch.bfloat16), normal((B, N, Hkv, d), 2, torch.bfloat16), normal((B, N, Hkv, d), 3, torch.bfloat16)
    o = torch.empty(B, N, Hq, d, dtype=torch.bfloat16, device="cuda")
    ctx.prefill(0, q.cuda(), k.cuda(), v.cuda(), o, 1 / math.sqrt(d))
    torch.cuda.synchronize()
    f = lambda t: t.to(torch.float64).cpu().numpy()
    O, _ = oracle.prefill(f(q), f(k), f(v), W, s, 1 / math.sqrt(d))
    print(N, d, "max err", float(np.abs(f(o) - O).max()), flush=True)
