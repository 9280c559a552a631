"""Time moa_attention_influence (NEXT-2) on a profiling-shaped item (CUDA events).

    python tools/time_influence.py [N] [heads] [d]

FLOP counts (per head):
  algorithmic -- the method's own products, S = Q K^T and G = dO V^T over the causal token
                 pairs: 4 d per pair, sum_i (i + 1) = N (N + 1) / 2 pairs;
  executed    -- what the kernel issues: both passes run both products on every 64-key tile
                 of the 128-row q tiles up to the diagonal (the diagonal tiles in full).
The roofline fraction uses the algorithmic count against the bf16 dense burst peak
(MEASURED_PEAKS.json).  MOA_INF_LEGACY=1 times the round-1 mma.sync kernel instead.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402


def main(N=8192, H=32, d=128):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = (torch.randn(1, N, H, d, device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    nb = (N + 63) // 64
    out = torch.empty(1, H, nb, nb, device=dev)
    sc = 1 / math.sqrt(d)
    for _ in range(2):
        moa.attention_influence(q, k, v, do, sc, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        moa.attention_influence(q, k, v, do, sc, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    alg = 4 * d * (N * (N + 1) // 2) * H
    ntile = (N + 127) // 128
    exe_tiles = sum(min((min(128 * qt + 127, N - 1)) // 64 + 1, nb) for qt in range(ntile))
    exe = 2 * 2 * 2 * 128 * 64 * d * exe_tiles * H
    peak = 1645.0
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peak = json.load(open(pk)).get("bf16_tflops", peak)
    kind = "mma.sync (legacy)" if os.environ.get("MOA_INF_LEGACY") == "1" else "tcgen05"
    print(f"influence N={N} heads={H} d={d} [{kind}]: {ms:.3f} ms per item-layer; algorithmic "
          f"{alg / ms / 1e9:.1f} TFLOP/s = {alg / ms / 1e9 / peak:.3f} of the {peak:.0f} TF bf16 burst; "
          f"executed {exe / ms / 1e9:.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
