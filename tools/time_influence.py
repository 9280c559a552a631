"""Time moa_attention_influence (NEXT-2) on a profiling-shaped item (CUDA events).

    python tools/time_influence.py [N] [heads] [d]

FLOP count: the two passes each run S = Q K^T and G = dO V^T on every causal 64 x 64
block pair: 4 GEMMs x 2 x 64 * 64 * d per pair.
"""
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
    reps = 3
    for _ in range(reps):
        moa.attention_influence(q, k, v, do, sc, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pairs = nb * (nb + 1) // 2
    flops = 4 * 2 * 64 * 64 * d * pairs * H
    print(f"influence N={N} heads={H} d={d}: {ms:.3f} ms per item-layer, {flops / ms / 1e9:.1f} TFLOP/s (mma.sync)")


if __name__ == "__main__":
    a = [int(x) for x in sys.argv[1:]]
    main(*a)
