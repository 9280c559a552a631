"""Worker of tests/test_gpu_prefill.py::test_prefill_bf16_clustered_kernel (run with
MOA_PP_CLUSTER=1 in its own process): the clustered bf16 prefill against the fp64 oracle."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_2406_14909_b200 as m  # noqa: E402
from moa_workloads import normal  # noqa: E402
from tests.gpu_util import check_cache_image, f64  # noqa: E402


def run(q, k, v, W, s, scale):
    B, N, Hq, d = q.shape
    Hkv = k.shape[2]
    ctx = m.MoAContext(1, Hq, Hkv, d, B, dtype=torch.bfloat16, device=0)
    ctx.set_spans(0, W, s, N)
    ctx.alloc_cache(B)
    o = torch.empty(B, N, Hq, d, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B, Hq, N, dtype=torch.float32, device="cuda")
    ctx.prefill(0, q.cuda(), k.cuda(), v.cuda(), o, scale, lse=lse)
    torch.cuda.synchronize()
    return ctx, o, lse


def main():
    assert os.environ.get("MOA_PP_CLUSTER") == "1"
    for d in (128, 64):
        for N in (100, 300, 513, 1100):
            B, Hq, Hkv, s = 2, 6, 3, 4
            W = [0, 1, 130, 257, 17, N + 3]
            q = normal((B, N, Hq, d), 211, torch.bfloat16)
            k = normal((B, N, Hkv, d), 212, torch.bfloat16)
            v = normal((B, N, Hkv, d), 213, torch.bfloat16)
            scale = 1 / math.sqrt(d)
            ctx, o, lse = run(q, k, v, W, s, scale)
            O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, scale)
            assert np.isfinite(f64(o)).all()
            err = float(np.abs(f64(o) - O).max())
            assert err < 2e-2, (d, N, err)
            assert float(np.abs(f64(lse) - L).max()) < 2e-3, (d, N)
            check_cache_image(ctx, 0, k, v, N - 1, W, s, B, 2)
            print(f"d={d} N={N} max err {err:.2e}", flush=True)
    # score spikes, dominant / vanishing sinks and a growing row max (the lazy reference moves
    # mid-row and is handed between the two softmax groups)
    B, N, H, d, s = 1, 900, 4, 128, 64
    W = [16, 200, 300, 900]
    u = torch.zeros(d)
    u[0] = 1.0
    for sink_score in (12.0, -12.0):
        spike = (torch.arange(N) % 16 == 0).float() * 8.0
        ramp = torch.linspace(0.0, 30.0, N)
        k = ((spike + ramp)[None, :, None, None] * u).expand(B, N, H, d).clone()
        k[:, :s] = sink_score * u
        k = (k + 0.01 * normal((B, N, H, d), 15)).to(torch.bfloat16)
        v = normal((B, N, H, d), 16, torch.bfloat16)
        q = u.expand(B, N, H, d).clone().to(torch.bfloat16)
        ctx, o, lse = run(q, k, v, W, s, 1.0)
        O, L = oracle.prefill(f64(q), f64(k), f64(v), W, s, 1.0)
        err = float(np.abs(f64(o) - O).max())
        assert err < 2e-2, (sink_score, err)
        assert float(np.abs(f64(lse) - L).max()) < 2e-3, sink_score
        print(f"structured sink {sink_score}: max err {err:.2e}", flush=True)
    print("clustered parity ok")


if __name__ == "__main__":
    main()
