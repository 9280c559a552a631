"""Decode timing study on the full C2 cache (all 32 layers resident, 8.6 GB).

    python tools/time_decode.py [--tokens 64] [--config C2]

Times the fused decode phase (tokens x layers launches) with CUDA events
around the whole phase, with and without an event pair around every launch,
and prints µs per launch and the in-window GB/s.  Diagnostic only.
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


def dump_trace():
    import ctypes

    import numpy as np

    from paper_2406_14909_b200 import _lib
    buf = np.zeros((2, 1024, 8), dtype=np.uint64)
    fn = _lib.lib().moa_debug_decode_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    names = ["entry", "prologue", "prod_start", "cons_wait", "first_tile", "loop_end", "end"]
    valid = [buf[s_][:, 0] > 0 for s_ in range(2)]
    t0 = min(int(buf[s_][valid[s_], 0].min()) for s_ in range(2))
    for s_ in range(2):
        b = buf[s_][valid[s_]].astype(np.int64)
        rel = (b[:, :7] - t0) / 1e3
        print(f"launch slot {s_}: {len(b)} CTAs (us from the first entry of both launches)")
        for i, n in enumerate(names):
            col = rel[:, i]
            print(f"  {n:11s} min {col.min():8.2f}  med {np.median(col):8.2f}  max {col.max():8.2f}")
        tiles = b[:, 7] & 0xffffffff
        npend = (b[:, 7] >> 32) & 0xff
        nseg = (b[:, 7] >> 40) & 0xff
        smid = (b[:, 7] >> 48) & 0xffff
        print(f"  tiles/CTA min {tiles.min()} max {tiles.max()}; pending combines max {npend.max()}")
        loop = rel[:, 5] - rel[:, 4]
        comb = rel[:, 6] - rel[:, 5]
        for k in sorted(set(nseg.tolist())):
            m = nseg == k
            print(f"  nseg={k}: {m.sum():3d} CTAs, loop us med {np.median(loop[m]):6.2f} max {loop[m].max():6.2f}, "
                  f"tiles med {np.median(tiles[m]):.0f}")
        for k in sorted(set(npend.tolist())):
            m = npend == k
            print(f"  npend={k}: {m.sum():3d} CTAs, combine us med {np.median(comb[m]):6.2f} max {comb[m].max():6.2f}")
        per_tile = loop / np.maximum(tiles, 1)
        order = np.argsort(-loop)[:8]
        print("  slowest CTAs (cta, sm, tiles, nseg, loop us, us/tile):",
              [(int(i), int(smid[i]), int(tiles[i]), int(nseg[i]), round(float(loop[i]), 2),
                round(float(per_tile[i]), 2)) for i in order])
        # per-SM: sum of loop of its CTAs
        sm_t = {}
        for i in range(len(b)):
            sm_t.setdefault(int(smid[i]), []).append(float(per_tile[i]))
        v = np.array([np.mean(x) for x in sm_t.values()])
        print(f"  us/tile by SM: min {v.min():.2f} med {np.median(v):.2f} max {v.max():.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--trace", action="store_true", help="read the per-CTA stamps (MOA_LIB=libmoa_trace.so)")
    ap.add_argument("--read-peak", action="store_true", help="also time a plain 4 GiB read (torch sum)")
    ap.add_argument("--graph", action="store_true", help="also replay a CUDA graph of one token step")
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    L = a.layers or cfg.layers
    B, N, s, d, G = a.batch or cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim, cfg.hq // cfg.hkv
    dev = torch.device("cuda")
    t = rule_table(cfg.name)
    ctx = moa.MoAContext(L, cfg.hq, cfg.hkv, d, B, dtype=torch.bfloat16)
    wins = []
    for l in range(L):
        w = moa.resolve_spans(t["alpha"][l], t["beta"][l], N, s)
        wins.append(w)
        ctx.set_spans(l, w, s, N)
    kc, vc = ctx.alloc_cache(B)
    kp = torch.randn(B, N, cfg.hkv, d, device=dev, dtype=torch.bfloat16)   # one prompt K/V for every layer
    vp = torch.randn(B, N, cfg.hkv, d, device=dev, dtype=torch.bfloat16)
    ws = ctx.alloc_workspace(B)
    T = a.tokens
    qd, kd, vd = decode_tokens(cfg, 0, T, batch=B, device=dev)
    od = torch.empty(B, cfg.hq, d, dtype=torch.bfloat16, device=dev)
    scale = 1 / math.sqrt(d)
    # in-window bytes per launch (mean over layers), p = N + t
    by = 0.0
    for t_ in range(T):
        p = N + t_
        for l in range(L):
            wg = [max(wins[l][g * G:(g + 1) * G]) for g in range(cfg.hkv)]
            by += sum(min(p + 1, s + w) for w in wg) * d * 2 * 2 * B + B * cfg.hq * d * 2 * 2 + B * cfg.hkv * d * 2 * 2 * 2
    by /= T * L
    stream = torch.cuda.current_stream()

    def phase(per_launch):
        evs = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t_ in range(T):
            for l in range(L):
                if per_launch:
                    x, y = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    x.record(stream)
                ctx.decode_step_fused(l, qd[t_], kd[t_], vd[t_], od, N + t_, scale, ws)
                if per_launch:
                    y.record(stream)
                    evs.append((x, y))
        e1.record(stream)
        torch.cuda.synchronize()
        tot = e0.elapsed_time(e1) * 1e3 / (T * L)
        k = sum(x.elapsed_time(y) for x, y in evs) * 1e3 / (T * L) if evs else float("nan")
        return tot, k

    # positions are replayed from N: cache_fill resets every layer to next_pos = N
    def reset():
        for l in range(L):
            ctx.cache_fill(l, kp, vp)
        torch.cuda.synchronize()

    for mode in (True, False, True, False):
        reset()
        phase(mode)          # warm
        reset()
        tot, k = phase(mode)
        print(f"per-launch events={mode!s:5}  phase {tot:7.2f} us/launch ({by / tot / 1e3:7.1f} GB/s)   "
              f"kernel events {k:7.2f} us ({by / k / 1e3 if k == k else float('nan'):7.1f} GB/s)", flush=True)
    if a.graph:
        # one token step (all layers, fused decode with device positions, then moa_advance_pos)
        # captured once in a CUDA graph and replayed T times
        pos = torch.full((B,), N, dtype=torch.int64, device=dev)
        q0, k0, v0 = qd[0].clone(), kd[0].clone(), vd[0].clone()
        g = torch.cuda.CUDAGraph()
        reset()
        s_ = torch.cuda.Stream()
        with torch.cuda.stream(s_):
            with torch.cuda.graph(g, stream=s_):
                for l in range(L):
                    ctx.decode_step_fused_ragged(l, q0, k0, v0, od, pos, scale, ws)
                moa.advance_pos(pos)
        for rep in range(3):
            reset()
            pos.fill_(N)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for t_ in range(T):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            tot = e0.elapsed_time(e1) * 1e3 / (T * L)
            print(f"graph replay (token step = {L} layers + advance)  {tot:7.2f} us/launch ({by / tot / 1e3:7.1f} GB/s)",
                  flush=True)
    if a.trace:
        dump_trace()
    print(f"bytes/launch {by / 1e6:.1f} MB, batch {B}, variant {os.environ.get('MOA_DEC_VARIANT', '0')}, "
          f"chunk {os.environ.get('MOA_DEC_CHUNK', 'default')}")
    if a.read_peak:
        del kp, vp
        x = torch.empty(2 * 1024**3, dtype=torch.bfloat16, device=dev).uniform_()
        for _ in range(3):
            x.sum(dtype=torch.float32)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            x.sum(dtype=torch.float32)
        e1.record()
        torch.cuda.synchronize()
        print(f"torch sum read: {10 * x.numel() * 2 / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
