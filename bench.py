#!/usr/bin/env python
"""MoA hot-path benchmark (BASELINE.json metric: decode + prefill tokens/s, % roofline).

One step = one pass of the whole hot path over one batch of the C2 workload
(configs[1], Vicuna-7B attention shape): span resolution is done once at
setup; the timed step is the prefill of all 32 layers (tcgen05 kernel with the
cache fill fused into it, N = 4096, B = 8) followed by 512 decode tokens x 32 layers (fused
append + split-KV decode + combine; one cross-layer launch per token,
moa_decode_step_fused_layers).  "decode_per_layer" reports the same decode with
one launch per layer-token (the order a model needs when layer l+1's query
depends on layer l's output).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): every rank serves its own batch of 8
sequences (data parallel over independent sequences, no collective on the
data path) -> "scaling": "weak".  At N > 1 (or with --kv-shard) the line also
carries "kv_shard": the north-star partition -- one batch of 8, its kv-groups
split over the ranks, the head outputs all-gathered with NCCL after every layer
(strong scaling, with and without the all-gather).  Timing: barrier + synchronize on both sides,
CUDA events on the launching stream, max over ranks.  The working set (8.6 GB
of cache cycled over 32 layers, 268 MB per layer) exceeds the 126 MB L2, so no
flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from moa_workloads import CONFIGS, decode_tokens, prefill_qkv, rule_table  # noqa: E402

CFG = CONFIGS["C2"]
DECODE_CHUNK = 512   # rows per rank-invariant decode chunk in the kv-sharded run (moa_set_decode_split)
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


# --------------------------------------------------------------------------------------------
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return dict(FALLBACK_PEAKS), "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------------------------
def windows_all_layers(moa):
    """Product path: Eq. 2 through the library's moa_resolve_spans."""
    t = rule_table("C2")
    return [moa.resolve_spans(t["alpha"][l], t["beta"][l], CFG.N, CFG.n_sink) for l in range(CFG.layers)]


def oracle_windows_all_layers():
    """Oracle legs: Eq. 2 through oracle.span_of / window_of (no libmoa on that path)."""
    import oracle
    t = rule_table("C2")
    return [[oracle.window_of(oracle.span_of(a, b, CFG.N), CFG.n_sink) for a, b in zip(t["alpha"][l], t["beta"][l])]
            for l in range(CFG.layers)]


def algorithmic_work(windows, B, N, T, s, d, G):
    """In-window work: prefill FLOPs = 4 d sum_{b,h} |V(h,i)| summed over i;
    decode bytes per layer-token = sum_{b,g} min(p+1, s+W_g) * d * 2 (K,V) * 2 B + q/o/new-token bytes."""
    def pairs(W):  # closed form of sum_i |V(h,i)| for W <= N, plain host arithmetic
        W = min(W, N)
        tot = W * (W + 1) // 2 + (N - W) * W
        tot += sum(min(s, i - W + 1) for i in range(W, N)) if W > 0 else min(s, N) * N - (min(s, N) * (min(s, N) - 1)) // 2
        return tot
    flops = 0
    dec_bytes = 0
    for wl in windows:
        flops += sum(4 * d * pairs(w) for w in wl) * B
        wg = [max(wl[g * G:(g + 1) * G]) for g in range(len(wl) // G)]
        rows = sum(min(N + T, s + w) for w in wg)  # ring full during decode (p >= N > s + W_g - 1)
        dec_bytes += B * (rows * d * 2 * 2 + len(wl) * d * 2 * 2 + len(wg) * d * 2 * 2 * 2)
    return flops, dec_bytes  # flops for all layers' prefill; bytes summed over layers for one token step


# --------------------------------------------------------------------------------------------
# Oracle CPU baseline on all host cores (SURVEY §8(d) "Oracle timing"): one process per core,
# each timing oracle.decode / oracle.prefill_rows on rows drawn uniformly at random over
# (layer, q-head, position) of the C2 workload until a shared deadline; the rates are
# extrapolated to the whole workload by the in-window work (decode: visible keys
# min(p+1, s+W_h) per row; prefill: sum |V(h,i)|, oracle.visible_pairs).  The oracle's cost
# does not depend on the values, so one seeded K/V history serves every sampled layer.
_ORC = {}


def _orc_init():
    try:
        import threadpoolctl
        threadpoolctl.threadpool_limits(1)
    except Exception:
        pass


def _orc_work(args):
    """One worker: rows (l, h, i) from its own seeded stream until the deadline."""
    import oracle

    kind, wid, deadline = args
    o = _ORC
    rng = np.random.default_rng(1000 + wid)
    L, Hq, N, T, s, tau = o["L"], o["Hq"], o["N"], o["T"], o["s"], o["tau"]
    K, V, Qp, qd = o["K"], o["V"], o["Q"], o["q"]
    rows = keys = 0
    while time.perf_counter() < deadline:
        l, h = int(rng.integers(L)), int(rng.integers(Hq))
        W = o["W"][l][h]
        if kind == "decode":
            n = int(rng.integers(T))
            p = N + n
            oracle.decode(qd[n][:, h:h + 1], K[:, :p + 1, h:h + 1], V[:, :p + 1, h:h + 1], p, [W], s, tau)
            keys += min(p + 1, s + W)
        else:
            i = int(rng.integers(N))
            oracle.prefill_rows(Qp[:, :, h:h + 1], K[:, :N, h:h + 1], V[:, :N, h:h + 1], [W], s, tau, [(0, 0, i)])
            keys += len(oracle.visible_keys(i, W, s))
        rows += 1
    return rows, keys


def cpu_oracle_baseline(seconds: float = 8.0, cores=None, full=True):
    """Decode and prefill tokens/s of the fp64 oracle on `cores` processes (default: all),
    `seconds` of wall time per phase, plus C1 run in full (`full=False`: decode only, no C1).
    Returns (decode tokens/s, block)."""
    import multiprocessing as mp

    import oracle

    cores = cores or os.cpu_count() or 1
    L, Hq, N, T, d, s = CFG.layers, CFG.hq, CFG.N, CFG.decode_steps, CFG.head_dim, CFG.n_sink
    W = oracle_windows_all_layers()
    g = torch.Generator().manual_seed(7)
    f64 = lambda *shape: torch.randn(*shape, generator=g).to(torch.bfloat16).double().numpy()  # noqa: E731
    _ORC.update(L=L, Hq=Hq, N=N, T=T, s=s, tau=1 / math.sqrt(d), W=W,
                K=f64(1, N + T, CFG.hkv, d), V=f64(1, N + T, CFG.hkv, d), Q=f64(1, N, Hq, d), q=f64(T, 1, Hq, d))
    out = {}
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_orc_init) as pool:
        for kind in (("decode", "prefill") if full else ("decode",)):
            t0 = time.perf_counter()
            res = pool.map(_orc_work, [(kind, w, t0 + seconds) for w in range(cores)])
            wall = time.perf_counter() - t0
            rows, keys = sum(r for r, _ in res), sum(k for _, k in res)
            out[kind] = (rows, keys, wall)
    # workload totals: decode keys per token step (all layers, heads, T positions averaged), prefill pairs
    dec_keys = sum(min(N + n + 1, s + W[l][h]) for l in range(L) for h in range(Hq) for n in range(T)) / T
    pre_pairs = sum(oracle.visible_pairs(N, W[l][h], s) for l in range(L) for h in range(Hq))
    rows, keys, wall = out["decode"]
    dec_tps = (keys / wall) / dec_keys            # tokens/s: one token of one sequence = dec_keys keys
    if not full:
        return dec_tps, {"kind": "oracle", "cores": cores, "value": dec_tps, "unit": "tokens/s",
                         "sample": f"fp64 oracle.decode on {cores} processes x {seconds:.1f} s, {rows} rows "
                                   f"drawn uniformly over the C2 workload's (layer, q-head, position), "
                                   f"{keys} visible keys, extrapolated by visible keys ({dec_keys:.0f} per token)"}
    rows_p, keys_p, wall_p = out["prefill"]
    pre_tps = N * (keys_p / wall_p) / pre_pairs    # N tokens of one sequence = pre_pairs pairs
    # C1 (BASELINE configs[0]) in full, one process: prefill + 64 decode steps
    from moa_workloads import prefill_qkv as pq
    c1 = CONFIGS["C1"]
    qh, kh, vh = (x.double().numpy() for x in pq(c1, 0))
    qd1, kd1, vd1 = (x.double().numpy() for x in decode_tokens(c1, 0, c1.decode_steps))
    t0 = time.perf_counter()
    oracle.prefill(qh, kh, vh, list(c1.windows), c1.n_sink, 1 / math.sqrt(c1.head_dim))
    t1 = time.perf_counter()
    Kh = np.concatenate([kh, kd1.transpose(1, 0, 2, 3)], 1)
    Vh = np.concatenate([vh, vd1.transpose(1, 0, 2, 3)], 1)
    for n in range(c1.decode_steps):
        oracle.decode(qd1[n], Kh, Vh, c1.N + n, list(c1.windows), c1.n_sink, 1 / math.sqrt(c1.head_dim))
    t2 = time.perf_counter()
    block = {
        "kind": "oracle", "cores": cores, "value": dec_tps, "unit": "tokens/s",
        "sample": (f"fp64 oracle (oracle.decode / oracle.prefill_rows) on {cores} processes x {seconds:.0f} s per "
                   f"phase, rows drawn uniformly over the C2 workload's (layer, q-head, position): decode "
                   f"{rows} rows / {keys} visible keys, prefill {rows_p} rows / {keys_p} visible pairs; "
                   f"extrapolated by in-window work (decode {dec_keys:.0f} keys per token step of one sequence, "
                   f"prefill {pre_pairs} pairs per sequence)"),
        "decode_tokens_per_s": dec_tps, "prefill_tokens_per_s": pre_tps,
        "prefill_extrapolation": "sum |V(h,i)| (oracle.visible_pairs)",
        "C1_full": {"prefill_s": t1 - t0, "decode_s": t2 - t1, "prefill_tokens_per_s": c1.N / (t1 - t0),
                    "decode_tokens_per_s": c1.decode_steps / (t2 - t1), "cores": 1,
                    "note": "C1 (configs[0]) run in full: prefill N=256 + 64 decode steps, 1 process"}}
    return dec_tps, block


# --------------------------------------------------------------------------------------------
def run_reference(args, rank, world):
    """--impl reference: the oracle (CPU) on the same workload/metric, bounded sample per step."""
    if rank != 0:
        return
    rates = []
    for _ in range(args.warmup):
        cpu_oracle_baseline(seconds=1.0, full=False)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, _ = cpu_oracle_baseline(seconds=3.0, full=False)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = float(statistics.median(rates))
    _, desc = cpu_oracle_baseline(seconds=6.0)   # prefill + C1 context, once, after the timed steps
    desc["value"] = value
    desc["sample"] = f"timed steps: decode, {args.steps} x 3 s on {desc['cores']} processes; " + desc["sample"]
    line = {
        "impl": "reference", "metric": "decode tokens/s", "value": value, "unit": "tokens/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_block(world),
        "cpu_baseline": desc,
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_block(world):
    return {"workload": "C2: Vicuna-7B attention shape, 32 layers x 32 heads, d=128, N=4096 prefill + 512 "
                        "decode tokens, batch 8 per GPU, MoA rule spans (mean density 0.50), 64 sinks",
            "model": "vicuna-7b-attention (random synthetic Q/K/V)", "global_batch": CFG.batch * world,
            "seq_len": CFG.N + CFG.decode_steps, "parallelism": f"dp{world}",
            "l2": "no flush: working set 8.6 GB cache + 25.8 GB prefill inputs cycled over 32 layers >> 126 MB L2"}


# --------------------------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import paper_2406_14909_b200 as moa

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # before any CUDA work: the worker processes are forked from this one
        _, cpu = cpu_oracle_baseline()

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    L, B, N, T, d, s = CFG.layers, CFG.batch, CFG.N, CFG.decode_steps, CFG.head_dim, CFG.n_sink
    scale = 1 / math.sqrt(d)
    windows = windows_all_layers(moa)
    ctx = moa.MoAContext(L, CFG.hq, CFG.hkv, d, B, dtype=torch.bfloat16, device=local_rank)
    for l in range(L):
        ctx.set_spans(l, windows[l], s, N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)          # single-layer launches
    ws_l = ctx.alloc_workspace(B, L)     # cross-layer launches (one slice per layer)
    # resident inputs (distinct per layer and per rank)
    Q, K, V = [], [], []
    for l in range(L):
        q, k, v = prefill_qkv(CFG, l + 1000 * rank, device=dev)
        Q.append(q), K.append(k), V.append(v)
    O = torch.empty_like(Q[0])
    qd, kd, vd = decode_tokens(CFG, 1000 * rank, T, device=dev)
    od = torch.empty(B, CFG.hq, d, dtype=torch.bfloat16, device=dev)
    od_l = torch.empty(L, B, CFG.hq, d, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream()
    ctx.prepare_layers()

    n_ev = T   # decode launches per step (one per token)
    ev_p = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]

    def step(record=False):
        for l in range(L):
            if record:
                ev_p[l][0].record(stream)
            ctx.prefill(l, Q[l], K[l], V[l], O, scale)   # attention + fused cache fill, one kernel
            if record:
                ev_p[l][1].record(stream)
        ph = torch.cuda.Event(enable_timing=True)
        ph.record(stream)
        # decode: one cross-layer launch per token (moa_decode_step_fused_layers: all 32 layers'
        # append + split-KV decode + combine; every layer reads this token's q -- layer stride 0).
        # No event between launches (an event record between two PDL launches stops the next
        # kernel's prologue from overlapping the previous one's tail); the phase events bracket them.
        for t in range(T):
            ctx.decode_step_fused_layers(0, qd[t].expand(L, *qd[t].shape), kd[t].expand(L, *kd[t].shape),
                                         vd[t].expand(L, *vd[t].shape), od_l, N + t, scale, ws_l)
        return ph

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    pre_ms, dec_ms, tot_ms, pk_ms = [], [], [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            barrier()
            torch.cuda.synchronize()
            e0, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ph = step(record=True)
            e2.record(stream)
            torch.cuda.synchronize()
            barrier()
            tot_ms.append(e0.elapsed_time(e2))
            pre_ms.append(e0.elapsed_time(ph))
            dec_ms.append(ph.elapsed_time(e2))
            pk_ms.append(sum(a.elapsed_time(b) for a, b in ev_p))
    tot = sum(tot_ms)
    pre = sum(pre_ms)
    dec = sum(dec_ms)
    if world > 1:
        t = torch.tensor([tot, pre, dec], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot, pre, dec = t.tolist()
    K_steps = args.steps
    decode_tps = B * T * world * K_steps / (dec / 1e3)
    prefill_tps = B * N * world * K_steps / (pre / 1e3)

    # roofline of the dominant kernel (decode: one cross-layer launch per token)
    flops, dec_bytes_per_token = algorithmic_work(windows, B, N, T, s, d, CFG.group)
    peaks, peak_src = load_peaks()
    dk_avg_ms = dec / (K_steps * n_ev)   # decode phase (max over ranks) / launches, gaps included
    dec_bytes_per_launch = dec_bytes_per_token
    achieved_gbs = dec_bytes_per_launch / (dk_avg_ms / 1e3) / 1e9
    pk_total_s = sum(pk_ms) / 1e3 / K_steps
    achieved_tf = flops / pk_total_s / 1e12
    clocks = clk.summary()
    traffic, traffic_note = None, None
    tp = os.path.join(ROOT, "profiles", "decode_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        traffic = tj.get("bytes_per_launch")
        traffic_note = (f"dram read+write of one {tj.get('launch')} launch ({tj.get('source')}); "
                        f"its algorithmic bytes {tj.get('algorithmic_bytes_same_launch')}, "
                        f"ratio {tj.get('traffic_over_algorithmic'):.3f}")

    # ---------------- the same decode with one launch per layer (a model whose layer l+1 query
    # depends on layer l's output cannot batch its layers): 64 tokens, same cache, same timing
    per_layer = run_per_layer(ctx, ws, K, V, qd, kd, vd, od, scale, world, dev, dec_bytes_per_token, peaks)
    # ---------------- e2e: host buffers through the public API, H2D/D2H inside the timed region
    e2e = run_e2e(ctx, ws_l, Q, K, V, qd, kd, vd, scale, world, dev)
    del Q, K, V, O
    ctx = ws = ws_l = None
    torch.cuda.empty_cache()
    kv_shard = None
    if world > 1 or args.kv_shard:
        try:
            kv_shard = run_kv_shard(rank, world, dev, scale)
        except Exception as exc:  # reported, never fatal for the main line
            kv_shard = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()

    configs = None
    if world == 1 and not args.no_configs:
        configs = run_configs(dev, peaks)

    if rank == 0:
        line = {
            "metric": "decode tokens/s", "value": decode_tps, "unit": "tokens/s", "n_gpus": world,
            "steps": K_steps, "warmup": args.warmup, "ms_per_step": tot / K_steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": config_block(world),
            "prefill": {"value": prefill_tps, "unit": "tokens/s", "ms_per_step": pre / K_steps,
                        "roofline": {"bound": "tensor", "achieved": achieved_tf,
                                     "peak": peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
                                     "unit": "TFLOP/s",
                                     "frac": achieved_tf / peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"]),
                                     "peak_source": peak_src + ", sustained bf16",
                                     "note": "in-window FLOPs 4*d*sum|V| over the event-timed launches of the "
                                             "tcgen05 prefill kernel (moa_prefill: attention + the cache fill "
                                             "fused into it)",
                                     "avg_launch_ms": pk_total_s * 1e3 / L}},
            "decode_ms_per_step": dec / K_steps,
            "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": achieved_gbs / peaks["hbm_gbs"], "traffic": traffic, "traffic_note": traffic_note,
                         "kernel": "decode_mma_kernel<128,2,2,ML=true>: one launch per token over all 32 layers "
                                   "(fused append + split-KV + last-CTA combine per layer)",
                         "bytes_per_launch": dec_bytes_per_launch, "avg_launch_ms": dk_avg_ms,
                         "avg_launch_note": "decode phase time (CUDA events on the launch stream, timed "
                                            "steps) / launches; inter-launch gaps count against the kernel",
                         "peak_source": peak_src},
            "e2e": e2e,
            "decode_per_layer": per_layer,
            "gpu_launches": K_steps * (L + T),
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        if kv_shard is not None:
            line["kv_shard"] = kv_shard
        if configs is not None:
            line["configs"] = configs
        print(json.dumps(line), flush=True)


def run_kv_shard(rank, world, dev, scale, T=64):
    """North-star partition across GPUs: the SAME batch of 8 sequences, its
    kv-groups split over the ranks in cost-balanced contiguous ranges (dist.plan_shards on
    the in-window rows of every group, summed over layers; each rank's cache holds only its
    groups), the rank-invariant decode split (so the gathered heads are the 1-GPU bits), and
    after every layer the head outputs all-gathered with NCCL (all_gather_into_tensor over
    NVLink, preallocated buffers: the kernel writes its heads straight into the send slab).
    Model-faithful order: layer l+1 starts after layer l's heads are gathered (its q would
    come from them).  Strong scaling: decode tokens/s of the whole job with and without the
    all-gather, device-timed, max over ranks."""
    import paper_2406_14909_b200 as moa
    from paper_2406_14909_b200 import dist as mdist

    L, B, N, d, s, G = CFG.layers, CFG.batch, CFG.N, CFG.head_dim, CFG.n_sink, CFG.group
    windows = windows_all_layers(moa)
    cost = mdist.group_costs(windows, s, G)
    shards = mdist.plan_shards(world, CFG.hkv, B, "kv", group_cost=cost)
    shard = shards[rank]
    ctx = mdist.make_context(shard, L, CFG.hq, CFG.hkv, d, device=dev.index)
    ctx.set_decode_split(DECODE_CHUNK)
    for l in range(L):
        ctx.set_spans(l, windows[l], s, N)
    ctx.alloc_cache(B)
    ws = ctx.alloc_workspace(B)
    g = torch.Generator(device=dev).manual_seed(77)
    kp = torch.randn(B, N, CFG.hkv, d, device=dev, generator=g).to(torch.bfloat16)  # prompt K/V (all groups)
    vp = torch.randn(B, N, CFG.hkv, d, device=dev, generator=g).to(torch.bfloat16)
    kl, vl = mdist.local_slice_kv(kp, shard), mdist.local_slice_kv(vp, shard)
    qd, kd, vd = decode_tokens(CFG, 0, T, device=dev)
    hg = mdist.HeadGather(shards, rank, B, G, d, device=dev)
    od = hg.local_out()
    stream = torch.cuda.current_stream()

    def phase(gather):
        for l in range(L):
            ctx.cache_fill(l, kl, vl)          # positions restart at N
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for t in range(T):
            ql = mdist.local_slice_q(qd[t], shard, G)
            kt, vt = mdist.local_slice_kv(kd[t], shard), mdist.local_slice_kv(vd[t], shard)
            for l in range(L):
                ctx.decode_step_fused(l, ql, kt, vt, od, N + t, scale, ws)
                if gather and world > 1:
                    ready = torch.cuda.Event()
                    ready.record(stream)
                    _, done = hg.gather(ready)      # comm stream: all-gather + head permute
                    stream.wait_event(done)         # layer l+1 consumes the gathered heads
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if world > 1:
            x = torch.tensor([ms], dtype=torch.float64, device=dev)
            torch.distributed.all_reduce(x, op=torch.distributed.ReduceOp.MAX)
            ms = x.item()
        return ms

    phase(True)
    with_ag = phase(True)
    compute = phase(False)
    fused, fused_err = None, None
    if world > 1:
        # fused head gather: the decode epilogue stores into every rank's symmetric-memory
        # buffer over NVLink; layer l+1 waits on this rank's counter of layer l
        try:
            pg = mdist.PeerGather.from_symmetric_memory(ctx, shard, G, CFG.hkv, L, B, CFG.hq, d, dev)

            def fused_phase():
                for l in range(L):
                    ctx.cache_fill(l, kl, vl)
                torch.cuda.synchronize()
                torch.distributed.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for t in range(T):
                    ql = mdist.local_slice_q(qd[t], shard, G)
                    kt, vt = mdist.local_slice_kv(kd[t], shard), mdist.local_slice_kv(vd[t], shard)
                    for l in range(L):
                        ctx.decode_step_fused(l, ql, kt, vt, od, N + t, scale, ws)
                        pg.wait(l)                  # layer l+1 consumes every rank's heads
                    pg.next_token()
                e1.record(stream)
                torch.cuda.synchronize()
                x = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
                torch.distributed.all_reduce(x, op=torch.distributed.ReduceOp.MAX)
                return x.item()

            fused_phase()
            fused = fused_phase()
            ctx.set_peer_outputs([], [], 0, 0, 0)
        except Exception as exc:  # reported; the NCCL numbers above stand
            fused_err = f"{type(exc).__name__}: {exc}"[:300]
    loads = [mdist.shard_cost(sh, cost) for sh in shards]
    return {"mode": f"kv-groups over {world} rank(s), cost-balanced contiguous ranges "
                    f"{[(sh.g0, sh.g1) for sh in shards]}, same batch of {B}",
            "rank_load_max_over_mean": max(loads) / (sum(loads) / len(loads)),
            "decode_split": f"rank-invariant, {DECODE_CHUNK}-row chunks (moa_set_decode_split)",
            "decode_tokens_per_s": B * T / (with_ag / 1e3),
            "decode_tokens_per_s_no_allgather": B * T / (compute / 1e3),
            "allgather_us_per_layer": (with_ag - compute) * 1e3 / (T * L),
            "fused_gather": ({"decode_tokens_per_s": B * T / (fused / 1e3),
                              "gather_us_per_layer": (fused - compute) * 1e3 / (T * L),
                              "note": "moa_set_peer_outputs: decode epilogue P2P-stores every head row into "
                                      "every rank's symmetric-memory buffer, per-layer counters + moa_wait_flag"}
                             if fused is not None else {"error": fused_err} if fused_err else None),
            "tokens": T, "scaling": "strong",
            "note": "NCCL all_gather_into_tensor of each layer's head outputs (torch.distributed, own stream, "
                    "preallocated), serialised before the next layer; device-timed, max over ranks"}


def _config_windows(moa, cfg, l):
    t = rule_table(cfg.name)
    return moa.resolve_spans(t["alpha"][l], t["beta"][l], cfg.N, cfg.n_sink)


def _bench_decode_cfg(moa, cfg, layers, T, dev, peaks):
    """Fused decode over `layers` (all resident) for T tokens; CUDA events around the phase."""
    L_all, B, N, s, d, G = cfg.layers, cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim, cfg.group
    wins = {l: _config_windows(moa, cfg, l) for l in range(L_all)}
    ctx = moa.MoAContext(len(layers), cfg.hq, cfg.hkv, d, B, dtype=torch.bfloat16, device=dev.index)
    for i, l in enumerate(layers):
        ctx.set_spans(i, wins[l], s, N)
    ctx.alloc_cache(B)
    nl = len(layers)
    ws = ctx.alloc_workspace(B, nl)
    ctx.prepare_layers()
    g = torch.Generator(device=dev).manual_seed(cfg.seed_base + 7)
    kp = torch.randn(B, N, cfg.hkv, d, device=dev, generator=g).to(torch.bfloat16)
    vp = torch.randn(B, N, cfg.hkv, d, device=dev, generator=g).to(torch.bfloat16)
    qd, kd, vd = decode_tokens(cfg, 0, T, device=dev)
    od = torch.empty(nl, B, cfg.hq, d, dtype=torch.bfloat16, device=dev)
    scale = 1 / math.sqrt(d)

    def layer_bytes(l, p):   # in-window bytes of one layer-token + q/o + new token
        wg = [max(wins[l][x * G:(x + 1) * G]) for x in range(cfg.hkv)]
        return B * (sum(min(p + 1, s + w) for w in wg) * d * 4 + cfg.hq * d * 4 + cfg.hkv * d * 8)

    def run(cross):
        for i in range(nl):
            ctx.cache_fill(i, kp, vp)  # positions restart at N
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for t in range(T):
            if cross:   # one launch per token over the resident layers
                ctx.decode_step_fused_layers(0, qd[t].expand(nl, *qd[t].shape), kd[t].expand(nl, *kd[t].shape),
                                             vd[t].expand(nl, *vd[t].shape), od, N + t, scale, ws)
            else:
                for i in range(nl):
                    ctx.decode_step_fused(i, qd[t], kd[t], vd[t], od[i], N + t, scale, ws)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    run(True)
    with ClockSampler(dev.index) as clk:
        sec = statistics.median(run(True) for _ in range(3))
    run(False)
    sec_pl = statistics.median(run(False) for _ in range(2))
    by_timed = sum(layer_bytes(l, N + t) for t in range(T) for l in layers)
    by_all = sum(layer_bytes(l, N + t) for t in range(T) for l in range(L_all))
    gbs = by_timed / sec / 1e9
    gbs_pl = by_timed / sec_pl / 1e9
    sec_model = by_all / (gbs * 1e9)          # all L layers at the measured in-window rate
    out = {"tokens_per_s": B * T / sec_model, "unit": "tokens/s", "batch": B, "tokens": T,
           "positions": [N, N + T - 1], "layers_timed": len(layers), "layers_model": L_all,
           "launch": "moa_decode_step_fused_layers: one launch per token over the resident layers",
           "us_per_layer_token": sec / (T * len(layers)) * 1e6,
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": gbs / peaks["hbm_gbs"], "traffic": None,
                        "bytes_per_launch": by_timed / T},
           "per_layer": {"tokens_per_s": B * T / (by_all / (gbs_pl * 1e9)), "achieved_gbs": gbs_pl,
                         "frac": gbs_pl / peaks["hbm_gbs"],
                         "note": "moa_decode_step_fused, one launch per layer-token"},
           "clocks": clk.summary()}
    if len(layers) < L_all:
        out["sampling"] = (f"{len(layers)} of {L_all} layers resident (every {layers[1] - layers[0]}th, "
                           f"{layers[0]}..{layers[-1]}: the whole density profile, not its densest end); "
                           f"tokens/s = B*T / (in-window bytes of all {L_all} layers / the measured GB/s)")
    del ctx, ws, kp, vp
    torch.cuda.empty_cache()
    return out


def _bench_prefill_cfg(moa, cfg, dev, peaks):
    """moa_prefill_attn + moa_cache_fill over every layer; per-layer events on the attention."""
    L, B, N, s, d = cfg.layers, cfg.batch, cfg.N, cfg.n_sink, cfg.head_dim
    wins = [_config_windows(moa, cfg, l) for l in range(L)]
    ctx = moa.MoAContext(L, cfg.hq, cfg.hkv, d, B, dtype=torch.bfloat16, device=dev.index)
    for l in range(L):
        ctx.set_spans(l, wins[l], s, N)
    ctx.alloc_cache(B)
    qkv = [prefill_qkv(cfg, l, device=dev) for l in range(L)]
    o = torch.empty_like(qkv[0][0])
    scale = 1 / math.sqrt(d)
    flops, _ = algorithmic_work(wins, B, N, 0, s, d, cfg.group)
    stream = torch.cuda.current_stream()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(L)]

    def run():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for l in range(L):
            ev[l][0].record(stream)
            ctx.prefill(l, *qkv[l], o, scale)   # attention + fused cache fill
            ev[l][1].record(stream)
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3, sum(a.elapsed_time(b) for a, b in ev) / 1e3

    run()
    with ClockSampler(dev.index) as clk:
        res = [run() for _ in range(3)]
    tot = statistics.median(r[0] for r in res)
    attn = statistics.median(r[1] for r in res)
    tf = flops / attn / 1e12
    pk = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    out = {"tokens_per_s": B * N / tot, "unit": "tokens/s", "batch": B, "N": N, "layers": L,
           "ms_all_layers": tot * 1e3, "attn_ms_all_layers": attn * 1e3,
           "roofline": {"bound": "tensor", "achieved": tf, "peak": pk, "unit": "TFLOP/s", "frac": tf / pk,
                        "frac_of_burst": tf / peaks["bf16_tflops"], "traffic": None,
                        "note": "in-window FLOPs 4*d*sum|V| over the event-timed moa_prefill launches "
                                "(attention + fused cache fill)"},
           "clocks": clk.summary()}
    del ctx, qkv, o
    torch.cuda.empty_cache()
    return out


def run_configs(dev, peaks):
    """BASELINE.json configs[2..4] on this GPU, as sub-blocks of the one JSON line:
    C3 GQA decode (all 32 layers, 64 tokens), C4 prefill (all 40 layers), C5 decode (16 of 80
    layers resident, strided over the density profile, 16 tokens; its 172 GB cache does not fit)."""
    import paper_2406_14909_b200 as moa
    out = {}
    for name, fn in (("C3", lambda c: _bench_decode_cfg(moa, c, list(range(c.layers)), 64, dev, peaks)),
                     ("C4", lambda c: _bench_prefill_cfg(moa, c, dev, peaks)),
                     ("C5", lambda c: _bench_decode_cfg(moa, c, list(range(0, c.layers, 5)), 16, dev, peaks))):
        try:
            out[name] = dict(mode="prefill" if name == "C4" else "decode", **fn(CONFIGS[name]))
        except Exception as exc:  # reported, never fatal for the main line
            out[name] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()
    return out


def run_per_layer(ctx, ws, K, V, qd, kd, vd, od, scale, world, dev, bytes_per_token, peaks, T=64):
    """Decode tokens/s with one moa_decode_step_fused launch per layer-token (the model-faithful
    order when layer l+1's query depends on layer l), on the same resident cache."""
    L, B, N = CFG.layers, CFG.batch, CFG.N
    for l in range(L):
        ctx.cache_fill(l, K[l], V[l])    # positions restart at N
    for t in range(4):                   # warm-up tokens (not timed)
        for l in range(L):
            ctx.decode_step_fused(l, qd[t], kd[t], vd[t], od, N + t, scale, ws)
    for l in range(L):
        ctx.cache_fill(l, K[l], V[l])
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(T):
        for l in range(L):
            ctx.decode_step_fused(l, qd[t], kd[t], vd[t], od, N + t, scale, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if world > 1:
        x = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(x, op=torch.distributed.ReduceOp.MAX)
        ms = x.item()
    gbs = bytes_per_token * T / (ms / 1e3) / 1e9
    return {"value": B * T * world / (ms / 1e3), "unit": "tokens/s", "tokens": T,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": gbs / peaks["hbm_gbs"], "avg_launch_ms": ms / (T * L)},
            "note": "moa_decode_step_fused, one launch per layer-token (decode_mma_kernel<128,2,2,ML=false>, "
                    "PDL-chained)"}


def run_e2e(ctx, ws, Q, K, V, qd, kd, vd, scale, world, dev):
    """Decode tokens/s through MoAContext with pinned HOST inputs and outputs.

    Every token's inputs (q, k_new, v_new of all layers, packed in one pinned buffer) are
    copied host->device and every token's outputs (o of all layers) device->host inside the
    timed region, on a copy stream double-buffered against the compute stream: the H2D of
    token t+1 and the D2H of token t-1 overlap the decode launches of token t.  The prefill
    inputs of each layer are staged from host as well (reported as prefill_ms)."""
    L, B, N, T, d = CFG.layers, CFG.batch, CFG.N, CFG.decode_steps, CFG.head_dim
    hq_, hkv_ = qd.shape[2], kd.shape[2]
    nq, nk = B * hq_ * d, B * hkv_ * d
    per_layer = nq + 2 * nk
    stream = torch.cuda.current_stream()
    cs = torch.cuda.Stream(device=dev)
    # host: [T, L, q|k|v] packed, pinned
    hin = torch.empty(T, L, per_layer, dtype=qd.dtype).pin_memory()
    hin[:, :, :nq] = qd.reshape(T, 1, nq).cpu()
    hin[:, :, nq:nq + nk] = kd.reshape(T, 1, nk).cpu()
    hin[:, :, nq + nk:] = vd.reshape(T, 1, nk).cpu()
    hout = torch.empty(T, L, B, hq_, d, dtype=qd.dtype).pin_memory()
    din = [torch.empty(L, per_layer, dtype=qd.dtype, device=dev) for _ in range(2)]
    dout = [torch.empty(L, B, hq_, d, dtype=qd.dtype, device=dev) for _ in range(2)]
    hQ, hK, hV = (x.cpu().pin_memory() for x in (Q[0], K[0], V[0]))
    hO = torch.empty(Q[0].shape, dtype=Q[0].dtype).pin_memory()
    dQ, dK, dV, dO = (torch.empty_like(x) for x in (Q[0], K[0], V[0], Q[0]))
    h2d = d2h = 0
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(stream)
    for l in range(L):
        dQ.copy_(hQ, non_blocking=True), dK.copy_(hK, non_blocking=True), dV.copy_(hV, non_blocking=True)
        h2d += 3 * hQ.numel() * 2
        ctx.prefill(l, dQ, dK, dV, dO, scale)
        hO.copy_(dO, non_blocking=True)
        d2h += hO.numel() * 2
    e1.record(stream)
    ev_in = [torch.cuda.Event() for _ in range(T)]
    ev_done = [torch.cuda.Event() for _ in range(T)]
    ev_out = [torch.cuda.Event() for _ in range(T)]
    cs.wait_event(e1)

    def h2d_token(t):
        nonlocal h2d
        with torch.cuda.stream(cs):
            din[t % 2].copy_(hin[t], non_blocking=True)
            ev_in[t].record(cs)
        h2d += hin[t].numel() * 2

    h2d_token(0)
    if T > 1:
        h2d_token(1)
    for t in range(T):
        stream.wait_event(ev_in[t])
        if t >= 2:
            stream.wait_event(ev_out[t - 2])       # dout[t % 2] drained to host
        buf, ob = din[t % 2], dout[t % 2]
        ctx.decode_step_fused_layers(0, buf[:, :nq].view(L, B, hq_, d), buf[:, nq:nq + nk].view(L, B, hkv_, d),
                                     buf[:, nq + nk:].view(L, B, hkv_, d), ob, N + t, scale, ws)
        ev_done[t].record(stream)
        cs.wait_event(ev_done[t])
        with torch.cuda.stream(cs):
            hout[t].copy_(ob, non_blocking=True)
            ev_out[t].record(cs)
        d2h += ob.numel() * 2
        if t + 2 < T:
            h2d_token(t + 2)                        # din[t % 2] is free once token t is done
    stream.wait_event(ev_out[T - 1])
    e2.record(stream)
    torch.cuda.synchronize()
    dec_ms = e1.elapsed_time(e2)
    if world > 1:
        x = torch.tensor([dec_ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(x, op=torch.distributed.ReduceOp.MAX)
        dec_ms = x.item()
    return {"value": B * T * world / (dec_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "prefill_ms": e0.elapsed_time(e1), "decode_ms": dec_ms,
            "note": "1 step; prefill inputs of one layer staged host->device per layer (o read back); "
                    "decode: per token one pinned H2D of q/k_new/v_new for all layers, one cross-layer "
                    "launch and one D2H of o for all layers, on a copy stream double-buffered against "
                    "the decode launches"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C3/C4/C5 sub-blocks")
    ap.add_argument("--kv-shard", action="store_true", help="also run the kv-group sharded decode at N = 1")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # self-launch: one rank per GPU under torchrun (the driver's own launch sets WORLD_SIZE)
        import socket
        import subprocess
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        # communicator evidence on stderr: NCCL prints "nranks N" when each rank's comm is built
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group(backend)
    try:
        if args.impl == "reference":
            run_reference(args, rank, world)
        else:
            run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
