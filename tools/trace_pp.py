"""Event timeline of CTA 0 of the two-tile prefill kernel (diagnostic build -DMOA_PP_DIAG_TRACE).

    python tools/build_variant.py trace -DMOA_PP_DIAG_TRACE
    MOA_LIB=tools/bin/libmoa_trace.so python tools/trace_pp.py [C2] [n_events]
    (MOA_PP_CLUSTER=1 MOA_TRACE_CL=1 ...: the clustered kernel -- S warp, softmax groups A/B, PV warp)
"""
import ctypes
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2406_14909_b200 as moa  # noqa: E402
from paper_2406_14909_b200 import _lib  # noqa: E402
from moa_workloads import CONFIGS, prefill_qkv, rule_table  # noqa: E402

TAGS = {1: "waits done, wait for turn", 2: "turn taken", 3: "dispatch done, pass turn", 4: "-",
        5: "-", 10: "mma PV waits done", 11: "mma p_full1 ok", 20: "mma PV issued", 21: "mma PV1 issued",
        30: "mma S issued", 31: "mma S1 issued", 40: "sm s_full seen", 41: "sm p_full arrive", 42: "sm S loaded+max", 43: "sm m_prev known", 44: "sm exps done", 45: "sm P buffer free", 46: "sm s_full probe (1 ready, 2 not)", 2: "mma S waits done", 3: "mma k_full ok", 4: "mma k_full probe (1 ready, 2 not)", 50: "K slot free, load issued"}


def main(name="C2", nev=120):
    cfg = CONFIGS[name]
    t = rule_table(name)
    dev = torch.device("cuda")
    ctx = moa.MoAContext(1, cfg.hq, cfg.hkv, cfg.head_dim, cfg.batch)
    ctx.set_spans(0, moa.resolve_spans(t["alpha"][8], t["beta"][8], cfg.N, cfg.n_sink), cfg.n_sink, cfg.N)
    ctx.alloc_cache(cfg.batch)
    q, k, v = prefill_qkv(cfg, 8, device=dev)
    o = torch.empty_like(q)
    sc = 1 / math.sqrt(cfg.head_dim)
    fn = _lib.lib().moa_debug_pp_trace
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_int)]
    buf = (ctypes.c_ulonglong * (4 * 4096))()
    cnt = (ctypes.c_int * 4)()
    ctx.prefill(0, q, k, v, o, sc)
    fn(buf, cnt)
    ctx.prefill(0, q, k, v, o, sc)
    fn(buf, cnt)
    ev = []
    for r in range(4):
        for i in range(cnt[r]):
            x = buf[r * 4096 + i]
            ev.append((x & ((1 << 48) - 1), r, x >> 56, (x >> 48) & 0xff))
    ev.sort()
    t0 = ev[0][0]
    start = len(ev) // 3
    prev = ev[start][0]
    for c, r, tag, arg in ev[start:start + nev]:
        who = ["MMA0", "SM0 ", "SM1 ", "MMA1"][r] if r != 2 or tag < 50 else "KPRD"
        if os.environ.get("MOA_TRACE_CL"):
            who = ["MMAS", "SMA ", "SMB ", "MMAV"][r]
        print(f"{c - t0:10d} (+{c - prev:5d})  {who} {TAGS.get(tag, tag)}" + (f" [{arg}]" if arg else ""))
        prev = c


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 120)
