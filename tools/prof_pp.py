"""Wait-time breakdown of the two-tile prefill kernel (diagnostic build -DMOA_PP_DIAG_PROF).

    python tools/build_variant.py prof -DMOA_PP_DIAG_PROF
    MOA_LIB=tools/bin/libmoa_prof.so python tools/prof_pp.py [C2|C4] [layers]

Prints, summed over CTAs, the clock64 cycles each role spent waiting on each barrier as a
share of that role's lifetime.
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

NAMES = {0: "mma: q_full", 1: "mma: v_full", 2: "mma: p_full0", 3: "mma: p_full1", 4: "mma: o_empty",
         5: "mma: k_full", 8: "sm0: s_full", 9: "sm1: s_full", 10: "sm0: o_full", 11: "sm1: o_full",
         16: "kv: k_empty", 17: "kv: v_empty",
         18: "sm0: ldtm S", 19: "sm0: max+rescale", 20: "sm0: exp+sttm", 21: "sm0: wait_st+arrive",
         26: "mma: issue S (8 MMA)", 27: "mma: issue PV (8 MMA)",
         22: "sm1: ldtm S", 23: "sm1: max+rescale", 24: "sm1: exp+sttm", 25: "sm1: wait_st+arrive"}


def main(name="C2", layers=4):
    cfg = CONFIGS[name]
    t = rule_table(name)
    dev = torch.device("cuda")
    L = list(range(8, 8 + layers))
    ctx = moa.MoAContext(len(L), cfg.hq, cfg.hkv, cfg.head_dim, cfg.batch)
    for i, l in enumerate(L):
        ctx.set_spans(i, moa.resolve_spans(t["alpha"][l], t["beta"][l], cfg.N, cfg.n_sink), cfg.n_sink, cfg.N)
    ctx.alloc_cache(cfg.batch)
    qkv = [prefill_qkv(cfg, l, device=dev) for l in L]
    o = torch.empty_like(qkv[0][0])
    sc = 1 / math.sqrt(cfg.head_dim)
    lib = _lib.lib()
    fn = lib.moa_debug_pp_prof
    fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 32)()
    for i in range(len(L)):
        ctx.prefill(i, *qkv[i], o, sc)
    fn(buf, 1)
    for i in range(len(L)):
        ctx.prefill(i, *qkv[i], o, sc)
    fn(buf, 1)
    v = list(buf)
    mma_tot, sm0_tot, sm1_tot = v[6], v[12], v[13]
    print(f"steps {v[7]}  S handshakes tile0 {v[14]} tile1 {v[15]}")
    print(f"mma role cycles/step {mma_tot / max(v[7], 1):.0f}")
    for k, n in NAMES.items():
        tot = mma_tot if n.startswith("mma") or n.startswith("kv") else (sm0_tot if n.startswith("sm0") else sm1_tot)
        print(f"  {n:16s} {v[k] / max(tot, 1) * 100:6.1f} %   {v[k] / max(v[7], 1):8.0f} cycles/step")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C2", int(sys.argv[2]) if len(sys.argv) > 2 else 4)
