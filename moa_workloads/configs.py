"""The five workloads of BASELINE.json ``configs`` as plain data.

This module holds shapes and recipe constants only -- none of the method's
arithmetic.  SURVEY.md §8(d) is the source of every field; "proposed" values
(not fixed by BASELINE.json) are marked and explained in DESIGN.md §"Input
recipe".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple


@dataclass(frozen=True)
class Config:
    name: str
    layers: int
    hq: int
    hkv: int
    head_dim: int
    N: int                    # prompt (prefill) length
    n_sink: int
    batch: int
    dtype: str                # "f32" | "bf16" (I/O dtype)
    decode_steps: int         # decode tokens per sequence (0 = prefill only)
    modes: Tuple[str, ...]    # which hot-path rows the bench/parity run
    target_density: Optional[float] = None   # rule-driven configs
    windows: Optional[Tuple[int, ...]] = None  # direct windows (C1)
    note: str = ""
    seed_base: int = field(default=0)

    @property
    def group(self) -> int:
        return self.hq // self.hkv


# C1: "1 layer, 4 heads, head_dim 64, N=256, per-head spans {16,32,64,256},
#      4 sink tokens, batch 1, fp32"
C1 = Config("C1", layers=1, hq=4, hkv=4, head_dim=64, N=256, n_sink=4, batch=1,
            dtype="f32", decode_steps=64, modes=("prefill", "decode"),
            windows=(16, 32, 64, 256), seed_base=1000)

# C2: "Vicuna-7B attention shape: 32 layers x 32 heads, head_dim 128,
#      N=4k prefill + 512-token decode, batch 8, MoA spans averaging N/2, bf16"
C2 = Config("C2", layers=32, hq=32, hkv=32, head_dim=128, N=4096, n_sink=64, batch=8,
            dtype="bf16", decode_steps=512, modes=("prefill", "decode"),
            target_density=0.5, seed_base=2000)

# C3: "Llama3-8B GQA shape: 32 q heads / 8 kv heads, head_dim 128, N=8k,
#      batch 16 decode, heterogeneous elastic spans, bf16"
#      (32 layers, density 0.5 and 512 decode steps are proposed)
C3 = Config("C3", layers=32, hq=32, hkv=8, head_dim=128, N=8192, n_sink=64, batch=16,
            dtype="bf16", decode_steps=512, modes=("decode",),
            target_density=0.5, seed_base=3000)

# C4: "Vicuna-13B shape: 40 layers x 40 heads, head_dim 128, N=16k prefill,
#      spans from alpha_h+beta_h*N rules with 25% average density, bf16"
#      (batch 1 proposed)
C4 = Config("C4", layers=40, hq=40, hkv=40, head_dim=128, N=16384, n_sink=64, batch=1,
            dtype="bf16", decode_steps=0, modes=("prefill",),
            target_density=0.25, seed_base=4000)

# C5: "Llama3-70B shape: 80 layers, 64 q / 8 kv heads, head_dim 128, N=32k,
#      batch 32 decode, kv-groups sharded across 8xB200"
#      (density 0.5 and 128 decode steps proposed)
C5 = Config("C5", layers=80, hq=64, hkv=8, head_dim=128, N=32768, n_sink=64, batch=32,
            dtype="bf16", decode_steps=128, modes=("decode",),
            target_density=0.5, seed_base=5000)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5)}

# Rule grid of the paper: 6 alpha values uniform in
# [-2048, 8192] and 9 beta values uniform in [0, 1].
ALPHA_GRID = (-2048.0, 0.0, 2048.0, 4096.0, 6144.0, 8192.0)
BETA_GRID = tuple(k / 8.0 for k in range(9))
