"""Seeded synthetic inputs shared by the tests, the oracle legs and bench.py.

Holds random-number streams and table loading only -- no span arithmetic,
no masking, no attention.  Values ~ N(0, 1) from a seeded ``torch.Generator``
(SURVEY.md §8(d) "Common settings"), cast to the config's I/O dtype.
"""
from __future__ import annotations

import json
import os

import torch

from .configs import CONFIGS, Config

_HERE = os.path.dirname(os.path.abspath(__file__))
_DTYPES = {"bf16": torch.bfloat16, "f32": torch.float32}


def torch_dtype(cfg: Config) -> torch.dtype:
    return _DTYPES[cfg.dtype]


def generator(seed: int, device="cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def normal(shape, seed: int, dtype=torch.float32, device="cpu") -> torch.Tensor:
    """N(0,1) samples from a seeded generator on ``device``, cast to dtype."""
    g = generator(seed, device)
    x = torch.randn(*shape, generator=g, dtype=torch.float32, device=device)
    return x.to(dtype)


def prefill_qkv(cfg: Config, layer: int, batch=None, N=None, device="cpu"):
    """Q [B,N,Hq,d], K,V [B,N,Hkv,d] of one layer (seed = 1000*config+layer,
    SURVEY.md §8(d)); separate sub-streams for Q, K, V."""
    B = cfg.batch if batch is None else batch
    n = cfg.N if N is None else N
    dt = torch_dtype(cfg)
    base = cfg.seed_base + 10 * layer
    q = normal((B, n, cfg.hq, cfg.head_dim), base + 1, dt, device)
    k = normal((B, n, cfg.hkv, cfg.head_dim), base + 2, dt, device)
    v = normal((B, n, cfg.hkv, cfg.head_dim), base + 3, dt, device)
    return q, k, v


def decode_tokens(cfg: Config, layer: int, steps: int, batch=None, device="cpu"):
    """Per-step decode inputs: q [T,B,Hq,d], k_new, v_new [T,B,Hkv,d]."""
    B = cfg.batch if batch is None else batch
    dt = torch_dtype(cfg)
    base = cfg.seed_base + 10 * layer + 500_000
    q = normal((steps, B, cfg.hq, cfg.head_dim), base + 1, dt, device)
    k = normal((steps, B, cfg.hkv, cfg.head_dim), base + 2, dt, device)
    v = normal((steps, B, cfg.hkv, cfg.head_dim), base + 3, dt, device)
    return q, k, v


def rule_table(name: str):
    """(alpha, beta) per (layer, q-head) of a rule-driven config, loaded from
    the committed table ``rules/<name>.json`` (written by
    ``tools/make_rule_tables.py``, which calls only ``oracle/``)."""
    with open(os.path.join(_HERE, "rules", f"{name}.json")) as f:
        t = json.load(f)
    return t


def config(name: str) -> Config:
    return CONFIGS[name]
