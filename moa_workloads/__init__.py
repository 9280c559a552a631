"""Seeded synthetic workloads (shapes, rule tables, random inputs).

Shared by tests, bench.py and the oracle legs; holds none of the method's
arithmetic (see DESIGN.md §"Input recipe").
"""
from .configs import ALPHA_GRID, BETA_GRID, CONFIGS, Config  # noqa: F401
from .inputs import (config, decode_tokens, generator, normal,  # noqa: F401
                     prefill_qkv, rule_table, torch_dtype)
