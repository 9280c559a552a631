"""B200 (sm_100a) MoA heterogeneous sliding-window attention (arXiv 2406.14909).

The hot path lives in libmoa.so (hand-written CUDA for sm_100a behind the C
ABI of include/moa.h); this package is its thin Python binding.  Importing it
does not require a GPU; using a context does, and there is no fallback.
"""
from ._lib import EXPORTED, MoAError, load  # noqa: F401
from .moa import MoAContext, advance_pos, attention_influence, plan_rules, resolve_spans, rule_losses, wait_flag  # noqa: F401

__all__ = ["MoAContext", "MoAError", "resolve_spans", "load", "EXPORTED"]
