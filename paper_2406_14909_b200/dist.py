"""Multi-GPU partitioning of the MoA hot path (one process per GPU).

Heads are masked independently ("Attention masks for all heads are applied in
parallel ... There is no overlap or sequential application between masks across
different heads") and sequences of a batch are independent,
so the work partitions without any exchange inside attention:

* ``"batch"`` -- every rank serves its own sequences with all kv-groups (the
  bench's weak-scaling mode: no data-path collective at all);
* ``"kv"``    -- every rank serves a contiguous range of kv-groups (and their
  q-heads) for the whole batch; the per-layer head outputs are all-gathered
  (NCCL over NVLink via torch.distributed) when a consumer needs every head.

A rank's ``MoAContext`` is created for its kv-group range, so its cache holds
only its groups' regions.  Rank order = head order, so the gathered layout is
the unsharded one after a fixed permute.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    mode: str
    g0: int        # kv-groups [g0, g1)
    g1: int
    b0: int        # sequences [b0, b1)
    b1: int


def plan_shards(world: int, num_kv_heads: int, batch: int, mode: str = "auto") -> List[Shard]:
    """Partition (sequence, kv-group) units over `world` ranks.

    ``auto`` prefers batch sharding (outputs gather contiguously, no permute)
    when the batch divides evenly, else kv-group sharding.  Both modes require
    an even split (the gathered tensors have equal-sized slabs).
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    if mode == "auto":
        mode = "batch" if batch % world == 0 else "kv"
    if mode == "batch":
        if batch % world:
            raise ValueError(f"batch {batch} not divisible by world {world}")
        per = batch // world
        return [Shard(r, world, mode, 0, num_kv_heads, r * per, (r + 1) * per) for r in range(world)]
    if mode == "kv":
        if num_kv_heads % world:
            raise ValueError(f"{num_kv_heads} kv-groups not divisible by world {world}")
        per = num_kv_heads // world
        return [Shard(r, world, mode, r * per, (r + 1) * per, 0, batch) for r in range(world)]
    raise ValueError(f"unknown shard mode {mode!r}")


def gather_heads(local: torch.Tensor, shard: Shard, group=None) -> torch.Tensor:
    """All-gather a rank's slab of head outputs into the unsharded layout.

    decode  local [B_local, Hq_local, d]     -> [B, Hq, d]
    prefill local [B_local, N, Hq_local, d]  -> [B, N, Hq, d]
    ``batch`` mode gathers along dim 0 (contiguous, no permute); ``kv`` mode
    gathers rank-major head slabs and moves the rank dim next to the heads.
    """
    import torch.distributed as dist

    world = shard.world
    if world == 1:
        return local
    local = local.contiguous()
    flat = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(flat, local, group=group)
    if shard.mode == "batch":
        return flat
    out = flat.view((world,) + tuple(local.shape))
    # kv: out [world, B, ..., Hq_local, d] -> [B, ..., world, Hq_local, d] -> merge heads
    nd = local.dim()
    perm = list(range(1, nd - 1)) + [0, nd - 1, nd]
    t = out.permute(*perm)
    return t.reshape(tuple(local.shape[:-2]) + (world * local.shape[-2], local.shape[-1]))


def local_slice_q(x: torch.Tensor, shard: Shard, group_size: int, head_dim: int = -2) -> torch.Tensor:
    """The rank's part of a full-batch, all-heads tensor (q/o: heads at dim -2)."""
    x = x[shard.b0:shard.b1]
    if shard.mode == "kv":
        x = x.narrow(x.dim() + head_dim if head_dim < 0 else head_dim, shard.g0 * group_size,
                     (shard.g1 - shard.g0) * group_size)
    return x


def local_slice_kv(x: torch.Tensor, shard: Shard) -> torch.Tensor:
    """The rank's part of a full-batch K/V tensor (kv-groups at dim -2)."""
    x = x[shard.b0:shard.b1]
    if shard.mode == "kv":
        x = x.narrow(x.dim() - 2, shard.g0, shard.g1 - shard.g0)
    return x


def make_context(shard: Shard, num_layers: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
                 dtype=torch.bfloat16, device: Optional[int] = 0):
    """MoAContext serving this rank's kv-groups and sequences (device -1: planning only)."""
    from .moa import MoAContext

    return MoAContext(num_layers, num_q_heads, num_kv_heads, head_dim, shard.b1 - shard.b0, dtype=dtype,
                      device=-1 if device is None else device, kv_group_begin=shard.g0, kv_group_end=shard.g1)
