"""Multi-GPU partitioning of the MoA hot path (one process per GPU).

Heads are masked independently ("Attention masks for all heads are applied in
parallel ... There is no overlap or sequential application between masks across
different heads") and sequences of a batch are independent,
so the work partitions without any exchange inside attention:

* ``"batch"`` -- every rank serves a contiguous range of sequences with all
  kv-groups (no data-path collective at all when each rank owns its sequences);
* ``"kv"``    -- every rank serves a contiguous range of kv-groups (and their
  q-heads) for the whole batch; the per-layer head outputs are all-gathered
  (NCCL over NVLink via torch.distributed) when a consumer needs every head.

kv ranges are COST-balanced (SURVEY §8(e) "assign units by cost"): the decode
cost of a kv-group is its in-window cache rows summed over the layers,
``sum_l min(p+1, s + W_g(l))`` (the bytes the decode kernel streams, §8(d)),
and the split is the contiguous partition of the groups that minimises the
heaviest rank (exact, by dynamic programming).  Contiguity keeps one context
per rank ([g0, g1) in moa_create) and the gathered layout a fixed permute.

A rank's ``MoAContext`` is created for its kv-group range, so its cache holds
only its groups' regions.  With the rank-invariant decode split (decode_mma.cu)
a shard computes exactly the bits the unsharded context computes for its heads,
so the gathered output equals the 1-GPU output bit for bit.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

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


def group_costs(windows_per_layer: Sequence[Sequence[int]], n_sink: int, group_size: int,
                pos: Optional[int] = None) -> List[int]:
    """Decode cost of every kv-group: in-window cache rows summed over layers,
    sum_l min(pos + 1, s + W_g(l)) with W_g = max over the group's q-heads (reading c10);
    pos None = a full ring (pos + 1 >= s + W_g)."""
    hkv = len(windows_per_layer[0]) // group_size
    cost = [0] * hkv
    for wl in windows_per_layer:
        for g in range(hkv):
            rows = n_sink + max(wl[g * group_size:(g + 1) * group_size])
            cost[g] += rows if pos is None else min(pos + 1, rows)
    return cost


def _min_max_partition(cost: Sequence[int], parts: int) -> List[int]:
    """Cut points 0 = c_0 < c_1 < ... < c_parts = n of the contiguous partition of `cost`
    into `parts` non-empty ranges minimising the largest range sum (exact DP, O(parts n^2));
    ties go to the earliest cuts."""
    n = len(cost)
    pre = [0]
    for c in cost:
        pre.append(pre[-1] + c)
    INF = float("inf")
    # best[k][i]: min over partitions of the first i units into k ranges of the max range sum
    best = [[INF] * (n + 1) for _ in range(parts + 1)]
    arg = [[0] * (n + 1) for _ in range(parts + 1)]
    best[0][0] = 0
    for k in range(1, parts + 1):
        for i in range(k, n - (parts - k) + 1):
            for j in range(k - 1, i):
                v = max(best[k - 1][j], pre[i] - pre[j])
                if v < best[k][i]:
                    best[k][i], arg[k][i] = v, j
    cuts = [n]
    for k in range(parts, 0, -1):
        cuts.append(arg[k][cuts[-1]])
    return cuts[::-1]


def plan_shards(world: int, num_kv_heads: int, batch: int, mode: str = "auto",
                group_cost: Optional[Sequence[int]] = None) -> List[Shard]:
    """Partition the (sequence, kv-group) units over `world` ranks.

    ``batch``: contiguous sequence ranges whose sizes differ by at most one (sequences
    of one batch share N and the spans, so they cost the same).  ``kv``: contiguous
    kv-group ranges minimising the heaviest rank's cost (`group_cost`, e.g.
    ``group_costs(...)``; equal costs when None).  ``auto`` prefers batch sharding
    (outputs gather contiguously, every rank holds every group's layout) when the batch
    divides evenly, else kv-group sharding.
    """
    if world < 1:
        raise ValueError("world must be >= 1")
    if mode == "auto":
        mode = "batch" if batch % world == 0 else "kv"
    if mode == "batch":
        if batch < world:
            raise ValueError(f"batch {batch} < world {world}: some rank would hold no sequence")
        sizes = [batch // world + (1 if r < batch % world else 0) for r in range(world)]
        out, b = [], 0
        for r in range(world):
            out.append(Shard(r, world, mode, 0, num_kv_heads, b, b + sizes[r]))
            b += sizes[r]
        return out
    if mode == "kv":
        if num_kv_heads < world:
            raise ValueError(f"{num_kv_heads} kv-groups < world {world}: some rank would hold no group")
        cost = list(group_cost) if group_cost is not None else [1] * num_kv_heads
        if len(cost) != num_kv_heads:
            raise ValueError("group_cost needs one entry per kv-group")
        cuts = _min_max_partition(cost, world)
        return [Shard(r, world, mode, cuts[r], cuts[r + 1], 0, batch) for r in range(world)]
    raise ValueError(f"unknown shard mode {mode!r}")


def shard_cost(shard: Shard, group_cost: Sequence[int]) -> int:
    return sum(group_cost[shard.g0:shard.g1]) * (shard.b1 - shard.b0)


def gather_heads(local: torch.Tensor, shard: Shard, shards: Optional[Sequence[Shard]] = None, group_size: int = 1,
                 group=None) -> torch.Tensor:
    """All-gather a rank's slab of head outputs into the unsharded layout.

    decode  local [B_local, Hq_local, d]     -> [B, Hq, d]
    prefill local [B_local, N, Hq_local, d]  -> [B, N, Hq, d]
    ``batch`` mode gathers along dim 0; ``kv`` mode gathers rank-major head slabs and
    concatenates them along the head dim.  Unequal slabs (uneven batch split, cost-balanced
    kv ranges) travel padded to the largest slab (`shards` = every rank's Shard, needed
    then; `group_size` = q-heads per kv-group).
    """
    import torch.distributed as dist

    world = shard.world
    if world == 1:
        return local
    if shards is None:  # equal slabs (the caller promises it)
        sizes = None
    elif shard.mode == "batch":
        sizes = [s.b1 - s.b0 for s in shards]
    else:
        sizes = [(s.g1 - s.g0) * group_size for s in shards]
    local = local.contiguous()
    dim = 0 if shard.mode == "batch" else local.dim() - 2
    mx = local.shape[dim] if sizes is None else max(sizes)
    if local.shape[dim] < mx:
        pad_shape = list(local.shape)
        pad_shape[dim] = mx - local.shape[dim]
        local = torch.cat([local, local.new_zeros(pad_shape)], dim=dim)
    flat = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(flat.view(-1), local.view(-1), group=group)
    parts = [flat[r].narrow(dim, 0, mx if sizes is None else sizes[r]) for r in range(world)]
    return torch.cat(parts, dim=dim)


class HeadGather:
    """Preallocated per-layer all-gather of decode head outputs ([B, Hq, d]) for kv-group
    shards, on its own stream.

    The rank's decode kernel writes its heads straight into ``send`` (``local_out()``, a
    [B, Hq_local, d] view with the unsharded batch stride of a padded slab), so no copy
    precedes the collective.  ``gather(layer_done_event)`` queues, on the comm stream, a
    wait for the layer's decode, one NCCL all_gather_into_tensor over NVLink and the
    fixed head permute into ``out``; it returns the event the consumer of ``out`` waits
    on, so the next layer's decode overlaps the collective (SURVEY §8(e) "on a dedicated
    stream")."""

    def __init__(self, shards: Sequence[Shard], rank: int, batch: int, group_size: int, head_dim: int,
                 dtype=torch.bfloat16, device=None, group=None, n_out: int = 2):
        self.shards, self.rank, self.group = list(shards), rank, group
        self.world = len(shards)
        self.sizes = [(s.g1 - s.g0) * group_size for s in shards]
        self.hmax = max(self.sizes)
        self.hq = sum(self.sizes)
        self.send = torch.zeros(batch, self.hmax, head_dim, dtype=dtype, device=device)
        self.recv = torch.empty(self.world, batch, self.hmax, head_dim, dtype=dtype, device=device)
        # double-buffered outputs: the consumer of layer l's heads reads out[l % n_out]
        self.outs = [torch.empty(batch, self.hq, head_dim, dtype=dtype, device=device) for _ in range(n_out)]
        self.stream = torch.cuda.Stream(device=device) if torch.cuda.is_available() and device is not None \
            and torch.device(device).type == "cuda" else None
        self.n = 0

    def local_out(self) -> torch.Tensor:
        return self.send[:, :self.sizes[self.rank]]

    def gather(self, ready: Optional["torch.cuda.Event"] = None):
        import torch.distributed as dist

        out = self.outs[self.n % len(self.outs)]
        self.n += 1
        ctx = torch.cuda.stream(self.stream) if self.stream is not None else _null()
        with ctx:
            if ready is not None and self.stream is not None:
                self.stream.wait_event(ready)
            dist.all_gather_into_tensor(self.recv.view(-1), self.send.view(-1), group=self.group)
            h = 0
            for r in range(self.world):
                out[:, h:h + self.sizes[r]].copy_(self.recv[r, :, :self.sizes[r]])
                h += self.sizes[r]
            done = None
            if self.stream is not None:
                done = torch.cuda.Event()
                done.record(self.stream)
        return out, done


class PeerGather:
    """Fused head-output all-gather for kv-group shards: the decode
    epilogue of every rank writes its finished head rows straight into every rank's gathered
    ``[L, B, Hq, d]`` buffer over NVLink (peer-mapped symmetric memory) and bumps that rank's
    per-layer counter; a rank waits on its own counter (``wait``) before it consumes layer l's
    heads.  No collective launch, no copy and no permute: each rank's heads land at their
    global offset directly.

    ``buffers``/``flags``: per-rank device addresses of the gathered buffers and counters as
    mapped on THIS device; built from torch symmetric memory by ``from_symmetric_memory``
    (multi-GPU), or from plain local tensors when several shard contexts share one GPU
    (tests)."""

    def __init__(self, ctx, shard: Shard, group_size: int, num_kv_heads: int, batch: int,
                 out: torch.Tensor, flags: torch.Tensor, buffers: Sequence[int], flag_ptrs: Sequence[int]):
        L, B, Hq, d = out.shape
        self.out, self.flags = out, flags
        self.per_layer_step = batch * num_kv_heads
        self.tokens = 0
        ctx.set_peer_outputs(list(buffers), list(flag_ptrs), batch_stride=Hq * d, layer_stride=B * Hq * d,
                             head0=shard.g0 * group_size)

    @classmethod
    def from_symmetric_memory(cls, ctx, shard: Shard, group_size: int, num_kv_heads: int, num_layers: int,
                              batch: int, num_q_heads: int, head_dim: int, device, group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        o_bytes = num_layers * batch * num_q_heads * head_dim * 2
        f_off = (o_bytes + 255) // 256 * 256
        buf = symm.empty(f_off + 4 * num_layers, dtype=torch.uint8, device=device)
        buf.zero_()
        grp = group if group is not None else dist.group.WORLD
        hdl = symm.rendezvous(buf, grp)
        torch.cuda.synchronize(device)
        dist.barrier(group=grp)   # every counter is zero before any rank writes
        ptrs = [int(p) for p in hdl.buffer_ptrs]
        out = buf[:o_bytes].view(torch.bfloat16).view(num_layers, batch, num_q_heads, head_dim)
        flags = buf[f_off:f_off + 4 * num_layers].view(torch.int32)
        pg = cls(ctx, shard, group_size, num_kv_heads, batch, out, flags, ptrs, [p + f_off for p in ptrs])
        pg._keep = (buf, hdl)
        return pg

    def wait(self, layer: int, stream=None):
        """Stream-ordered: later work waits until every rank's heads of `layer` of the
        current token have landed in this rank's buffer."""
        from .moa import wait_flag
        wait_flag(self.flags[layer:layer + 1], (self.tokens + 1) * self.per_layer_step, stream)

    def next_token(self):
        self.tokens += 1


class _null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


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
