"""Thin Python front-end over the C ABI (include/moa.h).

``MoAContext`` wraps one ``moa_ctx``: it turns torch tensors into device
pointers, element strides and the current CUDA stream, calls the library
function of the same name and raises ``MoAError`` on a non-OK status.  Every
step of the hot path runs in libmoa.so's CUDA kernels; PyTorch only supplies
memory and streams.
"""
from __future__ import annotations

import ctypes
from ctypes import byref, c_float, c_int32, c_int64, c_size_t, c_uint8, c_void_p
from typing import Optional, Sequence

import torch

from . import _lib
from ._lib import MOA_BF16, MOA_FP32, MOA_TILE, MoAError, check  # noqa: F401

_DT = {torch.bfloat16: MOA_BF16, torch.float32: MOA_FP32}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        if not torch.cuda.is_available():
            return None
        stream = torch.cuda.current_stream()
    return c_void_p(stream.cuda_stream)


def resolve_spans(alpha: Sequence[float], beta: Sequence[float], N: int, n_sink: int):
    """Elastic rules -> windows through ``moa_resolve_spans`` (Eq. 2)."""
    n = len(alpha)
    a = (c_float * n)(*alpha)
    b = (c_float * n)(*beta)
    w = (c_int32 * n)()
    check(_lib.lib().moa_resolve_spans(a, b, n, int(N), int(n_sink), w), "moa_resolve_spans")
    return list(w)


def attention_influence(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, dout: torch.Tensor, scale: float,
                        out: Optional[torch.Tensor] = None, block: int = 64, accumulate: bool = False,
                        stream=None) -> torch.Tensor:
    """Block-averaged attention influence (Eq. 3) of one calibration item through
    ``moa_attention_influence``: q, dout [B, N, Hq, d], k, v [B, N, Hkv, d] bf16 CUDA tensors
    (token-major, any token row stride); returns / fills fp32 [B, Hq, nb, nb]."""
    B, N, Hq, d = q.shape
    Hkv = k.shape[2]
    nb = (N + block - 1) // block
    if out is None:
        out = torch.empty(B, Hq, nb, nb, dtype=torch.float32, device=q.device)
    for t in (q, k, v, dout):
        if t.dtype != torch.bfloat16 or t.stride(3) != 1 or t.stride(2) != d:
            raise MoAError(1, "attention_influence", "bf16 tensors with contiguous heads x head_dim rows")
    if dout.stride(1) != q.stride(1) or v.stride(1) != k.stride(1):
        raise MoAError(1, "attention_influence", "dout/q and v/k must share their token row strides")
    check(_lib.lib().moa_attention_influence(_ptr(q), _ptr(k), _ptr(v), _ptr(dout), B, N, Hq, Hkv, d,
                                             q.stride(1), k.stride(1), float(scale), int(block), _ptr(out),
                                             int(bool(accumulate)), _stream(stream)), "moa_attention_influence")
    return out


def rule_losses(e_blocks: torch.Tensor, N: int, n_sink: int, alphas: Sequence[float], betas: Sequence[float],
                block: int = 64, stream=None) -> torch.Tensor:
    """Eq. 4 rule losses [heads, n_rules] (fp32, device) from one entry [heads, nb, nb] of
    attention_influence's output through ``moa_rule_losses``."""
    if e_blocks.dtype != torch.float32 or not e_blocks.is_contiguous() or e_blocks.dim() != 3:
        raise MoAError(1, "rule_losses", "e_blocks must be a contiguous fp32 [heads, nb, nb] tensor")
    n = len(alphas)
    a = (c_float * n)(*alphas)
    b = (c_float * n)(*betas)
    out = torch.empty(e_blocks.shape[0], n, dtype=torch.float32, device=e_blocks.device)
    check(_lib.lib().moa_rule_losses(_ptr(e_blocks), e_blocks.shape[0], int(N), int(block), int(n_sink), a, b, n,
                                     _ptr(out), _stream(stream)), "moa_rule_losses")
    return out


def plan_rules(loss, density, layers: int, heads_per_layer: int, density_budget: float, max_rules_per_layer: int = 2):
    """One rule per head under the density budget (``moa_plan_rules``).  loss: [H, R] host
    array-like (H = layers * heads_per_layer), density: [R].  Returns (rules [H], loss, density)."""
    import numpy as np
    L = np.ascontiguousarray(np.asarray(loss, dtype=np.float32))
    d = np.ascontiguousarray(np.asarray(density, dtype=np.float32))
    H, R = L.shape
    assert H == layers * heads_per_layer and d.shape == (R,)
    out = (c_int32 * H)()
    lo, do = c_float(), c_float()
    check(_lib.lib().moa_plan_rules(L.ctypes.data_as(ctypes.POINTER(c_float)), d.ctypes.data_as(ctypes.POINTER(c_float)),
                                    layers, heads_per_layer, R, float(density_budget), int(max_rules_per_layer), out,
                                    byref(lo), byref(do)), "moa_plan_rules")
    return list(out), lo.value, do.value


def advance_pos(pos: torch.Tensor, delta: int = 1, stream=None):
    """moa_advance_pos: pos[b] += delta on the device for active sequences (pos >= 0)."""
    assert pos.dtype == torch.int64 and pos.is_contiguous() and pos.is_cuda
    check(_lib.lib().moa_advance_pos(_ptr(pos), pos.numel(), int(delta), _stream(stream)), "moa_advance_pos")


class MoAContext:
    """One context per (process, device): span tables, cache layout, launches."""

    def __init__(self, num_layers: int, num_q_heads: int, num_kv_heads: int, head_dim: int,
                 max_batch: int, dtype: torch.dtype = torch.bfloat16, device: int = 0,
                 kv_group_begin: int = 0, kv_group_end: Optional[int] = None):
        self.lib = _lib.lib()
        self.dtype = dtype
        self.device = device
        self.L, self.Hq, self.Hkv, self.d = num_layers, num_q_heads, num_kv_heads, head_dim
        self.G = num_q_heads // num_kv_heads
        self.g0 = kv_group_begin
        self.g1 = num_kv_heads if kv_group_end is None else kv_group_end
        self.nql = (self.g1 - self.g0) * self.G
        self.ngl = self.g1 - self.g0
        ctx = c_void_p()
        check(self.lib.moa_create(byref(ctx), device, _DT[dtype], num_layers, num_q_heads, num_kv_heads,
                                  head_dim, max_batch, self.g0, self.g1), "moa_create")
        self.ctx = ctx
        self._cache = None

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.moa_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- planning ---------------------------------------------------------------------
    def set_spans(self, layer: int, windows: Sequence[int], n_sink: int, N: int, block: int = 0):
        """moa_set_spans (block = 0, token mask) / moa_set_spans_blocked (block-granular
        prefill mask of the paper)."""
        w = (c_int32 * len(windows))(*[int(x) for x in windows])
        if block:
            check(self.lib.moa_set_spans_blocked(self.ctx, layer, w, int(n_sink), int(N), int(block)),
                  "moa_set_spans_blocked")
        else:
            check(self.lib.moa_set_spans(self.ctx, layer, w, int(n_sink), int(N)), "moa_set_spans")

    def set_decode_split(self, chunk_rows: int):
        """moa_set_decode_split: 0 = balanced split (default), > 0 = rank-invariant chunks."""
        check(self.lib.moa_set_decode_split(self.ctx, int(chunk_rows)), "moa_set_decode_split")

    def set_ragged(self, layer: int, seq_len: Optional[Sequence[int]], windows=None):
        """moa_set_ragged: per-sequence prompt lengths N_b and windows W_{b,h} ([B][Hq] nested
        sequence or array, all heads; None = the layer's windows).  seq_len None clears."""
        if seq_len is None:
            check(self.lib.moa_set_ragged(self.ctx, layer, 0, None, None), "moa_set_ragged")
            return
        B = len(seq_len)
        n = (c_int64 * B)(*[int(x) for x in seq_len])
        w = None
        if windows is not None:
            flat = [int(x) for row in windows for x in row]
            w = (c_int32 * len(flat))(*flat)
        check(self.lib.moa_set_ragged(self.ctx, layer, B, n, w), "moa_set_ragged")

    def cache_bytes(self, batch: int):
        k, v = c_size_t(), c_size_t()
        check(self.lib.moa_cache_bytes(self.ctx, batch, byref(k), byref(v)), "moa_cache_bytes")
        return k.value, v.value

    def layer_cache_bytes(self, layer: int, batch: int):
        k, v = c_size_t(), c_size_t()
        check(self.lib.moa_layer_cache_bytes(self.ctx, layer, batch, byref(k), byref(v)), "moa_layer_cache_bytes")
        return k.value, v.value

    def workspace_bytes(self, batch: int) -> int:
        b = c_size_t()
        check(self.lib.moa_workspace_bytes(self.ctx, batch, byref(b)), "moa_workspace_bytes")
        return b.value

    def layer_offset(self, layer: int, batch: int) -> int:
        b = c_size_t()
        check(self.lib.moa_layer_offset(self.ctx, layer, batch, byref(b)), "moa_layer_offset")
        return b.value

    def window(self, layer: int, h: int) -> int:
        w = c_int32()
        check(self.lib.moa_get_window(self.ctx, layer, h, byref(w)), "moa_get_window")
        return w.value

    def group_window(self, layer: int, g: int) -> int:
        w = c_int32()
        check(self.lib.moa_get_group_window(self.ctx, layer, g, byref(w)), "moa_get_group_window")
        return w.value

    def slot_of(self, layer: int, g: int, pos: int) -> int:
        s = c_int64()
        check(self.lib.moa_slot_of(self.ctx, layer, g, int(pos), byref(s)), "moa_slot_of")
        return s.value

    def cache_region(self, layer: int, b: int, g: int):
        off, rows = c_int64(), c_int64()
        check(self.lib.moa_cache_region(self.ctx, layer, b, g, byref(off), byref(rows)), "moa_cache_region")
        return off.value, rows.value

    def prefill_tiles(self, layer: int, h: int, q_tile: int):
        n = c_int32()
        check(self.lib.moa_prefill_tiles(self.ctx, layer, h, q_tile, None, None, 0, byref(n)), "moa_prefill_tiles")
        tiles = (c_int32 * max(1, n.value))()
        edge = (c_uint8 * max(1, n.value))()
        check(self.lib.moa_prefill_tiles(self.ctx, layer, h, q_tile, tiles, edge, n.value, byref(n)),
              "moa_prefill_tiles")
        return list(tiles)[: n.value], [bool(e) for e in list(edge)[: n.value]]

    def prefill_items(self, layer: int):
        n = c_int32()
        check(self.lib.moa_prefill_items(self.ctx, layer, None, 0, byref(n)), "moa_prefill_items")
        buf = (c_int32 * max(1, 2 * n.value))()
        check(self.lib.moa_prefill_items(self.ctx, layer, buf, n.value, byref(n)), "moa_prefill_items")
        return [(buf[2 * i], buf[2 * i + 1]) for i in range(n.value)]

    def prefill_schedule(self, layer: int):
        """Per-CTA prefill schedule: (entries [(h | b << 16, q_block)], offsets per CTA)."""
        ne, nc = c_int32(), c_int32()
        check(self.lib.moa_prefill_schedule(self.ctx, layer, None, 0, None, 0, byref(ne), byref(nc)),
              "moa_prefill_schedule")
        ent = (c_int32 * max(1, 2 * ne.value))()
        off = (c_int32 * max(1, nc.value + 1))()
        check(self.lib.moa_prefill_schedule(self.ctx, layer, ent, ne.value, off, nc.value, byref(ne), byref(nc)),
              "moa_prefill_schedule")
        return [(ent[2 * i], ent[2 * i + 1]) for i in range(ne.value)], list(off)[: nc.value + 1]

    def decode_chunks(self, layer: int):
        n = c_int32()
        check(self.lib.moa_decode_chunks(self.ctx, layer, None, 0, byref(n)), "moa_decode_chunks")
        buf = (c_int32 * max(1, 3 * n.value))()
        check(self.lib.moa_decode_chunks(self.ctx, layer, buf, n.value, byref(n)), "moa_decode_chunks")
        return [tuple(buf[3 * i: 3 * i + 3]) for i in range(n.value)]

    def next_pos(self, layer: int) -> int:
        p = c_int64()
        check(self.lib.moa_next_pos(self.ctx, layer, byref(p)), "moa_next_pos")
        return p.value

    # ---- memory --------------------------------------------------------------------------
    def bind_cache(self, k_cache: torch.Tensor, v_cache: torch.Tensor, batch: int):
        check(self.lib.moa_bind_cache(self.ctx, _ptr(k_cache), _ptr(v_cache), batch), "moa_bind_cache")
        self._cache = (k_cache, v_cache)
        self._bound_batch = batch

    def bind_layer_cache(self, layer: int, k_cache: torch.Tensor, v_cache: torch.Tensor, batch: int):
        check(self.lib.moa_bind_layer_cache(self.ctx, layer, _ptr(k_cache), _ptr(v_cache), batch),
              "moa_bind_layer_cache")

    def alloc_cache(self, batch: int):
        """Allocate (with torch) and bind the cache of all layers; returns (K, V) byte tensors."""
        kb, vb = self.cache_bytes(batch)
        dev = torch.device("cuda", self.device)
        k = torch.empty(kb, dtype=torch.uint8, device=dev)
        v = torch.empty(vb, dtype=torch.uint8, device=dev)
        self.bind_cache(k, v, batch)
        return k, v

    def alloc_workspace(self, batch: int, n_layers: int = 1) -> torch.Tensor:
        """Decode workspace; n_layers > 1 sizes it for decode_step_fused_layers."""
        return torch.empty(self.workspace_bytes(batch) * n_layers, dtype=torch.uint8,
                           device=torch.device("cuda", self.device))

    # ---- launches ------------------------------------------------------------------------
    @staticmethod
    def _row_stride(t: torch.Tensor) -> int:
        return t.stride(1)

    def prefill(self, layer: int, q, k, v, o, scale: float, lse=None, workspace=None, stream=None):
        B, N = q.shape[0], q.shape[1]
        for t in (q, k, v, o):
            assert t.stride(-1) == 1 and t.stride(-2) == self.d and t.stride(0) == N * t.stride(1)
        ws = workspace
        check(self.lib.moa_prefill(self.ctx, layer, _ptr(q), _ptr(k), _ptr(v), _ptr(o), q.stride(1), k.stride(1),
                                   o.stride(1), B, N, float(scale), _ptr(lse), _ptr(ws),
                                   0 if ws is None else ws.numel() * ws.element_size(), _stream(stream)),
              "moa_prefill")

    def prefill_attn(self, layer: int, q, k, v, o, scale: float, lse=None, stream=None):
        B, N = q.shape[0], q.shape[1]
        for t in (q, k, v, o):
            assert t.stride(-1) == 1 and t.stride(-2) == self.d and t.stride(0) == N * t.stride(1)
        check(self.lib.moa_prefill_attn(self.ctx, layer, _ptr(q), _ptr(k), _ptr(v), _ptr(o), q.stride(1),
                                        k.stride(1), o.stride(1), B, N, float(scale), _ptr(lse), _stream(stream)),
              "moa_prefill_attn")

    def cache_fill(self, layer: int, k, v, stream=None):
        B, N = k.shape[0], k.shape[1]
        check(self.lib.moa_cache_fill(self.ctx, layer, _ptr(k), _ptr(v), k.stride(1), B, N, _stream(stream)),
              "moa_cache_fill")

    def kv_append(self, layer: int, k_new, v_new, pos: int, stream=None):
        B = k_new.shape[0]
        check(self.lib.moa_kv_append(self.ctx, layer, _ptr(k_new), _ptr(v_new), k_new.stride(0), B, int(pos),
                                     _stream(stream)), "moa_kv_append")

    def decode_step(self, layer: int, q, o, pos: int, scale: float, workspace, lse=None, stream=None):
        B = q.shape[0]
        check(self.lib.moa_decode_step(self.ctx, layer, _ptr(q), _ptr(o), q.stride(0), o.stride(0), B, int(pos),
                                       float(scale), _ptr(lse), _ptr(workspace),
                                       workspace.numel() * workspace.element_size(), _stream(stream)),
              "moa_decode_step")

    def decode_step_fused(self, layer: int, q, k_new, v_new, o, pos: int, scale: float, workspace, lse=None,
                          stream=None):
        B = q.shape[0]
        check(self.lib.moa_decode_step_fused(self.ctx, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(o),
                                             q.stride(0), k_new.stride(0), o.stride(0), B, int(pos), float(scale),
                                             _ptr(lse), _ptr(workspace),
                                             workspace.numel() * workspace.element_size(), _stream(stream)),
              "moa_decode_step_fused")

    def set_peer_outputs(self, peer_o: Sequence[int], peer_flags: Sequence[int], batch_stride: int,
                         layer_stride: int, head0: int):
        """moa_set_peer_outputs: destination buffers (device addresses as ints, e.g.
        ``t.data_ptr()`` of peer-mapped / symmetric-memory tensors) and their uint32 counters."""
        n = len(peer_o)
        arr_o = (ctypes.c_void_p * max(n, 1))(*[int(x) for x in peer_o])
        arr_f = (ctypes.c_void_p * max(n, 1))(*[int(x) for x in peer_flags])
        check(self.lib.moa_set_peer_outputs(self.ctx, n, arr_o, arr_f, int(batch_stride), int(layer_stride),
                                            int(head0)), "moa_set_peer_outputs")

    def prepare_layers(self):
        """moa_prepare_layers: upload the cross-layer descriptors (before graph capture)."""
        check(self.lib.moa_prepare_layers(self.ctx), "moa_prepare_layers")

    def decode_step_fused_layers(self, layer0: int, q, k_new, v_new, o, pos: int, scale: float, workspace,
                                 lse=None, stream=None):
        """moa_decode_step_fused_layers: q/o [n, B, Hq, d], k_new/v_new [n, B, Hkv, d] (layer-major),
        one launch for layers [layer0, layer0 + n); workspace >= n * workspace_bytes(B)."""
        n, B = q.shape[0], q.shape[1]
        check(self.lib.moa_decode_step_fused_layers(
            self.ctx, layer0, n, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(o), q.stride(0), k_new.stride(0),
            o.stride(0), q.stride(1), k_new.stride(1), o.stride(1), B, int(pos), float(scale), _ptr(lse),
            lse.stride(0) if lse is not None else 0, _ptr(workspace), workspace.numel() * workspace.element_size(),
            _stream(stream)), "moa_decode_step_fused_layers")

    def decode_step_fused_ragged(self, layer: int, q, k_new, v_new, o, pos, scale: float, workspace, lse=None,
                                 stream=None):
        """moa_decode_step_fused_ragged: pos is a device int64 tensor [B] (per-sequence positions,
        < 0 = inactive), read by the kernel; the caller advances it."""
        B = q.shape[0]
        assert pos.dtype == torch.int64 and pos.is_contiguous() and pos.numel() >= B and pos.device == q.device
        check(self.lib.moa_decode_step_fused_ragged(self.ctx, layer, _ptr(q), _ptr(k_new), _ptr(v_new), _ptr(o),
                                                    q.stride(0), k_new.stride(0), o.stride(0), B, _ptr(pos),
                                                    float(scale), _ptr(lse), _ptr(workspace),
                                                    workspace.numel() * workspace.element_size(),
                                                    _stream(stream)),
              "moa_decode_step_fused_ragged")

    # ---- cache inspection (tests) --------------------------------------------------------
    def cache_rows(self, layer: int, b: int, g: int, which: str = "k") -> torch.Tensor:
        """The (n_sink + W_g, d) rows of region (b, g) as a view of the cache bound by
        ``bind_cache``/``alloc_cache``."""
        k, v = self._cache
        buf = k if which == "k" else v
        es = torch.tensor([], dtype=self.dtype).element_size()
        off, rows = self.cache_region(layer, b, g)
        start = self.layer_offset(layer, self._bound_batch) + off * self.d * es
        return buf[start: start + rows * self.d * es].view(self.dtype).view(rows, self.d)


def wait_flag(flag: torch.Tensor, expected: int, stream=None):
    """moa_wait_flag: the next work on `stream` waits until the uint32 counter `flag`
    (a 1-element int32/uint32 device tensor view) reaches `expected` (mod 2^32)."""
    check(_lib.lib().moa_wait_flag(_ptr(flag), int(expected) & 0xffffffff, _stream(stream)), "moa_wait_flag")
