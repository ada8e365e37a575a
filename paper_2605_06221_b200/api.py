"""Host-side mirror of the reference operator API for the token-selection hot path.

Every function here validates its arguments, then calls the C ABI
(``include/uniprefill_b200.h``) on device buffers; all compute runs in the sm_100a kernels
of ``_lib/libuniprefill_b200.so``.  PyTorch only supplies device memory and the current CUDA
stream.  There is no CPU fallback: without the library, importing this package fails.

Two layers:

* varlen entry points used by an engine (``score_blocks_varlen``, ``select_varlen``,
  ``compact_varlen``, ``DropLayer``) -- device-resident metadata, no host syncs;
* reference-named mirrors with the reference's argument meaning and error behaviour
  (``score_tokens``, ``score_tokens_heads``, ``top_p_select``, ``sharded_block_scores``,
  ``allreduce_scores``, ``apply_drop``, ``patch_metadata``), each citing the reference
  declaration it mirrors, so parity tests read like ``/root/reference/proj/tests``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import torch

from . import _capi
from ._capi import (BatchC, HeadsC, PlaneC, ScoreConfigC, SelectionOutC, lib)


# --------------------------------------------------------------------------- errors
class ConfigError(ValueError):
    """Reference ConfigError (errors.hpp:15-18)."""


class ContractViolation(RuntimeError):
    """Reference ContractViolation (errors.hpp:22-25)."""


class UnsupportedError(RuntimeError):
    """Valid input outside the implemented envelope."""


class AllocationMissError(RuntimeError):
    """Reference AllocationMissError (errors.hpp:32-35): a KV slot whose page is absent."""


class CudaError(RuntimeError):
    """CUDA runtime / driver failure."""


def _check(status: int, what: str) -> None:
    if status == _capi.UP_OK:
        return
    msg = f"{what}: {_capi.status_string(status)}"
    if status == _capi.UP_ERR_CONFIG:
        raise ConfigError(msg)
    if status == _capi.UP_ERR_CONTRACT:
        raise ContractViolation(msg)
    if status == _capi.UP_ERR_UNSUPPORTED:
        raise UnsupportedError(msg)
    if status == _capi.UP_ERR_CUDA:
        raise CudaError(msg)
    if status == _capi.UP_ERR_ALLOCATION_MISS:
        raise AllocationMissError(msg)
    raise RuntimeError(msg)


# --------------------------------------------------------------------------- config
@dataclass
class ScoreConfig:
    """ScoreConfig (config.hpp:53-63): n=128, G=64, A=128, p=0.99."""

    query_window_n: int = 128
    block_size_g: int = 64
    sink_count_a: int = 128
    top_p: float = 0.99

    def c(self) -> ScoreConfigC:
        return ScoreConfigC(int(self.query_window_n), int(self.block_size_g),
                            int(self.sink_count_a), float(self.top_p))

    def validate(self) -> None:
        """ScoreConfig::validate (config.cpp:98-103) -> ConfigError."""
        _check(lib.up_config_validate(ctypes.byref(self.c())), "ScoreConfig.validate")


@dataclass
class HeadLayout:
    """Head layout of q / k on this rank (up_heads)."""

    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    gqa_group: Optional[int] = None  # global Hq / Hkv; defaults to local Hq / Hkv
    q_head_offset: int = 0
    kv_head_offset: int = 0

    def c(self, q_row_stride: int, k_row_stride: int) -> HeadsC:
        group = self.gqa_group if self.gqa_group is not None else self.num_q_heads // self.num_kv_heads
        return HeadsC(self.num_q_heads, self.num_kv_heads, self.head_dim, group, self.q_head_offset,
                      self.kv_head_offset, q_row_stride, k_row_stride)


def _stream_ptr(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _as_i32_cuda(x, device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.int32).contiguous()
    return torch.tensor(list(x), dtype=torch.int32, device=device)


def _batch(cu: torch.Tensor, max_tokens: int, drop_enabled: Optional[torch.Tensor]) -> BatchC:
    return BatchC(cu.numel() - 1, int(max_tokens), ctypes.c_void_p(cu.data_ptr()),
                  None if drop_enabled is None else ctypes.c_void_p(drop_enabled.data_ptr()))


class Workspace:
    """Device scratch shared by all entry points; grows on demand, zeroed once."""

    def __init__(self, device=None):
        self.device = torch.device(device if device is not None else "cuda")
        self.buf: Optional[torch.Tensor] = None

    def get(self, batch: BatchC, heads: Optional[HeadsC], cfg: ScoreConfigC) -> torch.Tensor:
        need = lib.up_workspace_bytes(ctypes.byref(batch),
                                      ctypes.byref(heads) if heads is not None else None,
                                      ctypes.byref(cfg))
        if self.buf is None or self.buf.numel() < need:
            self.buf = torch.zeros(max(int(need), 256), dtype=torch.uint8, device=self.device)
        return self.buf

    def device_status(self) -> None:
        """Raise the sticky device-side error (ContractViolation / UnsupportedError), if any."""
        if self.buf is None:
            return
        _check(lib.up_device_status(_stream_ptr(self.device), ctypes.c_void_p(self.buf.data_ptr())),
               "device status")


_default_ws: dict = {}


def _ws(device) -> Workspace:
    key = str(torch.device(device))
    if key not in _default_ws:
        _default_ws[key] = Workspace(device)
    return _default_ws[key]


# --------------------------------------------------------------------------- varlen API
@dataclass
class BlockScores:
    block_scores: torch.Tensor          # fp32 [>= Σ ceil(N_r/G)]
    cu_blocks: torch.Tensor             # int32 [R+1]
    token_scores: Optional[torch.Tensor] = None


def _heads_view(x: torch.Tensor, num_heads: int):
    """Accept [T, H, D] or [T, H*D]; return (tensor, row_stride_elements, D)."""
    if x.dim() == 3:
        if x.stride(2) != 1 or x.stride(1) != x.shape[2]:
            raise ContractViolation("q/k heads must be contiguous within a row")
        return x, x.stride(0), x.shape[2]
    if x.dim() == 2:
        if x.stride(1) != 1 or x.shape[1] % num_heads != 0:
            raise ContractViolation("score_tokens: bad head layout")
        return x, x.stride(0), x.shape[1] // num_heads
    raise ContractViolation("q/k must be [T, H, D] or [T, H*D]")


def score_blocks_varlen(q: torch.Tensor, k: torch.Tensor, cu_seqlens, config: ScoreConfig,
                        heads: Optional[HeadLayout] = None, drop_enabled=None,
                        want_token_scores: bool = False, max_tokens: Optional[int] = None,
                        workspace: Optional[Workspace] = None, out: Optional[BlockScores] = None,
                        check: bool = False) -> BlockScores:
    """Block scores of every drop-enabled segment (up_score_blocks).

    q: bf16 [T, Hq, D] (or [T, Hq*D]); k: bf16 [T, Hkv, D].  Returns the PARTIAL scores over
    the local heads (reduce across TP ranks before selection)."""
    if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16:
        raise ContractViolation("q and k must be bfloat16")
    dev = q.device
    cu = _as_i32_cuda(cu_seqlens, dev)
    R = cu.numel() - 1
    T = int(max_tokens if max_tokens is not None else q.shape[0])
    if heads is None:
        if q.dim() != 3 or k.dim() != 3:
            raise ContractViolation("pass heads= for 2-D q/k")
        heads = HeadLayout(q.shape[1], k.shape[1], q.shape[2])
    qv, qs, D = _heads_view(q, heads.num_q_heads)
    kv, ks, _ = _heads_view(k, heads.num_kv_heads)
    if D != heads.head_dim:
        raise ContractViolation("partial_scores: head dim mismatch")
    en = None if drop_enabled is None else drop_enabled.to(device=dev, dtype=torch.uint8).contiguous()
    b = _batch(cu, T, en)
    hc = heads.c(qs, ks)
    cfg = config.c()
    ws = workspace or _ws(dev)
    buf = ws.get(b, hc, cfg)
    nbmax = int(lib.up_max_blocks(ctypes.byref(b), ctypes.byref(cfg)))
    if out is None:
        out = BlockScores(torch.empty(nbmax, dtype=torch.float32, device=dev),
                          torch.empty(R + 1, dtype=torch.int32, device=dev),
                          torch.empty(T, dtype=torch.float32, device=dev) if want_token_scores else None)
    st = lib.up_score_blocks(_stream_ptr(dev), ctypes.byref(b), ctypes.byref(hc), ctypes.byref(cfg),
                             _ptr(qv), _ptr(kv), _ptr(out.block_scores), _ptr(out.cu_blocks),
                             _ptr(out.token_scores), ctypes.c_void_p(buf.data_ptr()), buf.numel())
    _check(st, "score_blocks")
    if check:
        ws.device_status()
    return out


@dataclass
class ShardedBlockScores:
    shard_scores: torch.Tensor          # fp32 [tp, >= Σ ceil(N_r/G)] per-shard partials
    block_scores: torch.Tensor          # fp32 ascending-shard sum (allreduce_scores)
    cu_blocks: torch.Tensor             # int32 [R+1]


def score_blocks_tp(q: torch.Tensor, k: torch.Tensor, cu_seqlens, config: ScoreConfig, tp_degree: int,
                    heads: Optional[HeadLayout] = None, drop_enabled=None, max_tokens: Optional[int] = None,
                    workspace: Optional[Workspace] = None, out: Optional[ShardedBlockScores] = None,
                    check: bool = False) -> ShardedBlockScores:
    """Head-sharded block scores in one call (up_score_blocks_tp): shard t scores q-heads
    [t*H/T, (t+1)*H/T) (sharded_block_scores, tp_sim.cpp:12-27) and block_scores is their
    ascending-shard fp32 sum (allreduce_scores, tp_sim.cpp:29-49) -- what a TP group of
    tp_degree ranks computes, on one device."""
    if q.dtype != torch.bfloat16 or k.dtype != torch.bfloat16:
        raise ContractViolation("q and k must be bfloat16")
    dev = q.device
    cu = _as_i32_cuda(cu_seqlens, dev)
    R = cu.numel() - 1
    T = int(max_tokens if max_tokens is not None else q.shape[0])
    if heads is None:
        if q.dim() != 3 or k.dim() != 3:
            raise ContractViolation("pass heads= for 2-D q/k")
        heads = HeadLayout(q.shape[1], k.shape[1], q.shape[2])
    qv, qs, D = _heads_view(q, heads.num_q_heads)
    kv, ks, _ = _heads_view(k, heads.num_kv_heads)
    if D != heads.head_dim:
        raise ContractViolation("partial_scores: head dim mismatch")
    en = None if drop_enabled is None else drop_enabled.to(device=dev, dtype=torch.uint8).contiguous()
    b = _batch(cu, T, en)
    hc = heads.c(qs, ks)
    cfg = config.c()
    ws = workspace or _ws(dev)
    buf = ws.get(b, hc, cfg)
    nbmax = int(lib.up_max_blocks(ctypes.byref(b), ctypes.byref(cfg)))
    if out is None:
        tpn = max(int(tp_degree), 1)
        out = ShardedBlockScores(torch.empty(tpn, nbmax, dtype=torch.float32, device=dev),
                                 torch.empty(nbmax, dtype=torch.float32, device=dev),
                                 torch.empty(R + 1, dtype=torch.int32, device=dev))
    st = lib.up_score_blocks_tp(_stream_ptr(dev), ctypes.byref(b), ctypes.byref(hc), ctypes.byref(cfg), _ptr(qv),
                                _ptr(kv), int(tp_degree), _ptr(out.shard_scores), out.shard_scores.stride(0),
                                _ptr(out.block_scores), _ptr(out.cu_blocks), ctypes.c_void_p(buf.data_ptr()),
                                buf.numel())
    _check(st, "score_blocks_tp")
    if check:
        ws.device_status()
    return out


@dataclass
class VarlenSelection:
    keep: torch.Tensor             # uint8 [T]
    cutoff_rank: torch.Tensor      # int64 [R] (-1 for pass-through segments)
    retained_count: torch.Tensor   # int64 [R]
    covered_mass: torch.Tensor     # float64 [R]
    degenerate: torch.Tensor       # uint8 [R]


def select_varlen(block_scores: torch.Tensor, cu_blocks: torch.Tensor, cu_seqlens, config: ScoreConfig,
                  veto: Optional[torch.Tensor] = None, drop_enabled=None,
                  max_tokens: Optional[int] = None, workspace: Optional[Workspace] = None,
                  out: Optional[VarlenSelection] = None, check: bool = False) -> VarlenSelection:
    """Top-p keep mask of every drop-enabled segment (up_select)."""
    dev = block_scores.device
    cu = _as_i32_cuda(cu_seqlens, dev)
    R = cu.numel() - 1
    if max_tokens is None and torch.cuda.is_current_stream_capturing():
        raise ContractViolation("select_varlen: pass max_tokens (the capacity) when capturing a CUDA graph "
                                "-- the default reads cu_seqlens[-1] on the host")
    T = int(max_tokens) if max_tokens is not None else int(cu[-1].item())
    en = None if drop_enabled is None else drop_enabled.to(device=dev, dtype=torch.uint8).contiguous()
    b = _batch(cu, T, en)
    cfg = config.c()
    ws = workspace or _ws(dev)
    buf = ws.get(b, None, cfg)
    if out is None:
        out = VarlenSelection(torch.empty(T, dtype=torch.uint8, device=dev),
                              torch.empty(R, dtype=torch.int64, device=dev),
                              torch.empty(R, dtype=torch.int64, device=dev),
                              torch.empty(R, dtype=torch.float64, device=dev),
                              torch.empty(R, dtype=torch.uint8, device=dev))
    so = SelectionOutC(_ptr(out.cutoff_rank), _ptr(out.retained_count), _ptr(out.covered_mass),
                       _ptr(out.degenerate))
    vt = None if veto is None else veto.to(device=dev, dtype=torch.uint8).contiguous()
    st = lib.up_select(_stream_ptr(dev), ctypes.byref(b), ctypes.byref(cfg), _ptr(block_scores),
                       _ptr(cu_blocks), _ptr(vt), _ptr(out.keep), ctypes.byref(so),
                       ctypes.c_void_p(buf.data_ptr()), buf.numel())
    _check(st, "select")
    if check:
        ws.device_status()
    return out


@dataclass
class Compacted:
    planes: List[torch.Tensor]     # compacted copies (capacity rows; first num_out valid)
    cu_seqlens: torch.Tensor       # int32 [R+1]
    retained_index: torch.Tensor   # int32 [capacity]
    num_out: torch.Tensor          # int32 [1] (device)

    def trimmed(self) -> "Compacted":
        n = int(self.num_out.item())
        return Compacted([p[:n] for p in self.planes], self.cu_seqlens, self.retained_index[:n],
                         self.num_out)


def compact_varlen(keep: torch.Tensor, cu_seqlens, planes: Sequence[torch.Tensor], drop_enabled=None,
                   max_tokens: Optional[int] = None, outs: Optional[Sequence[torch.Tensor]] = None,
                   workspace: Optional[Workspace] = None, result: Optional[Compacted] = None,
                   check: bool = False, after_select: bool = False) -> Compacted:
    """Segmented prefix sum + gather of retained rows (up_compact).  planes: [T, ...] tensors on
    the device, or in pinned host memory (read in place: only retained rows cross PCIe).
    after_select: `keep` is select_varlen's output on the same workspace, unmodified since
    (up_compact_selected: the selection already counted the rows per tile)."""
    dev = keep.device
    cu = _as_i32_cuda(cu_seqlens, dev)
    R = cu.numel() - 1
    T = int(max_tokens) if max_tokens is not None else int(keep.numel())
    en = None if drop_enabled is None else drop_enabled.to(device=dev, dtype=torch.uint8).contiguous()
    b = _batch(cu, T, en)
    ws = workspace or _ws(dev)
    before = ws.buf
    # block size only sizes the block-decision region, which compaction does not use: a
    # huge G keeps this layout inside the selection's (same offsets, no regrowth)
    buf = ws.get(b, None, ScoreConfig(1, 1 << 20, 0, 1.0).c())
    if buf is not before:
        after_select = False  # a fresh workspace holds no tile counts from a selection
    if result is None:
        if outs is None:
            outs = [torch.empty_like(p) for p in planes]
        result = Compacted(list(outs), torch.empty(R + 1, dtype=torch.int32, device=dev),
                           torch.empty(T, dtype=torch.int32, device=dev),
                           torch.empty(1, dtype=torch.int32, device=dev))
    arr = (PlaneC * max(len(planes), 1))()
    for i, (src, dst) in enumerate(zip(planes, result.planes)):
        if not (src.is_contiguous() and dst.is_contiguous()):
            raise ContractViolation("compact planes must be contiguous")
        if dst.device != dev or (src.device != dev and not (src.device.type == "cpu" and src.is_pinned())):
            # A source plane may live in pinned host memory: under unified addressing the
            # copy kernel reads it in place over PCIe, so only the retained rows cross the bus.
            raise ContractViolation("compact planes: sources on the keep mask's device or pinned host, "
                                    "destinations on the device")
        rb = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
        arr[i] = PlaneC(src.data_ptr(), dst.data_ptr(), rb, 0, 0)
    fn = lib.up_compact_selected if after_select else lib.up_compact
    st = fn(_stream_ptr(dev), ctypes.byref(b), _ptr(keep), arr, len(planes), _ptr(result.cu_seqlens),
            _ptr(result.retained_index), _ptr(result.num_out), ctypes.c_void_p(buf.data_ptr()), buf.numel())
    _check(st, "compact")
    if check:
        ws.device_status()
    return result


def scatter_rows(index: torch.Tensor, planes: Sequence[torch.Tensor], outs: Sequence[torch.Tensor],
                 num_rows: Optional[torch.Tensor] = None) -> None:
    """Row scatter (up_scatter_rows), the inverse of compact_varlen's gather:
    outs[p][index[o]] = planes[p][o] for o < num_rows (device int32 count; default: all
    rows of index), skipping index[o] < 0.  Destinations may be pinned host memory
    (written in place over PCIe, only the scattered rows cross the bus)."""
    if index.dtype != torch.int32 or not index.is_contiguous():
        raise ContractViolation("scatter_rows: index must be contiguous int32")
    dev = index.device
    arr = (PlaneC * max(len(planes), 1))()
    for i, (src, dst) in enumerate(zip(planes, outs)):
        if not (src.is_contiguous() and dst.is_contiguous()):
            raise ContractViolation("scatter planes must be contiguous")
        if src.device != dev or (dst.device != dev and not (dst.device.type == "cpu" and dst.is_pinned())):
            raise ContractViolation("scatter planes: sources on the index's device, destinations on the "
                                    "device or pinned host")
        rb = src[0].numel() * src.element_size() if src.dim() > 1 else src.element_size()
        if (dst[0].numel() * dst.element_size() if dst.dim() > 1 else dst.element_size()) != rb:
            raise ContractViolation("scatter planes: row size mismatch")
        arr[i] = PlaneC(src.data_ptr(), dst.data_ptr(), rb, 0, 0)
    _check(lib.up_scatter_rows(_stream_ptr(dev), _ptr(index), _ptr(num_rows), int(index.numel()), arr,
                               len(planes)), "scatter_rows")


def reconstitute_varlen(current_planes: Sequence[torch.Tensor], drop: "Compacted",
                        pre_drop_planes: Sequence[torch.Tensor]) -> None:
    """Undo one drop of a varlen batch in place: the current state of every row retained by
    `drop` (current_planes, row o = output row o of the drop, first drop.num_out rows) is
    written back over its row of the pre-drop buffer, which still holds the dropped rows as
    they were when parked.  Applied to a block's drops in reverse order this is the engine's
    reconstitution at a block boundary (scheduler.cpp:349-360 + reconstitute,
    propagation.cpp:79-100); the batch's cu_seqlens become the pre-drop ones again."""
    scatter_rows(drop.retained_index, current_planes, pre_drop_planes, num_rows=drop.num_out)


def slot_mapping(cu_seqlens: torch.Tensor, positions: torch.Tensor, block_tables: torch.Tensor, block_size: int,
                 num_rows: Optional[torch.Tensor] = None, out: Optional[torch.Tensor] = None,
                 workspace: Optional[Workspace] = None, check: bool = False) -> torch.Tensor:
    """Eq. 16 KV slot mapping of the retained rows for downstream layers (up_slot_mapping;
    recompute_slots_after_drop, kvcache.cpp:147-158).  cu_seqlens int32 [R+1] and positions
    int64 [rows] of the compacted batch, block_tables int32 [L, R, max_pages] (-1 = no
    page).  Returns int64 [L, rows]."""
    dev = positions.device
    cu = _as_i32_cuda(cu_seqlens, dev)
    R = cu.numel() - 1
    if block_tables.dim() != 3 or block_tables.shape[1] != R or block_tables.dtype != torch.int32:
        raise ContractViolation("slot_mapping: block_tables must be int32 [layers, R, max_pages]")
    L, _, max_pages = block_tables.shape
    rows = positions.numel()
    if out is None:
        out = torch.empty(L, rows, dtype=torch.int64, device=dev)
    ws = workspace or _ws(dev)
    b = _batch(cu, max(rows, 1), None)
    buf = ws.get(b, None, ScoreConfig(1, 1 << 20, 0, 1.0).c())  # only the error word is used
    _check(lib.up_slot_mapping(_stream_ptr(dev), _ptr(cu), R, _ptr(num_rows), rows,
                               _ptr(positions.contiguous()), _ptr(block_tables.contiguous()), L, max_pages,
                               int(block_size), _ptr(out), out.stride(0), ctypes.c_void_p(buf.data_ptr()),
                               buf.numel()), "slot_mapping")
    if check:
        ws.device_status()
    return out


def attention_varlen(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, cu_seqlens, positions: torch.Tensor,
                     heads: Optional[HeadLayout] = None, window: Optional[int] = None,
                     max_tokens: Optional[int] = None, out: Optional[torch.Tensor] = None,
                     workspace: Optional[Workspace] = None, check: bool = False) -> torch.Tensor:
    """Attention readout over the retained rows (up_attention_varlen; attention_readout,
    model.cpp:215-263, as prefill_layer_step calls it at a drop layer, propagation.cpp:195-205).

    q bf16 [T, Hq, D], k / v bf16 [T, Hkv, D] (or 2-D with heads=), cu_seqlens int32 [R+1]
    and positions int64 [T] of the compacted batch (``Compacted.cu_seqlens`` and its
    positions plane).  Row j of a segment attends to the segment's rows with position in
    (pos_j - window, pos_j].  Returns bf16 [T, Hq, D] (rows past cu_seqlens[-1] untouched)."""
    for t in (q, k, v):
        if t.dtype != torch.bfloat16:
            raise ContractViolation("attention_varlen: q, k, v must be bfloat16")
    if positions.dtype != torch.int64:
        raise ContractViolation("attention_varlen: positions must be int64")
    dev = q.device
    cu = _as_i32_cuda(cu_seqlens, dev)
    T = int(max_tokens if max_tokens is not None else q.shape[0])
    if heads is None:
        if q.dim() != 3 or k.dim() != 3:
            raise ContractViolation("pass heads= for 2-D q/k/v")
        heads = HeadLayout(q.shape[1], k.shape[1], q.shape[2])
    qv, qs, D = _heads_view(q, heads.num_q_heads)
    kv, ks, _ = _heads_view(k, heads.num_kv_heads)
    vv, vs, _ = _heads_view(v, heads.num_kv_heads)
    if D != heads.head_dim or vs != ks:
        raise ContractViolation("attention_varlen: head dim / k-v row stride mismatch")
    if out is None:
        out = torch.empty(T, heads.num_q_heads, D, dtype=torch.bfloat16, device=dev)
    ov, os_, _ = _heads_view(out, heads.num_q_heads)
    b = _batch(cu, T, None)
    hc = heads.c(qs, ks)
    ws = workspace or _ws(dev)
    buf = ws.get(b, hc, ScoreConfig().c())
    _check(lib.up_attention_varlen(_stream_ptr(dev), ctypes.byref(b), ctypes.byref(hc), _ptr(qv), _ptr(kv), _ptr(vv),
                                   _ptr(positions.contiguous()), int(window or 0), _ptr(ov), os_,
                                   ctypes.c_void_p(buf.data_ptr()), buf.numel()), "attention_varlen")
    if check:
        ws.device_status()
    return out


def decode_seqused(num_layers: int, cu_orig: torch.Tensor, drop_layers: Sequence[int],
                   cu_after: Sequence[torch.Tensor], decode_appended: Optional[torch.Tensor] = None,
                   out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Eq. 17 per-layer decode KV lengths (up_decode_seqused; decode_seqused,
    kvcache.cpp:182-186) for every request: int32 [num_layers, R]."""
    dev = cu_orig.device
    cu0 = _as_i32_cuda(cu_orig, dev)
    R = cu0.numel() - 1
    cus = [_as_i32_cuda(c, dev) for c in cu_after]
    if out is None:
        out = torch.empty(num_layers, R, dtype=torch.int32, device=dev)
    dl = (ctypes.c_int32 * max(len(drop_layers), 1))(*[int(x) for x in drop_layers])
    ptrs = (ctypes.c_void_p * max(len(cus), 1))(*[c.data_ptr() for c in cus])
    app = None if decode_appended is None else decode_appended.to(device=dev, dtype=torch.int32).contiguous()
    _check(lib.up_decode_seqused(_stream_ptr(dev), int(num_layers), R, _ptr(cu0), len(cus), dl, ptrs,
                                 _ptr(app), _ptr(out)), "decode_seqused")
    return out


def reduce_block_scores(shards: Sequence[torch.Tensor], out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Ascending-shard fp32 sum (up_reduce_block_scores), bitwise like allreduce_scores."""
    if len(shards) == 0:
        raise ContractViolation("allreduce_scores: no shards")
    n = shards[0].numel()
    if any(s.numel() != n for s in shards):
        raise ContractViolation("allreduce_scores: shard length mismatch")
    dev = shards[0].device
    out = torch.empty(n, dtype=torch.float32, device=dev) if out is None else out
    ptrs = (ctypes.c_void_p * len(shards))(*[s.data_ptr() for s in shards])
    _check(lib.up_reduce_block_scores(_stream_ptr(dev), ptrs, len(shards), n, _ptr(out)),
           "reduce_block_scores")
    return out


# --------------------------------------------------------------------------- engine hook
class DropLayer:
    """score -> select -> compact for one full-attention drop layer over a varlen batch.

    Buffers are preallocated for a capacity of ``max_tokens`` rows and ``num_requests``
    segments, so a layer step issues only kernel launches (capturable in a CUDA graph).
    Mirrors prefill_layer_step's drop section (propagation.cpp:163-202) followed by
    patch_metadata (scheduler.cpp:332)."""

    def __init__(self, config: ScoreConfig, heads: HeadLayout, max_tokens: int, num_requests: int,
                 plane_shapes: Sequence[tuple], plane_dtypes: Sequence[torch.dtype], device=None):
        config.validate()
        self.config = config
        self.heads = heads
        self.device = torch.device(device if device is not None else "cuda")
        self.max_tokens = int(max_tokens)
        self.R = int(num_requests)
        dev = self.device
        self.ws = Workspace(dev)
        cfg = config.c()
        G = config.block_size_g
        nb = self.max_tokens // G + self.R + 1
        self.scores = BlockScores(torch.empty(nb, dtype=torch.float32, device=dev),
                                  torch.empty(self.R + 1, dtype=torch.int32, device=dev))
        self.sel = VarlenSelection(torch.empty(self.max_tokens, dtype=torch.uint8, device=dev),
                                   torch.empty(self.R, dtype=torch.int64, device=dev),
                                   torch.empty(self.R, dtype=torch.int64, device=dev),
                                   torch.empty(self.R, dtype=torch.float64, device=dev),
                                   torch.empty(self.R, dtype=torch.uint8, device=dev))
        self.out = Compacted([torch.empty((self.max_tokens, *s), dtype=d, device=dev)
                              for s, d in zip(plane_shapes, plane_dtypes)],
                             torch.empty(self.R + 1, dtype=torch.int32, device=dev),
                             torch.empty(self.max_tokens, dtype=torch.int32, device=dev),
                             torch.empty(1, dtype=torch.int32, device=dev))
        self._cfg = cfg
        self.last_launches = 0

    def __call__(self, q: torch.Tensor, k: torch.Tensor, cu_seqlens: torch.Tensor,
                 planes: Sequence[torch.Tensor], drop_enabled: Optional[torch.Tensor] = None,
                 veto: Optional[torch.Tensor] = None, block_scores_hook=None) -> Compacted:
        """block_scores_hook(block_scores) runs between scoring and selection (TP all-reduce)."""
        score_blocks_varlen(q, k, cu_seqlens, self.config, self.heads, drop_enabled,
                            max_tokens=self.max_tokens, workspace=self.ws, out=self.scores)
        n = lib.up_last_launch_count()
        if block_scores_hook is not None:
            block_scores_hook(self.scores.block_scores)
        select_varlen(self.scores.block_scores, self.scores.cu_blocks, cu_seqlens, self.config, veto,
                      drop_enabled, max_tokens=self.max_tokens, workspace=self.ws, out=self.sel)
        n += lib.up_last_launch_count()
        compact_varlen(self.sel.keep, cu_seqlens, planes, drop_enabled, max_tokens=self.max_tokens,
                       workspace=self.ws, result=self.out, after_select=True)
        n += lib.up_last_launch_count()
        self.last_launches = n
        return self.out

    def check(self) -> None:
        self.ws.device_status()


# --------------------------------------------------------------------------- reference mirrors
@dataclass
class ImportanceScores:
    """ImportanceScores (importance.hpp:18-23)."""

    token_scores: torch.Tensor
    block_scores: torch.Tensor
    num_tokens: int
    effective_n: int


def score_tokens_heads(q: torch.Tensor, k: torch.Tensor, num_heads: int, head_begin: int,
                       head_end: int, config: ScoreConfig, num_kv_heads: Optional[int] = None,
                       want_token_scores: bool = True) -> ImportanceScores:
    """score_tokens_heads (importance.hpp:42-43) on one request.

    q: bf16 [N, num_heads*D] (head-blocked columns, already rotated); k: bf16
    [N, num_kv_heads*D] (num_kv_heads defaults to num_heads, as in the MHA reference)."""
    kvh = num_heads if num_kv_heads is None else num_kv_heads
    if q.dim() != 2 or k.dim() != 2 or q.shape[1] % num_heads != 0 or k.shape[1] % kvh != 0:
        raise ContractViolation("score_tokens: bad head layout")
    D = q.shape[1] // num_heads
    if k.shape[1] // kvh != D or num_heads % kvh != 0:
        raise ContractViolation("score_tokens: bad head layout")
    if head_begin < 0 or head_end > num_heads or head_begin >= head_end:
        raise ContractViolation("score_tokens: bad head range")
    if k.shape[0] != q.shape[0]:
        raise ContractViolation("score_tokens: q/k row mismatch")
    N = k.shape[0]
    if N < 1:
        raise ContractViolation("block_reduce: empty scores")
    if config.block_size_g <= 0:
        raise ContractViolation("block_reduce: block size must be positive")
    group = num_heads // kvh
    heads = HeadLayout(head_end - head_begin, kvh, D, group, head_begin, 0)
    qs = q[:, head_begin * D: head_end * D]
    res = score_blocks_varlen(qs, k, [0, N], config, heads, want_token_scores=want_token_scores,
                              check=True)
    nb = (N + config.block_size_g - 1) // config.block_size_g
    return ImportanceScores(res.token_scores[:N] if res.token_scores is not None else None,
                            res.block_scores[:nb], N, min(config.query_window_n, N))


def score_tokens(q: torch.Tensor, k: torch.Tensor, num_heads: int, config: ScoreConfig,
                 num_kv_heads: Optional[int] = None, want_token_scores: bool = True) -> ImportanceScores:
    """score_tokens (importance.hpp:46-47): all heads."""
    return score_tokens_heads(q, k, num_heads, 0, num_heads, config, num_kv_heads, want_token_scores)


@dataclass
class ShardScores:
    """ShardScores (tp_sim.hpp:16-19)."""

    shard_id: int
    block_scores: torch.Tensor


def sharded_block_scores(q: torch.Tensor, k: torch.Tensor, num_heads: int, config: ScoreConfig,
                         tp_degree: int, num_kv_heads: Optional[int] = None) -> List[ShardScores]:
    """sharded_block_scores (tp_sim.hpp:25-26): shard t scores heads [tH/T, (t+1)H/T)."""
    if tp_degree <= 0:
        raise ConfigError("tp_degree must be positive")
    if num_heads % tp_degree != 0:
        raise ConfigError("num_heads must be divisible by tp_degree")
    hps = num_heads // tp_degree
    return [ShardScores(t, score_tokens_heads(q, k, num_heads, t * hps, (t + 1) * hps, config,
                                              num_kv_heads, want_token_scores=False).block_scores.clone())
            for t in range(tp_degree)]


def allreduce_scores(shards: Sequence[ShardScores]) -> torch.Tensor:
    """allreduce_scores (tp_sim.hpp:31, tp_sim.cpp:29-49): ids exactly 0..T-1, fp32 ascending sum."""
    if len(shards) == 0:
        raise ContractViolation("allreduce_scores: no shards")
    T = len(shards)
    by_id: List[Optional[ShardScores]] = [None] * T
    for s in shards:
        if s.shard_id < 0 or s.shard_id >= T or by_id[s.shard_id] is not None:
            raise ContractViolation("allreduce_scores: shard ids must be exactly 0..T-1")
        if s.block_scores.numel() != shards[0].block_scores.numel():
            raise ContractViolation("allreduce_scores: shard length mismatch")
        by_id[s.shard_id] = s
    return reduce_block_scores([s.block_scores.contiguous() for s in by_id])


@dataclass
class Selection:
    """Selection (selection.hpp:34-57), device-resident."""

    keep_mask: torch.Tensor
    retained_indices: torch.Tensor
    retention_ratio: float
    covered_mass: float
    cutoff_rank: int
    degenerate_keep_all: bool

    def num_tokens(self) -> int:
        return int(self.keep_mask.numel())

    def retained_count(self) -> int:
        return int(self.retained_indices.numel())


def top_p_select(block_scores, config: ScoreConfig, num_tokens: int,
                 veto: Optional[torch.Tensor] = None, device=None) -> Selection:
    """top_p_select (selection.hpp:53-54) on one request (+ optional no-readmission veto)."""
    config.validate()
    if num_tokens < 1:
        raise ContractViolation("top_p_select: num_tokens must be positive")
    dev = torch.device(device) if device is not None else (
        block_scores.device if isinstance(block_scores, torch.Tensor) and block_scores.is_cuda
        else torch.device("cuda"))
    bs = torch.as_tensor(block_scores, dtype=torch.float32).to(dev).contiguous()
    nb = (num_tokens + config.block_size_g - 1) // config.block_size_g
    if bs.numel() != nb:
        raise ContractViolation("top_p_select: block score length must be ceil(N/G)")
    cu = torch.tensor([0, num_tokens], dtype=torch.int32, device=dev)
    cub = torch.tensor([0, nb], dtype=torch.int32, device=dev)
    sel = select_varlen(bs, cub, cu, config, veto=veto, max_tokens=num_tokens, check=True)
    idx = compact_varlen(sel.keep, cu, [], max_tokens=num_tokens, check=True)
    n_ret = int(idx.num_out.item())
    return Selection(sel.keep, idx.retained_index[:n_ret].to(torch.int64), n_ret / num_tokens,
                     float(sel.covered_mass[0].item()), int(sel.cutoff_rank[0].item()),
                     bool(sel.degenerate[0].item()))


# ---- propagation / scheduler mirrors ------------------------------------------------
@dataclass
class DropEvent:
    """DropEvent (drop_history.hpp:14-18)."""

    layer: int
    retained_length: int
    retained_positions: torch.Tensor


@dataclass
class DropHistory:
    """DropHistory (drop_history.hpp:20-31)."""

    events: List[DropEvent] = field(default_factory=list)
    original_length: int = 0
    decode_appended: int = 0


@dataclass
class TokenStream:
    """TokenStream (propagation.hpp:21-39).  Parked rows are kept as (positions, states)
    gathered out of the pre-drop buffer; the pre-drop buffer itself is left untouched
    (out-of-place compaction, propagation.cpp:64-67)."""

    active_states: torch.Tensor
    logical_positions: torch.Tensor
    parked_positions: List[torch.Tensor] = field(default_factory=list)
    parked_states: List[torch.Tensor] = field(default_factory=list)
    original_length: int = 0

    @staticmethod
    def from_prompt(prompt: torch.Tensor) -> "TokenStream":
        if prompt.shape[0] < 1:
            raise ContractViolation("TokenStream: prompt must be non-empty")
        pos = torch.arange(prompt.shape[0], dtype=torch.int64, device=prompt.device)
        return TokenStream(prompt, pos, [], [], prompt.shape[0])

    def active_count(self) -> int:
        return int(self.logical_positions.numel())


def reconstitute(stream: TokenStream) -> None:
    """reconstitute (propagation.hpp:43, propagation.cpp:79-100): rebuild the full-length
    stream -- parked rows with the state they had when dropped, active rows with their
    current state, positions 0..n-1 -- through up_scatter_rows.  No-op without parked rows."""
    if not stream.parked_states:
        return
    n = stream.original_length
    act = stream.active_states.contiguous()
    full = torch.empty((n, *act.shape[1:]), dtype=act.dtype, device=act.device)
    for pos, st in zip(stream.parked_positions, stream.parked_states):
        scatter_rows(pos.to(torch.int32).contiguous(), [st.contiguous()], [full])
    scatter_rows(stream.logical_positions.to(torch.int32).contiguous(), [act], [full])
    stream.active_states = full
    stream.logical_positions = torch.arange(n, dtype=torch.int64, device=act.device)
    stream.parked_positions = []
    stream.parked_states = []


def apply_drop(stream: TokenStream, selection: Selection, layer: int, history: DropHistory) -> None:
    """apply_drop (propagation.hpp:415, propagation.cpp:47-77) through up_compact."""
    rows = stream.active_count()
    if selection.num_tokens() != rows:
        raise ContractViolation("apply_drop: selection length disagrees with the active stream")
    keep = selection.keep_mask
    cu = torch.tensor([0, rows], dtype=torch.int32, device=keep.device)
    states = stream.active_states.contiguous()
    pos = stream.logical_positions.contiguous()
    res = compact_varlen(keep, cu, [states, pos], max_tokens=rows, check=True).trimmed()
    dropped = (keep == 0)
    if bool(dropped.any()):
        inv = (1 - keep).to(torch.uint8)
        park = compact_varlen(inv, cu, [states, pos], max_tokens=rows, check=True).trimmed()
        stream.parked_states.append(park.planes[0])
        stream.parked_positions.append(park.planes[1])
    stream.active_states = res.planes[0]
    stream.logical_positions = res.planes[1]
    history.events.append(DropEvent(layer, int(res.planes[1].numel()), res.planes[1]))


@dataclass
class PackedBatch:
    """PackedBatch (scheduler.hpp:33-46)."""

    tokens: torch.Tensor
    cu_seqlens: torch.Tensor       # int64 or int32 [R+1]
    phases: List[str]              # "prefill" / "decode"

    def num_requests(self) -> int:
        return len(self.phases)


def patch_metadata(batch: PackedBatch, selections: Sequence[Optional[Selection]], layer: int) -> None:
    """patch_metadata (scheduler.hpp:52-53, scheduler.cpp:50-90) through up_compact."""
    del layer
    R = batch.num_requests()
    if len(selections) != R:
        raise ContractViolation("patch_metadata: one selection slot per request required")
    cu_h = [int(x) for x in batch.cu_seqlens.tolist()]
    if len(cu_h) != R + 1 or cu_h[0] != 0:
        raise ContractViolation("PackedBatch: cu_seqlens must start at 0")
    if any(cu_h[i] <= cu_h[i - 1] for i in range(1, len(cu_h))):
        raise ContractViolation("PackedBatch: cu_seqlens must be strictly increasing")
    if cu_h[-1] != batch.tokens.shape[0]:
        raise ContractViolation("PackedBatch: cu_seqlens must end at the total token count")
    dev = batch.tokens.device
    T = cu_h[-1]
    keep = torch.ones(T, dtype=torch.uint8, device=dev)
    enabled = torch.zeros(R, dtype=torch.uint8, device=dev)
    for s, sel in enumerate(selections):
        if sel is None:
            continue
        if batch.phases[s] != "prefill":
            raise ContractViolation("patch_metadata: drops apply only to prefill segments")
        if sel.num_tokens() != cu_h[s + 1] - cu_h[s]:
            raise ContractViolation("patch_metadata: selection length disagrees with segment")
        keep[cu_h[s]:cu_h[s + 1]] = sel.keep_mask.to(dev)
        enabled[s] = 1
    res = compact_varlen(keep, batch.cu_seqlens, [batch.tokens.contiguous()], drop_enabled=enabled,
                         max_tokens=T, check=True).trimmed()
    batch.tokens = res.planes[0]
    batch.cu_seqlens = res.cu_seqlens.to(torch.int64)
