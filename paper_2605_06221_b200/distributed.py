"""Multi-GPU plumbing for the hot path (one process per GPU, torch.distributed).

Two ways the path shards:

* request sharding -- requests are independent, so a varlen batch is
  split across ranks by longest-processing-time bin packing on N_r and each rank runs the
  whole score -> select -> compact path on its own sub-batch.  No collective on the data
  path (weak scaling);
* head sharding (TP) -- each rank scores a contiguous slice of q-heads
  (sharded_block_scores, tp_sim.cpp:12-27) and the per-block partials are summed across
  ranks before selection (Eq. 15).  ``allreduce_block_scores`` uses one
  NCCL all-reduce (sum) over NVLink; ``deterministic=True`` instead all-gathers the
  partials and sums them in ascending rank order with the sm_100a reduce kernel, which
  reproduces allreduce_scores (tp_sim.cpp:43-47) bit for bit.  ``PeerScoreReducer`` does
  the same bitwise reduction as ONE sm_100a kernel over peer memory (CUDA IPC-mapped
  exchange buffers on every rank, P2P stores over NVLink / NVSwitch + device flags):
  no NCCL call and no separate gather on the data path.
"""
from __future__ import annotations

import ctypes
from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist

from . import _capi
from .api import ContractViolation, ConfigError, _check, _stream_ptr, reduce_block_scores


def lpt_partition(lengths: Sequence[int], parts: int) -> List[List[int]]:
    """Longest-processing-time bin packing of request indices onto `parts` ranks (the
    per-request cost of every stage is linear in N_r)."""
    if parts < 1:
        raise ConfigError("parts must be positive")
    order = sorted(range(len(lengths)), key=lambda i: (-int(lengths[i]), i))
    bins: List[List[int]] = [[] for _ in range(parts)]
    loads = [0] * parts
    for i in order:
        b = min(range(parts), key=lambda x: (loads[x], x))
        bins[b].append(i)
        loads[b] += int(lengths[i])
    return [sorted(b) for b in bins]


def shard_requests(cu_seqlens: Sequence[int], rank: int, world: int):
    """The rank's requests (global indices) and its local cu_seqlens under LPT sharding."""
    cu = [int(x) for x in cu_seqlens]
    lengths = [cu[i + 1] - cu[i] for i in range(len(cu) - 1)]
    mine = lpt_partition(lengths, world)[rank]
    local = [0]
    for i in mine:
        local.append(local[-1] + lengths[i])
    return mine, local


def head_slice(num_q_heads: int, num_kv_heads: int, tp_rank: int, tp_size: int):
    """q-head range [begin, end) and kv-head range of one TP rank (tp_sim.cpp:18-24).
    When Hkv < TP (Qwen3-Next: Hkv=2, TP=8) each kv-head is replicated on TP/Hkv ranks."""
    if tp_size < 1 or num_q_heads % tp_size != 0:
        raise ConfigError("num_heads must be divisible by tp_degree")
    hps = num_q_heads // tp_size
    qb, qe = tp_rank * hps, (tp_rank + 1) * hps
    group = num_q_heads // num_kv_heads
    kb, ke = qb // group, (qe - 1) // group + 1
    return (qb, qe), (kb, ke)


class PeerScoreReducer:
    """TP all-reduce of partial block scores over peer memory (up_peer_allreduce_scores).

    Collective constructor: every rank of `group` allocates an exchange buffer for up to
    `capacity` block scores, the CUDA IPC handles are all-gathered over `group` (any
    backend) and the peers' buffers are mapped into this process.  A call then runs one
    kernel: P2P stores of this rank's partial into every peer, device flags, and the
    ascending-rank fp32 sum (bitwise allreduce_scores, tp_sim.cpp:43-47) on every rank.
    Every rank must make the same sequence of calls with the same element counts."""

    def __init__(self, capacity: int, group=None, device=None):
        if not dist.is_initialized():
            raise ContractViolation("PeerScoreReducer: torch.distributed is not initialized")
        self.lib = _capi.lib
        self.group = group
        self.rank = dist.get_rank(group)
        self.tp = dist.get_world_size(group)
        self.capacity = int(capacity)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        own = ctypes.c_void_p()
        _check(self.lib.up_peer_buffer_alloc(self.tp, self.capacity, ctypes.byref(own)), "peer_buffer_alloc")
        self._own = own
        handle = (ctypes.c_char * 64)()
        _check(self.lib.up_ipc_get_handle(own, handle), "ipc_get_handle")
        handles: list = [None] * self.tp
        dist.all_gather_object(handles, bytes(handle), group=group)
        ptrs, self._opened = [], []
        for t, h in enumerate(handles):
            if t == self.rank:
                ptrs.append(own.value)
                continue
            p = ctypes.c_void_p()
            _check(self.lib.up_ipc_open_handle(ctypes.create_string_buffer(h, 64), ctypes.byref(p)),
                   "ipc_open_handle")
            self._opened.append(p)
            ptrs.append(p.value)
        self.buffers = (ctypes.c_void_p * self.tp)(*ptrs)
        self.err = torch.zeros(64, dtype=torch.int32, device=self.device)
        dist.barrier(group)

    def __call__(self, partial: torch.Tensor, out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Reduced scores of `partial` (fp32, contiguous, numel <= capacity) into `out`
        (default: in place)."""
        if partial.dtype != torch.float32 or not partial.is_contiguous():
            raise ContractViolation("PeerScoreReducer: partial must be contiguous float32")
        out = partial if out is None else out
        _check(self.lib.up_peer_allreduce_scores(
            _stream_ptr(partial.device), ctypes.c_void_p(partial.data_ptr()), partial.numel(), self.rank, self.tp,
            self.buffers, self.capacity, ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(self.err.data_ptr()),
            self.err.numel() * 4), "peer_allreduce_scores")
        return out

    def score_blocks(self, q: torch.Tensor, k: torch.Tensor, cu_seqlens, config, heads, max_tokens=None,
                     workspace=None, out=None):
        """This rank's head slice scored and all-reduced across the group in the scorer's own
        launches (up_score_blocks_peer): the combine kernel stores each block's partial into
        the peers and writes the ascending-rank sum.  Returns api.BlockScores with the
        REDUCED block scores (identical on every rank)."""
        from . import api
        dev = q.device
        cu = api._as_i32_cuda(cu_seqlens, dev)
        R = cu.numel() - 1
        T = int(max_tokens if max_tokens is not None else q.shape[0])
        qv, qs, D = api._heads_view(q, heads.num_q_heads)
        kv, ks, _ = api._heads_view(k, heads.num_kv_heads)
        if D != heads.head_dim:
            raise ContractViolation("score_blocks: head dim mismatch")
        b = api._batch(cu, T, None)
        hc = heads.c(qs, ks)
        cfg = config.c()
        ws = workspace or api._ws(dev)
        buf = ws.get(b, hc, cfg)
        nbmax = int(self.lib.up_max_blocks(ctypes.byref(b), ctypes.byref(cfg)))
        if nbmax > self.capacity:
            raise ContractViolation(f"score_blocks: {nbmax} blocks exceed the reducer capacity {self.capacity}")
        if out is None:
            out = api.BlockScores(torch.empty(nbmax, dtype=torch.float32, device=dev),
                                  torch.empty(R + 1, dtype=torch.int32, device=dev), None)
        _check(self.lib.up_score_blocks_peer(
            _stream_ptr(dev), ctypes.byref(b), ctypes.byref(hc), ctypes.byref(cfg), api._ptr(qv), api._ptr(kv),
            self.rank, self.tp, self.buffers, self.capacity, api._ptr(out.block_scores), api._ptr(out.cu_blocks),
            ctypes.c_void_p(buf.data_ptr()), buf.numel()), "score_blocks_peer")
        return out

    def check(self) -> None:
        """Raise if a peer's partial never arrived (sticky device flag)."""
        _check(self.lib.up_device_status(_stream_ptr(self.device), ctypes.c_void_p(self.err.data_ptr())),
               "peer_allreduce_scores")

    def close(self) -> None:
        torch.cuda.synchronize(self.device)
        dist.barrier(self.group)  # no peer still writes into a buffer about to go away
        for p in self._opened:
            self.lib.up_ipc_close_handle(p)
        self._opened = []
        dist.barrier(self.group)
        if self._own is not None:
            self.lib.up_peer_buffer_free(self._own)
            self._own = None


def allreduce_block_scores(partial: torch.Tensor, group=None, deterministic: bool = False,
                           reducer: Optional[Callable[[List[torch.Tensor]], torch.Tensor]] = None,
                           peer: Optional[PeerScoreReducer] = None) -> torch.Tensor:
    """Sum per-rank partial block scores across the TP group, in place (returns `partial`).

    deterministic=False: one all-reduce (NCCL sum over NVLink).
    deterministic=True : all-gather + ascending-rank fp32 sum (bitwise allreduce_scores).
    `reducer` overrides the ordered summation (tests pass the CPU oracle on gloo).
    `peer`: the one-kernel peer-memory reduction (bitwise, like deterministic=True)."""
    if peer is not None:
        return peer(partial)
    if not dist.is_initialized():
        raise ContractViolation("allreduce_block_scores: torch.distributed is not initialized")
    if not deterministic:
        dist.all_reduce(partial, op=dist.ReduceOp.SUM, group=group)
        return partial
    world = dist.get_world_size(group)
    shards = [torch.empty_like(partial) for _ in range(world)]
    dist.all_gather(shards, partial.contiguous(), group=group)
    # shards[t] is the partial of group rank t: the ascending order of tp_sim.cpp:43-47.
    if reducer is not None:
        out = reducer(shards)
    else:
        out = reduce_block_scores(shards)
    partial.copy_(out)
    return partial
