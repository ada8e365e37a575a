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
  reproduces allreduce_scores (tp_sim.cpp:43-47) bit for bit.
"""
from __future__ import annotations

from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist

from .api import ContractViolation, ConfigError, reduce_block_scores


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


def allreduce_block_scores(partial: torch.Tensor, group=None, deterministic: bool = False,
                           reducer: Optional[Callable[[List[torch.Tensor]], torch.Tensor]] = None
                           ) -> torch.Tensor:
    """Sum per-rank partial block scores across the TP group, in place (returns `partial`).

    deterministic=False: one all-reduce (NCCL sum over NVLink).
    deterministic=True : all-gather + ascending-rank fp32 sum (bitwise allreduce_scores).
    `reducer` overrides the ordered summation (tests pass the CPU oracle on gloo)."""
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
