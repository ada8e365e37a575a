"""Deterministic synthetic activations at real model shapes (data plumbing, not the product).

There is no network for checkpoints, so the benchmark and tests use random-init bf16
activations with the named models' head layouts.  Two regimes:

* ``iid``: q, k ~ N(0, 1) -- gives retention rho ~ 1.0 (worst case for compaction bytes);
* ``planted``: a unit-variance direction m per kv-head is added (times gamma) to every query
  row and to every key row of the "hot" blocks (block g hot with probability ``frac``),
  mirroring the reference's low-entropy prompts (report.cpp:108-129); gamma=0.8, frac=0.25
  gives rho ~ 0.28 at G=64.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

# Layer shapes named in BASELINE.json (public HF configs).
MODEL_SHAPES = {
    "llama3.1-8b": dict(num_q_heads=32, num_kv_heads=8, head_dim=128, hidden=4096),
    "qwen3-next-80b-a3b": dict(num_q_heads=16, num_kv_heads=2, head_dim=256, hidden=2048),
    "gemma3-12b": dict(num_q_heads=16, num_kv_heads=8, head_dim=256, hidden=3840),
}


@dataclass
class SyntheticBatch:
    q: torch.Tensor          # bf16 [T, Hq, D]
    k: torch.Tensor          # bf16 [T, Hkv, D]
    v: torch.Tensor          # bf16 [T, Hkv, D]
    hidden: torch.Tensor     # bf16 [T, hidden]
    positions: torch.Tensor  # int64 [T] (0..N_r-1 per request)
    cu_seqlens: torch.Tensor  # int32 [R+1]
    lengths: List[int]


def make_batch(lengths: Sequence[int], num_q_heads: int, num_kv_heads: int, head_dim: int,
               hidden: int, regime: str = "planted", gamma: float = 0.8, frac: float = 0.25,
               block_size_g: int = 64, seed: int = 0, device="cuda", with_v: bool = True,
               with_hidden: bool = True) -> SyntheticBatch:
    dev = torch.device(device)
    lengths = [int(x) for x in lengths]
    T = sum(lengths)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    group = num_q_heads // num_kv_heads

    def randn(*shape):
        return torch.randn(*shape, generator=gen, device=dev, dtype=torch.float32)

    q = randn(T, num_q_heads, head_dim)
    k = randn(T, num_kv_heads, head_dim)
    if regime == "planted":
        m = randn(num_kv_heads, head_dim)
        q += gamma * m.repeat_interleave(group, dim=0)[None]
        hot = torch.zeros(T, dtype=torch.bool, device=dev)
        start = 0
        for n in lengths:
            nb = (n + block_size_g - 1) // block_size_g
            hb = torch.rand(nb, generator=gen, device=dev) < frac
            hot[start:start + n] = hb.repeat_interleave(block_size_g)[:n]
            start += n
        k += gamma * m[None] * hot[:, None, None].float()
    elif regime != "iid":
        raise ValueError(regime)
    cu = torch.zeros(len(lengths) + 1, dtype=torch.int32)
    cu[1:] = torch.cumsum(torch.tensor(lengths, dtype=torch.int64), 0).to(torch.int32)
    pos = torch.cat([torch.arange(n, dtype=torch.int64) for n in lengths]).to(dev)
    v = randn(T, num_kv_heads, head_dim).to(torch.bfloat16) if with_v else None
    h = randn(T, hidden).to(torch.bfloat16) if with_hidden else None
    return SyntheticBatch(q.to(torch.bfloat16), k.to(torch.bfloat16), v, h, pos, cu.to(dev), lengths)


def loguniform_lengths(count: int, lo: int, hi: int, seed: int) -> List[int]:
    """Request lengths ~ log-uniform[lo, hi] (BASELINE config 5)."""
    g = torch.Generator().manual_seed(seed)
    u = torch.rand(count, generator=g, dtype=torch.float64)
    import math
    return [int(round(math.exp(math.log(lo) + float(x) * (math.log(hi) - math.log(lo))))) for x in u]


def lpt_partition(lengths: Sequence[int], parts: int) -> List[List[int]]:
    """Longest-processing-time bin packing of request indices onto `parts` GPUs."""
    order = sorted(range(len(lengths)), key=lambda i: -lengths[i])
    bins: List[List[int]] = [[] for _ in range(parts)]
    loads = [0] * parts
    for i in order:
        b = loads.index(min(loads))
        bins[b].append(i)
        loads[b] += lengths[i]
    return [sorted(b) for b in bins]
