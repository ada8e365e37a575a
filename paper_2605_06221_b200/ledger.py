"""Per-layer metadata snapshots and the FLOPs ledger of dropped work.

Host-side bookkeeping around the device path -- what the reference's engine records per
layer (``LayerMeta``, scheduler.hpp:25-30, snapshot scheduler.cpp:284-289) and the analytic
FLOPs accounting that audits the savings of token dropping (flops.hpp / flops.cpp:14-144):

* ``layer_meta`` reads the device-resident ``cu_seqlens`` a drop produced into a LayerMeta;
* ``layer_flops`` / ``scoring_flops`` / ``FlopsLedger`` / ``validate_savings`` restate the
  reference's integer formulas (uint64 arithmetic, the same telescoping drop-history replay)
  and are checked against the reference build in ``tests/test_ledger.py``.
"""
from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field
from typing import List, Sequence

_U64 = (1 << 64) - 1


class SublayerKind(enum.IntEnum):
    """SublayerKind (config.hpp:15-20)."""

    FullAttention = 0
    SlidingWindowAttention = 1
    LinearAttention = 2
    FFN = 3


@dataclass
class ModelConfig:
    """The ModelConfig fields the ledger reads (config.hpp:28-48)."""

    num_blocks: int
    sublayers_per_block: int
    layer_pattern: Sequence[SublayerKind]
    hidden_dim: int
    head_dim: int
    num_heads: int
    window_size: int
    ffn_dim: int

    def pattern_length(self) -> int:
        return 1 + self.sublayers_per_block

    def total_layers(self) -> int:
        return self.num_blocks * self.pattern_length()

    def kind(self, layer: int) -> SublayerKind:
        return SublayerKind(self.layer_pattern[layer % self.pattern_length()])


class ContractViolation(RuntimeError):
    """Reference ContractViolation (errors.hpp:22-25)."""


def layer_flops(kind: SublayerKind, tokens: int, cfg: ModelConfig) -> int:
    """layer_flops (flops.cpp:14-33): exact integer cost of one sublayer at a token count."""
    if tokens < 0:
        raise ContractViolation("layer_flops: negative token count")
    if tokens == 0:
        return 0
    n, d, dk, h = tokens, cfg.hidden_dim, cfg.head_dim, cfg.num_heads
    proj = 8 * n * d * d
    if kind == SublayerKind.FullAttention:
        f = 2 * n * n * dk * h + proj
    elif kind == SublayerKind.SlidingWindowAttention:
        f = 2 * n * min(n, cfg.window_size) * dk * h + proj
    elif kind == SublayerKind.LinearAttention:
        f = 2 * n * dk * dk * h + proj
    else:
        f = 4 * n * d * cfg.ffn_dim
    return f & _U64


def scoring_flops(effective_n: int, num_keys: int, cfg: ModelConfig) -> int:
    """scoring_flops (flops.cpp:35-39): 2 n_eff N d_k H (H = query heads)."""
    if effective_n < 0 or num_keys < 0:
        raise ContractViolation("scoring_flops: negative count")
    return (2 * effective_n * num_keys * cfg.head_dim * cfg.num_heads) & _U64


@dataclass
class LayerFlopsEntry:
    layer: int
    kind: SublayerKind
    tokens: int
    flops: int


@dataclass
class DropRecord:
    """DropRecord (flops.hpp:33-39)."""

    layer: int
    tokens_before: int
    tokens_after: int
    retention_ratio: float = 1.0
    covered_mass: float = 1.0


@dataclass
class FlopsLedger:
    """FlopsLedger (flops.hpp:44-60): layers charged at the token count they entered with."""

    entries: List[LayerFlopsEntry] = field(default_factory=list)
    drops: List[DropRecord] = field(default_factory=list)
    scoring_overhead: int = 0

    def add_layer(self, layer: int, kind: SublayerKind, tokens: int, cfg: ModelConfig) -> None:
        self.entries.append(LayerFlopsEntry(layer, kind, tokens, layer_flops(kind, tokens, cfg)))

    def add_drop(self, record: DropRecord) -> None:
        self.drops.append(record)

    def add_scoring(self, flops: int) -> None:
        self.scoring_overhead = (self.scoring_overhead + flops) & _U64

    def merge(self, other: "FlopsLedger") -> None:
        """FlopsLedger::merge (flops.cpp:47-51)."""
        self.entries.extend(other.entries)
        self.drops.extend(other.drops)
        self.scoring_overhead = (self.scoring_overhead + other.scoring_overhead) & _U64

    def total(self) -> int:
        return sum(e.flops for e in self.entries) & _U64


@dataclass
class SavingsReport:
    """SavingsReport (flops.hpp:62-78)."""

    dense_total: int = 0
    accel_total: int = 0
    scoring_overhead: int = 0
    measured_delta: int = 0
    formula_delta: int = 0
    exact_match: bool = False
    single_drop: bool = False
    retention_ratio: float = 1.0
    drop_layer: int = -1
    layers_after_drop: int = 0
    closed_linear_form: int = 0
    linear_form_exact: bool = False
    attention_only_ratio: float = 0.0

    def to_text(self) -> str:
        """SavingsReport::to_text (flops.cpp:146-159)."""
        t = (f"dense={self.dense_total} accel={self.accel_total} scoring_overhead={self.scoring_overhead} "
             f"delta={self.measured_delta} formula={self.formula_delta}"
             + (" [exact]" if self.exact_match else " [MISMATCH]"))
        if self.single_drop:
            t += (f" single_drop{{layer={self.drop_layer} rho={self.retention_ratio:g} "
                  f"downstream_layers={self.layers_after_drop} linear_form={self.closed_linear_form}"
                  + (" exact" if self.linear_form_exact else " approx")
                  + f" attention_only_ratio={self.attention_only_ratio:g}}}")
        return t


def validate_savings(dense: FlopsLedger, accel: FlopsLedger, cfg: ModelConfig) -> SavingsReport:
    """validate_savings (flops.cpp:58-144): replay the drop history against the accelerated
    ledger and cross-check the measured saving against the telescoping formula."""
    total_layers = cfg.total_layers()
    if len(dense.entries) != total_layers or len(accel.entries) != total_layers:
        raise ContractViolation("validate_savings: ledgers must cover every layer exactly once")
    if dense.drops:
        raise ContractViolation("validate_savings: dense ledger must not contain drop events")
    original = dense.entries[0].tokens
    for l in range(total_layers):
        de, ae = dense.entries[l], accel.entries[l]
        if de.layer != l or ae.layer != l or de.kind != ae.kind or de.tokens != original:
            raise ContractViolation("validate_savings: mismatched run identities")
    pattern = cfg.pattern_length()
    nxt = 0
    current = original
    for l in range(total_layers):
        if accel.entries[l].tokens != current:
            raise ContractViolation("validate_savings: per-layer token counts disagree with history")
        if nxt < len(accel.drops) and accel.drops[nxt].layer == l:
            d = accel.drops[nxt]
            if d.tokens_before != current:
                raise ContractViolation("validate_savings: drop record inconsistent with stream")
            current = d.tokens_after
            nxt += 1
        if (l + 1) % pattern == 0:
            current = original  # reconstitution boundary
    if nxt != len(accel.drops):
        raise ContractViolation("validate_savings: drop layers out of order")
    rep = SavingsReport()
    rep.dense_total = dense.total()
    rep.accel_total = accel.total()
    rep.scoring_overhead = accel.scoring_overhead
    rep.measured_delta = (rep.dense_total - rep.accel_total) & _U64
    formula = 0
    for d in accel.drops:
        sweep_end = (d.layer // pattern + 1) * pattern - 1
        for l in range(d.layer + 1, sweep_end + 1):
            kind = dense.entries[l].kind
            formula += layer_flops(kind, d.tokens_before, cfg) - layer_flops(kind, d.tokens_after, cfg)
    rep.formula_delta = formula & _U64
    rep.exact_match = rep.formula_delta == rep.measured_delta
    if len(accel.drops) == 1:
        d = accel.drops[0]
        rep.single_drop = True
        rep.retention_ratio = d.retention_ratio
        rep.drop_layer = d.layer
        sweep_end = (d.layer // pattern + 1) * pattern - 1
        rep.layers_after_drop = sweep_end - d.layer
        downstream = 0
        for l in range(d.layer + 1, sweep_end + 1):
            downstream += layer_flops(dense.entries[l].kind, d.tokens_before, cfg)
        x = (1.0 - d.retention_ratio) * float(downstream & _U64)
        r = int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))  # std::llround
        rep.closed_linear_form = r & _U64  # static_cast<uint64_t>
        rep.linear_form_exact = rep.closed_linear_form == rep.formula_delta
        n = float(original)
        rep.attention_only_ratio = (float(rep.layers_after_drop) * n * float(cfg.hidden_dim) *
                                    float(cfg.hidden_dim) / (n * n * float(cfg.head_dim)))
    return rep


@dataclass
class LayerMeta:
    """LayerMeta (scheduler.hpp:25-30): the attention metadata downstream layers read."""

    layer: int
    query_start_loc: List[int]
    seq_lens: List[int]
    num_actual_tokens: int


def layer_meta(layer: int, cu_seqlens) -> LayerMeta:
    """Snapshot a (device or host) cu_seqlens -- e.g. ``Compacted.cu_seqlens`` after a drop --
    into a LayerMeta (scheduler.cpp:284-289).  Reads the device array once."""
    cu = [int(x) for x in (cu_seqlens.tolist() if hasattr(cu_seqlens, "tolist") else cu_seqlens)]
    return LayerMeta(layer, cu, [cu[i + 1] - cu[i] for i in range(len(cu) - 1)], cu[-1] if cu else 0)


class BatchLedger:
    """Per-request FlopsLedgers and LayerMeta snapshots for a varlen batch, charged the way
    Engine::run_batch charges them (scheduler.cpp:283-310): every layer at the token count each
    request entered it with; at a drop layer also the scoring overhead
    (scoring_flops(min(n, rows), rows), propagation.cpp:186) and a DropRecord with the retained
    count the device path produced.  One device->host read of cu_seqlens per recorded layer."""

    def __init__(self, cfg: ModelConfig, query_window_n: int = 128):
        self.cfg = cfg
        self.query_window_n = query_window_n
        self.ledgers: List[FlopsLedger] = []
        self.layer_meta: List[LayerMeta] = []

    def record_layer(self, layer: int, cu_seqlens, cu_seqlens_out=None, covered_mass=None) -> LayerMeta:
        """Charge `layer` for the batch described by cu_seqlens (the rows each request entered
        with).  cu_seqlens_out (e.g. ``Compacted.cu_seqlens``) marks a drop at this layer."""
        meta = layer_meta(layer, cu_seqlens)
        self.layer_meta.append(meta)
        if not self.ledgers:
            self.ledgers = [FlopsLedger() for _ in meta.seq_lens]
        if len(self.ledgers) != len(meta.seq_lens):
            raise ContractViolation("BatchLedger: request count changed between layers")
        kind = self.cfg.kind(layer)
        for r, rows in enumerate(meta.seq_lens):
            self.ledgers[r].add_layer(layer, kind, rows, self.cfg)
        if cu_seqlens_out is not None:
            after = layer_meta(layer, cu_seqlens_out).seq_lens
            cm = [1.0] * len(after) if covered_mass is None else [float(x) for x in
                                                                   (covered_mass.tolist() if hasattr(covered_mass, "tolist") else covered_mass)]
            for r, (rows, kept) in enumerate(zip(meta.seq_lens, after)):
                if rows == 0:
                    continue
                self.ledgers[r].add_scoring(scoring_flops(min(self.query_window_n, rows), rows, self.cfg))
                self.ledgers[r].add_drop(DropRecord(layer, rows, kept, kept / rows, cm[r]))
        return meta
