"""B200-native UniPrefill token-selection hot path (score -> top-p keep mask -> compact).

The compute lives in hand-written sm_100a kernels behind the C ABI in
``include/uniprefill_b200.h`` (``_lib/libuniprefill_b200.so``); this package is the host-side
mirror of the reference's operator API (see ``api.py``).
"""
from .api import (AllocationMissError, attention_varlen, BlockScores, Compacted, ConfigError, ContractViolation, CudaError, DropEvent,
                  DropHistory, DropLayer, HeadLayout, ImportanceScores, PackedBatch, ScoreConfig,
                  Selection, ShardedBlockScores, ShardScores, TokenStream, UnsupportedError, VarlenSelection, Workspace,
                  allreduce_scores, apply_drop, compact_varlen, patch_metadata, reconstitute, reconstitute_varlen,
                  reduce_block_scores, scatter_rows, slot_mapping, decode_seqused,
                  score_blocks_tp, score_blocks_varlen, score_tokens, score_tokens_heads, select_varlen,
                  sharded_block_scores, top_p_select)
from ._capi import LIB_PATH, lib
from .ledger import (BatchLedger, DropRecord, FlopsLedger, LayerMeta, ModelConfig, SavingsReport, SublayerKind,
                     layer_flops, layer_meta, scoring_flops, validate_savings)

__all__ = [
    "AllocationMissError", "attention_varlen", "BlockScores", "Compacted", "ConfigError", "ContractViolation", "CudaError", "DropEvent",
    "DropHistory", "DropLayer", "HeadLayout", "ImportanceScores", "PackedBatch", "ScoreConfig",
    "Selection", "ShardedBlockScores", "ShardScores", "TokenStream", "UnsupportedError", "VarlenSelection", "Workspace",
    "allreduce_scores", "apply_drop", "compact_varlen", "patch_metadata", "reconstitute",
    "reconstitute_varlen", "reduce_block_scores", "scatter_rows", "slot_mapping", "decode_seqused",
    "score_blocks_tp", "score_blocks_varlen", "score_tokens", "score_tokens_heads", "select_varlen",
    "sharded_block_scores", "top_p_select", "LIB_PATH", "lib",
    "BatchLedger", "DropRecord", "FlopsLedger", "LayerMeta", "ModelConfig", "SavingsReport", "SublayerKind",
    "layer_flops", "layer_meta", "scoring_flops", "validate_savings",
]
