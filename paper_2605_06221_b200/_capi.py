"""ctypes binding of the C ABI declared in ``include/uniprefill_b200.h``.

Loads the in-tree ``_lib/libuniprefill_b200.so``.  There is deliberately no fallback: if the
library is missing or fails to load, importing this module raises, and every API call
fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libuniprefill_b200.so")

# Symbols the header declares (checked by tests/test_capi_symbols.py).
EXPORTED = (
    "up_abi_version", "up_status_string", "up_config_validate", "up_max_blocks",
    "up_workspace_bytes", "up_score_blocks", "up_score_blocks_tp", "up_reduce_block_scores", "up_select",
    "up_compact", "up_compact_selected", "up_scatter_rows", "up_slot_mapping", "up_decode_seqused", "up_drop_layer", "up_attention_varlen", "up_peer_buffer_bytes", "up_peer_buffer_alloc",
    "up_peer_buffer_free", "up_ipc_get_handle", "up_ipc_open_handle", "up_ipc_close_handle",
    "up_peer_allreduce_scores", "up_score_blocks_peer", "up_device_status", "up_scorer_kind", "up_last_launch_count",
)

UP_OK, UP_ERR_CONFIG, UP_ERR_CONTRACT, UP_ERR_UNSUPPORTED, UP_ERR_WORKSPACE, UP_ERR_CUDA, \
    UP_ERR_INVALID_ARGUMENT, UP_ERR_ALLOCATION_MISS = range(8)


class ScoreConfigC(ctypes.Structure):
    _fields_ = [("query_window_n", ctypes.c_int32), ("block_size_g", ctypes.c_int32),
                ("sink_count_a", ctypes.c_int32), ("top_p", ctypes.c_float)]


class BatchC(ctypes.Structure):
    _fields_ = [("num_requests", ctypes.c_int32), ("max_tokens", ctypes.c_int64),
                ("cu_seqlens", ctypes.c_void_p), ("drop_enabled", ctypes.c_void_p)]


class HeadsC(ctypes.Structure):
    _fields_ = [("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("gqa_group", ctypes.c_int32),
                ("q_head_offset", ctypes.c_int32), ("kv_head_offset", ctypes.c_int32),
                ("q_row_stride", ctypes.c_int64), ("k_row_stride", ctypes.c_int64)]


class PlaneC(ctypes.Structure):
    _fields_ = [("src", ctypes.c_void_p), ("dst", ctypes.c_void_p), ("row_bytes", ctypes.c_int64),
                ("src_stride_bytes", ctypes.c_int64), ("dst_stride_bytes", ctypes.c_int64)]


class SelectionOutC(ctypes.Structure):
    _fields_ = [("cutoff_rank", ctypes.c_void_p), ("retained_count", ctypes.c_void_p),
                ("covered_mass", ctypes.c_void_p), ("degenerate", ctypes.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2605_06221_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    sig = {
        "up_abi_version": ([], ctypes.c_int),
        "up_status_string": ([ctypes.c_int], ctypes.c_char_p),
        "up_config_validate": ([P(ScoreConfigC)], ctypes.c_int),
        "up_max_blocks": ([P(BatchC), P(ScoreConfigC)], i64),
        "up_workspace_bytes": ([P(BatchC), P(HeadsC), P(ScoreConfigC)], sz),
        "up_score_blocks": ([vp, P(BatchC), P(HeadsC), P(ScoreConfigC), vp, vp, vp, vp, vp, vp, sz],
                            ctypes.c_int),
        "up_score_blocks_tp": ([vp, P(BatchC), P(HeadsC), P(ScoreConfigC), vp, vp, i32, vp, i64, vp, vp, vp,
                                sz], ctypes.c_int),
        "up_reduce_block_scores": ([vp, P(vp), i32, i64, vp], ctypes.c_int),
        "up_select": ([vp, P(BatchC), P(ScoreConfigC), vp, vp, vp, vp, P(SelectionOutC), vp, sz],
                      ctypes.c_int),
        "up_compact": ([vp, P(BatchC), vp, P(PlaneC), i32, vp, vp, vp, vp, sz], ctypes.c_int),
        "up_compact_selected": ([vp, P(BatchC), vp, P(PlaneC), i32, vp, vp, vp, vp, sz], ctypes.c_int),
        "up_scatter_rows": ([vp, vp, vp, i64, P(PlaneC), i32], ctypes.c_int),
        "up_slot_mapping": ([vp, vp, i32, vp, i64, vp, vp, i32, i32, i32, vp, i64, vp, sz], ctypes.c_int),
        "up_decode_seqused": ([vp, i32, i32, vp, i32, P(i32), P(vp), vp, vp], ctypes.c_int),
        "up_drop_layer": ([vp, P(BatchC), P(HeadsC), P(ScoreConfigC), vp, vp, vp, vp, vp, vp,
                           P(SelectionOutC), P(PlaneC), i32, vp, vp, vp, vp, sz], ctypes.c_int),
        "up_attention_varlen": ([vp, P(BatchC), P(HeadsC), vp, vp, vp, vp, i64, vp, i64, vp, sz], ctypes.c_int),
        "up_peer_buffer_bytes": ([i32, i64], sz),
        "up_peer_buffer_alloc": ([i32, i64, P(vp)], ctypes.c_int),
        "up_peer_buffer_free": ([vp], ctypes.c_int),
        "up_ipc_get_handle": ([vp, vp], ctypes.c_int),
        "up_ipc_open_handle": ([vp, P(vp)], ctypes.c_int),
        "up_ipc_close_handle": ([vp], ctypes.c_int),
        "up_peer_allreduce_scores": ([vp, vp, i64, i32, i32, P(vp), i64, vp, vp, sz], ctypes.c_int),
        "up_score_blocks_peer": ([vp, P(BatchC), P(HeadsC), P(ScoreConfigC), vp, vp, i32, i32, P(vp), i64, vp, vp,
                                  vp, sz], ctypes.c_int),
        "up_device_status": ([vp, vp], ctypes.c_int),
        "up_scorer_kind": ([P(HeadsC), P(ScoreConfigC), ctypes.c_int], ctypes.c_int),
        "up_last_launch_count": ([], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def status_string(code: int) -> str:
    return lib.up_status_string(code).decode()
