"""CPU: the C-ABI library loads, exports every symbol include/uniprefill_b200.h declares,
and its host-side validation (no device work) behaves like the reference's exceptions."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "uniprefill_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(up_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2605_06221_b200 import _capi
    lib = ctypes.CDLL(_capi.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 13
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_capi.EXPORTED) == set(syms)


def test_abi_version_and_status_strings():
    from paper_2605_06221_b200._capi import lib, status_string
    assert lib.up_abi_version() == 3
    assert status_string(0) == "ok"
    assert "ConfigError" in status_string(1)
    assert "ContractViolation" in status_string(2)


def test_config_validation_maps_to_config_error():
    import paper_2605_06221_b200 as up
    up.ScoreConfig().validate()
    for bad in (dict(top_p=0.0), dict(top_p=1.01), dict(query_window_n=0), dict(block_size_g=0),
                dict(sink_count_a=-1)):
        with pytest.raises(up.ConfigError):
            up.ScoreConfig(**bad).validate()
    up.ScoreConfig(top_p=1.0).validate()  # p = 1 is allowed (config.cpp:102)


def test_workspace_and_block_bounds():
    from paper_2605_06221_b200._capi import BatchC, HeadsC, ScoreConfigC, lib
    b = BatchC(4, 131072, None, None)
    c = ScoreConfigC(128, 64, 128, 0.99)
    h = HeadsC(32, 8, 128, 4, 0, 0, 4096, 1024)
    assert lib.up_max_blocks(ctypes.byref(b), ctypes.byref(c)) == 131072 // 64 + 4 + 1
    ws = lib.up_workspace_bytes(ctypes.byref(b), ctypes.byref(h), ctypes.byref(c))
    assert ws > 32 * 2048 * 128 * 4  # P: [Hq][blocks][128] fp32
    assert ws % 256 == 0
    # bigger batches need more workspace
    b2 = BatchC(4, 262144, None, None)
    assert lib.up_workspace_bytes(ctypes.byref(b2), ctypes.byref(h), ctypes.byref(c)) > ws


def test_scorer_dispatch():
    from paper_2605_06221_b200._capi import HeadsC, ScoreConfigC, lib
    c = ScoreConfigC(128, 64, 128, 0.99)
    for D in (64, 128, 256):
        h = HeadsC(8, 2, D, 4, 0, 0, 8 * D, 2 * D)
        assert lib.up_scorer_kind(ctypes.byref(h), ctypes.byref(c), 0) == 1   # tcgen05 kernel
        assert lib.up_scorer_kind(ctypes.byref(h), ctypes.byref(c), 1) == 2   # token scores -> SIMT
    h = HeadsC(8, 8, 8, 1, 0, 0, 64, 64)
    assert lib.up_scorer_kind(ctypes.byref(h), ctypes.byref(ScoreConfigC(16, 8, 8, 0.9)), 0) == 2
    h = HeadsC(8, 2, 128, 4, 0, 0, 1024, 256)
    # n > 128: query tiles on the tensor cores up to 1024 rows (8 tiles), SIMT beyond
    assert lib.up_scorer_kind(ctypes.byref(h), ctypes.byref(ScoreConfigC(256, 64, 8, 0.9)), 0) == 1
    assert lib.up_scorer_kind(ctypes.byref(h), ctypes.byref(ScoreConfigC(1024, 64, 8, 0.9)), 0) == 1
    assert lib.up_scorer_kind(ctypes.byref(h), ctypes.byref(ScoreConfigC(1025, 64, 8, 0.9)), 0) == 2


def test_entry_points_reject_bad_arguments_before_device_work():
    from paper_2605_06221_b200._capi import (BatchC, HeadsC, ScoreConfigC, SelectionOutC,
                                             UP_ERR_CONFIG, UP_ERR_CONTRACT, UP_ERR_INVALID_ARGUMENT,
                                             UP_ERR_WORKSPACE, lib)
    fake = ctypes.c_void_p(0x1000)  # never dereferenced: validation fails first
    good_cfg = ScoreConfigC(128, 64, 128, 0.99)
    bad_cfg = ScoreConfigC(128, 64, 128, 0.0)
    b = BatchC(2, 1024, fake, None)
    h = HeadsC(8, 2, 128, 4, 0, 0, 1024, 256)
    st = lib.up_score_blocks(None, ctypes.byref(b), ctypes.byref(h), ctypes.byref(bad_cfg), fake, fake,
                             fake, fake, None, fake, 1 << 40)
    assert st == UP_ERR_CONFIG
    st = lib.up_score_blocks(None, ctypes.byref(b), ctypes.byref(h), ctypes.byref(good_cfg), fake, fake,
                             fake, fake, None, fake, 16)
    assert st == UP_ERR_WORKSPACE
    bad_heads = HeadsC(8, 1, 128, 4, 0, 0, 1024, 128)  # q-heads 4..7 map to a missing kv-head
    st = lib.up_score_blocks(None, ctypes.byref(b), ctypes.byref(bad_heads), ctypes.byref(good_cfg), fake,
                             fake, fake, fake, None, fake, 1 << 40)
    assert st == UP_ERR_CONTRACT
    st = lib.up_score_blocks(None, ctypes.byref(b), ctypes.byref(h), ctypes.byref(good_cfg), None, fake,
                             fake, fake, None, fake, 1 << 40)
    assert st == UP_ERR_INVALID_ARGUMENT
    out = SelectionOutC(None, None, None, None)
    st = lib.up_select(None, ctypes.byref(b), ctypes.byref(good_cfg), fake, fake, None, fake,
                       ctypes.byref(out), fake, 1 << 40)
    assert st == UP_ERR_INVALID_ARGUMENT
    st = lib.up_reduce_block_scores(None, (ctypes.c_void_p * 1)(fake), 0, 4, fake)
    assert st == UP_ERR_CONTRACT


def test_api_mirror_host_errors():
    import paper_2605_06221_b200 as up
    with pytest.raises(up.ConfigError):
        up.sharded_block_scores(None, None, 8, up.ScoreConfig(), 3)
    with pytest.raises(up.ConfigError):
        up.sharded_block_scores(None, None, 8, up.ScoreConfig(), 0)
    with pytest.raises(up.ContractViolation):
        up.allreduce_scores([])
    import torch
    z = torch.zeros(2)
    with pytest.raises(up.ContractViolation):
        up.allreduce_scores([up.ShardScores(0, z), up.ShardScores(0, z)])
    with pytest.raises(up.ContractViolation):
        up.allreduce_scores([up.ShardScores(0, z), up.ShardScores(2, z)])
    with pytest.raises(up.ContractViolation):
        up.allreduce_scores([up.ShardScores(0, z), up.ShardScores(1, torch.zeros(3))])


def test_product_path_has_no_oracle_dependency():
    """The package must never import the test oracle (no CPU fallback)."""
    pkg = os.path.join(ROOT, "paper_2605_06221_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "uniprefill_oracle" not in text, f
