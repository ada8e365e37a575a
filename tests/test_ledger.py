"""CPU: the FLOPs ledger and LayerMeta mirror (paper_2605_06221_b200/ledger.py) against the
unmodified reference (flops.cpp:14-144 through oracle/_ref), plus the reference's own
known answers for the formulas (flops.hpp:14-19)."""
import random

import pytest

from paper_2605_06221_b200 import ledger as L
from paper_2605_06221_b200.ledger import SublayerKind as K

import oracle

U64 = (1 << 64) - 1


def _cfg(rng):
    spb = rng.randint(1, 4)
    pattern = [K.FullAttention] + [K(rng.randint(0, 3)) for _ in range(spb)]
    return L.ModelConfig(num_blocks=rng.randint(1, 4), sublayers_per_block=spb, layer_pattern=pattern,
                         hidden_dim=rng.choice([64, 512, 4096]), head_dim=rng.choice([8, 64, 128]),
                         num_heads=rng.choice([4, 8, 32]), window_size=rng.choice([16, 4096]),
                         ffn_dim=rng.choice([128, 14336]))


def _history(cfg, rng, original, max_drops):
    """A drop history the reference engine could produce: drops at random layers, each
    keeping a random prefix count of the rows that entered, reset at every block boundary."""
    tokens, drops, cur = [], [], original
    pattern = cfg.pattern_length()
    for l in range(cfg.total_layers()):
        tokens.append(cur)
        if len(drops) < max_drops and rng.random() < 0.4:
            after = rng.randint(0, cur)
            drops.append((l, cur, after, after / cur if cur else 1.0))
            cur = after
        if (l + 1) % pattern == 0:
            cur = original
    return tokens, drops


def _ledgers(cfg, original, tokens, drops, scoring):
    dense, accel = L.FlopsLedger(), L.FlopsLedger()
    for l in range(cfg.total_layers()):
        dense.add_layer(l, cfg.kind(l), original, cfg)
        accel.add_layer(l, cfg.kind(l), tokens[l], cfg)
    for d in drops:
        accel.add_drop(L.DropRecord(*d))
    accel.add_scoring(scoring)
    return dense, accel


def test_known_answers():
    cfg = L.ModelConfig(2, 3, [K.FullAttention, K.SlidingWindowAttention, K.LinearAttention, K.FFN],
                        hidden_dim=64, head_dim=8, num_heads=8, window_size=16, ffn_dim=128)
    n = 100
    proj = 8 * n * 64 * 64
    assert L.layer_flops(K.FullAttention, n, cfg) == 2 * n * n * 8 * 8 + proj
    assert L.layer_flops(K.SlidingWindowAttention, n, cfg) == 2 * n * 16 * 8 * 8 + proj
    assert L.layer_flops(K.LinearAttention, n, cfg) == 2 * n * 8 * 8 * 8 + proj
    assert L.layer_flops(K.FFN, n, cfg) == 4 * n * 64 * 128
    assert L.layer_flops(K.FullAttention, 0, cfg) == 0
    assert L.scoring_flops(128, n, cfg) == 2 * 128 * n * 8 * 8
    with pytest.raises(L.ContractViolation):
        L.layer_flops(K.FFN, -1, cfg)
    # one drop at layer 0 keeping 25 of 100 rows: the three downstream sublayers of block 0
    dense, accel = _ledgers(cfg, n, [100, 25, 25, 25, 100, 100, 100, 100], [(0, 100, 25, 0.25)], 0)
    rep = L.validate_savings(dense, accel, cfg)
    assert rep.exact_match and rep.single_drop and rep.layers_after_drop == 3
    assert rep.measured_delta == sum(L.layer_flops(k, 100, cfg) - L.layer_flops(k, 25, cfg)
                                     for k in (K.SlidingWindowAttention, K.LinearAttention, K.FFN))
    assert "[exact]" in rep.to_text()


def test_contract_violations():
    cfg = L.ModelConfig(1, 1, [K.FullAttention, K.FFN], 64, 8, 8, 16, 128)
    dense, accel = _ledgers(cfg, 10, [10, 7], [], 0)  # counts disagree with the (empty) history
    with pytest.raises(L.ContractViolation):
        L.validate_savings(dense, accel, cfg)
    dense, accel = _ledgers(cfg, 10, [10, 5], [(0, 9, 5, 0.5)], 0)  # record inconsistent with stream
    with pytest.raises(L.ContractViolation):
        L.validate_savings(dense, accel, cfg)
    dense, accel = _ledgers(cfg, 10, [10, 10], [], 0)
    accel.entries.pop()  # a ledger missing a layer
    with pytest.raises(L.ContractViolation):
        L.validate_savings(dense, accel, cfg)


def test_layer_flops_match_reference(ref):
    rng = random.Random(7)
    for _ in range(300):
        cfg = _cfg(rng)
        kind = K(rng.randint(0, 3))
        n = rng.choice([0, 1, rng.randint(1, 1 << 20), rng.randint(1 << 30, 1 << 33)])  # last wraps uint64
        assert L.layer_flops(kind, n, cfg) == ref.layer_flops(kind, n, cfg)
        ne, nk = rng.randint(0, 256), rng.randint(0, 1 << 24)
        assert L.scoring_flops(ne, nk, cfg) == ref.scoring_flops(ne, nk, cfg)
    with pytest.raises(oracle.OracleContractViolation):
        ref.layer_flops(int(K.FFN), -1, cfg)


@pytest.mark.parametrize("seed", range(40))
def test_validate_savings_matches_reference(ref, seed):
    rng = random.Random(seed)
    cfg = _cfg(rng)
    original = rng.choice([1, 64, 1000, 32768, 1 << 20])
    tokens, drops = _history(cfg, rng, original, max_drops=1 if seed % 3 == 0 else 8)
    scoring = rng.randint(0, 1 << 40)
    rep = L.validate_savings(*_ledgers(cfg, original, tokens, drops, scoring), cfg)
    want = ref.validate_savings(cfg, original, tokens, drops, scoring)
    for key, val in want.items():
        got = getattr(rep, key)
        assert got == val, (key, got, val)
    assert rep.exact_match  # the telescoping identity holds for every consistent history


def test_validate_savings_rejects_like_reference(ref):
    cfg = L.ModelConfig(2, 1, [K.FullAttention, K.FFN], 64, 8, 8, 16, 128)
    bad = [10, 6, 10, 10]  # layer 1 entered with 6 rows but no drop was recorded
    with pytest.raises(oracle.OracleContractViolation):
        ref.validate_savings(cfg, 10, bad, [], 0)
    with pytest.raises(L.ContractViolation):
        L.validate_savings(*_ledgers(cfg, 10, bad, [], 0), cfg)


def test_batch_ledger_and_layer_meta(ref):
    """BatchLedger charges a varlen batch like Engine::run_batch: per request, layers at their
    entry counts, scoring + DropRecord at the drop layer; LayerMeta = the cu_seqlens snapshot."""
    cfg = L.ModelConfig(2, 2, [K.FullAttention, K.SlidingWindowAttention, K.FFN], 256, 64, 8, 512, 1024)
    lengths = [700, 0, 65, 4096]
    kept = [300, 0, 65, 1024]
    cu = [0]
    for n in lengths:
        cu.append(cu[-1] + n)
    cu_out = [0]
    for n in kept:
        cu_out.append(cu_out[-1] + n)
    bl = L.BatchLedger(cfg, query_window_n=128)
    for layer in range(cfg.total_layers()):
        if layer % cfg.pattern_length() == 0:
            meta = bl.record_layer(layer, cu, cu_out)  # drop at every block's full-attention layer
            assert meta.query_start_loc == cu and meta.seq_lens == lengths and meta.num_actual_tokens == cu[-1]
        else:
            meta = bl.record_layer(layer, cu_out)
            assert meta.seq_lens == kept
    for r, n in enumerate(lengths):
        dense = L.FlopsLedger()
        for layer in range(cfg.total_layers()):
            dense.add_layer(layer, cfg.kind(layer), n, cfg)
        acc = bl.ledgers[r]
        if n == 0:
            assert not acc.drops and acc.total() == 0
            continue
        rep = L.validate_savings(dense, acc, cfg)
        tokens = [e.tokens for e in acc.entries]
        drops = [(d.layer, d.tokens_before, d.tokens_after, d.retention_ratio) for d in acc.drops]
        want = ref.validate_savings(cfg, n, tokens, drops, acc.scoring_overhead)
        assert rep.exact_match and rep.measured_delta == want["measured_delta"]
        assert acc.scoring_overhead == 2 * ref.scoring_flops(min(128, n), n, cfg)
