"""GPU parity: downstream-layer metadata after a drop -- Eq. 16 KV slot mapping
(PagedKVCache::recompute_slots_after_drop, kvcache.cpp:147-158) and Eq. 17 decode seqused
(decode_seqused, kvcache.cpp:182-186) -- against the unmodified reference."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _compacted_positions(up, lengths, keep_frac, seed):
    rng = np.random.default_rng(seed)
    T = sum(lengths)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    pos = torch.cat([torch.arange(n, dtype=torch.int64) for n in lengths]).cuda()
    keep = (rng.random(T) < keep_frac).astype(np.uint8)
    keep[np.concatenate([[0], np.cumsum(lengths)[:-1]])] = 1  # every request keeps a row
    res = up.compact_varlen(torch.from_numpy(keep).cuda(), cu, [pos], check=True)
    return res, keep


@pytest.mark.parametrize("lengths,L,B", [([300, 17, 1000], 3, 16), ([64], 1, 64), ([5000, 33], 2, 128)])
def test_slot_mapping_matches_reference(up, ref, lengths, L, B):
    res, _ = _compacted_positions(up, lengths, 0.4, sum(lengths) + L)
    n = int(res.num_out.item())
    cu = res.cu_seqlens.cpu().numpy()
    pos = res.planes[0][:n].cpu().numpy()
    R = len(lengths)
    max_pages = max((x + B - 1) // B for x in lengths) + 1
    tables = np.full((L, R, max_pages), -1, np.int32)
    want = np.zeros((L, n), np.int64)
    for r in range(R):
        ret = pos[cu[r]:cu[r + 1]]
        # pages pre-allocated for the first half of the prompt, the rest on demand
        t, s = ref.recompute_slots(L, B, lengths[r] // 2, ret, max_pages)
        tables[:, r, :] = t
        want[:, cu[r]:cu[r + 1]] = s
    got = up.slot_mapping(res.cu_seqlens, res.planes[0][:n], torch.from_numpy(tables).cuda(), B,
                          num_rows=res.num_out, check=True)
    assert np.array_equal(got.cpu().numpy(), want)


def test_slot_mapping_missing_page_is_allocation_miss(up):
    cu = torch.tensor([0, 3], dtype=torch.int32, device="cuda")
    pos = torch.tensor([0, 17, 40], dtype=torch.int64, device="cuda")
    tables = torch.tensor([[[7, -1, 3]]], dtype=torch.int32, device="cuda")
    with pytest.raises(up.AllocationMissError):
        up.slot_mapping(cu, pos, tables, 16, check=True)
    ok = up.slot_mapping(cu, pos[[0, 2]], tables, 16, check=True)
    assert ok.cpu().tolist() == [[7 * 16 + 0, 3 * 16 + 8]]
    with pytest.raises(up.ConfigError):
        up.slot_mapping(cu, pos, tables, 0)


def test_decode_seqused_matches_reference(up, ref):
    lengths = [700, 1, 2500, 64]
    R = len(lengths)
    cu0 = torch.tensor(np.concatenate([[0], np.cumsum(lengths)]), dtype=torch.int32, device="cuda")
    # two drop events (layers 3 and 9) -> cu_seqlens after each
    res1, _ = _compacted_positions(up, lengths, 0.5, 1)
    l1 = np.diff(res1.cu_seqlens.cpu().numpy()).tolist()
    res2, _ = _compacted_positions(up, l1, 0.5, 2)
    l2 = np.diff(res2.cu_seqlens.cpu().numpy()).tolist()
    appended = torch.tensor([3, 0, 11, 1], dtype=torch.int32, device="cuda")
    L = 14
    got = up.decode_seqused(L, cu0, [3, 9], [res1.cu_seqlens, res2.cu_seqlens], appended).cpu().numpy()
    for layer in range(L):
        for r in range(R):
            want = ref.decode_seqused(lengths[r], int(appended[r]), [3, 9], [l1[r], l2[r]], layer)
            assert got[layer, r] == want, (layer, r)
    # no drops: every layer sees the prompt
    got0 = up.decode_seqused(4, cu0, [], []).cpu().numpy()
    assert (got0 == np.array(lengths)[None, :]).all()
    with pytest.raises(up.ContractViolation):  # drop layers must increase (DropHistory::validate)
        up.decode_seqused(L, cu0, [9, 3], [res1.cu_seqlens, res2.cu_seqlens])


def test_batch_ledger_over_device_drop_layers(up, ref):
    """§8f row 4: LayerMeta snapshots and per-request FLOPs ledgers read off the device path's
    own cu_seqlens through a 2-block hybrid model (drop at each block's full-attention layer,
    reconstitution at the boundary), audited by the reference's validate_savings."""
    from paper_2605_06221_b200.ledger import BatchLedger, FlopsLedger, ModelConfig, SublayerKind as K, validate_savings
    from paper_2605_06221_b200.synthetic import make_batch
    lengths = [3000, 129, 1500]
    sb = make_batch(lengths, 32, 8, 128, 64, regime="planted", seed=11, device="cuda")
    cfg = ModelConfig(2, 3, [K.FullAttention, K.SlidingWindowAttention, K.LinearAttention, K.FFN],
                      hidden_dim=4096, head_dim=128, num_heads=32, window_size=4096, ffn_dim=14336)
    layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(32, 8, 128), sum(lengths), len(lengths), [()],
                         [torch.int64])
    bl = BatchLedger(cfg)
    for l in range(cfg.total_layers()):
        if cfg.kind(l) == K.FullAttention:  # every block re-enters with the full prompt
            out = layer(sb.q, sb.k, sb.cu_seqlens, [sb.positions])
            layer.check()
            meta = bl.record_layer(l, sb.cu_seqlens, out.cu_seqlens, layer.sel.covered_mass)
            assert meta.seq_lens == lengths
            cu_after = out.cu_seqlens
        else:
            meta = bl.record_layer(l, cu_after)
    kept = np.diff(cu_after.cpu().numpy()).tolist()
    assert bl.layer_meta[1].seq_lens == kept and bl.layer_meta[1].num_actual_tokens == sum(kept)
    for r, n in enumerate(lengths):
        dense = FlopsLedger()
        for l in range(cfg.total_layers()):
            dense.add_layer(l, cfg.kind(l), n, cfg)
        acc = bl.ledgers[r]
        rep = validate_savings(dense, acc, cfg)
        want = ref.validate_savings(cfg, n, [e.tokens for e in acc.entries],
                                    [(d.layer, d.tokens_before, d.tokens_after, d.retention_ratio) for d in acc.drops],
                                    acc.scoring_overhead)
        assert rep.exact_match and want["exact_match"]
        for key in ("dense_total", "accel_total", "measured_delta", "formula_delta", "scoring_overhead"):
            assert getattr(rep, key) == want[key], key
        assert [d.tokens_after for d in acc.drops] == [kept[r]] * 2
