"""GPU parity against the reference's golden vectors and end to end (score -> select ->
compact) against the reference hot path on identical bf16-exact inputs.

Parity rules (north star):
  * selection on identical block scores: keep mask, k*, retained indices bit-exact;
  * end to end from q/k: block scores within rtol 1e-3; keep masks equal except for blocks
    whose reference score lies within rtol 1e-3 of the cutoff score (tie band);
  * compaction on an identical mask: byte-exact rows, cu_seqlens and index lists.
"""
import json
import os
import struct

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden.json")
RTOL = 1e-3


def unhex(xs):
    return np.array([struct.unpack("<f", bytes.fromhex(x))[0] for x in xs], np.float32)


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def test_gpu_selection_matches_reference_golden(up, golden):
    for case in golden["selection"]:
        s = torch.from_numpy(unhex(case["scores"])).cuda()
        sel = up.top_p_select(s, up.ScoreConfig(**case["cfg"]), case["num_tokens"])
        assert sel.retained_indices.cpu().tolist() == case["retained"], case["kind"]
        assert sel.cutoff_rank == case["cutoff_rank"]
        assert sel.degenerate_keep_all == case["degenerate"]
        want = float.fromhex(case["covered_mass"])
        assert abs(sel.covered_mass - want) <= 1e-12 * max(1.0, abs(want))


def test_gpu_selection_batched_golden(up, golden):
    """All c3 golden vectors in ONE varlen launch (one CTA per request)."""
    cases = [c for c in golden["selection"] if c["kind"] == "c3" and c["cfg"]["block_size_g"] == 1]
    # select_varlen takes one config; group by p.
    by_p = {}
    for c in cases:
        by_p.setdefault(c["cfg"]["top_p"], []).append(c)
    for p, group in by_p.items():
        scores = np.concatenate([unhex(c["scores"]) for c in group])
        lengths = [c["num_tokens"] for c in group]
        cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
        sel = up.select_varlen(torch.from_numpy(scores).cuda(), torch.from_numpy(cu).cuda(),
                               torch.from_numpy(cu).cuda(), up.ScoreConfig(**group[0]["cfg"]), check=True)
        keep = sel.keep.cpu().numpy()
        for r, c in enumerate(group):
            assert np.flatnonzero(keep[cu[r]:cu[r + 1]]).tolist() == c["retained"]
            assert int(sel.cutoff_rank[r]) == c["cutoff_rank"]


def test_gpu_compaction_matches_reference_golden(up, golden):
    for case in golden["compact"]:
        if case["name"] == "apply_drop_order":
            st = torch.from_numpy(unhex(case["states"]).reshape(case["rows"], case["cols"])).cuda()
            stream = up.TokenStream.from_prompt(st)
            keep = torch.tensor(case["keep"], dtype=torch.uint8, device="cuda")
            idx = torch.nonzero(keep).flatten()
            up.apply_drop(stream, up.Selection(keep, idx, 0.5, 1.0, 4, False), 0, up.DropHistory())
            assert np.array_equal(stream.active_states.cpu().numpy(), unhex(case["out"]).reshape(-1, case["cols"]))
            assert stream.logical_positions.cpu().tolist() == case["positions"]
            continue
        toks = torch.from_numpy(unhex(case["tokens"]).reshape(-1, case["cols"])).cuda()
        phases = ["decode" if (case["is_decode"] and case["is_decode"][s]) else "prefill"
                  for s in range(len(case["cu"]) - 1)]
        b = up.PackedBatch(toks, torch.tensor(case["cu"]), phases)
        sels = []
        for s in range(len(case["cu"]) - 1):
            if case["selected"][s]:
                k = torch.tensor(case["keep"][case["cu"][s]:case["cu"][s + 1]], dtype=torch.uint8, device="cuda")
                i = torch.nonzero(k).flatten()
                sels.append(up.Selection(k, i, 1.0, 1.0, i.numel(), False))
            else:
                sels.append(None)
        up.patch_metadata(b, sels, 0)
        assert b.cu_seqlens.tolist() == case["cu_out"]
        assert np.array_equal(b.tokens.cpu().numpy(), unhex(case["out"]).reshape(-1, case["cols"]))


def _rng_matrix(port, rows, cols, seed, stream, stddev):
    return port.rng_normal_array(seed, stream, rows * cols, stddev).reshape(rows, cols)


def test_gpu_scorer_golden_inputs(up, port, golden):
    """Golden scorer cases on bf16-rounded inputs: GPU vs oracle (same rounded inputs)."""
    for case in golden["scorer"]:
        N, H, Hkv, D = case["N"], case["H"], case["Hkv"], case["D"]
        q = torch.from_numpy(_rng_matrix(port, N, H * D, case["seed"], 0x696D70, case["stddev"])).to(torch.bfloat16)
        k = torch.from_numpy(_rng_matrix(port, N, Hkv * D, case["seed"], 0x696D71, case["stddev"])).to(torch.bfloat16)
        for want_tokens in (False, True):
            res = up.score_tokens(q.cuda(), k.cuda(), H, up.ScoreConfig(**case["cfg"]), num_kv_heads=Hkv,
                                  want_token_scores=want_tokens)
            tok, blk, _ = port.score_tokens(q.float().numpy(), k.float().numpy(), H, Hkv, **case["cfg"])
            np.testing.assert_allclose(res.block_scores.cpu().numpy(), blk, rtol=RTOL, atol=1e-7)
            if want_tokens:
                np.testing.assert_allclose(res.token_scores.cpu().numpy(), tok, rtol=RTOL, atol=1e-7)


def _tie_band_ok(gpu_keep, ref_keep, ref_blocks, G, cutoff_score):
    """Mismatched tokens must belong to blocks whose reference score is within rtol of the
    cutoff score s_{pi(k*)}."""
    bad = np.flatnonzero(gpu_keep != ref_keep)
    for i in bad:
        s = ref_blocks[i // G]
        if abs(s - cutoff_score) > RTOL * abs(cutoff_score):
            return False
    return True


@pytest.mark.parametrize("shape,lengths,regime", [
    ((32, 8, 128, 256), [4096], "planted"),            # C1: LLaMA-3.1-8B layer shape, 1 x 4K
    ((32, 8, 128, 256), [1500, 64, 2100, 1], "planted"),
    ((16, 2, 256, 128), [2048, 700], "planted"),       # Qwen3-Next FA head layout (D=256, GQA 8)
    ((16, 8, 256, 128), [1200, 900], "iid"),           # Gemma-3-12B head layout (D=256, GQA 2)
])
def test_drop_layer_end_to_end_vs_reference(up, port, shape, lengths, regime):
    import oracle
    from paper_2605_06221_b200.synthetic import make_batch
    Hq, Hkv, D, HID = shape
    cfgd = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
    cfg = up.ScoreConfig(**cfgd)
    sb = make_batch(lengths, Hq, Hkv, D, HID, regime=regime, seed=sum(lengths), device="cuda")
    T = sum(lengths)
    layer = up.DropLayer(cfg, up.HeadLayout(Hq, Hkv, D), T, len(lengths), [(HID,), (Hkv, D), (Hkv, D), ()],
                         [torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.int64])
    out = layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden, sb.k, sb.v, sb.positions])
    layer.check()
    checker = oracle.ref() if (oracle.ref_available() and T <= 4096) else port
    cu = sb.cu_seqlens.cpu().numpy()
    cub = layer.scores.cu_blocks.cpu().numpy()
    bs = layer.scores.block_scores.cpu().numpy()
    keep = layer.sel.keep.cpu().numpy()
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        q = sb.q[s:e].float().reshape(e - s, -1).cpu().numpy()
        k = sb.k[s:e].float().reshape(e - s, -1).cpu().numpy()
        _, ref_blk, _ = checker.score_tokens(q, k, Hq, Hkv, want_tokens=False, **cfgd)
        got = bs[cub[r]:cub[r + 1]]
        np.testing.assert_allclose(got, ref_blk, rtol=RTOL, atol=1e-6 * ref_blk.sum() / len(ref_blk))
        ref_sel = checker.top_p_select(ref_blk, e - s, **cfgd)
        # Rule 1: the GPU's own block scores select bit-exactly like the reference.
        own = port.top_p_select(got, e - s, **cfgd)
        assert np.array_equal(keep[s:e], own.keep_mask)
        assert int(layer.sel.cutoff_rank[r]) == own.cutoff_rank
        # Rule 2: vs the reference's scores, mismatches only inside the tie band.
        order = np.argsort(-ref_blk, kind="stable")
        cutoff_score = ref_blk[order[ref_sel.cutoff_rank - 1]]
        assert _tie_band_ok(keep[s:e], ref_sel.keep_mask, ref_blk, 64, cutoff_score)
    # Rule 3: compaction byte-exact given the mask.
    n = int(out.num_out.item())
    idx = np.flatnonzero(keep[:T])
    assert n == len(idx)
    ii = torch.from_numpy(idx).cuda()
    assert torch.equal(out.planes[0][:n], sb.hidden[ii])
    assert torch.equal(out.planes[1][:n], sb.k[ii])
    assert torch.equal(out.planes[2][:n], sb.v[ii])
    assert torch.equal(out.planes[3][:n], sb.positions[ii])
    assert np.array_equal(out.retained_index[:n].cpu().numpy(), idx)
    new_cu = [0] + [int(keep[cu[r]:cu[r + 1]].sum()) for r in range(len(lengths))]
    assert out.cu_seqlens.cpu().tolist() == np.cumsum(new_cu).tolist()


def test_tp_head_sharded_scores_and_ordered_reduce(up, port):
    """TP=2/4/8 head slices scored separately and reduced in ascending shard order on the GPU
    equal the reference's sharded_block_scores + allreduce_scores within rtol, and every
    TP degree selects the same tokens (acceptance c8)."""
    from paper_2605_06221_b200.distributed import head_slice
    from paper_2605_06221_b200.synthetic import make_batch
    Hq, Hkv, D = 16, 2, 256      # Qwen3-Next FA layer: TP=8 -> 2 q-heads, 1 kv-head per rank
    sb = make_batch([3000], Hq, Hkv, D, 64, regime="planted", seed=8, device="cuda")
    cfg = up.ScoreConfig()
    q2 = sb.q.reshape(3000, -1)
    full = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, up.HeadLayout(Hq, Hkv, D), check=True)
    nb = int(full.cu_blocks[-1].item())
    keeps = []
    for tp in (1, 2, 4, 8):
        parts = []
        for t in range(tp):
            (qb, qe), (kb, ke) = head_slice(Hq, Hkv, t, tp)
            qs = sb.q[:, qb:qe]
            ks = sb.k[:, kb:ke]
            # a rank holds only its slices: copy them out contiguously as a TP rank would
            res = up.score_blocks_varlen(qs.contiguous(), ks.contiguous(), sb.cu_seqlens, cfg,
                                         up.HeadLayout(qe - qb, ke - kb, D, Hq // Hkv, qb, kb), check=True)
            parts.append(res.block_scores[:nb].clone())
        red = up.reduce_block_scores(parts)
        np.testing.assert_allclose(red.cpu().numpy(), full.block_scores[:nb].cpu().numpy(), rtol=RTOL)
        want = np.zeros(nb, np.float32)
        for pt in parts:
            want = (want + pt.cpu().numpy()).astype(np.float32)
        assert np.array_equal(red.cpu().numpy(), want)  # ascending-rank fp32 order, bitwise
        sel = up.select_varlen(red, full.cu_blocks, sb.cu_seqlens, cfg, check=True)
        keeps.append(sel.keep.cpu().numpy())
        if tp == 1:
            red1 = red.cpu().numpy()
            cut1 = red1[np.argsort(-red1, kind="stable")[int(sel.cutoff_rank[0]) - 1]]
    # c8 (acceptance_main.cpp:445-478): identical selection for every TP degree -- tokens may
    # differ only in blocks whose TP=1 score lies within rtol of the TP=1 cutoff score (the
    # shard sums round differently, the tie band of north-star rule 2)
    for k in keeps[1:]:
        assert _tie_band_ok(k, keeps[0], red1, 64, cut1)


def test_cuda_graph_capture_of_drop_layer(up):
    """The whole layer is device-driven (no host syncs): it captures and replays in a graph."""
    from paper_2605_06221_b200.synthetic import make_batch
    sb = make_batch([2000, 1000], 32, 8, 128, 512, regime="planted", seed=3, device="cuda")
    layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(32, 8, 128), 3000, 2, [(512,)], [torch.bfloat16])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        eager = layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden])
        keep0 = layer.sel.keep.clone()
        n0 = int(eager.num_out.item())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden])
        layer.sel.keep.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(layer.sel.keep, keep0)
    assert int(layer.out.num_out.item()) == n0


def test_cuda_graph_capture_across_select_size_classes(up):
    """Requests in two select size classes (<= 512 and > 512 blocks): the larger class runs
    on the library's side stream (fork / join events), in eager mode and inside a graph."""
    from paper_2605_06221_b200.synthetic import make_batch
    sb = make_batch([36000, 3000, 500], 8, 2, 128, 256, regime="planted", seed=5, device="cuda")
    layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(8, 2, 128), 40000, 3, [(256,)], [torch.bfloat16])
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        eager = layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden])
        keep0 = layer.sel.keep.clone()
        cu0 = eager.cu_seqlens.clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden])
        layer.sel.keep.zero_()
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    T = 36000 + 3000 + 500  # keep past the batch (capacity 40000) is not written
    assert torch.equal(layer.sel.keep[:T], keep0[:T])
    assert torch.equal(layer.out.cu_seqlens, cu0)


def _random_case(seed):
    rng = np.random.default_rng(seed)
    Hq, Hkv, D = [(8, 2, 128), (4, 2, 256), (4, 4, 64), (16, 8, 256), (32, 8, 128), (2, 1, 256)][seed % 6]
    cfgd = dict(query_window_n=int(rng.choice([16, 64, 100, 128, 200])),
                block_size_g=int(rng.choice([8, 32, 64, 96, 128])),
                sink_count_a=int(rng.choice([0, 16, 128, 1000])),
                top_p=float(rng.choice([0.5, 0.9, 0.99, 1.0])))
    R = int(rng.integers(1, 6))
    lengths = [int(x) for x in rng.choice([1, 5, 40, 130, 700, 1500, 2600], size=R)]
    en = (rng.random(R) < 0.8).astype(np.uint8)
    veto_frac = float(rng.choice([0.0, 0.0, 0.05]))
    return (Hq, Hkv, D), cfgd, lengths, en, veto_frac


# 24 seeds in the default run; UP_SWEEP_SEEDS=N widens the sweep (profiles/parity_sweep_r01.txt)
@pytest.mark.parametrize("seed", list(range(int(os.environ.get("UP_SWEEP_SEEDS", "24")))))
def test_drop_layer_random_configs_vs_oracle(up, port, seed):
    """Seeded sweep over the knobs (n, G, A, p), head layouts (every scorer kernel), varlen
    segments incl. single-token and n > N, drop-disabled segments and a no-readmission veto:
    block scores within rtol of the oracle, the keep mask bit-exact with the reference's
    top_p_select (+ restrict_selection for the veto) on the GPU's own scores, compaction
    exact (SURVEY parity rules 1-3)."""
    from paper_2605_06221_b200.synthetic import make_batch
    (Hq, Hkv, D), cfgd, lengths, en, veto_frac = _random_case(seed)
    cfg = up.ScoreConfig(**cfgd)
    T = sum(lengths)
    sb = make_batch(lengths, Hq, Hkv, D, 32, regime="planted", block_size_g=cfgd["block_size_g"], seed=seed)
    rng = np.random.default_rng(100 + seed)
    veto = (rng.random(T) < veto_frac).astype(np.uint8) if veto_frac > 0 else None
    en_t = torch.from_numpy(en).cuda()
    veto_t = torch.from_numpy(veto).cuda() if veto is not None else None
    layer = up.DropLayer(cfg, up.HeadLayout(Hq, Hkv, D), T, len(lengths), [(32,), ()],
                         [torch.bfloat16, torch.int64])
    out = layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden, sb.positions], drop_enabled=en_t, veto=veto_t)
    layer.check()
    cu = sb.cu_seqlens.cpu().numpy()
    cub = layer.scores.cu_blocks.cpu().numpy()
    bs = layer.scores.block_scores.cpu().numpy()
    keep = layer.sel.keep.cpu().numpy()
    kst = layer.sel.cutoff_rank.cpu().numpy()
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        got = bs[cub[r]:cub[r + 1]]
        if not en[r]:  # pass-through segment: untouched, all kept
            assert (keep[s:e] == 1).all() and int(kst[r]) == -1 and not got.any()
            continue
        q = sb.q[s:e].float().reshape(e - s, -1).cpu().numpy()
        k = sb.k[s:e].float().reshape(e - s, -1).cpu().numpy()
        _, want, _ = port.score_tokens(q, k, Hq, Hkv, want_tokens=False, **cfgd)
        np.testing.assert_allclose(got, want, rtol=RTOL, atol=1e-6 * max(want.sum(), 1e-30) / len(want))
        own = port.top_p_select(got, e - s, **cfgd)
        if veto is not None:
            own = port.restrict_selection(own, veto[s:e], got, cfgd["block_size_g"])
        assert np.array_equal(keep[s:e], own.keep_mask), f"segment {r}"
        assert int(kst[r]) == own.cutoff_rank
    n = int(out.num_out.item())
    idx = np.flatnonzero(keep[:T])
    assert n == len(idx)
    ii = torch.from_numpy(idx).cuda()
    assert torch.equal(out.planes[0][:n], sb.hidden[ii])
    assert torch.equal(out.planes[1][:n], sb.positions[ii])


def test_run_to_run_bitwise_determinism(up):
    """Fixed reduction orders: two runs of the drop layer and of the attention
    over its retained rows on the same inputs agree bit for bit -- block scores, keep mask,
    compacted planes, attention output (the persistent kernels' work distribution does not
    leak into the arithmetic)."""
    from paper_2605_06221_b200.synthetic import make_batch
    lengths = [5000, 3000, 700]
    Hq, Hkv, D = 32, 8, 128
    sb = make_batch(lengths, Hq, Hkv, D, 64, regime="planted", seed=77)
    T = sum(lengths)
    outs = []
    for _ in range(2):
        layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(Hq, Hkv, D), T, len(lengths),
                             [(64,), (Hkv, D), (Hkv, D), (), (Hq, D)],
                             [torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.int64, torch.bfloat16])
        res = layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden, sb.k, sb.v, sb.positions, sb.q])
        layer.check()
        n = int(res.num_out.item())
        att = up.attention_varlen(res.planes[4], res.planes[1], res.planes[2], res.cu_seqlens, res.planes[3],
                                  max_tokens=T, check=True)
        nb = int(layer.scores.cu_blocks[-1])  # past it: capacity padding, never written
        outs.append([layer.scores.block_scores[:nb].clone(), layer.sel.keep[:T].clone(),
                     *[p[:n].clone() for p in res.planes], att[:n].clone()])
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_batching_transparency(up):
    """A request's block scores do not depend on what it is batched with (scheduler
    batching transparency, test_scheduler.cpp:85-119): each request of a varlen batch vs the
    same request scored alone, within 1e-5 relative (the persistent scorer's partition moves
    with the batch, so rounding may differ in the last bits), and the same keep mask."""
    from paper_2605_06221_b200.synthetic import make_batch
    lengths = [3000, 777, 5000, 64]
    Hq, Hkv, D = 32, 8, 128
    sb = make_batch(lengths, Hq, Hkv, D, 16, regime="planted", seed=5)
    cfg = up.ScoreConfig()
    heads = up.HeadLayout(Hq, Hkv, D)
    full = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, cfg, heads, check=True)
    fsel = up.select_varlen(full.block_scores, full.cu_blocks, sb.cu_seqlens, cfg, check=True)
    cu = sb.cu_seqlens.tolist()
    cub = full.cu_blocks.tolist()
    for r in range(len(lengths)):
        s, e = cu[r], cu[r + 1]
        one = up.score_blocks_varlen(sb.q[s:e].contiguous(), sb.k[s:e].contiguous(),
                                     torch.tensor([0, e - s], dtype=torch.int32, device="cuda"), cfg, heads,
                                     check=True)
        nb = cub[r + 1] - cub[r]
        a, b = full.block_scores[cub[r]:cub[r + 1]].double(), one.block_scores[:nb].double()
        assert bool(((a - b).abs() <= 1e-5 * b.abs() + 1e-12).all()), f"request {r}"
        osel = up.select_varlen(one.block_scores, one.cu_blocks,
                                torch.tensor([0, e - s], dtype=torch.int32, device="cuda"), cfg, check=True)
        if torch.equal(a, b):
            assert torch.equal(fsel.keep[s:e], osel.keep[:e - s])


def test_p_one_keeps_everything_and_counts_are_monotone_in_p(up):
    """p = 1 keeps every row and compaction is the identity (test_propagation.cpp:171-194);
    the retained count never decreases as p grows (:232-253); the query window and the
    sinks always survive (:310-327)."""
    from paper_2605_06221_b200.synthetic import make_batch
    lengths = [2500, 900, 4100]
    Hq, Hkv, D = 8, 2, 128
    sb = make_batch(lengths, Hq, Hkv, D, 32, regime="planted", seed=12)
    T = sum(lengths)
    cu = sb.cu_seqlens.tolist()
    prev = -1
    for p in (0.3, 0.6, 0.9, 0.99, 1.0):
        cfg = up.ScoreConfig(top_p=p)
        layer = up.DropLayer(cfg, up.HeadLayout(Hq, Hkv, D), T, len(lengths), [(32,), ()],
                             [torch.bfloat16, torch.int64])
        res = layer(sb.q, sb.k, sb.cu_seqlens, [sb.hidden, sb.positions])
        layer.check()
        n = int(res.num_out.item())
        assert n >= prev, (p, n, prev)
        prev = n
        keep = layer.sel.keep[:T].bool()
        for r in range(len(lengths)):
            s, e = cu[r], cu[r + 1]
            neff = min(cfg.query_window_n, e - s)
            assert bool(keep[e - neff:e].all()) and bool(keep[s:s + min(cfg.sink_count_a, e - s)].all())
        if p == 1.0:
            assert n == T
            assert torch.equal(res.planes[0][:T], sb.hidden) and torch.equal(res.planes[1][:T], sb.positions)


def test_batch_past_capacity_is_a_contract_violation(up):
    """cu_seqlens ending past max_tokens (a malformed batch): the device raises the sticky
    ContractViolation and no kernel reads or writes past the capacity-sized buffers."""
    from paper_2605_06221_b200.synthetic import make_batch
    lengths = [700, 500]
    Hq, Hkv, D = 8, 2, 128
    sb = make_batch(lengths, Hq, Hkv, D, 32, regime="planted", seed=3)
    T = sum(lengths)
    cap = T - 100  # the batch claims 100 rows more than the buffers hold
    layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(Hq, Hkv, D), cap, len(lengths),
                         [(32,), (Hkv, D), (Hkv, D), (), (Hq, D)],
                         [torch.bfloat16, torch.bfloat16, torch.bfloat16, torch.int64, torch.bfloat16])
    planes = [sb.hidden[:cap], sb.k[:cap], sb.v[:cap], sb.positions[:cap], sb.q[:cap]]
    res = layer(sb.q[:cap], sb.k[:cap], sb.cu_seqlens, planes)
    with pytest.raises(up.ContractViolation):
        layer.check()
    ws = up.Workspace("cuda")
    up.attention_varlen(sb.q[:cap], sb.k[:cap], sb.v[:cap], sb.cu_seqlens, sb.positions[:cap], max_tokens=cap,
                        workspace=ws)
    with pytest.raises(up.ContractViolation):
        ws.device_status()
    torch.cuda.synchronize()  # the context is still healthy (no out-of-bounds fault)
    assert int(res.num_out.item()) <= cap


def test_malformed_batch_after_a_good_one_compacts_to_nothing(up):
    """A well-formed short batch, then malformed batches on the SAME DropLayer (capacity of
    five 1024-row tiles, so stale per-tile counts and keep bytes from the first call are
    present): past capacity, cu[0] != 0, non-increasing.  Each raises the sticky
    ContractViolation (PackedBatch::validate, scheduler.cpp:33-48) and compacts to an empty
    result (cu_seqlens_out all zero, num_out 0) instead of deriving rows from stale state."""
    from paper_2605_06221_b200.synthetic import make_batch
    Hq, Hkv, D = 8, 2, 128
    cap = 5000
    sb = make_batch([2900, 2100], Hq, Hkv, D, 32, regime="planted", seed=31)
    layer = up.DropLayer(up.ScoreConfig(), up.HeadLayout(Hq, Hkv, D), cap, 2,
                         [(32,), (Hkv, D), ()], [torch.bfloat16, torch.bfloat16, torch.int64])
    planes = [sb.hidden, sb.k, sb.positions]
    short = torch.tensor([0, 1000, 1800], dtype=torch.int32, device="cuda")
    res = layer(sb.q, sb.k, short, planes)
    layer.check()
    assert 0 < int(res.num_out.item()) <= 1800
    for bad in ([0, 2900, 6000], [5, 2900, 5000], [0, 2900, 2900], [0, 3000, 2000]):
        res = layer(sb.q, sb.k, torch.tensor(bad, dtype=torch.int32, device="cuda"), planes)
        with pytest.raises(up.ContractViolation):
            layer.check()
        assert int(res.num_out.item()) == 0, bad
        assert res.cu_seqlens.tolist() == [0, 0, 0], bad
    res = layer(sb.q, sb.k, short, planes)  # and the layer still works afterwards
    layer.check()
    assert 0 < int(res.num_out.item()) <= 1800


@pytest.mark.parametrize("shape", ["token_scores", "simt_head_dim"])
def test_malformed_batch_on_the_simt_scorer(up, shape):
    """The SIMT scorer (per-token scores requested, or a head dim off the tensor-core
    envelope) under a batch ending past max_tokens: ContractViolation, cu_blocks zeroed, no
    out-of-bounds access (the context stays healthy)."""
    from paper_2605_06221_b200.synthetic import make_batch
    Hq, Hkv, D = (8, 2, 128) if shape == "token_scores" else (4, 2, 96)
    sb = make_batch([700, 500], Hq, Hkv, D, 16, regime="planted", seed=4)
    cap = 1100
    ws = up.Workspace("cuda")
    out = up.score_blocks_varlen(sb.q[:cap], sb.k[:cap], sb.cu_seqlens, up.ScoreConfig(), up.HeadLayout(Hq, Hkv, D),
                                 want_token_scores=shape == "token_scores", max_tokens=cap, workspace=ws)
    with pytest.raises(up.ContractViolation):
        ws.device_status()
    torch.cuda.synchronize()
    assert out.cu_blocks.tolist() == [0, 0, 0]
