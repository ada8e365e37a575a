"""GPU parity at the BASELINE.json configuration sizes -- against the reference itself
(oracle/_ref, the unmodified reference compiled from its sources) on full-length requests,
and through size-independent properties and an fp64 PyTorch restatement of the scorer:

* END TO END vs the reference (north-star rule 2): for full-length requests of every config
  (C1 4K is in test_gpu_golden_e2e.py; here 32K, 64K, 128K, the 64-request stream and a 1M
  TP-rank slice) the reference's score_tokens (or its sharded_block_scores +
  allreduce_scores, shards on host threads, bitwise the sequential reference) runs on the
  same bf16-exact q/k: GPU block scores within rtol 1e-3, keep masks equal except for
  blocks whose reference score is within rtol 1e-3 of the reference cutoff score (tie band);
* block scores vs an fp64 dense softmax of the same bf16 inputs (importance.cpp:17-90
  restated with torch.float64): rtol 1e-3;
* mass conservation: Σ_g b_g·|g| = #q-heads per request (each head's softmax rows sum to 1,
  averaged over n_eff rows; test_importance.cpp:111-126);
* keep masks bit-exact vs the reference's top_p_select (oracle port) on the GPU's block
  scores, for every request;
* compaction byte-exact vs torch gathers; cu_seqlens_out = per-segment kept counts;
* reconstitution round trip restores the pre-drop buffer exactly.
"""
import numpy as np
import pytest
import torch

from paper_2605_06221_b200.synthetic import MODEL_SHAPES, make_batch

pytestmark = pytest.mark.gpu

CFG = dict(query_window_n=128, block_size_g=64, sink_count_a=128, top_p=0.99)
RTOL = 1e-3


def _reference_requests(ref, sb, requests, Hq, Hkv, cfg, tp=1):
    """The reference's block scores and selection for each request in `requests`, run
    concurrently (one request per thread; each request's shards on further threads)."""
    import concurrent.futures as cf
    import os
    cu = sb.cu_seqlens.cpu().tolist()
    D = sb.q.shape[2]
    n = cfg["query_window_n"]
    threads = max(1, (os.cpu_count() or 1) // max(1, len(requests)))

    def one(r):
        s, e = cu[r], cu[r + 1]
        qt = sb.q[max(s, e - n):e].float().reshape(-1, Hq * D).cpu().numpy()
        kk = sb.k[s:e].float().reshape(e - s, Hkv * D).cpu().numpy()
        _, blk = ref.sharded_allreduce_mt(qt, kk, Hq, Hkv, tp, threads, **cfg)
        return r, blk, ref.top_p_select(blk, e - s, **cfg)

    with cf.ThreadPoolExecutor(len(requests)) as ex:
        return list(ex.map(one, requests))


def _check_vs_reference(ref, sb, res, keep, kstar, requests, Hq, Hkv, cfg, tp=1):
    """Rule 2 for the given requests: rtol on block scores, tie band on keep masks."""
    cu = sb.cu_seqlens.cpu().numpy()
    cub = res.cu_blocks.cpu().numpy()
    bs = res.block_scores.cpu().numpy()
    G = cfg["block_size_g"]
    for r, blk, rsel in _reference_requests(ref, sb, requests, Hq, Hkv, cfg, tp):
        s, e = int(cu[r]), int(cu[r + 1])
        got = bs[cub[r]:cub[r + 1]]
        np.testing.assert_allclose(got, blk, rtol=RTOL, atol=1e-6 * float(blk.sum()) / len(blk))
        order = np.argsort(-blk, kind="stable")
        cut = blk[order[rsel.cutoff_rank - 1]]
        diff = np.flatnonzero(keep[s:e] != rsel.keep_mask)
        off = [i for i in diff if abs(blk[i // G] - cut) > RTOL * abs(cut)]
        assert off == [], f"request {r}: {len(off)} keep decisions differ outside the tie band"
        print(f"request {r}: N={e - s} vs reference: k* {int(kstar[r])} / {rsel.cutoff_rank}, "
              f"{len(diff)} tie-band tokens differ, worst rel err "
              f"{float(np.max(np.abs(got - blk) / np.maximum(blk, 1e-30))):.2e}")


def _fp64_block_scores(q, k, s, e, Hq, Hkv, n, G):
    """importance.cpp:17-90 in float64 on the device: last-n queries vs all keys, causal
    mask in the tail, softmax over keys, mean over rows, sum over heads, mean per block."""
    N = e - s
    neff = min(n, N)
    D = q.shape[2]
    grp = Hq // Hkv
    qt = q[e - neff:e].to(torch.float64)            # [neff, Hq, D]
    kk = k[s:e].to(torch.float64)                   # [N, Hkv, D]
    tok = torch.zeros(N, dtype=torch.float64, device=q.device)
    rows = torch.arange(neff, device=q.device)
    cols = torch.arange(N, device=q.device)
    mask = cols[None, :] > (N - neff + rows)[:, None]
    for h in range(Hq):
        sc = qt[:, h, :] @ kk[:, h // grp, :].T / np.sqrt(D)
        sc.masked_fill_(mask, float("-inf"))
        tok += torch.softmax(sc, dim=1).sum(0) / neff
    nb = (N + G - 1) // G
    pad = torch.zeros(nb * G, dtype=torch.float64, device=q.device)
    pad[:N] = tok
    sizes = torch.full((nb,), G, dtype=torch.float64, device=q.device)
    sizes[-1] = N - (nb - 1) * G
    return pad.view(nb, G).sum(1) / sizes


def _check_layer(up, port, sb, Hq, Hkv, D, lengths, cfg, tp=1, exact_requests=(0,), ref=None, ref_requests=(),
                 ref_tp=None):
    sc = up.ScoreConfig(**cfg)
    heads = up.HeadLayout(Hq, Hkv, D)
    if tp > 1:
        res = up.score_blocks_tp(sb.q, sb.k, sb.cu_seqlens, sc, tp, heads, check=True)
    else:
        res = up.score_blocks_varlen(sb.q, sb.k, sb.cu_seqlens, sc, heads, check=True)
    cu = sb.cu_seqlens.cpu().numpy()
    cub = res.cu_blocks.cpu().numpy()
    bs = res.block_scores[:int(cub[-1])].double()
    G = cfg["block_size_g"]
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        b = bs[cub[r]:cub[r + 1]]
        sizes = torch.full_like(b, G)
        sizes[-1] = (e - s) - (b.numel() - 1) * G
        mass = float((b * sizes).sum())
        assert abs(mass - Hq) < 1e-3 * Hq, (r, mass)
        if r in exact_requests:
            want = _fp64_block_scores(sb.q, sb.k, s, e, Hq, Hkv, cfg["query_window_n"], G)
            err = (b - want).abs()
            atol = 1e-6 * float(want.sum()) / want.numel()
            bad = err > 1e-3 * want.abs() + atol
            assert not bool(bad.any()), f"request {r}: {int(bad.sum())} blocks off, worst {float((err / want).max()):.2e}"
            print(f"request {r}: N={e - s} mass={mass:.6f} worst rel err {float((err / want).max()):.2e}")
    # selection: bit-exact vs the reference top_p_select on the GPU's own block scores
    sel = up.select_varlen(res.block_scores, res.cu_blocks, sb.cu_seqlens, sc, check=True)
    keep = sel.keep.cpu().numpy()
    bsh = res.block_scores.cpu().numpy()
    kstar = sel.cutoff_rank.cpu().numpy()
    for r in range(len(lengths)):
        s, e = int(cu[r]), int(cu[r + 1])
        want = port.top_p_select(bsh[cub[r]:cub[r + 1]], e - s, **cfg)
        assert np.array_equal(keep[s:e], want.keep_mask), f"keep mask of request {r}"
        assert int(kstar[r]) == want.cutoff_rank
    if ref is not None and ref_requests:
        _check_vs_reference(ref, sb, res, keep, kstar, list(ref_requests), Hq, Hkv, cfg,
                            tp if ref_tp is None else ref_tp)
    # compaction: byte-exact gathers, new cu_seqlens, then the reconstitution round trip
    planes = [sb.hidden, sb.k, sb.v, sb.positions]
    out = up.compact_varlen(sel.keep, sb.cu_seqlens, planes, check=True)
    n = int(out.num_out.item())
    idx = out.retained_index[:n].long()
    assert bool((idx[1:] > idx[:-1]).all())
    for src, dst in zip(planes, out.planes):
        assert torch.equal(dst[:n], src[idx])
    kept = [int(keep[int(cu[r]):int(cu[r + 1])].sum()) for r in range(len(lengths))]
    assert out.cu_seqlens.cpu().tolist() == np.concatenate([[0], np.cumsum(kept)]).tolist()
    pre = sb.hidden.clone()
    pre[idx] = 0  # wipe the retained rows; the unwind must restore them exactly
    up.reconstitute_varlen([out.planes[0]], out, [pre])
    assert torch.equal(pre, sb.hidden)
    return n / sum(lengths)


def test_llama_4x32k_full_layer(up, port, ref):
    """BASELINE config 2 layer (LLaMA-3.1-8B shape, 4 x 32K); requests 0 and 3 end to end
    vs the reference's unsharded score_tokens."""
    shp = MODEL_SHAPES["llama3.1-8b"]
    lengths = [32768] * 4
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=11)
    rho = _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, CFG,
                       exact_requests=(0, 3), ref=ref, ref_requests=(0, 3))
    assert 0.1 < rho < 0.6


def test_qwen3_next_128k_tp8_full_layer(up, port, ref):
    """BASELINE config 3 layer (Qwen3-Next full-attention shape, 1 x 128K, TP=8 shards) end
    to end vs the reference's sharded_block_scores + allreduce_scores at T = 8."""
    shp = MODEL_SHAPES["qwen3-next-80b-a3b"]
    lengths = [131072]
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=12)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, CFG, tp=8,
                 ref=ref, ref_requests=(0,))


def test_gemma3_varlen_64k_layer(up, port, ref):
    """BASELINE config 4 shape (Gemma-3-12B, p = 0.98), four 64K requests; request 1 end to
    end vs the reference's unsharded score_tokens."""
    shp = MODEL_SHAPES["gemma3-12b"]
    lengths = [65536] * 4
    cfg = dict(CFG, top_p=0.98)
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=13)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, cfg,
                 exact_requests=(1,), ref=ref, ref_requests=(1,))


def test_mixed_stream_64_requests(up, port, ref):
    """BASELINE config 5 stream (64 requests, 4K-128K log-uniform): per-request checks; the
    longest and the shortest request end to end vs the reference (shards of 4 heads on host
    threads -- the reference's own TP path)."""
    from paper_2605_06221_b200.synthetic import loguniform_lengths
    shp = MODEL_SHAPES["llama3.1-8b"]
    lengths = loguniform_lengths(64, 4096, 131072, 5)
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=14)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, CFG,
                 exact_requests=(0, 31), ref=ref,
                 ref_requests=(int(np.argmax(lengths)), int(np.argmin(lengths))), ref_tp=8)


def test_one_million_token_request_tp_rank(up, port, ref):
    """Maximum request size: a 2^20-token (1M context) request at one Qwen3-Next TP=8 rank's
    head slice (2 q-heads, 1 kv-head, D = 256) -- 16384 blocks, the most the on-chip select
    sort holds -- through score (fp64 restatement), select (bit-exact), compaction and the
    reconstitution round trip; end to end vs the reference (its two heads as two shards on
    two threads)."""
    lengths = [1 << 20]
    sb = make_batch(lengths, 2, 1, 256, 512, regime="planted", seed=15)
    rho = _check_layer(up, port, sb, 2, 1, 256, lengths, CFG, ref=ref, ref_requests=(0,), ref_tp=2)
    assert 0.05 < rho < 0.8


def test_llama_32k_query_window_512(up, port, ref):
    """The paper's n = 512 ablation at a BASELINE request length (LLaMA-3.1-8B shape, 2 x
    32K): the query-tile scorer (4 tiles of 128 rows per q-head as virtual heads) vs an fp64
    restatement (request 0) and end to end vs the reference (request 1, its heads as 8
    shards on host threads)."""
    shp = MODEL_SHAPES["llama3.1-8b"]
    lengths = [32768] * 2
    cfg = dict(CFG, query_window_n=512)
    sb = make_batch(lengths, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], shp["hidden"],
                    regime="planted", seed=16)
    _check_layer(up, port, sb, shp["num_q_heads"], shp["num_kv_heads"], shp["head_dim"], lengths, cfg,
                 exact_requests=(0,), ref=ref, ref_requests=(1,), ref_tp=8)
